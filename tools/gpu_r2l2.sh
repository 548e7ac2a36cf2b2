# A/B: number of refinement steps captured as plain gated nodes (SOSADMM_WARM_UNCOND) on the mid-size configs
set -x
for u in 3 4 5 6; do
  for cfg in "pop20 500" "pop20 1200" "box24 600" "lyap10 800"; do
    set -- $cfg
    SOSADMM_WARM_UNCOND=$u timeout 300 python tools/kernel_times.py $1 50 $2 2>&1 | grep span | sed "s/^/unc=$u /" >> gpurun_out/r2l2_span.log
  done
done
for u in 3 5; do SOSADMM_WARM_UNCOND=$u timeout 300 python tools/kernel_times.py pop40 20 4000 2>&1 | grep span | sed "s/^/unc=$u /" >> gpurun_out/r2l2_span.log; done

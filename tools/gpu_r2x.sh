# warm-path experiments: per-evaluation trace, unconditional first steps
set -x
python -c "from paper_1708_04174_b200.build import build; build(force=True)" > gpurun_out/x_build.log 2>&1; echo build=$?
timeout 600 python tools/warm_trace.py pop40 8000 500 > gpurun_out/x_trace40.log 2>&1; echo trace=$?
timeout 300 python tools/warm_trace.py pop20 1500 250 > gpurun_out/x_trace20.log 2>&1; echo trace20=$?
for u in 0 1 2 3; do TAG=unc$u SOSADMM_WARM_UNCOND=$u timeout 300 python tools/span.py pop40 2000 200 3 >> gpurun_out/x_span.log 2>&1; echo unc$u=$?; done
for u in 0 3; do TAG=unc$u SOSADMM_WARM_UNCOND=$u timeout 300 python tools/span.py pop40 7000 200 3 >> gpurun_out/x_span.log 2>&1; done
for u in 0 3; do TAG=unc$u SOSADMM_WARM_UNCOND=$u timeout 300 python tools/span.py pop20 600 200 3 >> gpurun_out/x_span.log 2>&1; done
cat gpurun_out/x_span.log

# Jacobi thread-count sweep for N <= 32 (scratch copy edits only)
for NT in 512 1024; do
  sed -i "s/^constexpr int JAC_NT32 = [0-9]*;/constexpr int JAC_NT32 = $NT;/" paper_1708_04174_b200/csrc/psd_jacobi.cuh
  python -c "from paper_1708_04174_b200.build import build; build(force=True)" > gpurun_out/build_$NT.log 2>&1
  timeout 300 python bench.py --config pop6 --steps 20 --warmup 5 --no-ttt --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('NT=$NT', round(d['value'],1), d['phase_ms_per_iter']['jacobi'])" >> gpurun_out/jnt.log
done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "pop6 or ball4 or msos2 or box24" >> gpurun_out/jnt.log 2>&1

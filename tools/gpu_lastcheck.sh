# last sanity pass on the final tree: smoke, the whole GPU suite, the default bench line and the reference arm
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/last_smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/last_pytest_gpu.log 2>&1; echo pytest=$?
timeout 900 python bench.py > gpurun_out/last_bench_default.log 2>&1; echo bench=$?
timeout 300 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/last_reference.log 2>&1; echo ref=$?

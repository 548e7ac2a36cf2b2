set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2g_smoke.log 2>&1; echo smoke=$?
timeout 1800 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/r2g_pytest_gpu.log 2>&1; echo pytest=$?
timeout 300 python bench.py --steps 20 --warmup 5 --no-ttt > gpurun_out/r2g_bench.log 2>&1; echo bench=$?

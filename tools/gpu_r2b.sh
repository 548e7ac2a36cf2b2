# two-stage tridiagonalisation: stage tests, timing, then the parity suite on the default path
set -x
timeout 600 python -m pytest tests/test_gpu_stages.py -q -x -k "sy2sb or sb2st or two_stage" > gpurun_out/r2b_stages.log 2>&1; echo stages=$?
timeout 300 python tools/ts_prof.py > gpurun_out/r2b_ts_prof.log 2>&1; echo prof=$?
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r2b_pytest_gpu.log 2>&1; echo pytest=$?
timeout 300 python bench.py --steps 20 --warmup 5 --no-ttt > gpurun_out/r2b_bench.log 2>&1; echo bench=$?

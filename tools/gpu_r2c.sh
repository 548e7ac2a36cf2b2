set -x
timeout 300 python tools/ts_debug.py > gpurun_out/r2c_ts_debug.log 2>&1; echo dbg=$?
timeout 600 python -m pytest tests/test_gpu_sharded.py -q -x > gpurun_out/r2c_sharded.log 2>&1; echo sh=$?

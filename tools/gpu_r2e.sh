set -x
timeout 300 python tools/ts_debug.py > gpurun_out/r2e_ts_debug.log 2>&1; echo dbg=$?
timeout 300 python tools/ts_debug2.py > gpurun_out/r2e_ts_debug2.log 2>&1; echo dbg2=$?
timeout 600 python -m pytest tests/test_gpu_stages.py -q -x > gpurun_out/r2e_stages.log 2>&1; echo stages=$?

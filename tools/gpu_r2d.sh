set -x
timeout 300 python tools/ts_debug.py > gpurun_out/r2d_ts_debug.log 2>&1; echo dbg=$?
timeout 300 python tools/ts_debug2.py > gpurun_out/r2d_ts_debug2.log 2>&1; echo dbg2=$?

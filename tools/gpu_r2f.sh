set -x
timeout 600 ncu --set full --import-source on --clock-control none -k "regex:k_sy2sb" -c 1 -o gpurun_out/r2f_ts2 python tools/ts_debug.py 66 > gpurun_out/r2f_ncu2.log 2>&1; echo ncu=$?

#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stages.py -x -q -m gpu 2>&1 | tail -1
for c in pop20 lyap10 box24 pop40; do timeout 200 python tools/kernel_times.py $c 50 200 2>&1 | grep "qrnode\|span"; done

#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for c in pop6 pop20 pop40; do timeout 200 python tools/kernel_times.py $c 50 200 2>&1 | grep "tphase\|k_gather\|span"; done

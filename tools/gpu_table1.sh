#!/bin/bash
# Table I / II reproduction on one B200 plus the new GPU tests (tools/table1_gpu.py, tests/test_gpu_table2.py).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/t1_smi.log 2>&1
timeout 900 python -m pytest tests/test_gpu_table2.py -x -q > gpurun_out/t1_pytest.log 2>&1; echo pytest=$?
timeout 1500 python tools/table1_gpu.py --out gpurun_out/table1_gpu.jsonl > gpurun_out/t1.log 2>&1; echo table1=$?

set -x
timeout 900 python -m pytest tests/test_gpu_sharded.py -q -x > gpurun_out/r2j_sharded.log 2>&1; echo sh=$?

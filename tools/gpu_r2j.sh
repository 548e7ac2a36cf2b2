# shared-GPU hint: batch tests, batch rates, lone-instance rate
set -x
timeout 900 python -m pytest tests/test_gpu_batch.py -x -q > gpurun_out/r2j_pytest.log 2>&1; echo pytest=$?
timeout 300 python bench.py --batch 8 --start 2000 --steps 10 --warmup 3 > gpurun_out/r2j_batch_pop40_8.log 2>&1; echo b8=$?
timeout 300 python bench.py --batch 8 --steps 10 --warmup 3 > gpurun_out/r2j_batch_pop40_8_cold.log 2>&1; echo b8c=$?
timeout 300 python bench.py --config pop20 --batch 16 --start 500 --steps 20 --warmup 3 > gpurun_out/r2j_batch_pop20_16.log 2>&1; echo p16=$?
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu > gpurun_out/r2j_cfg_pop40.log 2>&1; echo pop40=$?

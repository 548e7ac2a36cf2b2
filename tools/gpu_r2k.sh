set -x
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/r2k_pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python bench.py --config pop40 --steps 20 --warmup 5 --no-ttt --no-cpu > gpurun_out/r2k_cfg_pop40.log 2>&1; echo b=$?
timeout 600 ncu --set full --clock-control none --cache-control all -k "regex:k_gather|k_scatter|k_pack" -c 6 -o gpurun_out/r2k_affine python bench.py --steps 1 --warmup 3 --no-ttt --no-cpu > gpurun_out/r2k_ncu.log 2>&1; echo ncu=$?

# fuse_low check: bit-identity + parity subset + small-config benches and in-graph kernel times
set -x
timeout 900 python -m pytest tests/test_gpu_batch.py tests/test_gpu_parity.py tests/test_gpu_sharded.py -x -q > gpurun_out/r2g_pytest.log 2>&1; echo pytest=$?
for c in pop6 pop20; do timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu > gpurun_out/r2g_cfg_$c.log 2>&1; echo $c=$?; done
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu > gpurun_out/r2g_cfg_pop40.log 2>&1; echo pop40=$?
timeout 300 python tools/kernel_times.py pop6 50 30 > gpurun_out/r2g_kernel_times_pop6.txt 2>&1; echo kt6=$?
timeout 300 python tools/kernel_times.py pop20 50 500 > gpurun_out/r2g_kernel_times_pop20.txt 2>&1; echo kt20=$?

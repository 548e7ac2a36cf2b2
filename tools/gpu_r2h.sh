# scan micro-changes: warm tests + parity + convergence subset, then in-graph kernel times and benches
set -x
timeout 1200 python -m pytest tests/test_gpu_warm.py tests/test_gpu_parity.py tests/test_gpu_convergence.py -x -q > gpurun_out/r2h_pytest.log 2>&1; echo pytest=$?
timeout 300 python tools/kernel_times.py pop40 20 2000 > gpurun_out/r2h_kernel_times_pop40.txt 2>&1; echo kt40=$?
timeout 300 python tools/kernel_times.py pop20 50 500 > gpurun_out/r2h_kernel_times_pop20.txt 2>&1; echo kt20=$?
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu > gpurun_out/r2h_cfg_pop40.log 2>&1; echo pop40=$?
for c in pop20 box24; do timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu > gpurun_out/r2h_cfg_$c.log 2>&1; echo $c=$?; done
timeout 300 python bench.py --batch 8 --start 2000 --steps 10 --warmup 3 > gpurun_out/r2h_batch_pop40_8.log 2>&1; echo b8=$?
timeout 300 python bench.py --batch 2 --start 2000 --steps 10 --warmup 3 > gpurun_out/r2h_batch_pop40_2.log 2>&1; echo b2=$?
timeout 300 python bench.py --config pop20 --batch 16 --start 500 --steps 20 --warmup 3 > gpurun_out/r2h_batch_pop20_16.log 2>&1; echo p16=$?

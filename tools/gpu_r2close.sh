# round-2 closing measurement set on the final tree (gpurun_out/close_*)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/close_smi.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/close_smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/close_pytest_gpu.log 2>&1; echo pytest=$?
timeout 900 python bench.py > gpurun_out/close_bench_default.log 2>&1; echo bench=$?
for c in pop6 pop20 lyap10 box24; do timeout 900 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/close_cfg_$c.log 2>&1; echo $c=$?; done
timeout 300 python bench.py --batch 8 --start 2000 --steps 10 --warmup 3 > gpurun_out/close_batch_pop40_8.log 2>&1; echo b8=$?
timeout 300 python bench.py --batch 8 --steps 10 --warmup 3 > gpurun_out/close_batch_pop40_8_cold.log 2>&1; echo b8c=$?
timeout 300 python bench.py --config pop20 --batch 16 --start 500 --steps 20 --warmup 3 > gpurun_out/close_batch_pop20_16.log 2>&1; echo p16=$?
timeout 300 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/close_reference.log 2>&1; echo ref=$?
timeout 300 python tools/kernel_times.py pop40 20 2000 > gpurun_out/close_kernel_times_pop40_k2000.txt 2>&1; echo kt=$?
timeout 300 python tools/kernel_times.py pop40 20 4000 > gpurun_out/close_kernel_times_pop40_k4000.txt 2>&1; echo kt4=$?
timeout 300 python tools/kernel_times.py pop6 50 30 > gpurun_out/close_kernel_times_pop6.txt 2>&1; echo kt6=$?
timeout 300 python tools/kernel_times.py pop20 50 500 > gpurun_out/close_kernel_times_pop20.txt 2>&1; echo kt20=$?
timeout 300 python tools/sanitize.py 30 > gpurun_out/close_allpaths.log 2>&1; echo allpaths=$?
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/close_launches.csv python tools/warm_launches.py pop40 2000 2 > gpurun_out/close_launches.log 2>&1; echo ncu1=$?
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k "regex:k_dgemm|k_warm_scan|k_warm_E" -c 6 -o gpurun_out/close_full python tools/warm_launches.py pop40 2000 1 > gpurun_out/close_full.log 2>&1; echo ncu2=$?

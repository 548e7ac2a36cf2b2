# round-2 closing measurement set on the final tree (gpurun_out/r2fin_*)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2fin_smi.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2fin_smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r2fin_pytest_gpu.log 2>&1; echo pytest=$?
timeout 900 python bench.py > gpurun_out/r2fin_bench_default.log 2>&1; echo bench=$?
for c in pop6 pop20 lyap10 box24; do timeout 900 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/r2fin_cfg_$c.log 2>&1; echo $c=$?; done
timeout 300 python bench.py --batch 8 --steps 10 --warmup 3 > gpurun_out/r2fin_batch_pop40_8.log 2>&1; echo b8=$?
timeout 300 python bench.py --config pop20 --batch 16 --steps 20 --warmup 3 > gpurun_out/r2fin_batch_pop20_16.log 2>&1; echo p16=$?
timeout 300 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r2fin_reference.log 2>&1; echo ref=$?
timeout 300 python tools/kernel_times.py pop40 20 2000 > gpurun_out/r2fin_kernel_times.txt 2>&1; echo kt=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2fin_launches.csv python bench.py --steps 3 --warmup 3 --no-ttt --no-cpu > gpurun_out/r2fin_ncu_list.log 2>&1; echo list=$?
timeout 300 python tools/kernel_times.py pop6 50 30 > gpurun_out/r2fin_kernel_times_pop6.txt 2>&1; echo kt6=$?
timeout 300 python tools/kernel_times.py pop20 50 500 > gpurun_out/r2fin_kernel_times_pop20.txt 2>&1; echo kt20=$?
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_dgemm" --launch-skip 600 -c 3 -o gpurun_out/r2fin_full python bench.py --steps 1 --warmup 3 --no-ttt --no-cpu > gpurun_out/r2fin_ncu_full.log 2>&1; echo ncu=$?

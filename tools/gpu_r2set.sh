# round-2 measurement set (outputs under gpurun_out/r2s_*)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2s_smi.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2s_smoke.log 2>&1; echo smoke=$?
timeout 1800 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/r2s_pytest_gpu.log 2>&1; echo pytest=$?
timeout 900 python bench.py > gpurun_out/r2s_bench_default.log 2>&1; echo bench=$?
for c in pop6 pop20 lyap10 box24; do timeout 900 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/r2s_cfg_$c.log 2>&1; echo $c=$?; done
timeout 300 python bench.py --batch 8 --steps 10 --warmup 3 > gpurun_out/r2s_batch_pop40_8.log 2>&1; echo b8=$?
timeout 300 python bench.py --config pop20 --batch 16 --steps 20 --warmup 3 > gpurun_out/r2s_batch_pop20_16.log 2>&1; echo p16=$?
timeout 300 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r2s_reference.log 2>&1; echo ref=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2s_launches.csv python bench.py --steps 3 --warmup 3 --no-ttt --no-cpu > gpurun_out/r2s_ncu_list.log 2>&1; echo list=$?
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_tridiag" -c 1 -o gpurun_out/r2s_tridiag python bench.py --steps 1 --warmup 3 --no-ttt --no-cpu > gpurun_out/r2s_ncu_trd.log 2>&1; echo trd=$?
timeout 600 ncu --set full --clock-control none --cache-control all -k "regex:k_gather|k_scatter|k_pack|k_kinv" -c 8 -o gpurun_out/r2s_affine python bench.py --steps 1 --warmup 3 --no-ttt --no-cpu > gpurun_out/r2s_ncu_aff.log 2>&1; echo aff=$?
timeout 600 ncu --set full --clock-control none -k "regex:k_gemm_f64|k_bt_apply" --launch-skip 20 -c 6 -o gpurun_out/r2s_gemm python bench.py --steps 1 --warmup 3 --no-ttt --no-cpu > gpurun_out/r2s_ncu_gemm.log 2>&1; echo gemm=$?

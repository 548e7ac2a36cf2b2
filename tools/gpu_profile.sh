# Round profile: clean bench (no ncu), launch list of the same command, one --set full capture of
# the dominant kernels with DRAM traffic.  Outputs under gpurun_out/.
python -c "from paper_1708_04174_b200.build import build; build(force=True)" > gpurun_out/build.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_full.log 2>&1; echo bench=$?
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-ttt --no-cpu > gpurun_out/ncu_list.log 2>&1; echo list=$?
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_tridiag|k_gemm_f64|k_gather|k_dc_prep|k_bt_apply" -c 6 -o gpurun_out/full python bench.py --steps 1 --warmup 3 --no-ttt --no-cpu > gpurun_out/ncu_full.log 2>&1; echo full=$?

# round-end measurement set (outputs under gpurun_out/final_*)
set -x
python -c "from paper_1708_04174_b200.build import build; build(force=True)" > gpurun_out/final_build.log 2>&1; echo build=$?
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/final_smi.log 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/final_pytest_gpu.log 2>&1; echo pytest=$?
timeout 900 python bench.py > gpurun_out/final_bench_default.log 2>&1; echo bench=$?
for c in pop6 pop20 lyap10 box24; do timeout 900 python bench.py --config $c --steps 20 --warmup 5 --no-cpu > gpurun_out/final_cfg_$c.log 2>&1; echo $c=$?; done
timeout 300 python bench.py --batch 8 --steps 10 --warmup 3 > gpurun_out/final_batch_pop40_8.log 2>&1; echo b8=$?
timeout 300 python bench.py --config pop20 --batch 16 --steps 20 --warmup 3 > gpurun_out/final_batch_pop20_16.log 2>&1; echo p16=$?
timeout 300 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/final_reference.log 2>&1; echo ref=$?
timeout 120 python tools/trd_prof.py 861 325 > gpurun_out/final_trd_prof.log 2>&1; echo prof=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final_launches.csv python bench.py --steps 3 --warmup 3 --no-ttt --no-cpu > gpurun_out/final_ncu_list.log 2>&1; echo list=$?
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_tridiag|k_gather|k_scatter|k_pack" -c 5 -o gpurun_out/final_full python bench.py --steps 1 --warmup 3 --no-ttt --no-cpu > gpurun_out/final_ncu_full.log 2>&1; echo full=$?
timeout 600 ncu --set full --clock-control none -k "regex:k_gemm_f64|k_dc_secular|k_dc_prep" --launch-skip 40 -c 8 -o gpurun_out/final_dc python bench.py --steps 1 --warmup 3 --no-ttt --no-cpu > gpurun_out/final_ncu_dc.log 2>&1; echo dc=$?
timeout 600 ncu --set full --clock-control none -k "regex:k_kinv" -c 1 -o gpurun_out/final_kinv python bench.py --config box24 --steps 1 --warmup 3 --no-ttt --no-cpu > gpurun_out/final_ncu_kinv.log 2>&1; echo kinv=$?
timeout 900 python tools/table1_gpu.py --out gpurun_out/final_table1_gpu.jsonl > gpurun_out/final_table1.log 2>&1; echo table1=$?

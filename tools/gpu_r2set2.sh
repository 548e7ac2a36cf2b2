# round-2 final measurement set (gpurun_out/r2t_*)
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2t_smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/r2t_bench_default.log 2>&1; echo bench=$?
for c in pop6 pop20 lyap10 box24; do timeout 900 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/r2t_cfg_$c.log 2>&1; echo $c=$?; done
timeout 300 python bench.py --batch 8 --steps 10 --warmup 3 > gpurun_out/r2t_batch_pop40_8.log 2>&1; echo b8=$?
timeout 300 python bench.py --config pop20 --batch 16 --steps 20 --warmup 3 > gpurun_out/r2t_batch_pop20_16.log 2>&1; echo p16=$?
timeout 300 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r2t_reference.log 2>&1; echo ref=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2t_launches.csv python bench.py --steps 3 --warmup 3 --no-ttt --no-cpu > gpurun_out/r2t_ncu_list.log 2>&1; echo list=$?

# round-2 final measurement set: GPU tests, default bench (config 4), configs 0-3, batches, reference arm,
# launch list and in-graph kernel times of a warm iteration, ncu --set full of the dominant kernel (k_dgemm)
set -x
python -c "from paper_1708_04174_b200.build import build; build(force=True)" > gpurun_out/build.log 2>&1; echo build=$?
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/f_gputests.log 2>&1; echo tests=$?
tail -3 gpurun_out/f_gputests.log
timeout 900 python bench.py > gpurun_out/f_bench.log 2>&1; echo bench=$?
for c in pop6 pop20 lyap10 box24; do timeout 900 python bench.py --config $c --steps 20 --warmup 5 --no-cpu > gpurun_out/f_cfg_$c.log 2>&1; echo $c=$?; done
timeout 600 python bench.py --config pop40 --batch 8 --steps 10 --warmup 3 > gpurun_out/f_batch_pop40.log 2>&1; echo batch=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/f_reference.log 2>&1; echo ref=$?
timeout 300 python tools/kernel_times.py pop40 20 2000 > gpurun_out/f_kernel_times_2000.log 2>&1
timeout 300 python tools/kernel_times.py pop40 20 4000 > gpurun_out/f_kernel_times_4000.log 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f_launches.csv python tools/warm_launches.py pop40 2000 2 > gpurun_out/f_launches.log 2>&1; echo ncu1=$?
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k "regex:k_dgemm|k_warm_scan|k_warm_E" -c 6 -o gpurun_out/f_full python tools/warm_launches.py pop40 2000 1 > gpurun_out/f_full.log 2>&1; echo ncu2=$?

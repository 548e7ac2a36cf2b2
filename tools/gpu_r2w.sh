# round-2 warm-start measurement set: GPU tests, the default bench line (config 4), configs 0-3, launch list
set -x
python -c "from paper_1708_04174_b200.build import build; build(force=True)" > gpurun_out/build.log 2>&1; echo build=$?
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/w_gputests.log 2>&1; echo tests=$?
tail -3 gpurun_out/w_gputests.log
timeout 900 python bench.py > gpurun_out/w_bench.log 2>&1; echo bench=$?
for c in pop6 pop20 lyap10 box24; do timeout 900 python bench.py --config $c --steps 20 --warmup 5 --no-cpu > gpurun_out/w_cfg_$c.log 2>&1; echo $c=$?; done
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/w_launches.csv python tools/warm_launches.py pop40 2000 2 > gpurun_out/w_launches.log 2>&1; echo ncu=$?

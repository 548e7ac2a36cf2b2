# weighted orthonormality test + unconditional first steps + backoff cap 3: GPU tests, bench lines
set -x
python -c "from paper_1708_04174_b200.build import build; build(force=True)" > gpurun_out/b_build.log 2>&1; echo build=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/b_smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/b_gputests.log 2>&1; echo tests=$?
tail -5 gpurun_out/b_gputests.log
timeout 900 python bench.py > gpurun_out/b_bench.log 2>&1; echo bench=$?
for c in pop6 pop20 lyap10 box24; do timeout 900 python bench.py --config $c --steps 20 --warmup 5 --no-cpu > gpurun_out/b_cfg_$c.log 2>&1; echo $c=$?; done

# dev loop (stops at the first failure; short per-step timeouts so a hang cannot eat the budget)
set -e
python -c "from paper_1708_04174_b200.build import build; build(force=True)" > gpurun_out/build.log 2>&1; echo build=$?
timeout 120 python -m pytest tests/test_gpu_stages.py -q -x > gpurun_out/pytest_stages.log 2>&1; echo stages=$?
timeout 120 python tools/trd_prof.py 861 325 > gpurun_out/trd_prof.log 2>&1; echo prof=$?
timeout 400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 300 python bench.py --steps 20 --warmup 5 --no-ttt --no-cpu > gpurun_out/bench.log 2>&1; echo bench=$?
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-ttt --no-cpu > gpurun_out/ncu.log 2>&1; echo ncu=$?

python -c "from paper_1708_04174_b200.build import build; build(force=True)" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python bench.py --steps 20 --warmup 5 --no-ttt --no-cpu > gpurun_out/bench_w5.log 2>&1; echo bench=$?
timeout 600 python bench.py --steps 20 --warmup 400 --no-ttt --no-cpu > gpurun_out/bench_w400.log 2>&1; echo bench=$?

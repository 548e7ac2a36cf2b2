python -c "from paper_1708_04174_b200.build import build; build(force=True)" > gpurun_out/build.log 2>&1; echo build=$?
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
for c in pop40 lyap10 box24; do timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-ttt --no-cpu > gpurun_out/bench_$c.log 2>&1; echo bench_$c=$?; done

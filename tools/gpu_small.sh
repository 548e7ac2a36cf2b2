# small-block (Jacobi) path: GPU tests + pop6 / box24 benches
set -x
python -c "from paper_1708_04174_b200.build import build; build(force=True)" > gpurun_out/build.log 2>&1; echo build=$?
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
for c in pop6 box24; do timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu > gpurun_out/cfg_$c.log 2>&1; echo $c=$?; done

set -x
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/r2i_pytest_gpu.log 2>&1; echo pytest=$?
for c in pop6 pop20 lyap10 box24 pop40; do timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-ttt --no-cpu > gpurun_out/r2i_cfg_$c.log 2>&1; echo $c=$?; done

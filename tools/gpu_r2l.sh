set -x
timeout 900 python -m pytest tests/test_gpu_stages.py -q -x -k "stedc" > gpurun_out/r2l_stedc.log 2>&1; echo stedc=$?
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/r2l_pytest_gpu.log 2>&1; echo pytest=$?
for c in pop20 lyap10 box24 pop40; do timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-ttt --no-cpu > gpurun_out/r2l_cfg_$c.log 2>&1; echo $c=$?; done

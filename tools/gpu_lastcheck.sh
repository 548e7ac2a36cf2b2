# last sanity pass on the final tree: smoke, the whole GPU suite, the default bench line, the config-0 / config-3
# lines (blocked Jacobi rounds) and the reference arm
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/last_smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/last_pytest_gpu.log 2>&1; echo pytest=$?
timeout 900 python bench.py > gpurun_out/last_bench_default.log 2>&1; echo bench=$?
for c in pop6 box24; do timeout 900 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/last_cfg_$c.log 2>&1; echo $c=$?; done
timeout 300 python tools/kernel_times.py pop6 50 30 > gpurun_out/last_kernel_times_pop6.txt 2>&1; echo kt6=$?
timeout 300 python tools/sanitize.py 30 > gpurun_out/last_allpaths.log 2>&1; echo allpaths=$?
timeout 300 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/last_reference.log 2>&1; echo ref=$?

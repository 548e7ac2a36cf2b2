# refresh after the Jacobi changes: checks, configs 0-3, full-size convergence parity
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/v11_smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/v11_pytest_gpu.log 2>&1; echo pytest=$?
for c in pop6 pop20 lyap10 box24; do timeout 900 python bench.py --config $c --steps 20 --warmup 5 --no-cpu > gpurun_out/v11_cfg_$c.log 2>&1; echo $c=$?; done
timeout 900 python tools/table1_gpu.py --out gpurun_out/v11_table1_gpu.jsonl > gpurun_out/v11_table1.log 2>&1; echo table1=$?
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/v11_smi.log 2>&1

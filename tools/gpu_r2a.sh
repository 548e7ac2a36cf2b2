# round 2, first GPU check: the new parity tests (DUAL_INFEASIBLE, per-component, NaN), smoke, FP64 probe
set -x
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/probe_fp64 tools/probe_fp64.cu > gpurun_out/r2a_probe_build.log 2>&1 && timeout 120 /tmp/probe_fp64 > gpurun_out/r2a_probe_fp64.log 2>&1; echo probe=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2a_smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/r2a_pytest_gpu.log 2>&1; echo pytest=$?

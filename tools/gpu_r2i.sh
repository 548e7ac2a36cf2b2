# early predictor branch: A/B of the in-graph span, then the tests that exercise the warm path
set -x
for e in 1 0; do SOSADMM_EARLY_PRED=$e timeout 300 python tools/kernel_times.py pop40 20 2000 > gpurun_out/r2i_kt_pop40_e$e.txt 2>&1; echo kt$e=$?; done
for e in 1 0; do SOSADMM_EARLY_PRED=$e timeout 300 python tools/kernel_times.py pop20 50 1000 > gpurun_out/r2i_kt_pop20_e$e.txt 2>&1; echo kt20$e=$?; done
timeout 1200 python -m pytest tests/test_gpu_warm.py tests/test_gpu_parity.py tests/test_gpu_convergence.py tests/test_gpu_batch.py tests/test_gpu_sharded.py -x -q > gpurun_out/r2i_pytest.log 2>&1; echo pytest=$?
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu > gpurun_out/r2i_cfg_pop40.log 2>&1; echo pop40=$?
for c in pop20 lyap10 box24; do timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu > gpurun_out/r2i_cfg_$c.log 2>&1; echo $c=$?; done

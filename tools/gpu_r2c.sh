# second-order predictor A/B
set -x
python -c "from paper_1708_04174_b200.build import build; build(force=True)" > gpurun_out/c_build.log 2>&1; echo build=$?
SOSADMM_WARM_PRED=2 timeout 600 python tools/warm_trace.py pop40 8500 500 0 > gpurun_out/c_trace40_p2.log 2>&1; echo trace=$?
for pr in 1 2; do for k in 1000 2000 5000 7000; do TAG=p$pr SOSADMM_WARM_PRED=$pr timeout 300 python tools/span.py pop40 $k 100 2 >> gpurun_out/c_span.log 2>&1; done; done
for pr in 1 2; do for k in 300 1000; do TAG=p$pr SOSADMM_WARM_PRED=$pr timeout 300 python tools/span.py pop20 $k 100 2 >> gpurun_out/c_span.log 2>&1; done; done
for pr in 1 2; do for k in 300 1000; do TAG=p$pr SOSADMM_WARM_PRED=$pr timeout 300 python tools/span.py box24 $k 100 2 >> gpurun_out/c_span.log 2>&1; done; done
SOSADMM_WARM_PRED=2 timeout 900 python -m pytest tests/test_gpu_warm.py -q -x > gpurun_out/c_warmtests.log 2>&1; echo wt=$?
tail -3 gpurun_out/c_warmtests.log

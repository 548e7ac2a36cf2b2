set -x
python -c "from paper_1708_04174_b200.build import build; build(force=True)" > gpurun_out/a_build.log 2>&1; echo build=$?
timeout 600 python tools/warm_trace.py pop40 8500 500 0 > gpurun_out/a_trace40.log 2>&1; echo trace=$?
for w in 1 0; do for k in 1000 2000 5000 7000; do TAG=w$w SOSADMM_WARM_WTEST=$w timeout 300 python tools/span.py pop40 $k 100 2 >> gpurun_out/a_span.log 2>&1; done; done
timeout 900 python -m pytest tests/test_gpu_warm.py -q -x > gpurun_out/a_warmtests.log 2>&1; echo wt=$?
tail -3 gpurun_out/a_warmtests.log
cat gpurun_out/a_span.log

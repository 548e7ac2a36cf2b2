set -x
python -c "from paper_1708_04174_b200.build import build; build(force=True)" > gpurun_out/z_build.log 2>&1; echo build=$?
timeout 600 python tools/warm_trace.py pop40 8500 500 0 > gpurun_out/z_trace40.log 2>&1; echo trace=$?
for u in 0 3; do TAG=unc$u SOSADMM_WARM_UNCOND=$u timeout 300 python tools/span.py pop40 2000 200 3 >> gpurun_out/z_span.log 2>&1; done
TAG=unc3 SOSADMM_WARM_UNCOND=3 timeout 300 python tools/span.py pop40 7000 200 3 >> gpurun_out/z_span.log 2>&1
for b in 6 3 1 0; do TAG=bo$b SOSADMM_WARM_BACKOFF=$b timeout 300 python tools/span.py pop40 0 300 1 >> gpurun_out/z_span.log 2>&1; done
timeout 900 python -m pytest tests/test_gpu_warm.py -q -x > gpurun_out/z_warmtests.log 2>&1; echo wt=$?
tail -3 gpurun_out/z_warmtests.log
cat gpurun_out/z_span.log

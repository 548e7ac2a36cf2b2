set -x
python -c "from paper_1708_04174_b200.build import build; build(force=True)" > gpurun_out/y_build.log 2>&1; echo build=$?
timeout 600 python tools/warm_trace.py pop40 8500 500 200 > gpurun_out/y_trace40.log 2>&1; echo trace=$?
timeout 300 python tools/warm_trace.py pop20 1500 250 100 > gpurun_out/y_trace20.log 2>&1; echo trace20=$?
timeout 300 python tools/warm_trace.py box24 1300 250 100 > gpurun_out/y_trace24.log 2>&1; echo trace24=$?

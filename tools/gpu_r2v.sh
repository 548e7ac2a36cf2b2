# re-entry verification: build, smoke, GPU tests, default bench line
set -x
python -c "from paper_1708_04174_b200.build import build; build(force=True)" > gpurun_out/v_build.log 2>&1; echo build=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v_smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/v_gputests.log 2>&1; echo tests=$?
tail -3 gpurun_out/v_gputests.log
timeout 900 python bench.py > gpurun_out/v_bench.log 2>&1; echo bench=$?
tail -1 gpurun_out/v_bench.log | cut -c1-600

set -x
python -c "from paper_1708_04174_b200.build import build; build(force=True)" > gpurun_out/build.log 2>&1; echo build=$?
timeout 300 python tools/eigh_lib.py > gpurun_out/eigh_lib.log 2>&1; echo eighlib=$?
timeout 120 python tools/trd_prof.py 861 325 > gpurun_out/trd_prof.log 2>&1; echo prof=$?

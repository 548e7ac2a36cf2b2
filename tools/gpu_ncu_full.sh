# one ncu --set full capture of the named kernels (regex in $1), from a short bench run
set -x
python -c "from paper_1708_04174_b200.build import build; build(force=True)" > gpurun_out/build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$1" -c ${2:-2} -o gpurun_out/full python bench.py --steps 1 --warmup 3 --no-ttt --no-cpu > gpurun_out/ncu_full.log 2>&1; echo ncu=$?

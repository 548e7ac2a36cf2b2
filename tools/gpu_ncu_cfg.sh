# one ncu --set full capture of kernel regex $1 on config $2 (launch-skip $3)
python -c "from paper_1708_04174_b200.build import build; build(force=True)" > gpurun_out/build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$1" --launch-skip ${3:-0} -c 1 -o gpurun_out/one python bench.py --config $2 --steps 1 --warmup 3 --no-ttt --no-cpu > gpurun_out/ncu_one.log 2>&1; echo ncu=$?

python -c "from paper_1708_04174_b200.build import build; build(force=True)" > gpurun_out/build.log 2>&1; echo build=$?
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
for c in box24 lyap10; do timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-ttt --no-cpu > gpurun_out/b_$c.log 2>&1; echo $c=$?; done
timeout 600 ncu --set full --clock-control none -k "regex:k_kinv" -c 2 -o gpurun_out/kinv2 python bench.py --config box24 --steps 1 --warmup 3 --no-ttt --no-cpu > gpurun_out/ncu_kinv.log 2>&1; echo ncu=$?

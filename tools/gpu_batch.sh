# f1 batch: GPU tests for the batch path, then aggregate throughput for B = 1, 2, 4, 8 (config 4) and pop20
set -x
python -c "from paper_1708_04174_b200.build import build; build(force=True)" > gpurun_out/build.log 2>&1; echo build=$?
timeout 600 python -m pytest tests/test_gpu_batch.py -x -q > gpurun_out/pytest_batch.log 2>&1; echo pytest=$?
for B in 2 4 8; do timeout 300 python bench.py --batch $B --steps 10 --warmup 3 > gpurun_out/batch_pop40_$B.log 2>&1; echo b$B=$?; done
for B in 2 8 16; do timeout 300 python bench.py --config pop20 --batch $B --steps 20 --warmup 3 > gpurun_out/batch_pop20_$B.log 2>&1; echo p$B=$?; done
timeout 300 python bench.py --config pop20 --steps 20 --warmup 3 --no-ttt --no-cpu > gpurun_out/batch_pop20_1.log 2>&1; echo p1=$?

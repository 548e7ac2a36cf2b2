# every BASELINE config through bench.py (1 GPU, time-to-1e-4 included), plus the dense K^-1 apply of
# config 3 (box24) under ncu for its DRAM bytes / bandwidth
set -x
python -c "from paper_1708_04174_b200.build import build; build(force=True)" > gpurun_out/build.log 2>&1; echo build=$?
for c in pop6 pop20 lyap10 box24; do timeout 900 python bench.py --config $c --steps 20 --warmup 5 --no-cpu > gpurun_out/cfg_$c.log 2>&1; echo $c=$?; done
timeout 600 ncu --set full --clock-control none -k "regex:k_kinv|k_gather|k_scatter" -c 3 -o gpurun_out/box24_aff python bench.py --config box24 --steps 1 --warmup 3 --no-ttt --no-cpu > gpurun_out/ncu_box24.log 2>&1; echo ncu=$?

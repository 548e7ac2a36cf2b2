# cluster size sweep for the mid-size blocks (tridiag phase of pop20 / lyap10 / box24)
python -c "from paper_1708_04174_b200.build import build; build(force=True)" > gpurun_out/build.log 2>&1
for C in 4 8 16; do for c in pop20 box24; do SOSADMM_TRD_C=$C timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-ttt --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C=$C', '$c', round(d['value'],1), d['phase_ms_per_iter']['tridiag'])"; done; done

#!/bin/bash
# full GPU tests + in-graph kernel times + bench lines for configs 1-4
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
for c in pop20 lyap10 box24 pop40; do timeout 200 python tools/kernel_times.py $c 50 200 2>&1 | grep -v -i warn | head -8; done
for C in pop20 lyap10 box24 pop40; do
  timeout 300 python bench.py --config $C --steps 300 --warmup 5 --no-ttt --no-cpu > gpurun_out/r2p_${C}.json 2> gpurun_out/r2p_${C}.err
  python - "$C" <<'PY'
import json,sys
d=json.loads(open(f"gpurun_out/r2p_{sys.argv[1]}.json").read().strip().splitlines()[-1])
ph=d.get("phase_ms_per_iter") or {}
print(sys.argv[1], round(d["value"],2), d.get("clocks",{}).get("sm_mhz"), {k: round(v,4) for k,v in ph.items()})
PY
done

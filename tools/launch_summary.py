"""Per-kernel summary of an ncu --metrics gpu__time_duration.sum --csv launch list (one warm iteration's
kernels are the active launches; gated-off launches are the ~3-4 us early exits).
usage: python tools/launch_summary.py launches.csv [iterations]"""
import collections
import csv
import io
import sys

txt = open(sys.argv[1]).read()
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 1
rows = list(csv.reader(io.StringIO(txt[txt.find('"ID"'):])))
h = rows[0]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
tot, cnt = collections.defaultdict(float), collections.Counter()
for r in rows[1:]:
    if len(r) <= vi:
        continue
    v = float(r[vi].replace(",", ""))
    us = v / 1000 if r[ui] in ("ns", "nsecond") else (v if r[ui] in ("us", "usecond") else v * 1000)
    n = r[ki].split("(")[0].replace("void ", "")
    tot[n] += us
    cnt[n] += 1
T = sum(tot.values())
print(f"{sum(cnt.values())} launches, {T / iters:.1f} us per iteration (serialised, cold cache)")
for n in sorted(tot, key=lambda x: -tot[x]):
    print(f"{n[:56]:56s} {cnt[n]:4d} x {tot[n] / cnt[n]:8.2f} us = {tot[n] / iters:8.1f} us/iter ({100 * tot[n] / T:.1f}%)")

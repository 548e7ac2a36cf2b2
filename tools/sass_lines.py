"""Attribute ncu SASS-level stall samples / executed instructions of one kernel to CUDA source lines.
usage: python tools/sass_lines.py <report.ncu-rep> <mangled kernel name> [top]"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

rep, fn = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
so = os.path.join(os.path.dirname(__file__), "..", "paper_1708_04174_b200", "libsosadmm.so")
with tempfile.TemporaryDirectory() as d:
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=d, capture_output=True)
    cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
    dis = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cub)], capture_output=True, text=True).stdout
sec, cur, offs = False, None, {}
for l in dis.splitlines():
    if l.startswith("//---") and ".text." in l:
        sec = (".text." + fn + " ") in (l + " ")
        continue
    if not sec:
        continue
    if "//##" in l:
        m = re.search(r'File "([^"]+)", line (\d+)', l)
        if m:
            cur = (os.path.basename(m.group(1)), int(m.group(2)))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
    if m and cur:
        offs[int(m.group(1), 16)] = cur
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout  # the report holds one kernel
r = list(csv.reader(io.StringIO(out)))
h = r[1]
rows = [dict(zip(h, x)) for x in r[2:] if len(x) >= len(h) - 1]


def f(x):
    try:
        return float(x.replace(",", ""))
    except Exception:
        return 0.0


base = min(int(d["Address"], 16) for d in rows)
agg, ins = collections.Counter(), collections.Counter()
for d in rows:
    key = offs.get(int(d["Address"], 16) - base, ("?", 0))
    agg[key] += f(d["Warp Stall Sampling (All Samples)"])
    ins[key] += f(d["Instructions Executed"])
tot, toti = sum(agg.values()), sum(ins.values())
srcs = {}
print(f"samples {tot:.0f}, warp instructions {toti / 1e6:.1f}M")
for key, s in agg.most_common(top):
    fpath = os.path.join(os.path.dirname(__file__), "..", "paper_1708_04174_b200", "csrc", key[0])
    if key[0] not in srcs:
        srcs[key[0]] = open(fpath).read().splitlines() if os.path.exists(fpath) else []
    txt = srcs[key[0]][key[1] - 1].strip()[:72] if key[1] <= len(srcs[key[0]]) and key[1] > 0 else ""
    print(f"{100 * s / tot:5.1f}% {100 * ins[key] / toti:5.1f}%i {key[0]}:{key[1]} {txt}")

"""Attribute shared-memory wavefronts (total / excessive) of one kernel in an ncu report to source lines.
usage: python tools/smem_lines.py <report.ncu-rep> <kernel regex> <mangled name> [top]"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

rep, kre, fn = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 20
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
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", "regex:" + kre],
                     capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
# one section per kernel launch: ["Kernel Name", name], header, rows...; keep the first matching one
rows, h, take = [], None, False
for x in r:
    if x and x[0] == "Kernel Name":
        if rows:
            break
        take = re.search(kre, x[1]) is not None
        h = None
        continue
    if not take:
        continue
    if h is None:
        h = x
        continue
    if len(x) >= len(h) - 1:
        rows.append(dict(zip(h, x)))


def f(x):
    try:
        return float(x.replace(",", ""))
    except Exception:
        return 0.0


base = min(int(d["Address"], 16) for d in rows)
wf, ex = collections.Counter(), collections.Counter()
for d in rows:
    key = offs.get(int(d["Address"], 16) - base, ("?", 0))
    wf[key] += f(d["L1 Wavefronts Shared"])
    ex[key] += f(d["L1 Wavefronts Shared Excessive"])
tw, te = sum(wf.values()), sum(ex.values())
print(f"shared wavefronts {tw / 1e6:.2f}M, excessive {te / 1e6:.2f}M")
src = {}
for key, v in wf.most_common(top):
    p = os.path.join(os.path.dirname(__file__), "..", "paper_1708_04174_b200", "csrc", key[0])
    if key[0] not in src:
        src[key[0]] = open(p).read().splitlines() if os.path.exists(p) else []
    t = src[key[0]][key[1] - 1].strip()[:70] if 0 < key[1] <= len(src[key[0]]) else ""
    print(f"{100 * v / tw:5.1f}% wf  {100 * ex[key] / max(te, 1):5.1f}% excess  {key[0]}:{key[1]} {t}")

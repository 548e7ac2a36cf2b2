"""Summarise an `ncu --set full` report: per kernel launch the duration, DRAM traffic, issue activity,
FP64 / DMMA pipe utilisation and the top warp-stall reasons; optionally write the per-kernel DRAM
traffic JSON that bench.py folds into its roofline lines.

usage: python tools/ncu_summary.py <report.ncu-rep> [--traffic-json out.json] [--source "..."]
"""
import argparse
import csv
import io
import json
import subprocess

ap = argparse.ArgumentParser()
ap.add_argument("rep")
ap.add_argument("--traffic-json")
ap.add_argument("--source", default="")
args = ap.parse_args()

out = subprocess.run(["ncu", "-i", args.rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
head, units = rows[0], rows[1]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "nsecond": 1e-6, "us": 1e-3,
         "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3}


def val(d, u, key):
    x = d.get(key, "")
    try:
        v = float(x.replace(",", ""))
    except ValueError:
        return None
    return v * SCALE.get(u.get(key, ""), 1.0)


STALL = "smsp__pcsamp_warps_issue_stalled_"
traffic = {}
for r in rows[2:]:
    d, u = dict(zip(head, r)), dict(zip(head, units))
    name = d["Kernel Name"].split("(")[0].replace("void ", "")
    ms = val(d, u, "gpu__time_duration.sum")
    rd = val(d, u, "dram__bytes_read.sum") or 0.0
    wr = val(d, u, "dram__bytes_write.sum") or 0.0
    ipc = val(d, u, "sm__inst_executed.avg.per_cycle_active")
    fp64 = val(d, u, "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active")
    dmma = val(d, u, "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active")
    fp64rt = val(d, u, "TPC.TriageCompute.sm__pipe_fp64_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed")
    st = {k[len(STALL):]: val(d, u, k) or 0.0 for k in head if k.startswith(STALL) and not k.endswith("not_issued")}
    tot = sum(st.values()) or 1.0
    top = sorted(st.items(), key=lambda kv: -kv[1])[:5]
    print(f"{name[:40]:40s} {ms:9.4f} ms  DRAM rd {rd / 1e6:8.3f} MB wr {wr / 1e6:8.3f} MB  IPC {ipc}  "
          f"fp64 pipe {fp64}%  dmma {dmma}%  fp64 active(rt) {fp64rt}%")
    print("    stalls: " + ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in top))
    traffic.setdefault(name, {"dram_read_bytes": rd, "dram_write_bytes": wr, "ms": ms})
if args.traffic_json:
    json.dump({"source": args.source, "kernels": traffic}, open(args.traffic_json, "w"), indent=1)

"""Summarise an ncu report: per-kernel headline metrics and per-source-line stall samples."""
import csv, collections, subprocess, sys, io

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
want = {"Duration", "Registers Per Thread", "Achieved Occupancy", "Executed Ipc Active", "DRAM Throughput",
        "L2 Cache Throughput", "Issue Slots Busy", "Warp Cycles Per Issued Instruction", "Grid Size", "Block Size",
        "Dynamic Shared Memory Per Block", "L1/TEX Hit Rate", "L2 Hit Rate", "Memory Throughput"}
rows = list(csv.reader(io.StringIO(det)))
hdr = rows[0]
for r in rows[1:]:
    d = dict(zip(hdr, r))
    if d.get("Metric Name") in want:
        print(d["ID"], d["Kernel Name"][:40], d["Metric Name"], d["Metric Value"], d["Metric Unit"])
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
agg = collections.defaultdict(lambda: [0, 0, ""])
cur = None
hdr = None
def num(x):
    try:
        return int(x)
    except ValueError:
        return 0
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]; continue
    if r[0] == "Line No":
        hdr = r; continue
    if hdr is None or len(r) < 8:
        continue
    try:
        ln = int(r[0])
    except ValueError:
        continue
    agg[(cur, ln)][0] += num(r[4]); agg[(cur, ln)][1] += num(r[7]); agg[(cur, ln)][2] = r[1][:110]
ts = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
print("samples", ts, "warp-instructions", ti)
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{k[0][:18]:18s}{k[1]:5d} samp {100*v[0]/ts:5.1f}% inst {100*v[1]/ti:5.1f}%  {v[2]}")

"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel.

    python tools/summarize_launches.py gpurun_out/launches.csv [skip_launches]
Per-launch times are cold-cache and serialised (ncu); compare SHARES, not absolutes.
"""
import collections
import csv
import sys


def main():
    path = sys.argv[1]
    skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    lines = [ln for ln in open(path) if ln.startswith('"')]
    rows = list(csv.reader(lines))
    hdr = rows[0]
    ki, vi, ui, ii = (hdr.index(k) for k in ("Kernel Name", "Metric Value", "Metric Unit", "ID"))
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    agg = collections.defaultdict(lambda: [0, 0.0])
    tot = 0.0
    for r in rows[1:]:
        if int(r[ii]) < skip:
            continue
        us = float(r[vi].replace(",", "")) * scale[r[ui]]
        name = r[ki].split("(")[0].strip()
        agg[name][0] += 1
        agg[name][1] += us
        tot += us
    print(f"{'kernel':44s} {'launches':>8s} {'total us':>10s} {'avg us':>9s} {'share':>6s}")
    for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k[:44]:44s} {n:8d} {us:10.1f} {us / n:9.1f} {100 * us / tot:5.1f}%")


if __name__ == "__main__":
    main()

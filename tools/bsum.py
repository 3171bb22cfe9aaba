#!/usr/bin/env python
"""Summarise bench.py JSON lines from stdin: label, ms/step, per-kernel solve time and GB/s."""
import json
import sys

label = sys.argv[1] if len(sys.argv) > 1 else ""
for line in sys.stdin:
    line = line.strip()
    if not line.startswith("{"):
        continue
    d = json.loads(line)
    ks = d.get("kernels", {})
    parts = [f"{k}: {v['avg_ms_per_solve']*1e3:.1f}us x{v['avg_iterations']:.1f}it {v['achieved_gbs']:.0f}GB/s"
             for k, v in ks.items()]
    print(label, f"{d.get('ms_per_step', 0):.3f} ms/step", f"value {d.get('value', 0):.3e}", "|", "; ".join(parts))

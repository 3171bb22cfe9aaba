#!/usr/bin/env python
"""Per-CTA phase stamps of iteration 3 of the streaming CG loop kernels (k_s_cg / k_t_cg).

    TLGPU_PROF=1 [TLGPU_TILED_MIN=1 ...] python tools/sweep_profile.py cfg4 local

Stamps (slot 1024 + 16 CTA + e, %globaltimer ns): 0 sweep A start, 1 first stage landed
(k_t_cg), 2 sweep A done, 3 past the grid barrier, 4 alpha known, 5 first stage of sweep B
landed (k_t_cg), 6 sweep B done, 7 past the grid barrier, 8 sums known.
"""
import ctypes as C
import os
import subprocess
import sys
from pathlib import Path

os.environ.setdefault("TLGPU_PROF", "1")
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402

sys.argv = [sys.argv[0], *sys.argv[1:3], "3"]
exec(open(ROOT / "tools" / "solve_tune.py").read())   # runs the solves, prints the timing line
from paper_2110_12932_b200 import _native as N  # noqa: E402

buf = (C.c_uint64 * 8192)()
cnt = C.c_int32()
N.check(N.lib().tl_debug_profile(buf, 8192, C.byref(cnt)))
raw = np.array(buf[:cnt.value], dtype=np.float64)[1024:].reshape(-1, 16)
ok = raw[:, 0] > 0
S = raw[ok]
t0 = S[:, 0].min()
names = {0: "A start", 1: "A first stage", 2: "A done", 3: "A barrier passed", 4: "alpha known",
         5: "B first stage", 6: "B done", 7: "B barrier passed", 8: "sums known"}
print(f"{ok.sum()} CTAs; times in us from the earliest sweep-A start")
for e, nm in names.items():
    v = S[:, e]
    v = v[v > 0]
    if v.size:
        v = (v - t0) / 1e3
        print(f"  {nm:18s} min {v.min():8.2f}  median {np.median(v):8.2f}  max {v.max():8.2f}")

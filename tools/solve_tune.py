#!/usr/bin/env python
"""Device time of one implicit solve on a BASELINE grid (tl_step_host, CUDA events around
the solve launches) for solver tuning; the TLGPU_* switches are read from the environment.

    python tools/solve_tune.py cfg4 local [repeats]

Prints one JSON line: median ms, iterations, algorithmic TB/s = N (64 k + 32) / t.
"""
import ctypes as C
import json
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2110_12932_b200 as P  # noqa: E402
from paper_2110_12932_b200 import _native as N, ops  # noqa: E402

cfgname, level = sys.argv[1], sys.argv[2]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
cfg = P.load_config(ROOT / "configs" / f"{cfgname}.cfg")
problem, lm = P.build_problem(cfg)
rng = np.random.default_rng(0)
if level == "global":
    grid = problem.global_mesh
    T = rng.uniform(293.0, 2293.0, grid.n_nodes)
    pts, pw = problem.global_source(0.0, cfg.dt_macro)
    load = ops.deposit_load(grid, pts, pw)
    run = lambda: ops.step(grid, 9.8, 8440 * 410.0, cfg.dt_macro, N.TL_DIRICHLET_BOTTOM, T,  # noqa: E731
                           g_const=293.0, load=load, rtol=1e-12)
else:
    grid = lm
    # a smooth hot spot under the beam (iteration counts like a real micro step)
    X = lm.coords
    c = np.asarray(problem.local_source(2e-6).center)
    T = 293.0 + 1500.0 * np.exp(-(((X - c) / np.array([1e-4, 1e-4, 5e-5])) ** 2).sum(axis=1))
    g = np.where(lm.gamma_mask(), 293.0, 0.0)
    src = problem.local_source(2e-6)
    run = lambda: ops.step(lm, 9.8, 8440 * 410.0, cfg.dt_macro / cfg.micro_steps,  # noqa: E731
                           N.TL_DIRICHLET_GAMMA, T, g=g, gaussian=src.device_args(), rtol=1e-12)
ms, its = [], None
for r in range(reps):
    x, info = run()
    f = C.c_float()
    N.check(N.lib().tl_step_last_ms(C.byref(f)), "ms")
    ms.append(f.value)
    its = info.iterations
    assert info.status == 0, info.status
n = grid.n_nodes
t = float(np.median(ms[1:] if len(ms) > 1 else ms))
env = {k: v for k, v in os.environ.items() if k.startswith("TLGPU_")}
print(json.dumps({"cfg": cfgname, "level": level, "n": n, "env": env, "ms": t, "all_ms": ms, "its": its,
                  "alg_tbs": n * (64 * its + 32) / (t / 1e3) / 1e12, "sum": float(x.sum())}), flush=True)

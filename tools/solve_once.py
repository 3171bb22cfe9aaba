#!/usr/bin/env python
"""One (or a few) device solves of a BASELINE grid through ops.step, for ncu captures.

    python tools/solve_once.py cfg3 global [repeats]
    python tools/solve_once.py cfg3 local  [repeats] [save.npy]
"""
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2110_12932_b200 as P  # noqa: E402
from paper_2110_12932_b200 import _native as N, ops  # noqa: E402

cfgname, level = sys.argv[1], sys.argv[2]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
cfg = P.load_config(ROOT / "configs" / f"{cfgname}.cfg")
problem, lm = P.build_problem(cfg)
rng = np.random.default_rng(0)
for r in range(reps):
    t = time.time()
    if level == "global":
        grid = problem.global_mesh
        T = rng.uniform(293.0, 2293.0, grid.n_nodes)
        pts, pw = problem.global_source(0.0, cfg.dt_macro)
        load = ops.deposit_load(grid, pts, pw)
        x, info = ops.step(grid, 9.8, 8440 * 410.0, cfg.dt_macro, N.TL_DIRICHLET_BOTTOM, T, g_const=293.0,
                           load=load, rtol=1e-12)
    else:
        T = rng.uniform(293.0, 2293.0, lm.n_nodes)
        g = np.where(lm.gamma_mask(), rng.uniform(293.0, 900.0, lm.n_nodes), 0.0)
        src = problem.local_source(2e-6)
        dt = cfg.dt_macro / cfg.micro_steps
        x, info = ops.step(lm, 9.8, 8440 * 410.0, dt, N.TL_DIRICHLET_GAMMA, T, g=g,
                           gaussian=src.device_args(), rtol=1e-12)
    if len(sys.argv) > 4 and r == reps - 1:
        np.save(sys.argv[4], x)
    print(f"{cfgname} {level} rep {r}: status {info.status} its {info.iterations} "
          f"true_resid {info.true_resid:.3e} wall {time.time() - t:.2f}s")

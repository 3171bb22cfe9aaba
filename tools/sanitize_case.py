#!/usr/bin/env python
"""One small (config-1-sized) run of one device code path, for compute-sanitizer.

    python tools/sanitize_case.py resident|exact|tiled|flat|vc|twoway|slab

The switches that select a path are environment variables read once per process
(DESIGN.md §4), so each path is its own process:
  resident  default: multi-solve CG-CG resident kernel (local), resident global solve,
            Gaussian precompute, interpolation, deposit
  exact     TLGPU_EXACT_CG=1: the two-barrier resident kernel
  tiled     TLGPU_STREAMING=1 TLGPU_TILED_MIN=1: k_s_rhs -> k_t_cg -> k_s_resid -> k_s_final
  flat      TLGPU_STREAMING=1 TLGPU_TILED=0: k_s_rhs -> k_s_cg -> k_s_resid -> k_s_final
  vc        temperature-dependent Picard passes (k_vc_tets / k_vc_assemble / k_vc_cg)
  twoway    two-way coupling: transmission load (sort + segment sums) + step solves
  slab      the z-slab global solve kernels on one rank
"""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
ENV = {"exact": {"TLGPU_EXACT_CG": "1"},
       "tiled": {"TLGPU_STREAMING": "1", "TLGPU_TILED_MIN": "1"},
       "flat": {"TLGPU_STREAMING": "1", "TLGPU_TILED": "0"}}
case = sys.argv[1]
os.environ.update(ENV.get(case, {}))
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

import paper_2110_12932_b200 as P  # noqa: E402

C = ROOT / "configs"
if case in ("resident", "exact", "tiled", "flat"):
    cfg = P.load_config(C / "cfg1_m4.cfg")
    cfg.t_end = 2 * cfg.dt_macro
    state, stats = P.two_level_run(cfg)
    print(case, stats.counters, float(state.local_field.values.max()))
elif case == "vc":
    cfg = P.load_config(C / "cfg1_tdep.cfg")
    cfg.t_end = cfg.dt_macro
    state, stats = P.two_level_run(cfg)
    print(case, stats.counters, float(state.local_field.values.max()))
elif case == "twoway":
    cfg = P.load_config(C / "cfg1_twoway.cfg")
    cfg.t_end = cfg.dt_macro
    state, stats = P.two_level_run(cfg)
    print(case, stats.counters, float(state.local_field.values.max()))
elif case == "slab":
    import torch
    from paper_2110_12932_b200 import ops
    from paper_2110_12932_b200 import slab as SL
    cfg = P.load_config(C / "cfg1_m4.cfg")
    problem, _ = P.build_problem(cfg)
    grid = problem.global_mesh
    T = np.random.default_rng(0).uniform(293.0, 2293.0, grid.n_nodes)
    pts, pw = problem.global_source(0.0, cfg.dt_macro)
    S = SL.SlabGlobalSolver(grid, 9.8, 8440 * 410.0, rank=0, world=1, device="cuda:0", rtol=1e-12)
    S.set_own(S.x, T)
    S.set_own(S.load, ops.deposit_load(grid, pts, pw))
    info = S.step(cfg.dt_macro, 293.0, with_load=True)
    torch.cuda.synchronize()
    print(case, info)
else:
    raise SystemExit(f"unknown case {case}")

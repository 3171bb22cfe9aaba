#!/usr/bin/env python
"""cProfile of one public run_spacetime(recorder=None) call (the bench's e2e leg) on a config.

    python tools/e2e_profile.py cfg4 20
"""
import cProfile
import pstats
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2110_12932_b200 as P  # noqa: E402
from paper_2110_12932_b200 import multirate as MR  # noqa: E402

name, K = sys.argv[1], int(sys.argv[2])
cfg = P.load_config(ROOT / "configs" / f"{name}.cfg")
problem, lmesh = P.build_problem(cfg)
T0 = P.uniform_field(problem.global_mesh, cfg.T_initial)
warm = MR.MacroSchedule(cfg.dt_macro, cfg.micro_steps, 0.0, 3 * cfg.dt_macro)
P.run_spacetime(problem, warm, lmesh, T0, path=cfg.path, policy=cfg.policy)
sched = MR.MacroSchedule(cfg.dt_macro, cfg.micro_steps, 0.0, K * cfg.dt_macro)
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
state = P.run_spacetime(problem, sched, lmesh, T0, path=cfg.path, policy=cfg.policy, recorder=None)
lv = state.local_field.values
pr.disable()
print(f"{name}: {K} steps, {time.perf_counter() - t0:.4f} s")
pstats.Stats(pr).sort_stats("cumulative").print_stats(28)

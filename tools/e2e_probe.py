#!/usr/bin/env python
"""Host wall time per macro step through DeviceRun for three read-back modes (cfg2)."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2110_12932_b200 as P  # noqa: E402
from paper_2110_12932_b200.schedule import plan_spacetime  # noqa: E402

cfg = P.load_config(ROOT / "configs" / "cfg2.cfg")
problem, lm = P.build_problem(cfg)
sched = P.MacroSchedule(cfg.dt_macro, cfg.micro_steps, 0.0, cfg.t_end)
plans, placement, tg, tl = [], lm.placement, 0.0, 0.0
for k in range(28):
    pl = plan_spacetime(problem, sched, placement, cfg.path, cfg.policy, tg, tl, k0=k, nsteps=1)
    plans.append(pl)
    placement, tg, tl = pl.final_placement, pl.final_t_global, pl.final_t_local
pins = [torch.empty(lm.n_nodes, dtype=torch.float64, pin_memory=True).numpy() for _ in range(2)]
for mode in ("none", "sync", "async", "none", "sync", "async"):
    run = P.DeviceRun(problem, lm)
    run.initial(P.uniform_field(problem.global_mesh, 293.0))
    for k in range(4):
        run.run(plans[k])
    run.sync()
    t0 = time.perf_counter()
    tr = 0.0
    for s, pl in enumerate(plans[4:]):
        a = time.perf_counter()
        run.run(pl)
        tr += time.perf_counter() - a
        if mode == "sync":
            run.field(1, out=pins[0])
        elif mode == "async":
            run.field_async(1, pins[s % 2], slot=s % 2)
            if s >= 1:
                run.field_wait((s - 1) % 2)
    if mode == "async":
        run.field_wait((len(plans) - 5) % 2)
    run.sync()
    dt = (time.perf_counter() - t0) / (len(plans) - 4)
    print(f"{mode:6s} {dt * 1e3:.3f} ms/step  (host time in run(): {tr / (len(plans) - 4) * 1e3:.3f} ms)")
    run.close()

#!/usr/bin/env python
"""SURVEY §8(d) CPU-baseline plan, run with the UNMODIFIED reference (imported from
/root/reference, so only in the build container; the GPU box has no copy):

  cfg1  run_spacetime over all 80 macro steps (m = 4) and run_space over all 80 uniform steps
  cfg2  run_spacetime over the first 20 macro steps, then DOF-timesteps/s extrapolates
        (the reference's cost per step is flat after the relocation warm-up)
  cfg3  infeasible here (its global mesh alone needs 55.8 GB)
  cfg4  infeasible
  cfg5  one process per host core, each running one seed-0 scenario for 10 macro steps

recorder=None, OPENBLAS_NUM_THREADS=1 (one core per run; scipy's sparse CG is single-
threaded).  Writes one JSON document (default profiles/r02_cpu_baseline_reference.json).

    python tools/cpu_baseline_reference.py [--only cfg1,cfg2,cfg5] [--procs N] [--out FILE]
"""
import argparse
import json
import multiprocessing as mp
import os
import platform
import subprocess
import sys
import time
from pathlib import Path

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("OMP_NUM_THREADS", "1")
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(ROOT))


def _ref():
    from lpbfsim import fem, multirate, runner
    from lpbfsim.config import load_config
    from lpbfsim.stats import RunStats
    return fem, multirate, runner, load_config, RunStats


def run_config(cfg, n_steps, spacetime=True):
    fem, multirate, runner, _, RunStats = _ref()
    cfg.t_end = n_steps * cfg.dt_macro if spacetime else cfg.t_end
    problem, lm = runner.build_problem(cfg)
    T0 = fem.uniform_field(problem.global_mesh, cfg.T_initial, time=0.0)
    Ng, Nl = problem.global_mesh.n_nodes, lm.n_nodes
    stats = RunStats()
    t0 = time.perf_counter()
    if spacetime:
        sched = multirate.MacroSchedule(cfg.dt_macro, cfg.micro_steps, 0.0, cfg.t_end)
        multirate.run_spacetime(problem, sched, lm, T0, path=cfg.path, policy=cfg.policy, stats=stats, recorder=None)
        dof = n_steps * (Ng + cfg.micro_steps * Nl)
    else:
        dt = cfg.dt_macro / cfg.micro_steps
        multirate.run_space(problem, dt, n_steps, lm, T0, path=cfg.path, policy=cfg.policy, stats=stats, recorder=None)
        dof = n_steps * (Ng + Nl)
    wall = time.perf_counter() - t0
    return {"steps": n_steps, "wall_s": wall, "dof_timesteps": dof, "dof_timesteps_per_s": dof / wall,
            "global_nodes": Ng, "local_nodes": Nl, "counters": stats.counters, "cores": 1}


def scenario_worker(idx):
    from paper_2110_12932_b200 import scenarios as S
    _, _, _, load_config, _ = _ref()
    sc = S.draw(0, 64)[idx]
    import tempfile
    tmp = Path(tempfile.mkdtemp())
    (tmp / "const.mat").write_text((ROOT / "configs" / "const.mat").read_text())
    (tmp / "s.cfg").write_text(sc.config_text() if hasattr(sc, "config_text") else "")
    cfg = load_config(tmp / "s.cfg") if (tmp / "s.cfg").stat().st_size else None
    if cfg is None:
        raise SystemExit("scenario has no config text")
    return run_config(cfg, 10)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="cfg1,cfg2,cfg5")
    ap.add_argument("--procs", type=int, default=max(1, (os.cpu_count() or 2) - 2))
    ap.add_argument("--out", default=str(ROOT / "profiles" / "r02_cpu_baseline_reference.json"))
    args = ap.parse_args()
    only = set(args.only.split(","))
    _, _, _, load_config, _ = _ref()
    cpu = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
    model = next((ln.split(":", 1)[1].strip() for ln in cpu.splitlines() if ln.startswith("Model name")), platform.processor())
    out = {"what": "unmodified reference lpbfsim 0.1.0 (imported from /root/reference) in the build container; "
                   "recorder=None, one core per run", "host": {"model": model, "cores": os.cpu_count()},
           "cfg3": "infeasible (55.8 GB for the global mesh alone, SURVEY §8d)", "cfg4": "infeasible"}
    p = Path(args.out)
    if p.exists():
        out.update({k: v for k, v in json.loads(p.read_text()).items() if k.startswith("cfg") and k not in ("cfg3", "cfg4")})

    def save():
        p.write_text(json.dumps(out, indent=1))

    if "cfg1" in only:
        out["cfg1_m4_80_steps"] = run_config(load_config(ROOT / "configs" / "cfg1_m4.cfg"), 80)
        save()
        cfg = load_config(ROOT / "configs" / "cfg1_uniform.cfg")
        out["cfg1_uniform_80_steps"] = run_config(cfg, int(round(cfg.t_end / (cfg.dt_macro / cfg.micro_steps))), spacetime=False)
        save()
    if "cfg2" in only:
        out["cfg2_first_20_macro_steps"] = run_config(load_config(ROOT / "configs" / "cfg2.cfg"), 20)
        save()
    if "cfg5" in only:
        n = args.procs
        t0 = time.perf_counter()
        with mp.get_context("spawn").Pool(n) as pool:
            res = pool.map(scenario_worker, list(range(n)))
        wall = time.perf_counter() - t0
        dof = sum(r["dof_timesteps"] for r in res)
        out["cfg5_10_macro_steps_per_core"] = {"processes": n, "scenarios": list(range(n)), "wall_s": wall,
                                               "dof_timesteps": dof, "aggregate_dof_timesteps_per_s": dof / wall,
                                               "per_process": res, "cores": n}
        save()
    print(json.dumps({k: (v.get("dof_timesteps_per_s") or v.get("aggregate_dof_timesteps_per_s")) if isinstance(v, dict) else v
                      for k, v in out.items() if k.startswith("cfg")}, indent=1))


if __name__ == "__main__":
    main()

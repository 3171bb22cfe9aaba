#!/usr/bin/env python
"""Benchmark: DOF-timesteps/s of the two-level multirate heat solve (BASELINE.json metric).

Workload (N=1, no flags): BASELINE config 4 at one GPU, the largest single-GPU
configuration — global 1001x1001x201 (201,402,201 nodes, h = 20 um), local 251x251x101
(6,363,101 nodes, h = 4 um), multirate m = 10, fp64, Jacobi-PCG rtol 1e-12.  One "step" =
one macro step of ``run_spacetime``: 1 global solve + 10 micro local solves + the
corrector re-solve + trace + relocation, i.e. N_g + m N_l = 265,033,211 DOF-timesteps
(the corrector re-solve is performed but not counted).
``--config cfg2|cfg3`` time the smaller BASELINE configs the same way, ``--config cfg5`` the
64-scenario sweep, ``--config picard`` the temperature-dependent step.

N > 1 (torchrun): the global grid in z-slabs over the ranks with the device-resident CG,
the local steps pipelined over the ranks in time (slab_bench; weak scaling on cfg4 grown in
depth, ``--strong`` for cfg4 itself); timing is the max over ranks of the device time.
``--impl reference`` times the reference's CPU algorithm (the literal P1-assembly +
scipy-CG port in oracle/assembly.py, pinned bit-for-bit to the reference) on rank 0.

Prints one JSON line.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

# Both CPU legs run the reference's algorithm single-threaded: its sparse CG (where the
# time goes) is single-threaded scipy, and BLAS threading only slows the small dense
# products down (measured here 35k vs 42k DOF-timesteps/s with 8 vs 1
# OpenBLAS threads on the cfg4 sample) — one thread is the reference's best configuration.
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

METRIC = "DOF-timesteps/sec (global+local solves, fp64)"
UNIT = "DOF-timesteps/s"


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def measured_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        time.sleep(0.25)
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        return False

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def cpu_sample(cfg_path, what: str = "global+local"):
    """Reference CPU algorithm (oracle/assembly.py, bitwise-pinned port) on a bounded sample.
    ``cfg_path``: a .cfg file or an already built ExperimentConfig."""
    import paper_2110_12932_b200 as P
    cfg = P.load_config(cfg_path) if isinstance(cfg_path, (str, Path)) else cfg_path
    smp = LocalSample(cfg, with_global="global" in what)
    return smp.once()


class LocalSample:
    """A bounded sample of a config's two-level step for the CPU port (oracle/assembly.py:
    the reference's own algorithm — explicit Kuhn tets, einsum element matrices, COO->CSR,
    symmetric Dirichlet elimination, scipy CG — bitwise equal to lpbfsim): one local micro
    solve (the first micro interval of macro step 0, uniform initial field; trace blend and
    Gaussian as run_spacetime has them) and optionally the global predictor before it.

    ``window``: lateral node count of a column cut out of the config's local grid (same h,
    same depth, same beam position relative to the box) when the whole local grid is too
    large for a bounded CPU sample (cfg4: 251 x 251 x 101 nodes)."""

    def __init__(self, cfg, with_global: bool = False, window: int | None = None):
        import dataclasses
        import paper_2110_12932_b200 as P
        from oracle import kuhn
        from oracle.twolevel import OracleRun
        if window is not None:
            pol = cfg.policy
            size = (window - 1) * cfg.h_local
            cfg = dataclasses.replace(cfg, policy=dataclasses.replace(
                pol, box_size=(size, size) + tuple(pol.box_size[2:])))
        self.cfg, self.with_global = cfg, with_global
        self.run = OracleRun(cfg, backend="assembly")
        self.L = kuhn.KuhnGrid.from_placement(self.run.placement0)
        self.Tg = np.full(self.run.G.n_nodes, cfg.T_initial) if with_global else None
        self.Tl = np.full(self.L.n_nodes, cfg.T_initial)
        self.sched = P.MacroSchedule(cfg.dt_macro, cfg.micro_steps, 0.0, cfg.t_end)
        self.trace0 = np.where(self.L.gamma_mask().ravel(), float(cfg.T_initial), 0.0)   # P1(uniform) on gamma
        self.shape = tuple(int(c) + 1 for c in self.run.placement0.ncells)

    def once(self):
        run, L, sched = self.run, self.L, self.sched
        t0 = time.perf_counter()
        dof = 0
        if self.with_global:
            Tg2 = run.solve_global(self.Tg, 0.0, self.cfg.dt_macro)
            dof += run.G.n_nodes
            trace = run.trace_of(L, Tg2)
            told = run.trace_of(L, self.Tg)
        else:
            trace = told = self.trace0          # uniform field: P1 of a constant
        w = 1.0 / sched.micro_per_macro
        run.solve_local(L, self.Tl, 0.0, sched.t_micro(0, 1), (1.0 - w) * told + w * trace)
        dof += L.n_nodes
        dt = time.perf_counter() - t0
        return dof, dt, run.iterations, (run.G.n_nodes, L.n_nodes, sched.micro_per_macro)


def _host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def _cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# CPU sample size per config: lateral nodes of the local-grid column (None: whole local grid)
# for our arm's 1-core cpu_baseline (~10-30 s) and for each step of the reference arm
# (~2-5 s, so --steps 20 --warmup 5 ends within a few minutes)
CPU_WINDOW = {"cfg4": (126, 80), "cfg3": (None, 80), "cfg2": (None, None)}


def slab_mode(args, world: int) -> bool:
    return (world > 1 or args.slabs) and args.config == "cfg4"


def workload(args, world: int):
    """The bench workload both arms report: config dict, grid sizes, DOF per step."""
    import paper_2110_12932_b200 as P
    from paper_2110_12932_b200.control import initial_local_box, structured_ncells
    slabs = slab_mode(args, world)
    if slabs and not args.strong:
        cfg = weak_config(world)
    else:
        cfg = P.load_config(ROOT / "configs" / f"{args.config}.cfg")
    gn = structured_ncells(cfg.global_box, cfg.h_global)
    lbox = initial_local_box(cfg.global_box, cfg.h_local, cfg.policy, cfg.path)
    ln = structured_ncells(lbox, cfg.h_local)
    Ng, Nl = int(np.prod(np.asarray(gn) + 1)), int(np.prod(np.asarray(ln) + 1))
    m = int(cfg.micro_steps)
    dof_step = Ng + m * Nl
    first = args.skip + args.warmup
    conf = {"workload": f"{args.config}: two-level multirate macro step (1 global + {m} local solves + "
                        f"corrector), global {Ng} + local {Nl} nodes",
            "config_file": f"configs/{args.config}.cfg", "dof_timesteps_per_step": dof_step,
            "macro_steps": f"{first}..{first + args.steps - 1}",
            "l2": ("inputs larger than L2 and flushed between timed steps" if Ng * 8 > 126e6
                   else "flushed between timed steps") if not args.no_flush else "not flushed",
            "parallelism": f"scenario replicas x{world}" if world > 1 else "single GPU"}
    if slabs:
        conf["workload"] = (f"{args.config}: two-level multirate macro step, global grid in z-slabs over {world} "
                            f"GPU(s) ({'strong scaling' if args.strong else 'weak scaling: ~201M global nodes per GPU'}),"
                            f" local steps pipelined over the GPUs in time; global {Ng} + local {Nl} nodes")
        conf["parallelism"] = f"z-slabs x{world} + local time pipeline"
    return cfg, conf, (Ng, Nl, m)


def reference_arm(args):
    """--impl reference: the reference's CPU algorithm (the literal P1-assembly + scipy-CG
    port, bitwise equal to lpbfsim) on the host cores, rank 0 only; same metric, unit and
    config as the device arm; each timed step is a bounded sample of the workload."""
    rank, world, _ = env_rank()
    if rank != 0:
        return
    cfg, conf, (Ng, Nl, m) = workload(args, world)
    win = CPU_WINDOW.get(args.config, (None, None))[1]
    if args.config == "cfg5":                 # config 5: a sample of its first scenario
        from paper_2110_12932_b200 import scenarios as S
        cfg = S.draw(0, 64)[0].config()
    smp = LocalSample(cfg, with_global=False, window=win)
    times, dofs = [], []
    for s in range(args.warmup + args.steps):
        dof, dt, _, _ = smp.once()
        if s >= args.warmup:
            times.append(dt)
            dofs.append(dof)
    total = sum(times)
    value = sum(dofs) / total
    what = (f"one {args.config} local micro solve (first micro interval, uniform initial field) on "
            + (f"a {smp.shape[0]}x{smp.shape[1]}x{smp.shape[2]}-node column of the {args.config} local grid "
               f"(same h and depth; the whole {Nl}-node local grid would take minutes per sample)"
               if win else f"the whole {smp.shape[0]}x{smp.shape[1]}x{smp.shape[2]} local grid")
            + f", {smp.L.n_nodes} DOF-timesteps")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "timed_step": what + "; ms_per_step is the time of that sample, value its DOF-timesteps/s",
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic (BASELINE {args.config} geometry and scan path)",
        "config": conf,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "port",
                         "sample": what + " per timed step via the literal P1-assembly + scipy-CG port "
                                   "(oracle/assembly.py, bitwise equal to lpbfsim); one thread: the reference is "
                                   "one sequential process (scipy's sparse CG is single-threaded) and BLAS threads "
                                   f"only slow it down; host: {_cpu_model()}, {_host_threads()} threads available"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def weak_config(world: int):
    """BASELINE config 4 grown in depth for weak scaling over z-slabs: the plate is
    20 x 20 x 4N mm (1001 x 1001 x (200 N + 1) global nodes, ~201M per GPU), the scan path
    on its top surface, the local box (251 x 251 x 101 nodes, h = 4 um) as in cfg4.  N = 1
    is cfg4 itself."""
    import paper_2110_12932_b200 as P
    text = (ROOT / "configs" / "cfg4.cfg").read_text()
    if world > 1:
        depth = 4 * world
        text = text.replace("global_max 20 20 4 mm", f"global_max 20 20 {depth} mm")
        text = text.replace("origin 2.5 9.55 4.0 mm", f"origin 2.5 9.55 {depth}.0 mm")
    return P.config_from_text(text, base_dir=ROOT / "configs", name=f"cfg4-weak-x{world}")


def slab_bench(args):
    """Multi-GPU (``--gpus N`` under torchrun, or ``--slabs``): the global grid in z-slabs
    with the device-resident CG (slab.py), the local steps pipelined over the ranks in time
    (multirate_dist.py).  Default workload: cfg4 grown in depth, ~201M global nodes per GPU
    (weak scaling); ``--strong``: cfg4 itself split over the ranks."""
    import torch
    import paper_2110_12932_b200 as P
    from paper_2110_12932_b200.multirate_dist import SlabRun, plan_superstep

    rank, world, local_rank = env_rank()
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    cfg, conf, (Ng, Nl, m) = workload(args, world)
    problem, lmesh = P.build_problem(cfg, device=local_rank)
    sched = P.MacroSchedule(cfg.dt_macro, cfg.micro_steps, 0.0, cfg.t_end)
    dof_step = Ng + m * Nl
    run = SlabRun(problem, lmesh, rank=rank, world=world, device=dev)
    run.initial(P.uniform_field(problem.global_mesh, cfg.T_initial))
    state = [lmesh.placement, 0.0, 0.0, 0]

    def steps(n):
        """Whole super-steps until at least n macro steps ran; returns the steps run."""
        done = 0
        while done < n:
            plans, nxt = plan_superstep(problem, sched, cfg.path, cfg.policy, *state, world, run.moved_before)
            if not plans:
                raise SystemExit("schedule exhausted")
            run.superstep(plans)
            state[:] = list(nxt)
            done += len(plans)
        return done

    steps(args.warmup)
    run.check_local()
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    run.timing = True
    run.global_ms.clear()
    l0 = run.solver.launches + run.local.launch_count()
    cur = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clocks:
        wall0 = time.perf_counter()
        e0.record(cur)
        nsteps = steps(args.steps)
        cur.wait_stream(run.local_stream)
        e1.record(cur)
        torch.cuda.synchronize()
        wall = time.perf_counter() - wall0
    run.check_local()
    dev_ms = e0.elapsed_time(e1)
    launches = run.solver.launches + run.local.launch_count() - l0
    S = run.solver
    own = (S.k1 - S.k0) * S.nxy
    gms = [a.elapsed_time(b) for a, b, _ in run.global_ms]
    gits = [k for _, _, k in run.global_ms]
    polls = S.polls
    if dist is not None:
        t = torch.tensor([dev_ms, wall], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dev_ms, wall = float(t[0]), float(t[1])
    value = dof_step * nsteps / (dev_ms / 1e3)
    peak, peak_src = measured_peak()
    alg = sum(own * (64 * k + 32) for k in gits)
    ach = alg / (sum(gms) / 1e3) / 1e9 if gms else None
    roofline = {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
                "frac": ach / peak if ach else None, "frac_of_8tbs_datasheet": ach / 8000.0 if ach else None,
                "traffic": None,
                "kernel": "z-slab global solve (rank 0): k_slab_rhs -> {k_sd_dir (bulk-copy sweep A), all-gather, "
                          "k_sd_upd_flat (boundary planes), halo || k_sd_upd (bulk-copy sweep B), all-gather} -> "
                          "k_sd_resid -> k_sd_finish; scalars on the device",
                "level": "global", "nodes": own, "peak_source": peak_src,
                "note": "rank 0's own nodes x (64 k + 32) bytes per solve / the solves' CUDA-event time "
                        "(incl. the collectives inside them)"}

    # e2e: the same driver with the host planning inside the clock and the final local
    # field read back (the public two_level_run_slabs / run_spacetime_slabs loop)
    T0 = P.uniform_field(problem.global_mesh, cfg.T_initial)
    run2 = run
    run2.check_local()
    h_lv = np.empty(lmesh.n_nodes)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    t0 = time.perf_counter()
    ne = steps(args.steps)
    run2.check_local()
    if rank == run2.last_rank:
        h_lv = run2.local.field(1)
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    if dist is not None:
        t = torch.tensor([e2e_s], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    del T0, h_lv
    e2e = {"value": dof_step * ne / e2e_s, "unit": UNIT, "h2d_bytes_per_step": 64 + 48 * (m + 1) + 8 * 4 * 144,
           "d2h_bytes_per_step": 40 * (m + 2) + 8 * Nl // max(ne, 1),
           "note": "host wall clock (max over ranks) of the next macro steps through the slab driver's "
                   "public loop (plan_superstep + SlabRun.superstep, as run_spacetime_slabs runs it): host "
                   "planning inside the clock, deposit samples H2D, solve records D2H, the last local field D2H"}
    # the global solve timed alone (no local step in flight on the other stream): three more
    # solves of the current field, all ranks together, CUDA events on the solve's stream
    run.check_local()
    alone = []
    for _ in range(3):
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(cur)
        inf = S.step(cfg.dt_macro, problem.bc.T_buildplate, with_load=False)
        b.record(cur)
        torch.cuda.synchronize()
        alone.append((a.elapsed_time(b), inf.iterations))
    alone_ms = float(np.mean([t for t, _ in alone]))
    alone_gbs = sum(own * (64 * k + 32) for _, k in alone) / (sum(t for t, _ in alone) / 1e3) / 1e9
    run.close()
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        win = CPU_WINDOW.get("cfg4", (None, None))[0]
        smp = LocalSample(cfg, with_global=False, window=win)
        dof, dt, _, _ = smp.once()
        cpu = {"value": dof / dt, "unit": UNIT, "cores": 1, "kind": "port",
               "sample": f"one local micro solve on a {smp.shape[0]}x{smp.shape[1]}x{smp.shape[2]}-node column of the "
                         f"cfg4 local grid ({dof} DOF-timesteps, {dt:.1f} s), literal P1-assembly + scipy-CG port; "
                         "the global solve is infeasible on the CPU port"}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": nsteps,
        "warmup": args.warmup, "ms_per_step": dev_ms / nsteps, "higher_is_better": True,
        "scaling": "strong" if args.strong else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (BASELINE config 4 scan path and geometry" + ("" if args.strong or world == 1 else
                f", plate {4 * world} mm deep for weak scaling") + ")",
        "config": conf,
        "global_solve": {"ms_mean": float(np.mean(gms)) if gms else None,
                         "iterations_mean": float(np.mean(gits)) if gits else None,
                         "host_syncs_per_solve": polls / max(len(run.global_infos), 1),
                         "alone_ms": alone_ms, "alone_iterations": float(np.mean([k for _, k in alone])),
                         "alone_gbs": alone_gbs, "alone_frac": alone_gbs / peak,
                         "note": "ms_mean: inside the step, with the previous step's local solves running "
                                 "concurrently on the local stream; alone_*: the same solve with nothing else "
                                 "on the device (rank 0's own nodes x (64 k + 32) bytes / its event time)"},
        "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
        "clocks": clocks.summary(), "wall_s_timed_region": wall,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def kernel_stats(rows, n, dev_ms):
    """Solve-launch timing rows [(ms, [iterations per solve])] on an n-node grid ->
    algorithmic HBM throughput N(64k+32) per solve."""
    if not rows:
        return None
    solves = sum(len(its) for _, its in rows)
    bytes_ = sum(n * (64 * k + 32) for _, its in rows for k in its)
    ms = sum(t for t, _ in rows)
    return {"launches": len(rows), "solves": solves, "avg_ms_per_solve": ms / solves,
            "avg_iterations": float(np.mean([k for _, its in rows for k in its])),
            "alg_bytes_per_solve": bytes_ / solves, "achieved_gbs": bytes_ / (ms / 1e3) / 1e9,
            "share_of_step": ms / dev_ms if dev_ms else None}


def split_timing(kt, infos):
    """Pair each timed solve launch with the solve records it produced -> (local, global)."""
    loc, glo, pos = [], [], 0
    for ms, lv, ns in kt:
        its = [inf["iterations"] for inf in infos[pos:pos + ns]]
        pos += ns
        (loc if lv == 1 else glo).append((ms, its))
    return loc, glo


def scenario_bench(args):
    """--config cfg5: BASELINE config 5, the batched scenario sweep.  64 independent runs of
    the config-2 geometry (parameters from seed 0, paper_2110_12932_b200/scenarios.py),
    LPT-sharded by DOF-timestep work across the ranks (no data-path collective).  Every
    scenario of the rank's group is resident at once (one tl_run each, ~0.1 GB); one "step"
    advances every scenario of the group by one macro step, issued back to back with the
    runs' streams chained by events so the device executes them in order with no host
    round trip between scenarios."""
    import torch
    import paper_2110_12932_b200 as P
    from paper_2110_12932_b200 import scenarios as S
    from paper_2110_12932_b200.schedule import plan_spacetime

    rank, world, local_rank = env_rank()
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    allsc = S.draw(0, 64)[:args.scenarios]
    group = S.shard(allsc, rank, world)
    nsteps = args.warmup + 2 * args.steps          # timed steps, then as many e2e steps
    runs, plans, dofs, nl_m = [], [], [], []
    for sc in group:
        cfg = sc.config()
        problem, lmesh = P.build_problem(cfg, device=local_rank)
        sched = P.MacroSchedule(cfg.dt_macro, cfg.micro_steps, 0.0, cfg.t_end)
        if nsteps > sched.n_macro:
            raise SystemExit(f"scenario {sc.index} has only {sched.n_macro} macro steps")
        pls, placement, tg, tl = [], lmesh.placement, 0.0, 0.0
        for k in range(nsteps):
            pl = plan_spacetime(problem, sched, placement, cfg.path, cfg.policy, tg, tl, k0=k, nsteps=1)
            pls.append(pl)
            placement, tg, tl = pl.final_placement, pl.final_t_global, pl.final_t_local
        run = P.DeviceRun(problem, lmesh)
        run.initial(P.uniform_field(problem.global_mesh, cfg.T_initial))
        runs.append(run)
        plans.append(pls)
        Ng, Nl = problem.global_mesh.n_nodes, lmesh.n_nodes
        dofs.append(Ng + sched.micro_per_macro * Nl)
        nl_m.append((Ng, Nl, sched.micro_per_macro))
    streams = [torch.cuda.ExternalStream(r.stream(), device=dev) for r in runs]
    dof_step = sum(dofs)
    batched = not args.no_batch
    batch = P.BatchedRuns(runs) if batched else None

    def one_step(k, plan_of=None, after=None):
        """Macro step k of every scenario.  Batched (default): one tl_runs_macro_step call, the
        i-th micro solve of all scenarios one streaming solve on the first run's stream (the
        other runs' streams are ordered after it).  --no-batch: one run after the other,
        device-ordered through event chaining."""
        if batched:
            batch.step([plans[i][k] if plan_of is None else plan_of(i, k) for i in range(len(runs))])
            if after is not None:
                for i in range(len(runs)):
                    after(i, k)
            prev = torch.cuda.Event()
            prev.record(streams[0])
            return prev
        prev = None
        for i, (run, st) in enumerate(zip(runs, streams)):
            if prev is not None:
                st.wait_event(prev)
            run.run(plans[i][k] if plan_of is None else plan_of(i, k))
            if after is not None:
                after(i, k)
            prev = torch.cuda.Event()
            prev.record(st)
        return prev

    for k in range(args.warmup):
        one_step(k)
    for r in runs:
        r.sync()
        r.check_solves(r.take_info())
        r.set_timing(True)
        r.take_timing()
    launches0 = sum(r.launch_count() for r in runs)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    ev = []
    with ClockSampler(local_rank) as clocks:
        wall0 = time.perf_counter()
        last = None
        for k in range(args.warmup, args.warmup + args.steps):
            if not args.no_flush:
                if last is not None:
                    streams[0].wait_event(last)
                runs[0].flush_l2()
            e0 = torch.cuda.Event(enable_timing=True)
            e0.record(streams[0])
            last = one_step(k)
            e1 = torch.cuda.Event(enable_timing=True)
            e1.record(streams[0] if batched else streams[-1])
            ev.append((e0, e1))
            last = e1
        for r in runs:
            r.sync()
        wall = time.perf_counter() - wall0
    torch.cuda.synchronize()
    launches = sum(r.launch_count() for r in runs) - launches0
    dev_ms = float(sum(a.elapsed_time(b) for a, b in ev))
    loc_rows, glo_rows = [], []
    for i, r in enumerate(runs):
        infos = r.take_info()
        r.check_solves(infos)
        if batched:
            # the batched solves are timed on the first run (level 0: the global solves of all
            # runs, level 1: one batched local solve); a run's records per step are
            # [global, micro..., corrector]
            per = 1 + nl_m[i][2] + 1
            assert len(infos) == per * args.steps, (len(infos), per)
            g_its = [infos[s_ * per]["iterations"] for s_ in range(args.steps)]
            l_its = [inf["iterations"] for s_ in range(args.steps) for inf in infos[s_ * per + 1:(s_ + 1) * per]]
            glo_rows.append((0.0, g_its))
            loc_rows.append((0.0, l_its))
            if i == 0:
                kt0 = r.take_timing()
        else:
            lo, gl = split_timing(r.take_timing(), infos)
            loc_rows.extend(lo)
            glo_rows.extend(gl)
        r.set_timing(False)
    if batched:
        # CUDA-event time of the batched launches (RHS -> CG loop -> residual -> finish), per level,
        # spread over the system-solves for the per-solve figures
        for rows, lv in ((glo_rows, 0), (loc_rows, 1)):
            ms = sum(t for t, l, _ in kt0 if l == lv)
            nsolve = sum(len(its) for _, its in rows)
            rows[:] = [(ms * len(its) / nsolve, its) for _, its in rows]
    if dist is not None:
        t = torch.tensor([dev_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dev_ms = float(t.item())
    total_dof = dof_step * args.steps
    if dist is not None:
        t = torch.tensor([float(total_dof)], device=dev, dtype=torch.float64)
        dist.all_reduce(t)
        total_dof = float(t.item())
    value = total_dof / (dev_ms / 1e3)

    # all scenarios share the config-2 grids: pool the solve launches per level
    Ng, Nl = nl_m[0][0], nl_m[0][1]
    share_ms = dev_ms if world == 1 else None
    kloc, kglo = kernel_stats(loc_rows, Nl, share_ms), kernel_stats(glo_rows, Ng, share_ms)
    peak, peak_src = measured_peak()
    roofline = {"bound": "hbm", "achieved": kloc["achieved_gbs"], "peak": peak, "unit": "GB/s",
                "frac": kloc["achieved_gbs"] / peak, "frac_of_8tbs_datasheet": kloc["achieved_gbs"] / 8000.0,
                "traffic": None,
                "kernel": ("batched local-grid PCG solves: the i-th micro solve of every scenario of the group in "
                           "one launch sequence k_sb_rhs -> k_tb_cg (bulk-copy z-march CG loop over all systems, in "
                           "lockstep) -> k_sb_resid -> k_sb_final") if batched else
                          ("local-grid PCG solves (k_pcg_resident_cg, SMEM-resident bricks, all micro solves "
                           "+ corrector of a macro step in one launch), pooled over the group's scenarios"),
                "level": "local", "nodes": Nl, "peak_source": peak_src,
                "note": ("algorithmic bytes N(64k+32) per system-solve (SURVEY §8d) / the CUDA-event time of the "
                         "batched solve launches") if batched else
                        ("algorithmic bytes N(64k+32) per solve (SURVEY §8d); each scenario's grids are "
                         "L2/SMEM-resident within its own macro step")}

    # ---- e2e through DeviceRun.run: pinned plan uploads, every scenario's local field read back ----
    def pin(arr, dtype):
        arr = np.ascontiguousarray(arr, dtype=dtype).reshape(-1)
        buf = torch.empty(max(arr.nbytes, 1), dtype=torch.uint8, pin_memory=True).numpy().view(dtype)[:arr.size]
        buf[:] = arr
        return buf

    ks = list(range(args.warmup + args.steps, nsteps))
    e2e_plans, h2d = {}, 0
    for i in range(len(runs)):
        for k in ks:
            pl = plans[i][k]
            pp = type(pl)(macro=pin(pl.macro, pl.macro.dtype), micro=pin(pl.micro, pl.micro.dtype),
                          dep_points=pin(pl.dep_points, np.float64).reshape(-1, 3),
                          dep_power=pin(pl.dep_power, np.float64))
            e2e_plans[i, k] = pp
            h2d += pp.macro.nbytes + pp.micro.nbytes + pp.dep_points.nbytes + pp.dep_power.nbytes
    pins = [[torch.empty(nl, dtype=torch.float64, pin_memory=True).numpy() for _ in range(2)]
            for (_, nl, _) in nl_m]
    for i, r in enumerate(runs):                  # staging buffers registered before the clock
        for s in range(2):
            r.field_async(1, pins[i][s], slot=s)
            r.field_wait(s)
    d2h = 0

    def readback(i, k):
        runs[i].field_async(1, pins[i][k % 2], slot=k % 2)

    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for s, k in enumerate(ks):
        one_step(k, plan_of=lambda i, kk: e2e_plans[i, kk], after=readback)
        d2h += sum(p[k % 2].nbytes for p in pins)
        if s >= 1:
            for r in runs:
                r.field_wait((k - 1) % 2)
    for r in runs:
        r.field_wait(ks[-1] % 2)
    e2e_s = time.perf_counter() - t0
    for r in runs:
        r.check_solves(r.take_info())
    if dist is not None:
        t = torch.tensor([e2e_s], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e = {"value": total_dof / e2e_s, "unit": UNIT, "h2d_bytes_per_step": h2d // len(ks),
           "d2h_bytes_per_step": d2h // len(ks),
           "note": "host wall clock (max over ranks) through DeviceRun.run, the next macro steps of every "
                   "scenario: plan arrays H2D from pinned memory, every scenario's local field D2H to "
                   "pinned memory each step (double-buffered, overlapped with the following scenarios)"}
    for r in runs:
        r.close()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        dof, dt, its, _ = cpu_sample(group[0].config(), what="local")
        cpu = {"value": dof / dt, "unit": UNIT, "cores": 1, "kind": "port",
               "sample": f"one local micro solve of scenario {group[0].index} ({dof} DOF-timesteps, {dt:.1f} s) "
                         "via the literal P1-assembly + scipy-CG port (oracle/assembly.py, bitwise equal to "
                         "lpbfsim); OPENBLAS_NUM_THREADS=1"}
    ms = [m for (_, _, m) in nl_m]
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dev_ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (BASELINE config 5: 64 config-2 scenarios, parameters drawn from seed 0)",
        "config": {"workload": f"cfg5: batched scenario sweep, {len(allsc)} scenarios of the config-2 geometry "
                               f"(global {Ng} + local {Nl} nodes, m in {{5,10,20}}) split over {world} GPU(s); "
                               f"one step = one macro step of every scenario of the group",
                   "scenarios_rank0": [s.index for s in group],
                   "micro_rank0": {str(v): ms.count(v) for v in sorted(set(ms))},
                   "dof_timesteps_per_step_rank0": dof_step,
                   "macro_steps": f"{args.warmup}..{args.warmup + args.steps - 1} (e2e: the next {args.steps})",
                   "l2": ("flushed between timed steps; each step also streams every scenario's fields "
                          f"({len(group)} x ~0.1 GB, larger than L2)") if not args.no_flush else "not flushed",
                   "batched_solves": batched,
                   "parallelism": f"scenario groups x{world}" if world > 1 else "single GPU"},
        "roofline": roofline, "kernels": {"local_pcg": kloc, "global_pcg": kglo},
        "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
        "clocks": clocks.summary(), "wall_s_timed_region": wall,
        "iterations": {"local": kloc["avg_iterations"], "global": kglo["avg_iterations"] if kglo else None},
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def picard_bench(args):
    """--config picard: SURVEY §8f row 1 on a cfg2-local-sized grid (101 x 101 x 51 nodes,
    h = 5 um): temperature-dependent implicit steps (configs/tdep.mat: kappa(T), c(T),
    latent heat; convection + lagged radiation on the top face; moving Gaussian beam;
    bottom Dirichlet) through the public seam fem.step_backward_euler, the field left on the
    device between steps.  One step = one Picard-converged implicit step: one
    tl_vc_picard_nodes_host call whose
    passes (assembly + one cooperative Jacobi-PCG launch + the increment reduction) run on
    the device.  value is the host wall clock around the public call, e2e the same with the
    field read back after every step; the roofline is
    the PCG launch timed with CUDA events: N (96 k + 32) algorithmic bytes per pass
    (SURVEY §8d's 64 B/node/iteration plus the 4 per-node coefficient arrays)."""
    import torch
    import paper_2110_12932_b200 as P
    from oracle import varcoef, kuhn

    rank, world, local_rank = env_rank()
    torch.cuda.set_device(local_rank)
    if rank != 0:
        return
    mat = P.load_material(ROOT / "configs" / "tdep.mat")
    box = P.Box((0.0, 0.0, 0.0), (5e-4, 5e-4, 2.5e-4))
    grid = P.build_structured_grid(box, 5e-6)
    n = grid.n_nodes
    X = grid.coords
    c0 = np.array([2.0e-4, 2.5e-4, 2.5e-4])
    r2 = ((X - c0) ** 2 / np.array([1.0e-4, 0.8e-4, 0.6e-4]) ** 2).sum(axis=1)
    T = 293.0 + 1900.0 * np.exp(-r2)
    bc = P.ThermalBC(10.0, 0.8, 293.0, 293.0)
    bounds = P.BoundarySpec(bc=bc, robin_tags=(P.TOP,), radiation=True,
                            dirichlet_nodes=grid.nodes_on(P.BOTTOM), dirichlet_values=293.0)
    beam = P.LaserBeam(200.0, 0.35, 5e-5, 5e-5, 0.8)
    settings = P.SolverSettings(picard_tol=1e-8, picard_max_iter=60, linear_tol=1e-12, linear_solver="cg")
    dt = 2e-6
    state = P.FieldState(grid, T, 0.0)
    T_first = T.copy()

    def step(st, k, stats):
        center = (2.0e-4 + beam.speed * dt * (k + 1), 2.5e-4, 2.5e-4)
        return P.step_backward_euler(st, dt, mat, P.GaussianSource(beam, center), bounds, settings,
                                     latent=True, stats=stats)

    for k in range(args.warmup):
        state = step(state, k, None)
    from paper_2110_12932_b200 import _native as N
    stats = P.RunStats()
    stats.device_log = []
    walls = []
    N.host_traffic(reset=True)
    with ClockSampler(local_rank) as clocks:
        for k in range(args.warmup, args.warmup + args.steps):
            t0 = time.perf_counter()
            state = step(state, k, stats)
            walls.append(time.perf_counter() - t0)
    wall = sum(walls)
    dev_h2d, dev_d2h = N.host_traffic(reset=True)
    # e2e: the same steps with the converged field read back to the host after every step
    e2e_walls = []
    for k in range(args.warmup + args.steps, args.warmup + 2 * args.steps):
        t0 = time.perf_counter()
        state = step(state, k, None)
        _ = state.values
        e2e_walls.append(time.perf_counter() - t0)
    e2e_wall = sum(e2e_walls)
    e2e_h2d, e2e_d2h = N.host_traffic(reset=True)
    passes = stats.counters.get("picard_iterations", 0)
    cg_ms = sum(ms for ms, _ in stats.device_log)
    its = [it for _, it in stats.device_log]
    alg = sum(n * (96 * k + 32) for k in its)
    peak, peak_src = measured_peak()
    value = n * args.steps / wall
    cpu = None
    if not args.no_cpu_baseline:
        G = kuhn.KuhnGrid(box.lo, box.hi, grid.ncells)
        dmask = np.zeros(n, dtype=bool)
        dmask[grid.nodes_on(P.BOTTOM)] = True
        g = np.full(n, 293.0)
        robin = (10.0, bc.sigma_sb * 0.8, 293.0)
        t0 = time.perf_counter()
        _, npass, _ = varcoef.step(G, mat, T_first, dt, P.GaussianSource(beam, (2.0e-4 + beam.speed * dt, 2.5e-4,
                                   2.5e-4)), dmask, g, True, robin, picard_max=60)
        tc = time.perf_counter() - t0
        cpu = {"value": n / tc, "unit": UNIT, "cores": 1, "kind": "port",
               "sample": f"the first step ({npass} Picard passes, {tc:.1f} s) via oracle/varcoef.py (the stencil "
                         "restatement pinned to the reference's step_backward_euler); OPENBLAS_NUM_THREADS=1"}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * wall / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (temperature-dependent material configs/tdep.mat, moving Gaussian beam, hot-spot T0)",
        "config": {"workload": f"picard: temperature-dependent implicit steps on {tuple(int(v) + 1 for v in grid.ncells)} "
                               f"nodes (cfg2 local grid), Picard loop over device passes",
                   "picard_passes_per_step": passes / args.steps,
                   "cg_iterations_per_pass": float(np.mean(its)) if its else None,
                   "l2": "not flushed (step-level seam: the field goes from step to step on the device)",
                   "pcie_bytes_per_step": {"h2d": dev_h2d // args.steps, "d2h": dev_d2h // args.steps},
                   "parallelism": "single GPU"},
        "roofline": {"bound": "hbm", "achieved": alg / (cg_ms / 1e3) / 1e9 if cg_ms else None, "peak": peak,
                     "unit": "GB/s", "frac": (alg / (cg_ms / 1e3) / 1e9) / peak if cg_ms else None, "traffic": None,
                     "kernel": "k_vc_cg (one cooperative Jacobi-PCG launch per Picard pass)",
                     "share_of_step": cg_ms / 1e3 / wall, "peak_source": peak_src,
                     "note": "N (96 k + 32) bytes per pass; working set L2-resident at this size"},
        "cpu_baseline": cpu,
        "e2e": {"value": n * args.steps / e2e_wall, "unit": UNIT, "h2d_bytes_per_step": int(e2e_h2d // args.steps),
                "d2h_bytes_per_step": int(e2e_d2h // args.steps),
                "note": "host wall clock around fem.step_backward_euler plus the read-back of the converged "
                        "field after every step (bytes from tl_host_traffic: the Dirichlet node list and "
                        "values up, the field down); value is the same loop without the read-back (the "
                        "field stays in a device vector between steps)"},
        # per pass: k_vc_tets, k_vc_assemble, k_vc_constrain_b/_w, k_vc_cg, k_vc_inc, k_vc_lag (not after
        # the last pass of a step); per step: k_scatter_dirichlet (profiles/r02_picard_launches_summary.txt)
        "gpu_launches": int(passes * 7), "clocks": clocks.summary(),
    }
    print(json.dumps(line), flush=True)


def device_arm(args):
    """Our arm at N = 1 (and scenario replicas at N > 1): ``value`` from per-step CUDA events
    around DeviceRun.run on the run's stream (inputs resident, L2 flushed between steps);
    ``e2e`` through the public ``run_spacetime`` (recorder=None) over a K-step schedule."""
    import torch
    import paper_2110_12932_b200 as P
    from paper_2110_12932_b200.schedule import plan_spacetime

    rank, world, local_rank = env_rank()
    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))

    cfg, conf, (Ng, Nl, m) = workload(args, world)
    problem, lmesh = P.build_problem(cfg, device=local_rank)
    sched = P.MacroSchedule(cfg.dt_macro, cfg.micro_steps, 0.0, cfg.t_end)
    assert (problem.global_mesh.n_nodes, lmesh.n_nodes, sched.micro_per_macro) == (Ng, Nl, m)
    dof_step = Ng + m * Nl
    nsteps = args.skip + args.warmup + args.steps
    if nsteps > sched.n_macro:
        raise SystemExit(f"{args.config} has only {sched.n_macro} macro steps")

    # per-step plans (host, outside the timed region of `value`)
    plans = []
    placement, tg, tl = lmesh.placement, 0.0, 0.0
    for k in range(nsteps):
        pl = plan_spacetime(problem, sched, placement, cfg.path, cfg.policy, tg, tl, k0=k, nsteps=1)
        plans.append(pl)
        placement, tg, tl = pl.final_placement, pl.final_t_global, pl.final_t_local

    run = P.DeviceRun(problem, lmesh)
    run.initial(P.uniform_field(problem.global_mesh, cfg.T_initial))
    stream = torch.cuda.ExternalStream(run.stream(), device=torch.device("cuda", local_rank))
    for k in range(args.skip + args.warmup):
        run.run(plans[k])
    run.sync()
    run.check_solves(run.take_info())

    # ---- timed region: K macro steps, per-step CUDA events on the run's stream ----
    timed = plans[args.skip + args.warmup:]
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in timed]
    run.set_timing(True)
    run.take_timing()
    launches0 = run.launch_count()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clocks:
        wall0 = time.perf_counter()
        for (e0, e1), pl in zip(ev, timed):
            if not args.no_flush:
                run.flush_l2()
            e0.record(stream)
            run.run(pl)
            e1.record(stream)
        run.sync()
        wall = time.perf_counter() - wall0
    torch.cuda.synchronize()
    launches = run.launch_count() - launches0
    dev_ms = float(sum(a.elapsed_time(b) for a, b in ev))
    infos = run.take_info()
    run.check_solves(infos)
    kt = run.take_timing()
    run.set_timing(False)
    run.close()
    if dist is not None:
        t = torch.tensor([dev_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dev_ms = float(t.item())
    value = dof_step * len(timed) * world / (dev_ms / 1e3)

    # ---- roofline of the dominant kernel ----
    peak, peak_src = measured_peak()
    loc, glo = split_timing(kt, infos)
    share_ms = dev_ms if world == 1 else None
    kloc, kglo = kernel_stats(loc, Nl, share_ms), kernel_stats(glo, Ng, share_ms)
    lev = "global" if kglo and (not kloc or sum(t for t, _ in glo) > sum(t for t, _ in loc)) else "local"
    kdom, ndom = (kglo, Ng) if lev == "global" else (kloc, Nl)
    kname = kernel_name(problem, lev, Ng if lev == "global" else Nl)
    traffic, tnote = None, None
    tfile = ROOT / "profiles" / "traffic.json"
    if tfile.exists():
        tj = json.loads(tfile.read_text())
        dram = tj.get(f"{args.config}_{lev}_pcg_dram_bytes_per_launch")
        alg = tj.get(f"{args.config}_{lev}_pcg_alg_bytes_per_launch")
        if dram and alg:
            # ncu's launch may run another iteration count: scale its DRAM/algorithmic ratio
            # to this run's algorithmic bytes per launch
            per_launch = kdom["alg_bytes_per_solve"] * kdom["solves"] / kdom["launches"]
            traffic = dram / alg * per_launch
            tnote = f"ncu DRAM/algorithmic = {dram / alg:.3f} ({tj.get(f'{args.config}_{lev}_pcg_kernel', '')})"
    if tfile.exists():                   # ncu DRAM / algorithmic bytes of each level's CG launch
        for kk, lv in ((kloc, "local"), (kglo, "global")):
            d_, a_ = tj.get(f"{args.config}_{lv}_pcg_dram_bytes_per_launch"), tj.get(f"{args.config}_{lv}_pcg_alg_bytes_per_launch")
            if kk and d_ and a_:
                kk["ncu_dram_over_algorithmic"] = d_ / a_
    roofline = {"bound": "hbm", "achieved": kdom["achieved_gbs"], "peak": peak, "unit": "GB/s",
                "frac": kdom["achieved_gbs"] / peak, "frac_of_8tbs_datasheet": kdom["achieved_gbs"] / 8000.0,
                "traffic": traffic, "traffic_note": tnote,
                "kernel": kname, "level": lev, "nodes": ndom, "peak_source": peak_src,
                "note": "algorithmic bytes N(64k+32) per solve (SURVEY §8d) / the solve launches' CUDA-event "
                        "time on the run's stream"}

    # ---- e2e through the public API: run_spacetime(recorder=None) over a K-step schedule ----
    e2e = e2e_run_spacetime(args, cfg, problem, lmesh, dof_step, world, local_rank)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        win = CPU_WINDOW.get(args.config, (None, None))[0]
        smp = LocalSample(cfg, with_global=win is None, window=win)
        dof, dt, _, _ = smp.once()
        what = ("one global + one local implicit step" if win is None else
                f"one local micro solve on a {smp.shape[0]}x{smp.shape[1]}x{smp.shape[2]}-node column of the "
                f"{args.config} local grid (same h and depth)")
        note = "" if win is None else (f"; the {Ng}-node global solve is infeasible on the CPU port (SURVEY §8d: "
                                       "cfg3's global mesh alone needed 55.8 GB and 87-149 s per step)"
                                       if args.config == "cfg4" else "")
        cpu = {"value": dof / dt, "unit": UNIT, "cores": 1, "kind": "port",
               "sample": f"{what} of {args.config} ({dof} DOF-timesteps, {dt:.1f} s) via the literal P1-assembly + "
                         "scipy-CG port (oracle/assembly.py, bitwise equal to lpbfsim); OPENBLAS_NUM_THREADS=1"
                         + note + f"; host CPU: {_cpu_model()}"}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": len(timed),
        "warmup": args.warmup, "ms_per_step": dev_ms / len(timed), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic (BASELINE {args.config} scan path and geometry; no dataset involved)",
        "config": conf,
        "roofline": roofline, "kernels": {"local_pcg": kloc, "global_pcg": kglo},
        "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
        "clocks": clocks.summary(), "wall_s_timed_region": wall,
        "iterations": {"local": kloc["avg_iterations"] if kloc else None,
                       "global": kglo["avg_iterations"] if kglo else None},
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def kernel_name(problem, level: str, n: int) -> str:
    tiled = "k_s_rhs -> k_t_cg (bulk-copy z-march CG loop) -> k_s_resid -> k_s_final"
    flat = "k_s_rhs -> k_s_cg (flat streaming CG loop) -> k_s_resid -> k_s_final"
    if n >= 20_000_000:
        return f"{level}-grid PCG solve: {tiled}"
    if n >= 1_000_000:
        return f"{level}-grid PCG solve: {flat} (k_t_cg from 20M nodes)"
    if level == "local":
        return ("local-grid PCG solves: k_pcg_resident_cg (SMEM-resident bricks, all micro solves + corrector "
                "of a macro step in one launch)")
    return "global-grid PCG solve: k_pcg_resident_cg (SMEM-resident bricks, x in global memory)"


def e2e_run_spacetime(args, cfg, problem, lmesh, dof_step, world, local_rank):
    """Wall clock of the public call a user makes, ``run_spacetime(problem, schedule,
    local_mesh, T0, path, policy, recorder=None)`` over a K-macro-step schedule from the
    initial state: host planning (overlapped with the device by windows), the plan arrays
    H2D every step, the device run, every step's solve records D2H (checked against
    non-convergence), the final local field and trace D2H (the global field stays on the
    device until read: DeviceFieldState).  One untimed call over W steps first (allocation,
    setup caches); the device run is reused from the driver's pool."""
    import torch
    import paper_2110_12932_b200 as P
    from paper_2110_12932_b200 import multirate as MR
    T0 = P.uniform_field(problem.global_mesh, cfg.T_initial)
    K, W = args.steps, max(1, args.warmup)
    warm = MR.MacroSchedule(cfg.dt_macro, cfg.micro_steps, 0.0, W * cfg.dt_macro)
    st = P.run_spacetime(problem, warm, lmesh, T0, path=cfg.path, policy=cfg.policy)
    del st
    sched = MR.MacroSchedule(cfg.dt_macro, cfg.micro_steps, 0.0, K * cfg.dt_macro)
    stats = P.RunStats()
    pooled = list(MR._POOL.values())
    for r in pooled:
        r.h2d_bytes = r.d2h_bytes = 0
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    state = P.run_spacetime(problem, sched, lmesh, T0, path=cfg.path, policy=cfg.policy, stats=stats,
                            recorder=None)
    lv = state.local_field.values
    e2e_s = time.perf_counter() - t0
    assert np.isfinite(lv).all() and stats.counters["global_solves"] == K
    h2d = sum(r.h2d_bytes for r in MR._POOL.values()) // K
    d2h = sum(r.d2h_bytes for r in MR._POOL.values()) // K
    del state
    MR.release_device_runs()
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([e2e_s], device=torch.device("cuda", local_rank), dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    return {"value": dof_step * K * world / e2e_s, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "seconds": e2e_s, "steps": K,
            "note": f"host wall clock (max over ranks) of one public run_spacetime(..., recorder=None) call over a "
                    f"{K}-macro-step schedule from the initial state (macro steps 0..{K - 1}; value times steps "
                    f"{args.skip + args.warmup}..): host planning overlapped with the device in windows, the plan "
                    "arrays (macro/micro records, <=144 deposit samples) H2D every step, the solve records D2H and "
                    "checked, the final local field + trace D2H; the global field stays device-resident until read"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg4")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-flush", action="store_true")
    ap.add_argument("--skip", type=int, default=0, help="macro steps to run before warm-up")
    ap.add_argument("--slabs", action="store_true",
                    help="the multi-GPU driver (z-slab global solve, time-pipelined local steps) even at N = 1")
    ap.add_argument("--strong", action="store_true",
                    help="multi-GPU: cfg4 itself split over the ranks instead of the weak-scaling plate")
    ap.add_argument("--no-batch", action="store_true",
                    help="cfg5: one scenario after the other (SMEM-resident kernels) instead of batched solves")
    ap.add_argument("--scenarios", type=int, default=64,
                    help="cfg5: how many of the 64 seed-0 scenarios to run (split over the ranks)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        return reference_arm(args)
    if slab_mode(args, env_rank()[1]):
        return slab_bench(args)
    if args.config == "cfg5":
        return scenario_bench(args)
    if args.config == "picard":
        return picard_bench(args)
    return device_arm(args)


if __name__ == "__main__":
    main()

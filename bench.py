#!/usr/bin/env python
"""Benchmark: DOF-timesteps/s of the two-level multirate heat solve (BASELINE.json metric).

Workload (N=1): BASELINE config 2 — 5-track alternating scan, global 121x121x41
(600,281 nodes, h = 25 um), local 101x101x51 (520,251 nodes, h = 5 um), multirate
m = 10, fp64, Jacobi-PCG rtol 1e-12.  One "step" = one macro step of
``run_spacetime``: 1 global solve + 10 micro local solves + the corrector
re-solve + trace + relocation, i.e. N_g + m N_l = 5,802,791 DOF-timesteps
(the corrector re-solve is performed but not counted).

N > 1 (torchrun): every rank runs its own independent scenario replica on its GPU
(scenario sharding, no data-path collective, weak scaling); timing is the max
over ranks of the device time.  ``--impl reference`` times the reference's CPU
algorithm (the literal P1-assembly + scipy-CG port in oracle/assembly.py, pinned
bit-for-bit to the reference) on rank 0.

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

# the CPU baseline leg of our arm is single-threaded (a 1-core port timing); the reference
# arm runs with the library defaults, i.e. every host thread BLAS can use
_REFERENCE_ARM = "--impl=reference" in sys.argv or (
    "--impl" in sys.argv and sys.argv[sys.argv.index("--impl") + 1:][:1] == ["reference"])
if not _REFERENCE_ARM:
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
    from oracle import kuhn
    from oracle.twolevel import OracleRun
    cfg = P.load_config(cfg_path) if isinstance(cfg_path, (str, Path)) else cfg_path
    run = OracleRun(cfg, backend="assembly")
    Tg = np.full(run.G.n_nodes, cfg.T_initial)
    L = kuhn.KuhnGrid.from_placement(run.placement0)
    Tl = kuhn.interpolate(run.G, Tg, L.coords())
    sched = P.MacroSchedule(cfg.dt_macro, cfg.micro_steps, 0.0, cfg.t_end)
    t0 = time.perf_counter()
    dof = 0
    if "global" in what:
        Tg2 = run.solve_global(Tg, 0.0, cfg.dt_macro)
        dof += run.G.n_nodes
    else:
        Tg2 = Tg
    trace = run.trace_of(L, Tg2)
    w = 1.0 / sched.micro_per_macro
    run.solve_local(L, Tl, 0.0, sched.t_micro(0, 1), (1.0 - w) * run.trace_of(L, Tg) + w * trace)
    dof += L.n_nodes
    dt = time.perf_counter() - t0
    return dof, dt, run.iterations, (run.G.n_nodes, L.n_nodes, sched.micro_per_macro)


def _host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def reference_arm(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return
    cfg_path = ROOT / "configs" / f"{args.config}.cfg"
    if args.config == "cfg5":                 # config 5: a sample of its first scenario
        from paper_2110_12932_b200 import scenarios as S
        cfg_path = S.draw(0, 64)[0].config()
    times, dofs = [], []
    for s in range(args.warmup + args.steps):
        dof, dt, _, (Ng, Nl, m) = cpu_sample(cfg_path, what="local")
        if s >= args.warmup:
            times.append(dt)
            dofs.append(dof)
    total = sum(times)
    value = sum(dofs) / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic (BASELINE {args.config} geometry; uniform initial field, first micro step)",
        # the same workload as the device arm; each timed step is a bounded sample of it
        "config": {"workload": f"{args.config}: two-level multirate macro step (1 global + {m} local "
                               f"solves + corrector), global {Ng} + local {Nl} nodes",
                   "config_file": f"configs/{args.config}.cfg", "dof_timesteps_per_step": Ng + m * Nl,
                   "parallelism": "host CPU"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": _host_threads(), "kind": "port",
                         "sample": f"one {args.config} local micro solve ({Nl} DOF-timesteps) per timed step via the literal "
                                   "P1-assembly + scipy-CG port (oracle/assembly.py, bitwise equal to lpbfsim); "
                                   "library-default threading (BLAS may use every host thread; scipy's sparse "
                                   "CG itself is single-threaded)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def slab_bench(args):
    """--slabs: the global grid z-slab-decomposed over the ranks (strong scaling of one run),
    local problem on the top rank.  Default workload cfg4 (201M-node global grid)."""
    import torch
    import paper_2110_12932_b200 as P
    from paper_2110_12932_b200.multirate_dist import SlabRun
    from paper_2110_12932_b200.schedule import plan_spacetime

    rank, world, local_rank = env_rank()
    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    name = args.config if args.config != "cfg2" else "cfg4"
    cfg = P.load_config(ROOT / "configs" / f"{name}.cfg")
    problem, lmesh = P.build_problem(cfg, device=local_rank)
    sched = P.MacroSchedule(cfg.dt_macro, cfg.micro_steps, 0.0, cfg.t_end)
    m = sched.micro_per_macro
    Ng, Nl = problem.global_mesh.n_nodes, lmesh.n_nodes
    dof_step = Ng + m * Nl
    nsteps = args.warmup + args.steps
    plans = []
    placement, tg, tl = lmesh.placement, 0.0, 0.0
    for k in range(nsteps):
        pl = plan_spacetime(problem, sched, placement, cfg.path, cfg.policy, tg, tl, k0=k, nsteps=1)
        plans.append(pl)
        placement, tg, tl = pl.final_placement, pl.final_t_global, pl.final_t_local
    run = SlabRun(problem, lmesh, rank=rank, world=world, device=f"cuda:{local_rank}")
    run.initial(P.uniform_field(problem.global_mesh, cfg.T_initial))
    for k in range(args.warmup):
        run.step(plans[k])
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    l0 = run.solver.launches + (run.local.launch_count() if run.local is not None else 0)
    gi0 = len(run.global_infos)
    run.timing = True
    with ClockSampler(local_rank) as clocks:
        for (e0, e1), pl in zip(ev, plans[args.warmup:]):
            e0.record()
            run.step(pl)          # host-orchestrated: returns after the step's work completed
            e1.record()
        torch.cuda.synchronize()
    launches = run.solver.launches + (run.local.launch_count() if run.local is not None else 0) - l0
    dev_ms = float(sum(a.elapsed_time(b) for a, b in ev))
    if dist is not None:
        t = torch.tensor([dev_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dev_ms = float(t.item())
    gits = [inf.iterations for inf in run.global_infos[gi0:]]
    peak, peak_src = measured_peak()
    S = run.solver
    own = (S.k1 - S.k0) * S.nxy
    line = {
        "metric": METRIC, "value": dof_step * args.steps / (dev_ms / 1e3), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dev_ms / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic (BASELINE {name} scan path and geometry)",
        "config": {"workload": f"{name}: two-level multirate macro step, global grid on {world} z-slab(s), "
                               f"local problem on the top rank; global {Ng} + local {Nl} nodes",
                   "config_file": f"configs/{name}.cfg", "dof_timesteps_per_step": dof_step,
                   "parallelism": f"z-slabs x{world}", "l2": f"inputs larger than L2 ({Ng * 8 / 1e9:.1f} GB per vector)"},
        "global_iterations": float(np.mean(gits)) if gits else None,
        "phase_ms_per_step": {"deposit+global slab solve": float(np.mean([a for a, _ in run.phase_ms])),
                              "gather+local part": float(np.mean([b for _, b in run.phase_ms]))},
        "rank0_own_nodes": own, "gpu_launches": launches, "clocks": clocks.summary(),
        "roofline": None, "cpu_baseline": None, "e2e": None,
        "note": "slab mode is host-orchestrated per CG phase (two rank-ordered sums per iteration); "
                "peak for reference " + f"{peak:.0f} GB/s ({peak_src})",
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    run.close()
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

    def one_step(k, plan_of=None, after=None):
        """Macro step k of every scenario, device-ordered through event chaining."""
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
            e1.record(streams[-1])
            ev.append((e0, e1))
            last = e1
        for r in runs:
            r.sync()
        wall = time.perf_counter() - wall0
    torch.cuda.synchronize()
    launches = sum(r.launch_count() for r in runs) - launches0
    dev_ms = float(sum(a.elapsed_time(b) for a, b in ev))
    loc_rows, glo_rows = [], []
    for r in runs:
        infos = r.take_info()
        r.check_solves(infos)
        lo, gl = split_timing(r.take_timing(), infos)
        loc_rows.extend(lo)
        glo_rows.extend(gl)
        r.set_timing(False)
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
                "frac": kloc["achieved_gbs"] / peak, "traffic": None,
                "kernel": "local-grid PCG solves (k_pcg_resident_cg, SMEM-resident bricks, all micro solves "
                          "+ corrector of a macro step in one launch), pooled over the group's scenarios",
                "level": "local", "nodes": Nl, "peak_source": peak_src,
                "note": "algorithmic bytes N(64k+32) per solve (SURVEY §8d); each scenario's grids are "
                        "L2/SMEM-resident within its own macro step"}

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
    bottom Dirichlet) through the public seam fem.step_backward_euler, host buffers in and
    out.  One step = one Picard-converged implicit step: one tl_vc_picard_host call whose
    passes (assembly + one cooperative Jacobi-PCG launch + the increment reduction) run on
    the device.  value and e2e are the
    host wall clock around the public call (the seam takes host arrays); the roofline is
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
    stats = P.RunStats()
    stats.device_log = []
    walls = []
    with ClockSampler(local_rank) as clocks:
        for k in range(args.warmup, args.warmup + args.steps):
            t0 = time.perf_counter()
            state = step(state, k, stats)
            walls.append(time.perf_counter() - t0)
    wall = sum(walls)
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
                   "l2": "not flushed (host-buffer seam: each step uploads its fields and reads the result back)",
                   "parallelism": "single GPU"},
        "roofline": {"bound": "hbm", "achieved": alg / (cg_ms / 1e3) / 1e9 if cg_ms else None, "peak": peak,
                     "unit": "GB/s", "frac": (alg / (cg_ms / 1e3) / 1e9) / peak if cg_ms else None, "traffic": None,
                     "kernel": "k_vc_cg (one cooperative Jacobi-PCG launch per Picard pass)",
                     "share_of_step": cg_ms / 1e3 / wall, "peak_source": peak_src,
                     "note": "N (96 k + 32) bytes per pass; working set L2-resident at this size"},
        "cpu_baseline": cpu,
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": int(n * (8 + 8 + 1)),
                "d2h_bytes_per_step": int(n * 8),
                "note": "host wall clock around fem.step_backward_euler (the seam takes host arrays: T_old, "
                        "Dirichlet values and mask up, the converged field down, the Picard loop in between "
                        "on the device); value is the same"},
        "gpu_launches": int(passes * 7 - 2 * args.steps), "clocks": clocks.summary(),
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-flush", action="store_true")
    ap.add_argument("--skip", type=int, default=0, help="macro steps to run before warm-up")
    ap.add_argument("--slabs", action="store_true",
                    help="global grid split into z-slabs over the ranks (default config cfg4)")
    ap.add_argument("--scenarios", type=int, default=64,
                    help="cfg5: how many of the 64 seed-0 scenarios to run (split over the ranks)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        return reference_arm(args)
    if args.slabs:
        return slab_bench(args)
    if args.config == "cfg5":
        return scenario_bench(args)
    if args.config == "picard":
        return picard_bench(args)

    import torch
    import paper_2110_12932_b200 as P
    from paper_2110_12932_b200.schedule import plan_spacetime

    rank, world, local_rank = env_rank()
    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))

    cfg_path = ROOT / "configs" / f"{args.config}.cfg"
    cfg = P.load_config(cfg_path)
    problem, lmesh = P.build_problem(cfg, device=local_rank)
    sched = P.MacroSchedule(cfg.dt_macro, cfg.micro_steps, 0.0, cfg.t_end)
    m = sched.micro_per_macro
    Ng, Nl = problem.global_mesh.n_nodes, lmesh.n_nodes
    dof_step = Ng + m * Nl
    nsteps = args.skip + args.warmup + args.steps
    if nsteps > sched.n_macro:
        raise SystemExit(f"{args.config} has only {sched.n_macro} macro steps")

    # per-step plans (host, outside the timed region)
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
    step_ms = [a.elapsed_time(b) for a, b in ev]
    dev_ms = float(sum(step_ms))
    infos = run.take_info()
    run.check_solves(infos)
    kt = run.take_timing()
    run.set_timing(False)
    if dist is not None:
        t = torch.tensor([dev_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dev_ms = float(t.item())

    value = dof_step * len(timed) * world / (dev_ms / 1e3)

    # ---- roofline of the dominant kernel (k_pcg on the local grid) ----
    peak, peak_src = measured_peak()
    # pair each timed launch with the solve records it produced (a persistent local
    # launch runs all micro solves + corrector of a macro step)
    loc, glo = split_timing(kt, infos)
    share_ms = dev_ms if world == 1 else None
    kloc, kglo = kernel_stats(loc, Nl, share_ms), kernel_stats(glo, Ng, share_ms)
    # the dominant kernel: the level whose solves take the larger share of the step
    lev = "global" if kglo and (not kloc or sum(t for t, _ in glo) > sum(t for t, _ in loc)) else "local"
    kdom, ndom = (kglo, Ng) if lev == "global" else (kloc, Nl)
    streaming = "k_s_rhs -> k_t_cg (bulk-copy z-march CG loop, grids of 20M+ nodes) or k_s_cg -> k_s_resid -> k_s_final"
    kname = {"local": ("local-grid PCG solve: k_pcg_resident_cg (SMEM-resident bricks, all micro solves + corrector "
                       "of a macro step in one launch) where the grid fits on chip, else the streaming " + streaming),
             "global": "global-grid PCG solve: k_pcg_resident(_cg) where the grid fits on chip, else the streaming "
                       + streaming}[lev]
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
    roofline = {"bound": "hbm", "achieved": kdom["achieved_gbs"], "peak": peak, "unit": "GB/s",
                "frac": kdom["achieved_gbs"] / peak, "traffic": traffic, "traffic_note": tnote,
                "kernel": kname, "level": lev, "nodes": ndom,
                "peak_source": peak_src,
                "note": "algorithmic bytes N(64k+32) per solve (SURVEY §8d); cfg2 vectors are L2-resident"}

    # ---- e2e through the public API: pinned plan upload + field read-back every step ----
    e2e = None
    if rank == 0 or True:
        pin_local = torch.empty(Nl, dtype=torch.float64, pin_memory=True).numpy()
        e2e_plans = []
        for pl in timed:
            pinned = {}
            for key in ("macro", "micro"):
                arr = getattr(pl, key)
                buf = torch.empty(arr.nbytes, dtype=torch.uint8, pin_memory=True).numpy().view(arr.dtype)
                buf[:] = arr
                pinned[key] = buf
            for key in ("dep_points", "dep_power"):
                arr = np.ascontiguousarray(getattr(pl, key), dtype=np.float64).reshape(-1)
                buf = torch.empty(max(arr.size, 1), dtype=torch.float64, pin_memory=True).numpy()[:arr.size]
                buf[:] = arr
                pinned[key] = buf
            e2e_plans.append(pinned)
        # restart from the state after the timed region would differ; rewind a fresh run
        run2 = P.DeviceRun(problem, lmesh)
        run2.initial(P.uniform_field(problem.global_mesh, cfg.T_initial))
        for k in range(args.skip + args.warmup):
            run2.run(plans[k])
        run2.sync()
        h2d = d2h = 0
        # pipelined read-back: step s's local field goes to pinned buffer s % 2 on a copy
        # stream while step s+1 computes; the host waits for step s-1's field after
        # enqueueing step s, and for the last one before the clock stops
        pins = [pin_local, torch.empty(Nl, dtype=torch.float64, pin_memory=True).numpy()]
        for k in range(2):                       # staging buffers allocated before the clock
            run2.field_async(1, pins[k], slot=k)
            run2.field_wait(k)
        t0 = time.perf_counter()
        for s, (pl, pin) in enumerate(zip(timed, e2e_plans)):
            pl2 = type(pl)(macro=pin["macro"], micro=pin["micro"],
                           dep_points=pin["dep_points"].reshape(-1, 3), dep_power=pin["dep_power"])
            run2.run(pl2)
            run2.field_async(1, pins[s % 2], slot=s % 2)
            if s >= 1:
                run2.field_wait((s - 1) % 2)
            h2d += pin["macro"].nbytes + pin["micro"].nbytes + pin["dep_points"].nbytes + pin["dep_power"].nbytes
            d2h += pins[s % 2].nbytes
        run2.field_wait((len(timed) - 1) % 2)
        e2e_s = time.perf_counter() - t0
        run2.check_solves(run2.take_info())
        run2.close()
        e2e = {"value": dof_step * len(timed) * world / e2e_s, "unit": UNIT,
               "h2d_bytes_per_step": h2d // len(timed), "d2h_bytes_per_step": d2h // len(timed),
               "note": "host wall clock through DeviceRun.run per macro step: plan arrays from pinned "
                       "memory H2D, local field (the melt-pool grid) D2H to pinned memory every step "
                       "(DeviceRun.field_async, double-buffered: overlapped with the next step; "
                       "the last step's field is waited for inside the timed region)"}
    run.close()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        dof, dt, its, _ = cpu_sample(cfg_path)
        cpu = {"value": dof / dt, "unit": UNIT, "cores": 1, "kind": "port",
               "sample": f"one global + one local implicit step of {args.config} ({dof} DOF-timesteps, "
                         f"{dt:.1f} s) via the literal P1-assembly + scipy-CG port (oracle/assembly.py, "
                         "bitwise equal to lpbfsim); OPENBLAS_NUM_THREADS=1"}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": len(timed),
        "warmup": args.warmup, "ms_per_step": dev_ms / len(timed), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (BASELINE config 2 scan path and geometry; no dataset involved)",
        "config": {"workload": f"{args.config}: two-level multirate macro step (1 global + {m} local "
                               f"solves + corrector), global {Ng} + local {Nl} nodes",
                   "config_file": f"configs/{args.config}.cfg", "dof_timesteps_per_step": dof_step,
                   "macro_steps": f"{args.skip + args.warmup}..{nsteps - 1}",
                   "l2": "flushed between timed steps" if not args.no_flush else "not flushed",
                   "parallelism": f"scenario replicas x{world}" if world > 1 else "single GPU"},
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


if __name__ == "__main__":
    main()

"""Multirate / uniform two-level drivers — the device-resident hot loop.

Drop-in for ``lpbfsim.multirate`` (``lpbfsim/multirate.py``):

- ``run_spacetime(problem, schedule, local_mesh, T0, path, policy, stats, recorder)``
  (``:167-191``) and ``run_space(problem, dt, n_steps, ...)`` (``:194-217``) keep
  their signatures, recorder protocol (kinds ``initial``/``predictor``/``micro``/
  ``macro`` at the same points) and ``RunStats`` counters, but run the whole
  schedule as one device-resident ``tl_run``: fields never leave the GPU unless a
  recorder asks for them.
- ``macro_step`` (``:105-164``) and ``predictor_global`` / ``interpolate_trace``
  keep the reference's step-level behaviour on top of the seam-2 solves.
"""

from __future__ import annotations

import ctypes as C
import threading
import time
import weakref

import numpy as np

from . import _native as N
from .control import LocalPlacement, MacroSchedule
from .errors import CouplingError, NonConvergence, SolverError
from .fem import FieldState, device_rtol
from .grid import StructuredGrid
from .ops import raise_for
from .schedule import Plan, plan_space, plan_spacetime
from .errors import UnsupportedOnDevice
from .twolevel import (
    TwoLevelProblem, TwoLevelState, extract_interface, initial_state, relocate_local, solve_global,
    solve_local, two_level_iterate,
)

__all__ = ["MacroSchedule", "DeviceRun", "DeviceFieldState", "run_spacetime", "run_space", "macro_step",
           "predictor_global", "interpolate_trace", "release_device_runs"]


def _run_desc(problem: TwoLevelProblem, local_mesh: StructuredGrid, external_planes: int = 0) -> N.RunDesc:
    kappa, rcg, rcl = problem.constants()
    beam = problem.beam
    desc = N.RunDesc()
    desc.global_grid = problem.global_mesh.desc()
    desc.local_grid = local_mesh.desc()
    desc.kappa = kappa
    desc.rho_c_global = rcg
    desc.rho_c_local = rcl
    desc.T_buildplate = problem.bc.T_buildplate
    if beam is not None:
        desc.beam_peak, desc.beam_radius, desc.beam_depth = beam.gaussian_peak, beam.radius, beam.depth
    desc.rtol = device_rtol(problem.solver)
    desc.maxiter_factor = 20                 # fem.py:285
    desc.max_micro = 64
    desc.max_deposit = 512
    desc.device = problem.device
    desc.external_planes = int(external_planes)
    return desc


class DeviceRun:
    """Owns one ``tl_run``: both grids' fields and solver workspace on the GPU."""

    def __init__(self, problem: TwoLevelProblem, local_mesh: StructuredGrid, external_planes: int = 0):
        """``external_planes`` > 0: a local-only run of the multi-GPU driver (the global field
        arrives from the z-slab solve; only its top ``external_planes`` planes are stored)."""
        problem.check_device_supported()
        if not problem.one_way:
            raise UnsupportedOnDevice("the device-resident run is one-way; two-way coupling runs "
                                      "through the step-level drivers (run_spacetime / run_space)")
        self.problem = problem
        self.local_mesh = local_mesh
        desc = _run_desc(problem, local_mesh, external_planes)
        self.external_planes = int(external_planes)
        self._h = C.c_void_p()
        N.check(N.lib().tl_run_create(C.byref(desc), C.byref(self._h)), "tl_run_create")
        self.n_global = problem.global_mesh.n_nodes
        self.n_local = local_mesh.n_nodes
        self.solve_log: list = []
        self.key = bytes(desc)
        self.h2d_bytes = 0                # host->device bytes issued (plans, uploads)
        self.d2h_bytes = 0                # device->host bytes read (fields, solve records)
        # device-backed result fields not yet read back: materialised before the run's
        # state changes (initial / run / close), so they always see the values they named
        self._lazy = weakref.WeakSet()

    # -- lifecycle -----------------------------------------------------------------

    def close(self):
        if self._h:
            self._materialize_lazy()
            N.lib().tl_run_destroy(self._h)
            self._h = C.c_void_p()

    def _materialize_lazy(self):
        for f in list(self._lazy):
            f._materialize()
        self._lazy.clear()

    def lazy_field(self, which: int, mesh, time: float) -> "DeviceFieldState":
        """The run's current field `which` as a FieldState whose values are read back on
        first access (or before the run's state next changes)."""
        f = DeviceFieldState(mesh, time, self, which)
        self._lazy.add(f)
        return f

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
        return False

    # -- state -----------------------------------------------------------------------

    def initial(self, T0: FieldState):
        self._materialize_lazy()
        u = getattr(T0, "uniform_value", None)
        if u is not None:
            N.check(N.lib().tl_run_initial(self._h, float(u)), "tl_run_initial")
            return
        v = np.asarray(T0.values)
        if v.size and np.all(v == v.flat[0]):
            N.check(N.lib().tl_run_initial(self._h, float(v.flat[0])), "tl_run_initial")
        else:
            a = np.ascontiguousarray(v, dtype=np.float64)
            N.check(N.lib().tl_run_set_global(self._h, N.dptr(a), a.size), "tl_run_set_global")

    def field(self, which: int, out: np.ndarray | None = None) -> np.ndarray:
        n = self.n_global if which == 0 else self.n_local
        out = np.empty(n) if out is None else out
        N.check(N.lib().tl_run_get_field(self._h, which, N.dptr(out), n), "tl_run_get_field")
        self.d2h_bytes += out.nbytes
        return out

    def field_at(self, which: int, nodes: np.ndarray) -> np.ndarray:
        """Selected entries of a field, gathered on the device (only len(nodes) values cross)."""
        idx = np.ascontiguousarray(nodes, dtype=np.int32)
        out = np.empty(len(idx))
        N.check(N.lib().tl_run_get_field_at(self._h, which, idx.ctypes.data_as(C.c_void_p), len(idx), N.dptr(out)),
                "tl_run_get_field_at")
        self.d2h_bytes += out.nbytes
        self.h2d_bytes += idx.nbytes
        return out

    def field_async(self, which: int, out: np.ndarray, slot: int = 0) -> None:
        """Enqueue the read-back of a field into `out` (pinned memory for full overlap)
        and return at once; the run may continue.  Complete with field_wait(slot)."""
        n = self.n_global if which == 0 else self.n_local
        if out.shape != (n,) or out.dtype != np.float64 or not out.flags.c_contiguous:
            raise ValueError(f"out must be a contiguous float64 array of {n} values")
        N.check(N.lib().tl_run_field_async(self._h, which, N.dptr(out), n, slot), "tl_run_field_async")

    def field_wait(self, slot: int = 0) -> None:
        N.check(N.lib().tl_run_field_wait(self._h, slot), "tl_run_field_wait")

    def snapshot(self, which: int, index: int = 0) -> np.ndarray:
        n = self.n_global if which == 0 else self.n_local
        out = np.empty(n)
        self.d2h_bytes += out.nbytes
        N.check(N.lib().tl_run_get_snapshot(self._h, which, index, N.dptr(out), n), "snapshot")
        return out

    def run(self, plan: Plan):
        if self._lazy:
            self._materialize_lazy()
        macro = np.ascontiguousarray(plan.macro)
        micro = np.ascontiguousarray(plan.micro)
        pts = np.ascontiguousarray(plan.dep_points.reshape(-1), dtype=np.float64)
        pw = np.ascontiguousarray(plan.dep_power, dtype=np.float64)
        self.h2d_bytes += macro.nbytes + micro.nbytes + pts.nbytes + pw.nbytes
        N.check(N.lib().tl_run_macro_steps(
            self._h, macro.ctypes.data_as(C.c_void_p), len(macro), micro.ctypes.data_as(C.c_void_p),
            len(micro), N.dptr(pts), N.dptr(pw), len(pw)), "tl_run_macro_steps")

    def sync(self):
        N.check(N.lib().tl_run_sync(self._h), "tl_run_sync")

    def take_info(self) -> list:
        out = []
        buf = (N.SolveInfo * 4096)()
        cnt = C.c_int32()
        while True:
            N.check(N.lib().tl_run_take_info(self._h, buf, 4096, C.byref(cnt)), "take_info")
            out.extend({"iterations": buf[e].iterations, "status": buf[e].status,
                        "bnorm": buf[e].bnorm, "rnorm": buf[e].rnorm,
                        "true_resid": buf[e].true_resid} for e in range(cnt.value))
            self.d2h_bytes += cnt.value * C.sizeof(N.SolveInfo)
            if cnt.value < 4096:
                break
        self.solve_log.extend(out)
        return out

    def check_solves(self, infos):
        for inf in infos:
            raise_for(inf)

    def melt_summary(self, T_liquidus: float):
        out = np.empty(4)
        N.check(N.lib().tl_run_melt_summary(self._h, float(T_liquidus), N.dptr(out)), "melt")
        return {"global_max": out[0], "local_max": out[1], "global_melt_nodes": int(out[2]),
                "local_melt_nodes": int(out[3])}

    def stream(self) -> int:
        s = C.c_void_p()
        N.check(N.lib().tl_run_stream(self._h, C.byref(s)), "stream")
        return s.value or 0

    def launch_count(self) -> int:
        return int(N.lib().tl_run_launch_count(self._h))

    def set_timing(self, on: bool = True):
        N.check(N.lib().tl_run_set_timing(self._h, int(on)), "set_timing")

    def take_timing(self):
        """[(ms, level, nsolve)] of the solve launches since the last call (level 0 global,
        1 local; nsolve = solves run by that launch, in the order of take_info's records)."""
        out = []
        ms = (C.c_float * 4096)()
        lv = (C.c_int32 * 4096)()
        ns = (C.c_int32 * 4096)()
        cnt = C.c_int32()
        while True:
            N.check(N.lib().tl_run_take_timing(self._h, ms, lv, ns, 4096, C.byref(cnt)), "take_timing")
            out.extend((float(ms[e]), int(lv[e]), int(ns[e])) for e in range(cnt.value))
            if cnt.value < 4096:
                break
        return out

    def flush_l2(self):
        N.check(N.lib().tl_run_flush_l2(self._h), "flush")


class DeviceFieldState(FieldState):
    """A FieldState whose values still live on the device (device-resident
    fields are materialised as numpy only when asked).  ``values`` reads the field back on
    first access; the owning run materialises it before its state changes.  The device
    solve already checked the field for non-finite values (the true-residual pass counts
    them, ``fem.py:50-51``)."""

    def __init__(self, mesh, time: float, run: "DeviceRun", which: int):
        object.__setattr__(self, "mesh", mesh)
        object.__setattr__(self, "time", float(time))
        object.__setattr__(self, "_run", run)
        object.__setattr__(self, "_which", which)
        object.__setattr__(self, "_v", None)

    def _materialize(self):
        if self._v is None:
            v = self._run.field(self._which)
            v.setflags(write=False)
            object.__setattr__(self, "_v", v)
            object.__setattr__(self, "_run", None)
        return self._v

    @property
    def values(self) -> np.ndarray:
        return self._materialize()

    @property
    def on_device(self) -> bool:
        return self._v is None

    def __reduce__(self):
        return (FieldState, (self.mesh, self.values, self.time))

    __hash__ = object.__hash__          # identity: the owning run tracks it in a WeakSet

    def __repr__(self):
        return (f"DeviceFieldState(mesh={self.mesh!r}, time={self.time!r}, "
                f"{'on device' if self._v is None else 'read back'})")


class BatchedRuns:
    """BASELINE config 5 (``runner.py:376-380`` is the reference's concurrency point): a group
    of resident runs on local grids of ONE shape, advanced one macro step at a time with the
    i-th micro solve (and the corrector) of all runs batched into one streaming solve
    (``tl_runs_macro_step``, ``k_tb_cg``).  The systems advance in lockstep, each with its
    own scalars, stop test and iteration count; outcomes go to every run's info log."""

    def __init__(self, runs):
        self.runs = list(runs)
        if not 1 <= len(self.runs) <= 64:
            raise ValueError("a batch holds 1..64 runs")
        self._handles = (C.c_void_p * len(self.runs))(*[r._h for r in self.runs])

    def step(self, plans):
        """One macro step of every run; ``plans[r]`` is a one-step Plan of run r (no recorder)."""
        n = len(self.runs)
        if len(plans) != n:
            raise ValueError("one plan per run")
        keep = []
        macro = np.zeros(n, dtype=plans[0].macro.dtype)
        micro_p, nmicro, pts_p, pw_p, ndep = ((C.c_void_p * n)(), (C.c_int32 * n)(), (C.c_void_p * n)(),
                                              (C.c_void_p * n)(), (C.c_int32 * n)())
        for r, (run, pl) in enumerate(zip(self.runs, plans)):
            if pl.n_steps != 1:
                raise ValueError("batched steps take one-step plans")
            if run._lazy:
                run._materialize_lazy()
            macro[r] = pl.macro[0]
            mi = np.ascontiguousarray(pl.micro)
            pts = np.ascontiguousarray(pl.dep_points.reshape(-1), dtype=np.float64)
            pw = np.ascontiguousarray(pl.dep_power, dtype=np.float64)
            keep.extend((mi, pts, pw))
            micro_p[r], nmicro[r] = mi.ctypes.data, len(mi)
            pts_p[r], pw_p[r], ndep[r] = (pts.ctypes.data if len(pw) else None, pw.ctypes.data if len(pw) else None,
                                          len(pw))
            run.h2d_bytes += macro[r:r + 1].nbytes + mi.nbytes + pts.nbytes + pw.nbytes
        N.check(N.lib().tl_runs_macro_step(self._handles, n, macro.ctypes.data_as(C.c_void_p), micro_p, nmicro,
                                           pts_p, pw_p, ndep), "tl_runs_macro_step")

    def sync(self):
        for r in self.runs:
            r.sync()

    def check(self):
        for r in self.runs:
            r.check_solves(r.take_info())


# One idle tl_run per problem descriptor, reused by the next run_spacetime / run_space call
# of the same problem (a cfg4 run holds ~10 GB: allocation and release are not per call).
_POOL: dict = {}
_POOL_LOCK = threading.Lock()
_POOL_MAX = 2


def _acquire_run(problem, local_mesh) -> DeviceRun:
    key = bytes(_run_desc(problem, local_mesh))
    with _POOL_LOCK:
        run = _POOL.pop(key, None)
    if run is None or not run._h:
        return DeviceRun(problem, local_mesh)
    run.problem, run.local_mesh = problem, local_mesh      # same device descriptor
    return run


def _release_run(run: DeviceRun) -> None:
    evict = []
    with _POOL_LOCK:
        old = _POOL.pop(run.key, None)
        if old is not None and old is not run:
            evict.append(old)
        _POOL[run.key] = run
        while len(_POOL) > _POOL_MAX:
            evict.append(_POOL.pop(next(iter(_POOL))))
    for r in evict:
        r.close()


def release_device_runs() -> None:
    """Free the idle device runs kept for reuse (results not yet read back are read first)."""
    with _POOL_LOCK:
        runs = list(_POOL.values())
        _POOL.clear()
    for r in runs:
        r.close()


def _merge_counters(stats, counters: dict):
    if stats is None:
        return
    for k, v in counters.items():
        stats.count(k, v)


def _drive(problem, run: DeviceRun, plan_fn, local_mesh, T0, stats, recorder, t_initial,
           batch: int | None):
    """Shared driver: plan on the host, execute on the device, deliver records.

    Without a recorder the schedule is planned in growing windows (1, 2, 4, ... up to
    ``batch`` or 32 macro steps) and each window is enqueued before the next one is
    planned, so the host planning overlaps the device executing the previous window;
    a window's solve records are checked after the next window has been planned.  With
    a recorder every macro step is one window (its snapshots are delivered before the
    next step overwrites them)."""
    gmesh = problem.global_mesh
    run.initial(T0)
    if recorder is not None:
        lv = run.field(1)
        recorder("initial", t_initial, FieldState(local_mesh, lv, T0.time), T0, 0)
    t0 = time.perf_counter()
    k = 0
    placement, tg, tl = local_mesh.placement, T0.time, T0.time
    last_plan = pending = None
    window, cap = 1, (batch or 32)
    while True:
        nsteps = 1 if recorder is not None else window
        plan = plan_fn(placement, tg, tl, k, nsteps, recorder is not None)
        if pending is not None:                  # the previous window: outcome + counters
            infos = run.take_info()
            run.check_solves(infos)
            _merge_counters(stats, pending.counters)
            pending = None
        if plan.n_steps == 0:
            break
        keep = None
        if recorder is not None:
            keep = _decimate(plan, recorder)
        run.run(plan)
        if recorder is not None:
            infos = run.take_info()
            run.check_solves(infos)
            _merge_counters(stats, plan.counters)
            _deliver(run, problem, plan, infos, recorder, keep)
        else:
            pending = plan
        placement, tg, tl = plan.final_placement, plan.final_t_global, plan.final_t_local
        k += plan.n_steps
        last_plan = plan
        window = min(2 * window, cap)
    if stats is not None:
        stats.seconds["device_run"] = stats.seconds.get("device_run", 0.0) + time.perf_counter() - t0
    final_local = StructuredGrid(placement)
    gamma = extract_interface(final_local, gmesh)
    trace = run.field_at(2, gamma.trace_nodes)          # gathered on the device: only the trace crosses
    # both fields stay on the device until the caller reads them
    gfield = run.lazy_field(0, gmesh, tg)
    lfield = run.lazy_field(1, final_local, tl)
    return TwoLevelState(gfield, lfield, gamma, trace), last_plan


def _decimate(plan: Plan, recorder):
    """Snapshot decimation (``runner.py:216-233``: the experiment modes write every 10th micro
    field, or none): a recorder with a ``wants(kind, time) -> bool`` method is asked once per
    micro record, in order, whether it will read that record's field; the answers go to the
    device as the macro plan's ``record`` mask (fields nobody reads are neither snapshotted
    on the device nor copied to the host; their records arrive with ``local=None``).
    Returns the answers, or None for a plain recorder (every field delivered)."""
    wants = getattr(recorder, "wants", None)
    if wants is None or plan.mode != "spacetime":
        return None
    keep = [bool(wants("micro", ti)) for ti in plan.micro_times[0]]
    mask = 1
    for i, k in enumerate(keep):
        if k or i >= 30:
            mask |= 1 << (i + 1)
            keep[i] = True
    if all(keep):
        mask = 1
    plan.macro["record"][0] = mask
    return keep


def _deliver(run: DeviceRun, problem, plan: Plan, infos, recorder, keep=None):
    """Replay the recorder calls of one macro step from the device snapshots."""
    gmesh = problem.global_mesh
    mp = plan.macro[0]
    local_mesh = StructuredGrid(plan.placements[0])
    spacetime = plan.mode == "spacetime"
    gpred = run.snapshot(0)
    t_next = plan.t_next[0]
    if spacetime:
        recorder("predictor", t_next, None, FieldState(gmesh, gpred, plan.t_global[0]), 0)
        for i, ti in enumerate(plan.micro_times[0]):
            if keep is not None and not keep[i]:
                recorder("micro", ti, None, None, 0)          # decimated: nobody reads this field
                continue
            recorder("micro", ti, FieldState(local_mesh, run.snapshot(1, i), ti), None, 0)
    n = int(mp["n_micro"]) - 1 + int(mp["corrector"])
    lfinal = run.snapshot(1, n)
    recorder("macro", t_next, FieldState(local_mesh, lfinal, t_next),
             FieldState(gmesh, gpred, plan.t_global[0] if spacetime else t_next), 1)


def run_spacetime(problem: TwoLevelProblem, schedule: MacroSchedule, local_mesh: StructuredGrid,
                  T0: FieldState, path=None, policy=None, stats=None, recorder=None,
                  batch: int | None = None) -> TwoLevelState:
    """Multirate driver over the whole schedule (``multirate.py:167-191``) on the device.

    One-way constant-material problems run device-resident (``DeviceRun``); two-way
    coupling and temperature-dependent physics run the reference's loop over the
    step-level device solves (``_run_spacetime_steps``)."""
    if not problem.device_resident:
        return _run_spacetime_steps(problem, schedule, local_mesh, T0, path, policy, stats, recorder)
    extract_interface(local_mesh, problem.global_mesh)
    run = _acquire_run(problem, local_mesh)
    try:
        def plan_fn(placement, tg, tl, k, nsteps, record):
            return plan_spacetime(problem, schedule, placement, path, policy, tg, tl, k0=k,
                                  nsteps=nsteps, record=record)
        state, _ = _drive(problem, run, plan_fn, local_mesh, T0, stats, recorder,
                          schedule.t_start, batch)
    finally:
        _release_run(run)
    return state


def run_space(problem: TwoLevelProblem, dt: float, n_steps: int, local_mesh: StructuredGrid,
              T0: FieldState, path=None, policy=None, stats=None, recorder=None,
              batch: int | None = None) -> TwoLevelState:
    """Uniform-step driver (``multirate.py:194-217``) on the device (two-way coupling: the
    reference's loop over the step-level device solves, ``_run_space_steps``)."""
    if not problem.device_resident:
        return _run_space_steps(problem, dt, n_steps, local_mesh, T0, path, policy, stats, recorder)
    extract_interface(local_mesh, problem.global_mesh)
    run = _acquire_run(problem, local_mesh)
    try:
        def plan_fn(placement, tg, tl, k, nsteps, record):
            return plan_space(problem, dt, n_steps, placement, path, policy, T0.time, tg, k0=k,
                              nsteps=nsteps, record=record)
        state, _ = _drive(problem, run, plan_fn, local_mesh, T0, stats, recorder, T0.time, batch)
    finally:
        _release_run(run)
    return state


# -- step-level API (reference behaviour on the seam-2 solves) ----------------------------

def predictor_global(problem, state, dt, stats=None) -> FieldState:
    """``multirate.py:78-89``."""
    if stats is not None:
        stats.count("predictor_solves")
    return solve_global(problem, state, dt, state.local_field, stats=stats, predictor=True)


def interpolate_trace(i: int, m: int, trace_old, trace_pred):
    """``multirate.py:92-102``."""
    if not 0 <= i <= m:
        raise CouplingError(f"micro index {i} outside 0..{m}")
    w = i / m
    return (1.0 - w) * trace_old + w * trace_pred


def macro_step(problem, state: TwoLevelState, schedule: MacroSchedule, k: int, stats=None,
               recorder=None) -> TwoLevelState:
    """One predictor / micro / corrector cycle (``multirate.py:105-164``); the one-way +
    interval-source corrector re-solves only the last local interval, otherwise the
    corrector is the relaxed two-level fixed point (``two_level_iterate``)."""
    m = schedule.micro_per_macro
    delta = schedule.dt_micro
    t_next = schedule.t_macro(k + 1)
    predicted = predictor_global(problem, state, schedule.dt_macro, stats=stats)
    if recorder is not None:
        recorder("predictor", t_next, None, predicted, 0)
    trace_old = state.trace
    trace_pred = state.gamma.trace_of(predicted, problem.global_mesh)
    local = state.local_field
    before_final = state.local_field
    for i in range(m):
        t_i = schedule.t_micro(k, i + 1)
        trace_i = interpolate_trace(i + 1, m, trace_old, trace_pred)
        if i == m - 1:
            before_final = local
        local = solve_local(problem, local, t_i - local.time, state.gamma, trace_i, stats=stats)
        local = local.retimed(t_i)
        if recorder is not None:
            recorder("micro", t_i, local, None, 0)
    if problem.one_way and problem.interval_source:
        corrected = solve_local(problem, before_final, delta, state.gamma, trace_pred, stats=stats)
        corrected = corrected.retimed(t_next)
        if stats is not None:
            stats.count("coupling_iterations")
        new_state = TwoLevelState(predicted, corrected, state.gamma, trace_pred)
        iters = 1
    else:
        new_state, iters = two_level_iterate(problem, state, schedule.dt_macro, local_from=before_final,
                                             local_dt=delta, transmission_seed=local, trace_start=trace_pred,
                                             stats=stats)
    if recorder is not None:
        recorder("macro", t_next, new_state.local_field, new_state.global_field, iters)
    return new_state


def _restamp(state: TwoLevelState, t: float) -> TwoLevelState:
    return TwoLevelState(state.global_field.retimed(t), state.local_field.retimed(t),
                         state.gamma, state.trace)


def _run_spacetime_steps(problem, schedule, local_mesh, T0, path, policy, stats, recorder):
    """``run_spacetime`` (``multirate.py:167-191``) over the step-level device solves."""
    problem.check_device_supported(resident=False)
    state = initial_state(problem, local_mesh, T0)
    if recorder is not None:
        recorder("initial", schedule.t_start, state.local_field, state.global_field, 0)
    n = schedule.n_macro
    for k in range(n):
        state = macro_step(problem, state, schedule, k, stats=stats, recorder=recorder)
        if policy is not None and path is not None and k < n - 1:
            t = min(schedule.t_macro(k + 1), path.t_end)
            moved = relocate_local(state, policy, path.position(t), path.direction(t), problem)
            if moved is not state and stats is not None:
                stats.count("relocations")
            state = moved
    return state


def _run_space_steps(problem, dt, n_steps, local_mesh, T0, path, policy, stats, recorder):
    """``run_space`` (``multirate.py:194-217``) over the step-level device solves."""
    problem.check_device_supported(resident=False)
    state = initial_state(problem, local_mesh, T0)
    if recorder is not None:
        recorder("initial", T0.time, state.local_field, state.global_field, 0)
    for k in range(n_steps):
        t_next = T0.time + (k + 1) * dt
        state, iters = two_level_iterate(problem, state, t_next - state.time, stats=stats)
        state = _restamp(state, t_next)
        if recorder is not None:
            recorder("macro", t_next, state.local_field, state.global_field, iters)
        if policy is not None and path is not None and k < n_steps - 1:
            t = min(t_next, path.t_end)
            moved = relocate_local(state, policy, path.position(t), path.direction(t), problem)
            if moved is not state and stats is not None:
                stats.count("relocations")
            state = moved
    return state

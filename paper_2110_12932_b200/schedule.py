"""Host precomputation of the temperature-independent control schedule.

Everything the device loop needs besides the fields depends only on the scan
path and the time bookkeeping: the global step length,
the swept-track deposit samples of each macro interval, the local step length,
trace weight and Gaussian centre of every micro solve, and the local-box
placement after every relocation.  The loops below mirror the reference's own
float bookkeeping so every scalar lands on the same bits:

- spacetime:  ``run_spacetime`` / ``macro_step`` one-way branch
              (``lpbfsim/multirate.py:105-191``): global time accumulates
              ``t + dt_macro`` (``fem.py:326``); micro instants come from
              ``MacroSchedule.t_micro``; local step = ``t_i - local.time``; the
              corrector re-solves ``[before_final.time, +dt_micro]``.
- uniform:    ``run_space`` + one-way ``two_level_iterate``
              (``lpbfsim/multirate.py:194-217``, ``twolevel.py:299-358``).
- sources:    ``_local_source_factory`` / ``_global_source_factory``
              (``lpbfsim/runner.py:49-81``), ``SweptTrackDeposit.sample_points``
              (``lpbfsim/sources.py:137-162``).
- relocation: ``relocate_local`` shift/clamp (``lpbfsim/scanpath.py:219-241``)
              after every macro step except the last (``multirate.py:184-190``).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from ._native import MACRO_DTYPE, MICRO_DTYPE
from .control import LocalPlacement, MacroSchedule, check_immersed


def swept_samples(beam, pieces, dt: float):
    """8 x 3 x 3 samples per swept piece, each carrying P*eta*(len/v)/dt/72."""
    na, nc, nd = 8, 3, 3
    pts_all, pw_all = [], []
    r, d, v = beam.radius, beam.depth, beam.speed
    for a, b in pieces:
        a = np.asarray(a, dtype=float)
        b = np.asarray(b, dtype=float)
        track = b - a
        length = float(np.linalg.norm(track))
        if length == 0.0:
            continue
        that = track / length
        lat = np.array([-that[1], that[0], 0.0])
        u = (np.arange(na) + 0.5) / na * length
        w = ((np.arange(nc) + 0.5) / nc - 0.5) * r
        s = (np.arange(nd) + 0.5) / nd * d
        U, W, S = np.meshgrid(u, w, s, indexing="ij")
        pts = (a[None, :] + U.reshape(-1, 1) * that[None, :] + W.reshape(-1, 1) * lat[None, :]
               - S.reshape(-1, 1) * np.array([0.0, 0.0, 1.0]))
        power = beam.power * beam.absorptivity * (length / v) / dt
        pts_all.append(pts)
        pw_all.append(np.full(len(pts), power / len(pts)))
    if not pts_all:
        return np.empty((0, 3)), np.empty(0)
    return np.vstack(pts_all), np.concatenate(pw_all)


@dataclass
class Plan:
    """Device schedule for a window of macro steps."""

    macro: np.ndarray                 # MACRO_DTYPE
    micro: np.ndarray                 # MICRO_DTYPE
    dep_points: np.ndarray            # (n, 3)
    dep_power: np.ndarray             # (n,)
    t_next: list = field(default_factory=list)           # macro-instant time stamps
    t_global: list = field(default_factory=list)         # global FieldState times
    micro_times: list = field(default_factory=list)      # per step: micro instants
    placements: list = field(default_factory=list)       # placement in force during each step
    placement_after: list = field(default_factory=list)  # placement after each step
    moved: list = field(default_factory=list)            # relocation happened after step
    final_placement: LocalPlacement | None = None
    final_t_global: float = 0.0
    final_t_local: float = 0.0
    counters: dict = field(default_factory=dict)
    mode: str = "spacetime"

    @property
    def n_steps(self) -> int:
        return len(self.macro)


class _Builder:
    def __init__(self, problem, path, policy, record: bool):
        self.problem = problem
        self.path = path
        self.policy = policy
        self.record = record
        self.macro = []
        self.micro = []
        self.pts = []
        self.pw = []
        self.ndep = 0
        self.counters = {}
        tend = path.t_end if path is not None else 0.0
        self.tol = 1e-12 * max(tend, 1.0)

    def count(self, key, inc=1):
        self.counters[key] = self.counters.get(key, 0) + inc

    def center(self, t):
        """Gaussian centre at t, or None outside the path (``runner.py:49-61``)."""
        path = self.problem.path
        if path is None or self.problem.beam is None:
            return None
        if t > path.t_end + self.tol or t < path.t_start - self.tol:
            return None
        return path.position(t)

    def deposit(self, t0, t1):
        path = self.problem.path
        if path is None or self.problem.beam is None:
            return 0, 0
        pieces = path.swept_pieces(t0, t1)
        if not pieces:
            return self.ndep, 0
        pts, pw = swept_samples(self.problem.beam, pieces, t1 - t0)
        off = self.ndep
        self.pts.append(pts)
        self.pw.append(pw)
        self.ndep += len(pts)
        return off, len(pts)

    def add_micro(self, dt, w, t1):
        c = self.center(t1)
        self.micro.append((dt, w, (0.0, 0.0, 0.0) if c is None else tuple(float(v) for v in c),
                           0 if c is None else 1))

    def relocate(self, placement, t, k, n):
        if self.policy is None or self.path is None or k >= n - 1:
            return placement, False
        tt = min(t, self.path.t_end)
        moved = placement.relocate(self.policy, self.path.position(tt), self.path.direction(tt),
                                   self.problem.global_mesh.box)
        if moved is None:
            return placement, False
        # relocate_local re-extracts the interface (scanpath.py:244): strict immersion
        gm = self.problem.global_mesh
        check_immersed(moved.box, gm.box, gm.h)
        self.count("relocations")
        return moved, True

    def finish(self, plan_kw) -> Plan:
        macro = np.zeros(len(self.macro), dtype=MACRO_DTYPE)
        for e, row in enumerate(self.macro):
            for key, v in row.items():
                macro[e][key] = v
        micro = np.zeros(len(self.micro), dtype=MICRO_DTYPE)
        for e, (dt, w, c, on) in enumerate(self.micro):
            micro[e] = (dt, w, c, on)
        pts = np.vstack(self.pts) if self.pts else np.zeros((0, 3))
        pw = np.concatenate(self.pw) if self.pw else np.zeros(0)
        return Plan(macro=macro, micro=micro, dep_points=np.ascontiguousarray(pts),
                    dep_power=np.ascontiguousarray(pw), counters=self.counters, **plan_kw)


def plan_spacetime(problem, schedule: MacroSchedule, placement: LocalPlacement, path, policy,
                   t_global: float, t_local: float, k0: int = 0, nsteps: int | None = None,
                   record: bool = False) -> Plan:
    """Schedule of macro steps k0 .. k0+nsteps-1 of ``run_spacetime``."""
    n = schedule.n_macro
    stop = n if nsteps is None else min(n, k0 + nsteps)
    m, delta = schedule.micro_per_macro, schedule.dt_micro
    B = _Builder(problem, path, policy, record)
    kw = dict(t_next=[], t_global=[], micro_times=[], placements=[], placement_after=[], moved=[])
    corrector = 1 if problem.resolve_corrector else 0
    tg, tl = t_global, t_local
    for k in range(k0, stop):
        t_next = schedule.t_macro(k + 1)
        dep_off, dep_cnt = B.deposit(tg, tg + schedule.dt_macro)
        B.count("predictor_solves")
        B.count("global_solves")
        tg = tg + schedule.dt_macro
        micro_off = len(B.micro)
        times = []
        t_before = tl
        for i in range(m):
            t_i = schedule.t_micro(k, i + 1)
            if i == m - 1:
                t_before = tl
            dt_i = t_i - tl
            B.add_micro(dt_i, (i + 1) / m, tl + dt_i)
            B.count("local_solves")
            B.count("picard_iterations")
            times.append(t_i)
            tl = t_i
        # corrector: re-solve [before_final.time, +delta] with the predicted trace
        B.add_micro(delta, 1.0, t_before + delta)
        # counted as the reference counts it even when the device reuses the last
        # micro field instead of re-solving
        B.count("local_solves")
        B.count("picard_iterations")
        B.count("picard_iterations")          # the global solve's Picard pass
        B.count("coupling_iterations")
        tl = t_next
        kw["placements"].append(placement)
        placement, moved = B.relocate(placement, t_next, k, n)
        B.macro.append(dict(dt_global=schedule.dt_macro, dep_offset=dep_off, dep_count=dep_cnt,
                            micro_offset=micro_off, n_micro=m, corrector=corrector,
                            relocate=int(moved), record=int(record),
                            new_offset=tuple(placement.offset)))
        kw["t_next"].append(t_next)
        kw["t_global"].append(tg)
        kw["micro_times"].append(times)
        kw["placement_after"].append(placement)
        kw["moved"].append(moved)
    plan = B.finish(kw)
    plan.final_placement = placement
    plan.final_t_global = tg
    plan.final_t_local = tl
    return plan


def plan_space(problem, dt: float, n_steps: int, placement: LocalPlacement, path, policy,
               t0: float, t_state: float, k0: int = 0, nsteps: int | None = None,
               record: bool = False) -> Plan:
    """Schedule of steps k0 .. of ``run_space`` (uniform step on both levels)."""
    stop = n_steps if nsteps is None else min(n_steps, k0 + nsteps)
    B = _Builder(problem, path, policy, record)
    kw = dict(t_next=[], t_global=[], micro_times=[], placements=[], placement_after=[], moved=[])
    for k in range(k0, stop):
        t_next = t0 + (k + 1) * dt
        dtk = t_next - t_state
        dep_off, dep_cnt = B.deposit(t_state, t_state + dtk)
        B.count("global_solves")
        micro_off = len(B.micro)
        B.add_micro(dtk, 1.0, t_state + dtk)
        B.count("local_solves")
        B.count("picard_iterations", 2)
        B.count("coupling_iterations")
        t_state = t_next
        kw["placements"].append(placement)
        placement, moved = B.relocate(placement, t_next, k, n_steps)
        B.macro.append(dict(dt_global=dtk, dep_offset=dep_off, dep_count=dep_cnt,
                            micro_offset=micro_off, n_micro=1, corrector=0, relocate=int(moved),
                            record=int(record), new_offset=tuple(placement.offset)))
        kw["t_next"].append(t_next)
        kw["t_global"].append(t_next)
        kw["micro_times"].append([t_next])
        kw["placement_after"].append(placement)
        kw["moved"].append(moved)
    plan = B.finish(kw)
    plan.mode = "space"
    plan.final_placement = placement
    plan.final_t_global = t_state
    plan.final_t_local = t_state
    return plan

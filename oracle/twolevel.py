"""Two-level multirate / uniform drivers over the oracle discretization.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

Restates, for the one-way + interval-source branch every BASELINE config
takes (equal materials => ``TwoLevelProblem.one_way``, distributed global
source => ``interval_source``):

- ``initial_state``   — ``lpbfsim/twolevel.py:145-156``
- ``solve_global``    — ``lpbfsim/twolevel.py:242-271`` (transmission load is
                        identically zero for equal conductivities, ``:175``)
- ``solve_local``     — ``lpbfsim/twolevel.py:274-288``
- ``macro_step``      — ``lpbfsim/multirate.py:105-164`` (one-way branch ``:144-155``)
- ``run_spacetime``   — ``lpbfsim/multirate.py:167-191``
- ``run_space``       — ``lpbfsim/multirate.py:194-217`` with the one-way pass of
                        ``two_level_iterate`` (``lpbfsim/twolevel.py:299-358``)
- ``relocate_local``  — ``lpbfsim/scanpath.py:208-248``
- ``run_reference``   — ``lpbfsim/runner.py:126-163`` → ``fem.solve_monolithic``
                        (``lpbfsim/fem.py:386-423``): the true beam on one fine grid

Times follow the reference's float bookkeeping exactly (global time accumulates
``t + dt``; local micro times come from ``MacroSchedule.t_micro``).
"""

from __future__ import annotations

import numpy as np

from paper_2110_12932_b200.control import (
    LocalPlacement, MacroSchedule, initial_local_box, material_constants, structured_ncells,
)

from . import kuhn
from .pcg import solve_constrained


class OracleRun:
    """Holds the grids and the per-level solver for one experiment config."""

    def __init__(self, cfg, backend: str = "stencil"):
        self.cfg = cfg
        gbox = cfg.global_box
        self.G = kuhn.KuhnGrid(gbox.lo, gbox.hi, structured_ncells(gbox, cfg.h_global))
        if cfg.policy is not None:
            lbox = initial_local_box(gbox, cfg.h_local, cfg.policy, cfg.path)
        else:
            lbox = cfg.local_box
        self.placement0 = LocalPlacement(lbox, structured_ncells(lbox, cfg.h_local))
        self.kappa, self.rhoc = material_constants(cfg.material)
        self.rtol = cfg.solver.linear_tol
        self.backend = backend
        self.iterations = []          # (kind, its) per solve
        self.counters = {}
        tol = 1e-12 * max(cfg.path.t_end, 1.0)
        self._src_tol = tol
        if backend == "assembly":
            from . import assembly
            self._assembly = assembly

    # -- sources --------------------------------------------------------------

    def local_center(self, t: float):
        """``_local_source_factory`` (``lpbfsim/runner.py:49-61``)."""
        path = self.cfg.path
        if t > path.t_end + self._src_tol or t < path.t_start - self._src_tol:
            return None
        return path.position(t)

    def deposit(self, t0: float, t1: float):
        """``_global_source_factory`` distributed branch (``lpbfsim/runner.py:75-79``)."""
        pieces = self.cfg.path.swept_pieces(t0, t1)
        if not pieces:
            return None
        pts, pw = kuhn.swept_samples(self.cfg.beam, pieces, t1 - t0)
        return kuhn.deposit_load(self.G, pts, pw)

    def _count(self, key):
        self.counters[key] = self.counters.get(key, 0) + 1

    # -- the two solves ---------------------------------------------------------

    def solve_global(self, Tg: np.ndarray, t0: float, dt: float) -> np.ndarray:
        load = self.deposit(t0, t0 + dt)
        g = np.full(self.G.n_nodes, self.cfg.bc.T_buildplate)
        if self.backend == "assembly":
            x, its = self._assembly.step(self.G, self.kappa, self.rhoc, dt, self.G.bottom_mask(),
                                         Tg, None, load, g, self.rtol)
        else:
            op = kuhn.StencilOperator(self.G, self.kappa, self.rhoc, dt, self.G.bottom_mask())
            b = op.rhs(Tg, load, g)
            x, its, _ = solve_constrained(op, b, g, self.rtol)
        self.iterations.append(("global", its))
        self._count("global_solves")
        return x

    def solve_local(self, L: kuhn.KuhnGrid, Tl: np.ndarray, t_from: float, dt: float,
                    trace: np.ndarray) -> np.ndarray:
        t1 = t_from + dt
        center = self.local_center(t1)
        if self.backend == "assembly":
            x, its = self._assembly.step(L, self.kappa, self.rhoc, dt, L.gamma_mask(), Tl,
                                         (self.cfg.beam, center) if center is not None else None,
                                         None, trace, self.rtol)
        else:
            load = kuhn.gaussian_load(L, self.cfg.beam, center) if center is not None else None
            op = kuhn.StencilOperator(L, self.kappa, self.rhoc, dt, L.gamma_mask())
            b = op.rhs(Tl, load, trace)
            x, its, _ = solve_constrained(op, b, trace, self.rtol)
        self.iterations.append(("local", its))
        self._count("local_solves")
        return x

    def trace_of(self, L: kuhn.KuhnGrid, Tg: np.ndarray) -> np.ndarray:
        """Dense local array holding P1(Tg) on the gamma nodes (0 elsewhere)."""
        out = np.zeros(L.n_nodes)
        gam = L.gamma_mask().ravel()
        out[gam] = kuhn.interpolate(self.G, Tg, L.coords()[gam])
        return out

    # -- drivers ---------------------------------------------------------------

    def initial(self, T0_value: float):
        Tg = np.full(self.G.n_nodes, float(T0_value))
        L = kuhn.KuhnGrid.from_placement(self.placement0)
        Tl = kuhn.interpolate(self.G, Tg, L.coords())
        return Tg, Tl, self.trace_of(L, Tg)

    def _relocate(self, placement, Tg, t_macro_next):
        cfg = self.cfg
        t = min(t_macro_next, cfg.path.t_end)
        moved = placement.relocate(cfg.policy, cfg.path.position(t), cfg.path.direction(t),
                                   cfg.global_box)
        if moved is None:
            return placement, None
        L = kuhn.KuhnGrid.from_placement(moved)
        Tl = kuhn.interpolate(self.G, Tg, L.coords())
        self._count("relocations")
        return moved, (Tl, self.trace_of(L, Tg))

    def run_spacetime(self, n_steps: int | None = None, recorder=None, resolve_corrector=True):
        """Yields per macro step; ``recorder(kind, t, local, global, placement)``."""
        cfg = self.cfg
        sched = MacroSchedule(cfg.dt_macro, cfg.micro_steps, 0.0, cfg.t_end)
        n = sched.n_macro
        steps = n if n_steps is None else min(n_steps, n)
        m, delta = sched.micro_per_macro, sched.dt_micro
        Tg, Tl, trace = self.initial(cfg.T_initial)
        tg = 0.0
        placement = self.placement0
        if recorder:
            recorder("initial", 0.0, Tl, Tg, placement)
        for k in range(steps):
            t_next = sched.t_macro(k + 1)
            L = kuhn.KuhnGrid.from_placement(placement)
            Tg_pred = self.solve_global(Tg, tg, cfg.dt_macro)
            self._count("predictor_solves")
            tg = tg + cfg.dt_macro
            trace_pred = self.trace_of(L, Tg_pred)
            tl = sched.t_macro(k) if k > 0 else 0.0
            local = Tl
            before_final, t_before = Tl, tl
            for i in range(m):
                t_i = sched.t_micro(k, i + 1)
                w = (i + 1) / m
                trace_i = (1.0 - w) * trace + w * trace_pred
                if i == m - 1:
                    before_final, t_before = local, tl
                local = self.solve_local(L, local, tl, t_i - tl, trace_i)
                tl = t_i
            if resolve_corrector:
                local = self.solve_local(L, before_final, t_before, delta, trace_pred)
            self._count("coupling_iterations")
            Tg, Tl, trace = Tg_pred, local, trace_pred
            if recorder:
                recorder("macro", t_next, Tl, Tg, placement)
            if cfg.policy is not None and k < n - 1:
                placement, moved = self._relocate(placement, Tg, t_next)
                if moved is not None:
                    Tl, trace = moved
        return Tg, Tl, placement

    def run_reference(self, h: float | None = None, dt: float | None = None,
                      n_steps: int | None = None):
        """Monolithic fine-grid reference: uniform steps on the plate at ``h_reference`` with
        the Gaussian beam at each target time and the bottom Dirichlet set.  Returns
        (times, fields)."""
        cfg = self.cfg
        h = cfg.h_reference if h is None else h
        dt = cfg.dt_reference if dt is None else dt
        n = int(round(cfg.t_end / dt)) if n_steps is None else n_steps
        gbox = cfg.global_box
        R = kuhn.KuhnGrid(gbox.lo, gbox.hi, structured_ncells(gbox, h))
        g = np.full(R.n_nodes, cfg.bc.T_buildplate)
        T = np.full(R.n_nodes, cfg.T_initial)
        times, fields = [0.0], [T]
        for k in range(1, n + 1):
            t_new = 0.0 + k * dt
            center = self.local_center(t_new)
            step_dt = t_new - times[-1]
            load = kuhn.gaussian_load(R, cfg.beam, center) if center is not None else None
            op = kuhn.StencilOperator(R, self.kappa, self.rhoc, step_dt, R.bottom_mask())
            T, its, _ = solve_constrained(op, op.rhs(T, load, g), g, self.rtol)
            self.iterations.append(("reference", its))
            self._count("reference_solves")
            times.append(t_new)
            fields.append(T)
        return times, fields

    def run_space(self, n_steps: int | None = None, recorder=None):
        cfg = self.cfg
        dt = cfg.dt_macro / cfg.micro_steps
        n = int(round(cfg.t_end / dt))
        steps = n if n_steps is None else min(n_steps, n)
        Tg, Tl, trace = self.initial(cfg.T_initial)
        t_state = 0.0
        placement = self.placement0
        if recorder:
            recorder("initial", 0.0, Tl, Tg, placement)
        for k in range(steps):
            t_next = 0.0 + (k + 1) * dt
            dtk = t_next - t_state
            L = kuhn.KuhnGrid.from_placement(placement)
            Tg = self.solve_global(Tg, t_state, dtk)
            trace = self.trace_of(L, Tg)
            Tl = self.solve_local(L, Tl, t_state, dtk, trace)
            self._count("coupling_iterations")
            t_state = t_next
            if recorder:
                recorder("macro", t_next, Tl, Tg, placement)
            if cfg.policy is not None and k < n - 1:
                placement, moved = self._relocate(placement, Tg, t_next)
                if moved is not None:
                    Tl, trace = moved
        return Tg, Tl, placement

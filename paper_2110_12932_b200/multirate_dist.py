"""Multirate two-level run with the global grid split into z-slabs across ranks.

Multi-GPU form of ``run_spacetime`` (``lpbfsim/multirate.py:167-191``, one-way
branch ``:144-155``), one process per GPU.  Per macro step:

1. every rank deposits the swept-track load of the interval on its own nodes
   (``SweptTrackDeposit.load``, ``sources.py:164-172``) and takes part in the
   global backward-Euler solve (``twolevel.solve_global``, ``twolevel.py:242-271``)
   through :class:`~.slab.SlabGlobalSolver`;
2. the planes of the new global field that lie under the local box (the only part
   trace and relocation read) are gathered on the top rank;
3. the top rank runs the local part of the macro step on its ``tl_run`` in
   external-global mode: interface trace, the m micro solves, the corrector,
   relocation (``multirate.py:129-162``, ``scanpath.py:208-248``).

Coupling is one way, so the local part never feeds back into the global solve.
The host schedule (deposit samples, micro instants, relocation offsets) is the
same deterministic plan every rank computes (``schedule.plan_spacetime``).
"""

from __future__ import annotations

import time

import numpy as np

from . import _native as N
from .fem import FieldState, device_rtol
from .grid import StructuredGrid
from .multirate import DeviceRun, _merge_counters
from .ops import raise_for
from .schedule import plan_spacetime
from .slab import SlabGlobalSolver, _dist
from .twolevel import TwoLevelState, extract_interface


def _first_plane_under(global_mesh, local_mesh) -> int:
    """Lowest global node plane a P1 location inside the local box can touch."""
    zg = np.asarray(global_mesh.axis(2))
    zlo = float(np.asarray(local_mesh.axis(2))[0])
    return max(0, int(np.searchsorted(zg, zlo, side="right")) - 2)


class SlabRun:
    """One rank's share of a slab-decomposed two-level run."""

    def __init__(self, problem, local_mesh, *, rank: int = 0, world: int = 1, group=None, device=None):
        problem.check_device_supported()
        extract_interface(local_mesh, problem.global_mesh)
        self.problem = problem
        self.rank, self.world, self.group = rank, world, group
        self.root = world - 1                      # owns the top plane, hosts the local problem
        kappa, rcg, _ = problem.constants()
        self.solver = SlabGlobalSolver(problem.global_mesh, kappa, rcg, rank=rank, world=world, group=group,
                                       device=device, rtol=device_rtol(problem.solver))
        self.local = None
        if rank == self.root:
            self.local = DeviceRun(problem, local_mesh)
            N.check(N.lib().tl_run_set_external_global(self.local._h, 1), "external global")
        self.global_infos: list = []
        self.phase_ms: list = []       # (global ms, local ms) per step when timing is on
        self.timing = False

    def close(self):
        if self.local is not None:
            self.local.close()
            self.local = None

    def initial(self, T0: FieldState):
        v = np.asarray(T0.values)
        n = self.problem.global_mesh.n_nodes
        full = v if v.size == n else np.full(n, float(v.flat[0]))
        self.solver.set_own(self.solver.x, np.ascontiguousarray(full, dtype=np.float64))
        if self.local is not None:
            self.local.initial(T0)

    def step(self, plan) -> None:
        """Execute one macro step of ``plan`` (a one-step ``plan_spacetime`` window)."""
        import torch
        mp = plan.macro[0]
        a, n = int(mp["dep_offset"]), int(mp["dep_count"])
        S = self.solver
        if self.timing:
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            ev[0].record()
        S.deposit(plan.dep_points[a:a + n], plan.dep_power[a:a + n])
        info = S.step(float(mp["dt_global"]), self.problem.bc.T_buildplate, with_load=True)
        raise_for(info)
        self.global_infos.append(info)
        if self.timing:
            ev[1].record()
        k_lo = min(_first_plane_under(self.problem.global_mesh, StructuredGrid(p))
                   for p in (plan.placements[0], plan.placement_after[0]))
        block = S.gather_planes(k_lo, self.root)
        if self.local is not None:
            torch.cuda.current_stream(S.device).synchronize()
            N.check(N.lib().tl_run_put_global_planes(self.local._h, block.data_ptr(), k_lo, S.nz),
                    "put global planes")
            self.local.run(plan)
            infos = self.local.take_info()
            self.local.check_solves(infos)
        if self.timing:
            ev[2].record()
            ev[2].synchronize()
            self.phase_ms.append((ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2])))


def run_spacetime_slabs(problem, schedule, local_mesh: StructuredGrid, T0: FieldState, path=None,
                        policy=None, stats=None, *, group=None, device=None):
    """``run_spacetime`` across the ranks of the current process group.

    Returns the final :class:`TwoLevelState` on the top rank (which holds the local
    problem; its global field is the gathered whole grid) and ``None`` elsewhere.
    """
    d = _dist()
    rank = d.get_rank(group) if d is not None else 0
    world = d.get_world_size(group) if d is not None else 1
    run = SlabRun(problem, local_mesh, rank=rank, world=world, group=group, device=device)
    try:
        run.initial(T0)
        t0 = time.perf_counter()
        placement, tg, tl, k = local_mesh.placement, T0.time, T0.time, 0
        while True:
            plan = plan_spacetime(problem, schedule, placement, path, policy, tg, tl, k0=k, nsteps=1)
            if plan.n_steps == 0:
                break
            run.step(plan)
            if rank == run.root:
                _merge_counters(stats, plan.counters)
            placement, tg, tl = plan.final_placement, plan.final_t_global, plan.final_t_local
            k += 1
        if stats is not None and rank == run.root:
            stats.seconds["device_run"] = stats.seconds.get("device_run", 0.0) + time.perf_counter() - t0
        gv = run.solver.gather_field(run.root)
        if rank != run.root:
            return None
        gmesh = problem.global_mesh
        final_local = StructuredGrid(placement)
        lv = run.local.field(1)
        gamma = extract_interface(final_local, gmesh)
        trace = run.local.field(2)[gamma.trace_nodes]
        return TwoLevelState(FieldState(gmesh, gv, tg), FieldState(final_local, lv, tl), gamma, trace)
    finally:
        run.close()

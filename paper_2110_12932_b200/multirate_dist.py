"""Multirate two-level run on several GPUs: global grid in z-slabs, local problem
pipelined over the ranks in time.

Multi-GPU form of ``run_spacetime`` (``lpbfsim/multirate.py:167-191``, one-way branch
``:144-155``), one process per GPU.

Global level.  Every macro step every rank deposits the swept-track load of the
interval on its own nodes (``SweptTrackDeposit.load``, ``sources.py:164-172``) and
takes part in the global backward-Euler solve (``twolevel.solve_global``,
``twolevel.py:242-271``) through the device-resident :class:`~.slab.SlabGlobalSolver`.

Local level.  Coupling is one way, so the local part of macro step k reads only the
global fields T_g(k) and T_g(k+1) and, when the box did not move after step k-1, the
local field of step k-1.  In every BASELINE config the box moves after every step
(``relocate_local`` re-interpolates the WHOLE local field from the global one,
``scanpath.py:243-248``), so the local parts of different macro steps are independent.
The run is cut into *chains* (a chain starts at step 0 and after every relocation) and
chain c runs on rank c mod world.  A *super-step* is `world` consecutive chains: all
ranks solve the super-step's global steps together, then each rank runs its chain's
local steps (trace, m micro solves, corrector) on its own ``tl_run`` in local-only mode
— concurrently on all ranks, with no collective — so the local work, which does not
grow with the global grid, is divided by the number of GPUs instead of serialising on
the rank under the laser.

Data movement per macro step: the planes of T_g(k+1) under the local box (from the
owning rank(s), ``[k_win, nz)``, ``_first_plane_under``) go to the rank running step k
(its predicted trace) and, if step k+1 starts a chain, to that chain's rank (its
re-anchored initial field, ``tl_run_reanchor``).  The host schedule (deposit samples,
micro instants, relocation offsets) is the same deterministic plan on every rank
(``schedule.plan_spacetime``).
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
from .slab import SlabGlobalSolver, _dist, plane_partition
from .twolevel import TwoLevelState, extract_interface


def _first_plane_under(global_mesh, local_mesh) -> int:
    """Lowest global node plane a P1 location inside the local box can touch."""
    zg = np.asarray(global_mesh.axis(2))
    zlo = float(np.asarray(local_mesh.axis(2))[0])
    return max(0, int(np.searchsorted(zg, zlo, side="right")) - 2)


def chain_ranks(moved_before: bool, moved: list, first_chain: int, world: int):
    """Chain starts and ranks of a window of steps.  ``moved_before``: the box moved after
    the step preceding the window (True for step 0); ``moved[i]``: it moves after step i.
    Returns (starts, ranks, chains used)."""
    starts, ranks = [], []
    c = first_chain - 1
    prev = moved_before
    for mv in moved:
        if prev:
            c += 1
        starts.append(bool(prev))
        ranks.append(c % world)
        prev = mv
    return starts, ranks, c + 1 - first_chain


class SlabRun:
    """One rank's share of a slab-decomposed, time-pipelined two-level run."""

    def __init__(self, problem, local_mesh, *, rank: int = 0, world: int = 1, group=None, device=None):
        import torch
        problem.check_device_supported()
        extract_interface(local_mesh, problem.global_mesh)
        self.problem = problem
        self.rank, self.world, self.group = rank, world, group
        kappa, rcg, _ = problem.constants()
        self.solver = SlabGlobalSolver(problem.global_mesh, kappa, rcg, rank=rank, world=world, group=group,
                                       device=device, rtol=device_rtol(problem.solver))
        S = self.solver
        self.k_win = _first_plane_under(problem.global_mesh, local_mesh)
        self.local = DeviceRun(problem, local_mesh, external_planes=S.nz - self.k_win)
        self.local_stream = torch.cuda.ExternalStream(self.local.stream(), device=S.device)
        self.parts = plane_partition(S.nz, world)
        self.chains = 0                 # chains started so far
        self.moved_before = True        # step 0 starts a chain
        self.step_index = 0             # macro steps executed
        self.old: dict = {}             # step -> T_g(step) window (chain starts on this rank)
        self.pending_infos = 0          # local steps whose solve records are not yet checked
        self.global_infos: list = []
        self.global_ms: list = []       # per global solve (timing on)
        self.timing = False
        self.last_rank = 0
        d = _dist()
        if world > 1 and d is not None:
            # a collective before the first point-to-point transfer (NCCL requires every
            # rank of the group in the first call; the first window involves two ranks)
            d.barrier(group=group)

    def close(self):
        if self.local is not None:
            # the window buffers were recorded on the local run's stream (record_stream):
            # release them to the allocator while that stream still exists
            import torch
            self.old.clear()
            torch.cuda.synchronize(self.solver.device)
            torch.cuda.empty_cache()
            self.local.close()
            self.local = None

    # -- global -> local window ----------------------------------------------------------
    def _window(self, dsts) -> "object":
        """Planes [k_win, nz) of the solver's current x to every rank in ``dsts``; returns
        this rank's copy (None if it is not a destination).  Owners send their planes;
        NCCL moves them device to device, other backends through host memory."""
        import torch
        S, me = self.solver, self.rank
        nxy, kw = S.nxy, self.k_win
        buf = torch.empty((S.nz - kw) * nxy, dtype=torch.float64, device=S.device) if me in dsts else None
        d = _dist()
        staged, ops = [], []
        for dst in sorted(dsts):
            for o, (k0, k1) in enumerate(self.parts):
                a, b = max(k0, kw), k1
                if a >= b:
                    continue
                if o == me and dst == me:
                    buf[(a - kw) * nxy:(b - kw) * nxy].copy_(S.plane_block(a, b))
                elif o == me:
                    if S.comm.nccl:
                        ops.append(d.P2POp(d.isend, S.plane_block(a, b), dst, self.group))
                    else:
                        ops.append(d.isend(S.plane_block(a, b).detach().cpu(), dst, group=self.group))
                elif dst == me:
                    if S.comm.nccl:
                        ops.append(d.P2POp(d.irecv, buf[(a - kw) * nxy:(b - kw) * nxy], o, self.group))
                    else:
                        t = torch.empty((b - a) * nxy, dtype=torch.float64)
                        ops.append(d.irecv(t, o, group=self.group))
                        staged.append((a, b, t))
        if ops:
            works = d.batch_isend_irecv(ops) if S.comm.nccl else ops
            for w in works:
                w.wait()
        for a, b, t in staged:
            buf[(a - kw) * nxy:(b - kw) * nxy].copy_(t.to(S.device))
        return buf

    def _put(self, buf) -> None:
        import torch
        # the window was written on the current stream; the local run's stream reads it
        self.local_stream.wait_stream(torch.cuda.current_stream(self.solver.device))
        buf.record_stream(self.local_stream)
        N.check(N.lib().tl_run_put_global_planes(self.local._h, buf.data_ptr(), self.k_win, self.solver.nz),
                "put global planes")

    # -- state ---------------------------------------------------------------------------
    def initial(self, T0: FieldState):
        S = self.solver
        u = getattr(T0, "uniform_value", None)
        if u is not None:
            S.own_view(S.x).fill_(float(u))
        else:
            S.set_own(S.x, np.ascontiguousarray(np.asarray(T0.values), dtype=np.float64))

    # -- one super-step ------------------------------------------------------------------
    def superstep(self, plans) -> None:
        """Global solves of the consecutive one-step ``plans`` (all ranks), then every
        rank's local steps.  ``plans`` should hold whole chains (``plan_superstep``)."""
        import torch
        problem, S, me = self.problem, self.solver, self.rank
        moved = [bool(pl.moved[0]) for pl in plans]
        starts, ranks, used = chain_ranks(self.moved_before, moved, self.chains, self.world)
        k_first = self.step_index
        pred = {}
        if starts[0]:                       # T_g(k_first): the first chain's initial field
            buf = self._window({ranks[0]})
            if buf is not None:
                self.old[k_first] = buf
        for i, pl in enumerate(plans):
            mp = pl.macro[0]
            a, n = int(mp["dep_offset"]), int(mp["dep_count"])
            if self.timing:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
            S.deposit(pl.dep_points[a:a + n], pl.dep_power[a:a + n])
            info = S.step(float(mp["dt_global"]), problem.bc.T_buildplate, with_load=True)
            if self.timing:
                e1.record()
                self.global_ms.append((e0, e1, info.iterations))
            raise_for(info)
            self.global_infos.append(info)
            # T_g(k+1): the predicted global field of step k, and the initial field of the
            # next chain when one starts at k+1 (its rank: the next chain's)
            dsts = {ranks[i]}
            nxt_rank = None
            if moved[i]:
                nxt_rank = ranks[i + 1] if i + 1 < len(plans) else (self.chains + used) % self.world
                dsts.add(nxt_rank)
            buf = self._window(dsts)
            if buf is not None:
                if me == ranks[i]:
                    pred[k_first + i] = buf
                if nxt_rank == me:
                    self.old[k_first + i + 1] = buf
        # local phase: this rank's steps, in order, on the local run's stream
        for i, pl in enumerate(plans):
            if ranks[i] != me:
                continue
            k = k_first + i
            if starts[i]:
                self._put(self.old.pop(k))
                off = np.ascontiguousarray(pl.placements[0].offset, dtype=np.float64)
                N.check(N.lib().tl_run_reanchor(self.local._h, off.ctypes.data), "reanchor")
            self._put(pred.pop(k))
            macro = pl.macro.copy()
            macro["relocate"] = 0               # the next chain's rank re-anchors itself
            pl2 = type(pl)(macro=macro, micro=pl.micro, dep_points=pl.dep_points, dep_power=pl.dep_power)
            self.local.run(pl2)
            self.pending_infos += 1
        self.last_rank = ranks[-1]
        self.chains += used
        self.moved_before = moved[-1]
        self.step_index += len(plans)

    def check_local(self) -> None:
        """Solve records of the local steps run so far (synchronises the local stream)."""
        if self.pending_infos:
            self.local.check_solves(self.local.take_info())
            self.pending_infos = 0


def plan_superstep(problem, schedule, path, policy, placement, tg, tl, k, world, moved_before):
    """One-step plans from macro step k covering up to ``world`` whole chains."""
    plans, chains = [], 0
    prev = moved_before
    while True:
        pl = plan_spacetime(problem, schedule, placement, path, policy, tg, tl, k0=k, nsteps=1)
        if pl.n_steps == 0:
            break
        if prev:
            if chains == world:
                break
            chains += 1
        plans.append(pl)
        prev = bool(pl.moved[0])
        placement, tg, tl = pl.final_placement, pl.final_t_global, pl.final_t_local
        k += 1
    return plans, (placement, tg, tl, k)


def run_spacetime_slabs(problem, schedule, local_mesh: StructuredGrid, T0: FieldState, path=None,
                        policy=None, stats=None, *, group=None, device=None):
    """``run_spacetime`` across the ranks of the current process group.

    Returns the final :class:`TwoLevelState` on the rank that ran the last macro step's
    local part (its global field is the gathered whole grid) and ``None`` elsewhere.
    """
    import torch
    d = _dist()
    rank = d.get_rank(group) if d is not None else 0
    world = d.get_world_size(group) if d is not None else 1
    run = SlabRun(problem, local_mesh, rank=rank, world=world, group=group, device=device)
    try:
        run.initial(T0)
        t0 = time.perf_counter()
        placement, tg, tl, k = local_mesh.placement, T0.time, T0.time, 0
        while True:
            plans, (placement, tg, tl, k) = plan_superstep(problem, schedule, path, policy, placement, tg, tl,
                                                           k, world, run.moved_before)
            if not plans:
                break
            run.superstep(plans)
            for pl in plans:
                _merge_counters(stats, pl.counters)
        run.check_local()
        torch.cuda.synchronize(run.solver.device)
        if stats is not None:
            stats.seconds["device_run"] = stats.seconds.get("device_run", 0.0) + time.perf_counter() - t0
        root = run.last_rank
        gv = run.solver.gather_field(root)
        if rank != root:
            return None
        gmesh = problem.global_mesh
        final_local = StructuredGrid(placement)
        lv = run.local.field(1)
        gamma = extract_interface(final_local, gmesh)
        trace = run.local.field(2)[gamma.trace_nodes]
        return TwoLevelState(FieldState(gmesh, gv, tg), FieldState(final_local, lv, tl), gamma, trace)
    finally:
        run.close()

"""Multi-GPU global solve: z-slab decomposition of the global grid.

One process per GPU (``torch.distributed``, NCCL between GPUs; gloo with host
staging for CPU-side tests).  Rank r owns the node planes ``[k0, k1)`` of the
global grid and stores ``[h0, h1)`` = its planes plus one halo plane per
neighbour.  Node planes are contiguous in the reference node order
(``id = i + NX (j + NY k)``, ``lpbfsim/mesh.py:406-409``), so each halo is one
contiguous ``NX*NY`` run that send/recv moves without packing.

The global step it distributes is ``twolevel.solve_global``
(``lpbfsim/twolevel.py:242-271``): one backward-Euler solve with the bottom face
held at the build-plate temperature, CG mirroring ``scipy.sparse.linalg.cg``
(``fem.py:271-298``) with Jacobi preconditioning.

The CG loop is device-resident (``csrc/tl_slabdev.cuh``): per iteration the host
enqueues the direction sweep, an all-gather of the ranks' 8 partial sums into device
memory, the update of the planes the neighbours read, the r halo exchange (overlapped
with the update of the remaining planes), the update of the rest and a second
all-gather.  Every scalar (alpha, beta, the stop test) is computed by the kernels from
the gathered sums, added in rank order, so all ranks take bitwise the same branch.
The host never reads a value inside the loop: it enqueues the previous solve's
iteration count + 1 (iterations after the stop test are no-ops) and synchronises once
per solve (``tl_slab_poll``).  The halo p is advanced on every rank by the owner's own
recurrence, so p never crosses ranks.

Why z rather than x slabs (SURVEY §8e suggests x): z planes are contiguous, so
halos go straight from the solve arrays into NCCL with no pack/unpack kernels,
and the laser's local box sits under the top surface, so the two-level
coupling touches only the top rank(s).  The price is a larger halo (cfg4:
8 MB per plane against 1.6 MB), about 10-20 us per plane over NVLink 5, hidden behind
the interior update sweep.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .errors import SolverError

SUMS = 8                                   # partial sums per rank (tl_slabdev.cuh kSdSums)


def plane_partition(n_planes: int, world: int) -> list[tuple[int, int]]:
    """Balanced contiguous plane ranges [k0, k1) for ``world`` ranks (lower ranks get the extra)."""
    if world < 1 or n_planes < world:
        raise ValueError(f"cannot split {n_planes} planes over {world} ranks")
    q, rem = divmod(n_planes, world)
    out, k = [], 0
    for r in range(world):
        n = q + (1 if r < rem else 0)
        out.append((k, k + n))
        k += n
    return out


def stored_planes(k0: int, k1: int, n_planes: int) -> tuple[int, int]:
    """Planes a rank stores: its own plus one halo plane per existing neighbour."""
    return max(k0 - 1, 0), min(k1 + 1, n_planes)


def _dist():
    import torch.distributed as dist
    return dist if (dist.is_available() and dist.is_initialized()) else None


class HaloExchange:
    """One-plane halo exchange of a stored-plane array between z neighbours.

    With NCCL the planes move device to device; with any other backend they are
    staged through host tensors (gloo CPU tests, several ranks sharing one GPU).
    """

    def __init__(self, rank: int, world: int, k0: int, k1: int, h0: int, nxy: int, group=None):
        self.rank, self.world, self.group = rank, world, group
        self.nxy = nxy
        self.k0, self.k1, self.h0 = k0, k1, h0
        d = _dist()
        self.nccl = d is not None and d.get_backend(group) == "nccl"

    def _plane(self, buf, k):
        o = (k - self.h0) * self.nxy
        return buf[o:o + self.nxy]

    def exchange(self, buf) -> None:
        for w in self.start(buf) or ():
            w.wait()

    def start(self, buf):
        """NCCL: enqueue the sends / receives and return the works (w.wait() orders the
        caller's stream after them; the host does not block).  Other backends: stage
        through the host and complete before returning (None)."""
        if self.world == 1:
            return None
        d = _dist()
        if d is None:
            raise SolverError("halo exchange needs an initialised process group")
        lo, hi = self.rank - 1, self.rank + 1
        # (peer, plane to send, plane to receive)
        pairs = []
        if lo >= 0:
            pairs.append((lo, self.k0, self.k0 - 1))
        if hi < self.world:
            pairs.append((hi, self.k1 - 1, self.k1))
        if self.nccl:
            ops = []
            for peer, ks, kr in pairs:
                ops.append(d.P2POp(d.isend, self._plane(buf, ks), peer, self.group))
                ops.append(d.P2POp(d.irecv, self._plane(buf, kr), peer, self.group))
            return d.batch_isend_irecv(ops)
        staged = []
        reqs = []
        for peer, ks, kr in pairs:
            s = self._plane(buf, ks).detach().to("cpu", copy=True)
            r = s.new_empty(s.shape)
            reqs.append(d.isend(s, peer, group=self.group))
            reqs.append(d.irecv(r, peer, group=self.group))
            staged.append((kr, r, s))
        for q in reqs:
            q.wait()
        for kr, r, _ in staged:
            self._plane(buf, kr).copy_(r)
        return None


def rank_sum(sums, world: int, group=None) -> np.ndarray:
    """Sum each rank's partial sums in rank order (bitwise identical on every rank) on the
    host: the reference order the device control replicates (tests, diagnostics)."""
    import torch
    d = _dist()
    if world == 1 or d is None:
        return sums.detach().cpu().numpy().astype(np.float64)
    local = sums.detach().cpu()
    lst = [torch.empty_like(local) for _ in range(world)]
    d.all_gather(lst, local, group=group)
    parts = np.stack([t.numpy() for t in lst])
    tot = np.zeros(parts.shape[1])
    for r in range(world):
        tot = tot + parts[r]
    return tot


class SlabComm:
    """The slab solve's collectives: the all-gather of every rank's partial sums into a
    device buffer (rank order) and the one-plane halo exchanges.  With NCCL both stay on
    the device: the collective is ordered after the kernels that produced its input and
    before the ones that read its output, and the host does not wait.  Other backends
    (gloo: CPU tests, several ranks sharing one GPU) stage through host memory."""

    def __init__(self, rank: int, world: int, k0: int, k1: int, h0: int, nxy: int, group=None):
        self.rank, self.world, self.group = rank, world, group
        self.halo = HaloExchange(rank, world, k0, k1, h0, nxy, group)
        self.nccl = self.halo.nccl

    def allgather(self, sums, gath) -> None:
        if self.world == 1:
            return
        d = _dist()
        if self.nccl:
            d.all_gather_into_tensor(gath, sums, group=self.group)
            return
        import torch
        local = sums.detach().cpu()
        lst = [torch.empty_like(local) for _ in range(self.world)]
        d.all_gather(lst, local, group=self.group)
        gath.copy_(torch.cat(lst).to(gath.device))

    def halo_start(self, buf):
        """Start the halo exchange of `buf`; NCCL: returns the pending works (the transfer
        runs while the caller enqueues more kernels), else completes it."""
        return self.halo.start(buf)

    def halo_wait(self, works) -> None:
        for w in works or ():
            w.wait()


@dataclass
class SlabInfo:
    iterations: int
    status: int
    bnorm: float
    rnorm: float
    true_resid: float


def _aligned(n: int, first_id: int, device):
    """Zeroed fp64 device array of n values for stored node ids [first_id, first_id + n):
    the address of global node 0 is 16-byte aligned (the bulk copies read 16-byte
    ranges by global id) and one value before / two after are readable."""
    import torch
    e = 2 - (first_id % 2)
    buf = torch.zeros(n + 4, dtype=torch.float64, device=device)
    return buf[e:e + n]


class SlabGlobalSolver:
    """This rank's share of the global backward-Euler step (bottom Dirichlet).

    ``x`` (stored planes) holds T_old on the owned planes before :meth:`step` and the
    solution after it; ``load`` (stored planes) is the deposit load.  Both are device
    tensors the caller may fill in place.
    """

    def __init__(self, grid, kappa: float, rho_c: float, *, rank: int = 0, world: int = 1,
                 group=None, device=None, rtol: float = 1e-12, maxiter: int | None = None):
        import torch
        self.grid = grid
        self.kappa, self.rho_c = float(kappa), float(rho_c)
        self.rank, self.world, self.group = rank, world, group
        nx, ny, nz = (int(c) + 1 for c in grid.ncells)
        self.nxy, self.nz = nx * ny, nz
        self.k0, self.k1 = plane_partition(nz, world)[rank]
        self.h0, self.h1 = stored_planes(self.k0, self.k1, nz)
        self.device = torch.device(device if device is not None else "cuda")
        n = (self.h1 - self.h0) * self.nxy
        self.n_stored = n
        st0 = self.h0 * self.nxy
        self.x, self.b, self.r = (_aligned(n, st0, self.device) for _ in range(3))
        self.p0, self.p1, self.load = (_aligned(n, st0, self.device) for _ in range(3))
        self.work = torch.zeros(int(N.lib().tl_slab_work_len()), dtype=torch.float64, device=self.device)
        self.sums = torch.zeros(SUMS, dtype=torch.float64, device=self.device)
        self.gath = torch.zeros(world * SUMS, dtype=torch.float64, device=self.device)
        self.rtol = float(rtol)
        nn = int(np.prod([int(c) + 1 for c in grid.ncells]))
        self.maxiter = min(20 * nn, 2_000_000_000) if maxiter is None else int(maxiter)
        self.comm = SlabComm(rank, world, self.k0, self.k1, self.h0, self.nxy, group)
        self.launches = 0
        self.polls = 0                 # host synchronisations (one per solve when predicted well)
        self.k_pred = 20               # iterations to enqueue: the previous solve's count + 1

    # -- index helpers --------------------------------------------------------
    @property
    def own_ids(self) -> slice:
        """Global node ids this rank owns."""
        return slice(self.k0 * self.nxy, self.k1 * self.nxy)

    @property
    def own_local(self) -> slice:
        """The owned part of the stored-plane arrays."""
        o = (self.k0 - self.h0) * self.nxy
        return slice(o, o + (self.k1 - self.k0) * self.nxy)

    def set_own(self, tensor, values) -> None:
        """Copy this rank's share of a full-grid (host or device) array into ``tensor``."""
        import torch
        v = torch.as_tensor(np.array(values[self.own_ids]) if isinstance(values, np.ndarray)
                            else values[self.own_ids])
        tensor[self.own_local].copy_(v)

    def own_view(self, tensor):
        return tensor[self.own_local]

    # -- solve ----------------------------------------------------------------
    def _desc(self, dt: float, g_const: float, with_load: bool):
        import torch
        s = N.Slab()
        s.grid = self.grid.desc()
        s.dirichlet_kind = N.TL_DIRICHLET_BOTTOM
        s.k0, s.k1 = self.k0, self.k1
        s.kappa, s.rho_c, s.dt, s.g_const = self.kappa, self.rho_c, float(dt), float(g_const)
        s.x, s.b, s.r = self.x.data_ptr(), self.b.data_ptr(), self.r.data_ptr()
        s.p0, s.p1 = self.p0.data_ptr(), self.p1.data_ptr()
        s.load = self.load.data_ptr() if with_load else None
        s.work, s.sums = self.work.data_ptr(), self.sums.data_ptr()
        s.gath = self.gath.data_ptr() if self.world > 1 else None
        s.world = self.world
        s.maxiter = self.maxiter
        s.rtol = self.rtol
        s.stream = torch.cuda.current_stream(self.device).cuda_stream
        return s

    def _iteration(self, L, ps) -> None:
        """One CG iteration, enqueued: no host synchronisation (NCCL)."""
        N.check(L.tl_slab_direction(ps), "slab direction")
        self.comm.allgather(self.sums, self.gath)
        N.check(L.tl_slab_update(ps, 0), "slab update (boundary planes)")
        works = self.comm.halo_start(self.r)
        N.check(L.tl_slab_update(ps, 1), "slab update")
        self.comm.allgather(self.sums, self.gath)
        self.comm.halo_wait(works)
        self.launches += 3

    def step(self, dt: float, g_const: float, with_load: bool = True, gaussian=None) -> SlabInfo:
        """One global solve; x holds the new field on the owned planes afterwards."""
        L = N.lib()
        s = self._desc(dt, g_const, with_load)
        ps = C.byref(s)
        src = None
        if gaussian is not None:
            peak, radius, depth, center = gaussian
            src = N.Gaussian(float(peak), float(radius), float(depth),
                             (C.c_double * 3)(*map(float, center)), 1)
        N.check(L.tl_slab_begin(ps, C.byref(src) if src is not None else None), "slab begin")
        self.launches += 2
        self.comm.allgather(self.sums, self.gath)
        self.comm.halo_wait(self.comm.halo_start(self.r))
        state = C.c_int32(0)
        info = N.SolveInfo()
        enqueued, k = 0, max(1, self.k_pred)
        while True:
            for _ in range(k):
                self._iteration(L, ps)
            enqueued += k
            # no-ops until the stop test fired inside the enqueued iterations
            self.comm.halo_wait(self.comm.halo_start(self.x))
            N.check(L.tl_slab_residual(ps), "slab residual")
            self.comm.allgather(self.sums, self.gath)
            N.check(L.tl_slab_finish(ps), "slab finish")
            self.launches += 2
            N.check(L.tl_slab_poll(ps, C.byref(state), C.byref(info)), "slab poll")
            self.polls += 1
            if state.value == 2:
                break
            if enqueued > self.maxiter + 1:
                raise SolverError("slab solve did not stop")
            k = max(2, min(k, 8))
        self.k_pred = (info.iterations if info.status == 0 else 0) + 1
        return SlabInfo(int(info.iterations), int(info.status), float(info.bnorm), float(info.rnorm),
                        float(info.true_resid))

    def deposit(self, points, power) -> None:
        """Swept-track deposit of one macro interval into ``load`` (own nodes only)."""
        import torch
        pts = torch.as_tensor(np.ascontiguousarray(points, dtype=np.float64).reshape(-1)).to(self.device)
        pw = torch.as_tensor(np.ascontiguousarray(power, dtype=np.float64)).to(self.device)
        s = self._desc(1.0, 0.0, True)
        N.check(N.lib().tl_slab_deposit(C.byref(s), pts.data_ptr() if pw.numel() else None,
                                        pw.data_ptr() if pw.numel() else None, int(pw.numel())),
                "slab deposit")
        self.launches += 1

    def plane_block(self, a: int, b: int):
        """Device view of owned planes [a, b) of x."""
        return self.x[(a - self.h0) * self.nxy:(b - self.h0) * self.nxy]

    def gather_planes(self, k_lo: int, root: int):
        """Planes [k_lo, nz) of the solution on ``root`` as one device tensor (None elsewhere)."""
        import torch
        d = _dist()
        parts = plane_partition(self.nz, self.world)

        def mine(r):
            k0, k1 = parts[r]
            return max(k0, k_lo), k1

        if self.world == 1 or d is None:
            a, b = mine(0)
            return self.plane_block(a, b)
        dev = self.device if self.comm.nccl else torch.device("cpu")
        if self.rank == root:
            out = torch.empty((self.nz - k_lo) * self.nxy, dtype=torch.float64, device=self.device)
            for r in range(self.world):
                a, b = mine(r)
                if a >= b:
                    continue
                dst = out[(a - k_lo) * self.nxy:(b - k_lo) * self.nxy]
                if r == self.rank:
                    dst.copy_(self.plane_block(a, b))
                else:
                    t = torch.empty(dst.numel(), dtype=torch.float64, device=dev)
                    d.recv(t, r, group=self.group)
                    dst.copy_(t)
            return out
        a, b = mine(self.rank)
        if a < b:
            d.send(self.plane_block(a, b).detach().to(dev).contiguous(), root, group=self.group)
        return None

    def gather_field(self, root: int = 0) -> np.ndarray | None:
        """Whole-grid field on ``root`` (None elsewhere): host copy for checks and output."""
        t = self.gather_planes(0, root)
        return None if t is None else t.detach().cpu().numpy().copy()

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
(``fem.py:271-298``) with Jacobi preconditioning.  Per CG iteration the ranks
exchange the r halo (one plane each way) and combine two sets of partial sums
(p.q; r.z and r.r).  The halo p is advanced on every rank by the owner's own
recurrence, so p never crosses ranks.  Partial sums are gathered and added in
rank order, so every rank computes bitwise the same scalars and the iteration
count does not depend on the backend's reduction algorithm.

Why z rather than x slabs (SURVEY §8e suggests x): z planes are contiguous, so
halos go straight from the solve arrays into NCCL with no pack/unpack kernels,
and the laser's local box sits under the top surface, so the two-level
coupling touches only the top rank(s).  The price is a larger halo (cfg4:
8 MB per plane against 1.6 MB), about 10 us per plane over NVLink 5 against
~350 us of per-rank stencil work per iteration at 8 GPUs.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .errors import SolverError


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
        if self.world == 1:
            return
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
            for w in d.batch_isend_irecv(ops):
                w.wait()
            return
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


def rank_sum(sums, world: int, group=None) -> np.ndarray:
    """Sum each rank's 4 partial sums in rank order (bitwise identical on every rank)."""
    import torch
    d = _dist()
    if world == 1 or d is None:
        return sums.detach().cpu().numpy().astype(np.float64)
    if d.get_backend(group) == "nccl":
        out = torch.empty(world * sums.numel(), dtype=sums.dtype, device=sums.device)
        d.all_gather_into_tensor(out, sums, group=group)
        parts = out.view(world, -1).cpu().numpy()
    else:
        local = sums.detach().cpu()
        lst = [torch.empty_like(local) for _ in range(world)]
        d.all_gather(lst, local, group=group)
        parts = np.stack([t.numpy() for t in lst])
    tot = np.zeros(parts.shape[1])
    for r in range(world):
        tot = tot + parts[r]
    return tot


@dataclass
class SlabInfo:
    iterations: int
    status: int
    bnorm: float
    rnorm: float
    true_resid: float


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
        z = lambda m: torch.zeros(m, dtype=torch.float64, device=self.device)  # noqa: E731
        self.x, self.b, self.r, self.p0, self.p1 = z(n), z(n), z(n), z(n), z(n)
        self.load = z(n)
        self.work = z(int(N.lib().tl_slab_work_len()))
        self.sums = z(4)
        self.rtol = float(rtol)
        nn = int(np.prod([int(c) + 1 for c in grid.ncells]))
        self.maxiter = min(20 * nn, 2_000_000_000) if maxiter is None else int(maxiter)
        self.halo = HaloExchange(rank, world, self.k0, self.k1, self.h0, self.nxy, group)
        self.launches = 0

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
        s.stream = torch.cuda.current_stream(self.device).cuda_stream
        return s

    def _sum(self) -> np.ndarray:
        return rank_sum(self.sums, self.world, self.group)

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
        N.check(L.tl_slab_rhs(ps, C.byref(src) if src is not None else None), "slab rhs")
        self.launches += 1
        tot = self._sum()
        bb, rz = tot[0], tot[1]
        self.halo.exchange(self.r)
        bnorm = math.sqrt(bb)
        atol = self.rtol * bnorm
        rnorm = bnorm
        it, status, rho_prev = 0, 0, 1.0
        if bb != 0.0:
            while True:
                if rnorm < atol:
                    status = 0
                    break
                if not math.isfinite(rnorm):
                    status = 3
                    break
                if it >= self.maxiter:
                    status = 1
                    break
                rho = rz
                beta = rho / rho_prev if it > 0 else 0.0
                par = it & 1
                N.check(L.tl_slab_direction(ps, int(it == 0), float(beta), par), "slab direction")
                pq = self._sum()[2]
                alpha = rho / pq
                N.check(L.tl_slab_update(ps, float(alpha), par), "slab update")
                self.launches += 2
                tot = self._sum()
                rz, rnorm = tot[0], math.sqrt(tot[1])
                self.halo.exchange(self.r)
                rho_prev = rho
                it += 1
        self.halo.exchange(self.x)
        N.check(L.tl_slab_residual(ps), "slab residual")
        tot = self._sum()
        tres = math.sqrt(tot[0]) / bnorm if bnorm > 0.0 else 0.0
        N.check(L.tl_slab_finish(ps), "slab finish")
        self.launches += 2
        if status == 0 and tot[3] > 0.0:
            status = 3
        if status == 0 and (not math.isfinite(tres) or tres > 1e2 * self.rtol):
            status = 2
        return SlabInfo(self.maxiter if status == 1 else it, status, bnorm, rnorm, tres)

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

    def gather_planes(self, k_lo: int, root: int):
        """Planes [k_lo, nz) of the solution on ``root`` as one device tensor (None elsewhere).

        Used to hand the global sub-block under the local box to the rank that runs the
        local problem (trace and relocation need only that block)."""
        import torch
        d = _dist()
        parts = plane_partition(self.nz, self.world)

        def mine(r):
            k0, k1 = parts[r]
            return max(k0, k_lo), k1

        if self.world == 1 or d is None:
            a, b = mine(0)
            return self.x[(a - self.h0) * self.nxy:(b - self.h0) * self.nxy]
        dev = self.device if self.halo.nccl else torch.device("cpu")
        if self.rank == root:
            out = torch.empty((self.nz - k_lo) * self.nxy, dtype=torch.float64, device=self.device)
            for r in range(self.world):
                a, b = mine(r)
                if a >= b:
                    continue
                dst = out[(a - k_lo) * self.nxy:(b - k_lo) * self.nxy]
                if r == self.rank:
                    dst.copy_(self.x[(a - self.h0) * self.nxy:(b - self.h0) * self.nxy])
                else:
                    t = torch.empty(dst.numel(), dtype=torch.float64, device=dev)
                    d.recv(t, r, group=self.group)
                    dst.copy_(t)
            return out
        a, b = mine(self.rank)
        if a < b:
            d.send(self.x[(a - self.h0) * self.nxy:(b - self.h0) * self.nxy].detach().to(dev).contiguous(),
                   root, group=self.group)
        return None

    def gather_field(self, root: int = 0) -> np.ndarray | None:
        """Whole-grid field on ``root`` (None elsewhere): host copy for checks and output."""
        t = self.gather_planes(0, root)
        return None if t is None else t.detach().cpu().numpy().copy()

"""Literal element-by-element P1 assembly + scipy CG — the reference's CPU algorithm.

TEST INFRASTRUCTURE / CPU BASELINE ONLY (see ``oracle/__init__.py``).

This is the algorithm the reference runs for every implicit step, restated
from its published structure (not its source): build the six Kuhn tets per
cell (``lpbfsim/mesh.py:84-102,406-439``, orientation fixed by swapping the
last two vertices of inverted tets), element geometry by inverting the edge
matrices (``mesh.py:263-277``), the 4-point rule at every tet
(``mesh.py:105-128,279-283``), einsum element matrices with a row-sum lumped
mass (``fem.py:156-178``), COO -> CSR (``fem.py:180-184``), symmetric Dirichlet
elimination (``fem.py:89-105``) and ``scipy.sparse.linalg.cg`` with a Jacobi
preconditioner and ``maxiter = 20 n`` (``fem.py:271-298``).  ``bench.py``
times it as the CPU baseline ("port", one core); the tests use it as a
second pin next to the matrix-free restatement in ``kuhn.py``.
"""

from __future__ import annotations

import itertools

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from .kuhn import QPHI, QW


class KuhnMesh:
    """Explicit tet mesh of a structured grid (node order x fastest)."""

    def __init__(self, grid):
        self.grid = grid
        n = grid.n
        X = grid.coords()
        nn = n + 1
        strides = np.array([1, nn[0], nn[0] * nn[1]], dtype=np.int64)
        ci = [np.arange(v) for v in n]
        CZ, CY, CX = np.meshgrid(ci[2], ci[1], ci[0], indexing="ij")
        corner0 = (np.stack([CX.ravel(), CY.ravel(), CZ.ravel()], axis=1) @ strides)
        offsets = np.array([[(b >> a) & 1 for a in range(3)] for b in range(8)])  # x fastest
        corner_ids = corner0[:, None] + offsets @ strides
        pats = []
        for perm in itertools.permutations(range(3)):
            verts, acc = [0], 0
            for ax in perm:
                acc += 1 << ax
                verts.append(acc)
            pats.append(verts)
        elems = corner_ids[:, np.array(pats)].reshape(-1, 4)
        J = X[elems[:, 1:]] - X[elems[:, [0]]]
        det = np.linalg.det(J)
        flip = det < 0
        elems[flip, 2:] = elems[flip, 2:][:, ::-1]
        J = X[elems[:, 1:]] - X[elems[:, [0]]]
        self.X = X
        self.elems = elems
        self.vol = np.linalg.det(J) / 6.0
        invJ = np.linalg.inv(J)
        g = np.empty((len(elems), 4, 3))
        g[:, 1:, :] = np.swapaxes(invJ, 1, 2)
        g[:, 0, :] = -g[:, 1:, :].sum(axis=1)
        self.grads = g
        self.rows = np.repeat(elems, 4, axis=1).reshape(-1)
        self.cols = np.tile(elems, (1, 4)).reshape(-1)

    def quad_points(self):
        return np.einsum("qi,eid->eqd", QPHI, self.X[self.elems])


_CACHE: dict = {}


def _mesh(grid) -> KuhnMesh:
    key = (tuple(grid.lo0), tuple(grid.hi0), tuple(grid.n), tuple(grid.offset))
    m = _CACHE.get(key)
    if m is None:
        _CACHE.clear()
        m = KuhnMesh(grid)
        _CACHE[key] = m
    return m


def gaussian_pointwise(beam, center, pts):
    c = np.asarray(center, dtype=float)
    ex = 3.0 * ((pts[:, 0] - c[0]) / beam.radius) ** 2
    ey = 3.0 * ((pts[:, 1] - c[1]) / beam.radius) ** 2
    ez = 3.0 * ((pts[:, 2] - c[2]) / beam.depth) ** 2
    peak = 6.0 * np.sqrt(3.0) * beam.power * beam.absorptivity / (2.0 * np.pi * beam.radius**2 * beam.depth)
    return peak * np.exp(-(ex + ey + ez))


def step(grid, kappa, rhoc, dt, dirichlet_mask, T_old, source, extra_load, g, rtol):
    """One implicit step exactly as the reference's CPU path does it; returns (x, iterations)."""
    M = _mesh(grid)
    conn = M.elems
    coeff = np.full((len(conn), 4), rhoc)
    kbar = np.full((len(conn), 4), kappa) @ QW
    mass = np.einsum("q,eq,qi->ei", QW, coeff / dt, QPHI) * M.vol[:, None]
    stiff = np.einsum("e,eid,ejd->eij", kbar * M.vol, M.grads, M.grads)
    data = stiff.copy()
    d4 = np.arange(4)
    data[:, d4, d4] += mass
    rhs_e = mass * T_old[conn]
    if source is not None:
        beam, center = source
        Q = gaussian_pointwise(beam, center, M.quad_points().reshape(-1, 3)).reshape(len(conn), 4)
        rhs_e += np.einsum("q,eq,qi->ei", QW, Q, QPHI) * M.vol[:, None]
    n = grid.n_nodes
    A = sp.coo_matrix((data.reshape(-1), (M.rows, M.cols)), shape=(n, n)).tocsr()
    b = np.zeros(n)
    np.add.at(b, conn.reshape(-1), rhs_e.reshape(-1))
    if extra_load is not None:
        b = b + extra_load
    D = np.nonzero(np.asarray(dirichlet_mask).ravel())[0]
    gfull = np.zeros(n)
    gfull[D] = np.asarray(g).ravel()[D]
    b -= A @ gfull
    keep = np.ones(n)
    keep[D] = 0.0
    Dm = sp.diags(keep)
    A = (Dm @ A @ Dm + sp.diags(1.0 - keep)).tocsr()
    b = keep * b
    b[D] = gfull[D]
    bnorm = np.linalg.norm(b)
    if bnorm == 0.0:
        return np.zeros(n), 0
    diag = A.diagonal()
    Minv = sp.diags(np.where(diag > 0, 1.0 / diag, 1.0))
    count = [0]

    def cb(_x):
        count[0] += 1

    x, info = spla.cg(A, b, rtol=rtol, M=Minv, maxiter=20 * n, callback=cb)
    res = np.linalg.norm(A @ x - b) / bnorm
    if info != 0 or res > 1e2 * rtol:
        raise RuntimeError(f"conjugate gradients did not converge (info={info}, res={res:.3e})")
    x[D] = gfull[D]
    return x, count[0]

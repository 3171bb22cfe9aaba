"""2D restatement of the reference's P1-triangle discretization in stencil form (TEST
INFRASTRUCTURE ONLY, see ``oracle/__init__.py``).

The reference's 2D meshes split every cell of a structured grid into the two triangles
``[0, 1, 3]`` and ``[0, 3, 2]`` (corner index = dx + 2 dy; ``lpbfsim/mesh.py:84-93``), both
positively oriented, so ``build_structured_mesh`` keeps their vertex order
(``mesh.py:388-439``):

    tri 0: (0,0) (1,0) (1,1)        tri 1: (0,0) (1,1) (0,1)

Both are right triangles with axis-aligned legs, so the P1 gradients are axis-aligned and
the element stiffness ``kbar * area * grad_i . grad_j`` (``fem.py:170``) couples only the
leg endpoints (``-kbar area / h_a^2`` on the leg along axis a); the hypotenuse carries no
coupling.  With the row-sum lumped mass (``fem.py:167-169``) the assembled operator is a
5-point stencil with per-edge weights:

    (A x)_p = diag_p x_p - sum_a (w_a[p] x_{p+e_a} + w_a[p-e_a] x_{p-e_a}),   a in {x, y}

Quadrature: the three edge midpoints with weights 1/3 (``mesh.py:107-110``); boundary
edges: two Gauss points (``mesh.py:129-131``).  The vertical axis is y: BOTTOM / TOP are
the edges y = lo / y = hi (``mesh.py:206-209`` tag the LAST coordinate).  The 2D beam is
``gaussian_source_2d`` (``sources.py:57-64``).

Node order: x fastest (``id = i + NX j``).
"""

from __future__ import annotations

import numpy as np

from .varcoef import latent_slope

# barycentric quadrature points of a triangle (rows) and their weights (mesh.py:107-110)
QPHI2 = np.array([[0.5, 0.5, 0.0], [0.0, 0.5, 0.5], [0.5, 0.0, 0.5]])
QW2 = np.full(3, 1.0 / 3.0)
# vertex offsets (dx, dy) of the two triangles of a cell, in the reference's vertex order
TRIS = (((0, 0), (1, 0), (1, 1)), ((0, 0), (1, 1), (0, 1)))
# legs of each triangle: (vertex a, vertex b, axis, vertex that holds w_axis = the lower one)
LEGS = (((0, 1, 0), (1, 2, 1)),          # tri 0: x leg v0-v1, y leg v1-v2
        ((0, 2, 1), (2, 1, 0)))          # tri 1: y leg v0-v2, x leg v2-v1
_G2 = 0.5 / np.sqrt(3.0)
FPHI = np.array([[0.5 + _G2, 0.5 - _G2], [0.5 - _G2, 0.5 + _G2]])     # mesh.py:129-131
FW = np.full(2, 0.5)


class Grid2D:
    """Structured 2D node lattice: construction box, cell counts, accumulated offset."""

    def __init__(self, lo0, hi0, ncells, offset=(0.0, 0.0)):
        self.lo0 = np.asarray(lo0, dtype=float)
        self.hi0 = np.asarray(hi0, dtype=float)
        self.n = np.asarray(ncells, dtype=np.int64)
        self.offset = np.asarray(offset, dtype=float)
        self.h = (self.hi0 - self.lo0) / self.n
        self.NX, self.NY = int(self.n[0]) + 1, int(self.n[1]) + 1
        self.n_nodes = self.NX * self.NY

    def axis(self, a: int) -> np.ndarray:
        return np.linspace(self.lo0[a], self.hi0[a], int(self.n[a]) + 1) + self.offset[a]

    @property
    def coords(self) -> np.ndarray:
        X, Y = np.meshgrid(self.axis(0), self.axis(1), indexing="xy")
        return np.stack([X.ravel(), Y.ravel()], axis=1)

    def cells(self):
        ci = np.stack(np.meshgrid(np.arange(self.n[0]), np.arange(self.n[1]), indexing="ij"), axis=-1)
        return ci.reshape(-1, 2)


def gaussian2d(beam_args, points):
    """``gaussian_source_2d`` (``sources.py:57-64``); beam_args = (power*absorptivity, radius, depth, center)."""
    pe, radius, depth, center = beam_args
    p = np.atleast_2d(np.asarray(points, dtype=float))
    ex = ((p[:, 0] - center[0]) / radius) ** 2
    ey = ((p[:, 1] - center[1]) / depth) ** 2
    return pe / (radius * depth) * np.exp(-(ex + ey))


def assemble(G: Grid2D, mat, T_old, T_lag, dt, source=None, latent=False, robin=None):
    """(diag, w (2, n), b) of the unconstrained system (``assemble_system``,
    ``fem.py:129-194``, + ``_add_robin``, ``:241-268``, on the top edge).
    ``source(points) -> Q``; ``robin = (h_conv, sigma*eps or 0, T_ambient)``."""
    n, NX = G.n_nodes, G.NX
    h = G.h
    area = 0.5 * float(h[0] * h[1])
    diag = np.zeros(n)
    w = np.zeros((2, n))
    b = np.zeros(n)
    T_old = np.asarray(T_old, dtype=float)
    T_lag = np.asarray(T_lag, dtype=float)
    ci = G.cells()
    x, y = G.axis(0), G.axis(1)
    for tri, legs in zip(TRIS, LEGS):
        ids = np.stack([(ci[:, 0] + a) + NX * (ci[:, 1] + bb) for a, bb in tri], axis=1)          # (E, 3)
        Tq = T_lag[ids] @ QPHI2.T
        Tq_old = T_old[ids] @ QPHI2.T
        kq = np.interp(Tq, mat.conductivity_table[:, 0], mat.conductivity_table[:, 1])
        cq = np.interp(Tq, mat.heat_capacity_table[:, 0], mat.heat_capacity_table[:, 1])
        if latent and mat.chi > 0.0:
            cq = cq + latent_slope(mat, Tq, Tq_old)
        coeff = mat.rho * cq
        kbar = kq @ QW2
        ml = np.einsum("q,eq,qi->ei", QW2, coeff / dt, QPHI2) * area
        np.add.at(diag, ids.reshape(-1), ml.reshape(-1))
        np.add.at(b, ids.reshape(-1), (ml * T_old[ids]).reshape(-1))
        if source is not None:
            X = np.stack([np.stack([x[ci[:, 0] + a], y[ci[:, 1] + bb]], axis=1) for a, bb in tri], axis=1)
            qp = np.einsum("qi,eid->eqd", QPHI2, X)
            Q = np.asarray(source(qp.reshape(-1, 2))).reshape(-1, 3)
            np.add.at(b, ids.reshape(-1), (np.einsum("q,eq,qi->ei", QW2, Q, QPHI2) * area).reshape(-1))
        for va, vb, ax in legs:
            we = kbar * area / h[ax] ** 2
            np.add.at(diag, ids[:, va], we)
            np.add.at(diag, ids[:, vb], we)
            lower = np.minimum(ids[:, va], ids[:, vb])
            np.add.at(w[ax], lower, we)
    if robin is not None:
        hc, se, T_amb = robin
        j = int(G.n[1])
        i = np.arange(int(G.n[0]))
        # top edge of tri 1 of each top cell, facet nodes in the reference's order:
        # the facet omitting vertex 0 of [n00, n11, n01] is (n11, n01) (mesh.py:190-192)
        fn = np.stack([(i + 1) + NX * j, i + NX * j], axis=1)
        Tq = T_lag[fn] @ FPHI.T
        coeff = hc + se * Tq ** 3
        load = np.full_like(coeff, hc * T_amb + se * T_amb ** 4)
        mdat = np.einsum("q,fq,qi->fi", FW, coeff, FPHI) * h[0]
        fdat = np.einsum("q,fq,qi->fi", FW, load, FPHI) * h[0]
        np.add.at(diag, fn.reshape(-1), mdat.reshape(-1))
        np.add.at(b, fn.reshape(-1), fdat.reshape(-1))
    return diag, w, b


def apply(G: Grid2D, diag, w, x):
    st = [1, G.NX]
    y = diag * x
    for a in range(2):
        y[:-st[a]] -= w[a][:-st[a]] * x[st[a]:]
        y[st[a]:] -= w[a][:-st[a]] * x[:-st[a]]
    return y


def constrained(G: Grid2D, diag, w, b, dmask, g):
    """``SparseSystem.constrained`` (``fem.py:89-105``) in stencil form."""
    st = [1, G.NX]
    free = ~dmask
    gD = np.where(dmask, g, 0.0)
    bc = b.copy()
    for a in range(2):
        bc[:-st[a]] += w[a][:-st[a]] * gD[st[a]:]
        bc[st[a]:] += w[a][:-st[a]] * gD[:-st[a]]
    bc[dmask] = g[dmask]
    wc = w.copy()
    for a in range(2):
        keep = free[:-st[a]] & free[st[a]:]
        wc[a][:-st[a]] *= keep
    dc = np.where(dmask, 1.0, diag)
    return dc, wc, bc


def step(G: Grid2D, mat, T_old, dt, source, dmask, g, latent, robin, rtol=1e-12, picard_tol=1e-8,
         picard_max=25):
    """``step_backward_euler`` (``fem.py:307-355``) in 2D: (x, picard passes, [CG iterations])."""
    from .pcg import cg_mirror
    T_lag = np.asarray(T_old, dtype=float)
    prev_inc, theta = np.inf, 1.0
    cg_its = []
    for it in range(1, picard_max + 1):
        diag, w, b = assemble(G, mat, T_old, T_lag, dt, source, latent, robin)
        dc, wc, bc = constrained(G, diag, w, b, dmask, g)
        x, info, its = cg_mirror(lambda v: apply(G, dc, wc, v), bc, 1.0 / dc, rtol, 20 * bc.size)
        if info != 0:
            raise RuntimeError("oracle CG did not converge")
        x = np.where(dmask, g, x)
        cg_its.append(its)
        inc = np.linalg.norm(x - T_lag) / max(np.linalg.norm(x), 1e-300)
        if inc < picard_tol:
            return x, it, cg_its
        if inc >= 0.9 * prev_inc:
            theta = max(0.25, 0.5 * theta)
        prev_inc = inc
        T_lag = T_lag + theta * (x - T_lag)
    raise RuntimeError("oracle Picard did not converge")


def interpolate(G: Grid2D, values, points):
    """``Mesh.interpolate`` (``mesh.py:308-361``) on the triangle lattice: cell by floor
    (clipped), triangle 0 where xi >= eta (the first candidate wins ties), P1 in it."""
    pts = np.atleast_2d(np.asarray(points, dtype=float))
    lo = np.array([G.axis(0)[0], G.axis(1)[0]])
    cell = np.floor((pts - lo) / G.h).astype(np.int64)
    cell = np.clip(cell, 0, G.n - 1)
    x, y = G.axis(0), G.axis(1)
    xi = (pts[:, 0] - x[cell[:, 0]]) / G.h[0]
    eta = (pts[:, 1] - y[cell[:, 1]]) / G.h[1]
    v = np.asarray(values, dtype=float)
    i00 = cell[:, 0] + G.NX * cell[:, 1]
    v00, v10, v01, v11 = v[i00], v[i00 + 1], v[i00 + G.NX], v[i00 + G.NX + 1]
    t0 = (1.0 - xi) * v00 + (xi - eta) * v10 + eta * v11
    t1 = (1.0 - eta) * v00 + xi * v11 + (eta - xi) * v01
    return np.where(xi >= eta, t0, t1)


def mass_norm2(G: Grid2D, v) -> float:
    """v^T M v with the consistent P1 mass matrix (``fem.mass_matrix``, ``fem.py:434-446``):
    per triangle area/12 (sum v_i^2 + (sum v_i)^2)."""
    v = np.asarray(v, dtype=float)
    ci = G.cells()
    area = 0.5 * float(G.h[0] * G.h[1])
    tot = 0.0
    for tri in TRIS:
        ids = np.stack([(ci[:, 0] + a) + G.NX * (ci[:, 1] + bb) for a, bb in tri], axis=1)
        ve = v[ids]
        tot += float(np.sum(area / 12.0 * ((ve ** 2).sum(axis=1) + ve.sum(axis=1) ** 2)))
    return tot

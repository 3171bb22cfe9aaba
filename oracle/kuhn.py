"""Matrix-free CPU restatement of the reference's Kuhn-P1 discretization (oracle).

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

The reference assembles P1 elements on a structured grid whose cells are each
split into the six Kuhn tetrahedra ``{0, e_a, e_a+e_b, 1}``
(``lpbfsim/mesh.py:84-102,388-439``).  With a constant material, the
row-sum-lumped mass (``lpbfsim/fem.py:167-169``) and the P1 stiffness
(``lpbfsim/fem.py:170``) reduce exactly to

    (A x)_p = m_p x_p + sum_axis sum_{q = p +- e_a} c_pq (x_p - x_q)
    m_p  = (rho c / dt) * V * n_p / 24        n_p = tets incident to node p
    c_pq = kappa * V / h_a^2 * n_e / 6        n_e = tets incident to edge pq

(non-axis couplings are zero analytically and
~1e-20 rounding noise in the reference CSR).  Dirichlet rows are eliminated
symmetrically as in ``SparseSystem.constrained`` (``lpbfsim/fem.py:89-105``).

Arrays are stored 3D as ``[k, j, i]`` (z slowest), so ``ravel()`` gives the
reference node order ``i + (nx+1)(j + (ny+1)k)`` (``lpbfsim/mesh.py:406-409``).
"""

from __future__ import annotations

import itertools

import numpy as np

# 4-point tetrahedron rule of the reference (``lpbfsim/mesh.py:116-128``)
ALPHA = (5.0 + 3.0 * np.sqrt(5.0)) / 20.0
BETA = (5.0 - np.sqrt(5.0)) / 20.0
QPHI = np.array([[ALPHA, BETA, BETA, BETA],
                 [BETA, ALPHA, BETA, BETA],
                 [BETA, BETA, ALPHA, BETA],
                 [BETA, BETA, BETA, ALPHA]])
QW = np.full(4, 0.25)

# Kuhn tetrahedra as axis permutations; vertex r of permutation (a, b, c) is the
# sum of e_perm[0..r-1]  (``lpbfsim/mesh.py:94-101``)
PERMS = list(itertools.permutations(range(3)))


def tet_vertices(perm) -> np.ndarray:
    """(4, 3) fractional offsets (x, y, z) of the Kuhn tet's vertices."""
    v = np.zeros((4, 3), dtype=np.int64)
    for r, ax in enumerate(perm, start=1):
        v[r:, ax] += 1
    return v


class KuhnGrid:
    """Structured node lattice: construction box, cell counts, accumulated offset."""

    def __init__(self, lo0, hi0, ncells, offset=(0.0, 0.0, 0.0)):
        self.lo0 = np.asarray(lo0, dtype=float)
        self.hi0 = np.asarray(hi0, dtype=float)
        self.n = np.asarray(ncells, dtype=np.int64)
        self.offset = np.asarray(offset, dtype=float)
        self.h = (self.hi0 - self.lo0) / self.n          # ``Mesh.spacing`` (mesh.py:162)
        self.shape = tuple(int(v) for v in (self.n[2] + 1, self.n[1] + 1, self.n[0] + 1))

    @classmethod
    def from_placement(cls, placement) -> "KuhnGrid":
        return cls(placement.box0.lo, placement.box0.hi, placement.ncells, placement.offset)

    @property
    def n_nodes(self) -> int:
        return int(np.prod(self.shape))

    @property
    def box_lo(self) -> np.ndarray:
        return self.lo0 + self.offset

    def axis(self, a: int) -> np.ndarray:
        """Node coordinates along axis a (linspace of construction box + offset)."""
        return np.linspace(self.lo0[a], self.hi0[a], int(self.n[a]) + 1) + self.offset[a]

    def coords(self) -> np.ndarray:
        x, y, z = self.axis(0), self.axis(1), self.axis(2)
        Z, Y, X = np.meshgrid(z, y, x, indexing="ij")
        return np.stack([X.ravel(), Y.ravel(), Z.ravel()], axis=1)

    # -- incidence counts ----------------------------

    def _has(self, a: int):
        idx = np.arange(int(self.n[a]) + 1)
        has0 = (idx < self.n[a]).astype(np.int64)   # cell idx exists   (offset 0)
        has1 = (idx > 0).astype(np.int64)           # cell idx-1 exists (offset 1)
        return has0, has1

    def _bcast(self, arr, a):
        shape = [1, 1, 1]
        shape[2 - a] = arr.size
        return arr.reshape(shape)

    def node_incidence(self) -> np.ndarray:
        """Number of Kuhn tets containing each node (interior 24)."""
        h0 = [self._bcast(self._has(a)[0], a) for a in range(3)]
        h1 = [self._bcast(self._has(a)[1], a) for a in range(3)]
        cnt = [h0[a] + h1[a] for a in range(3)]
        n_p = 2 * cnt[0] * cnt[1] * cnt[2] + 4 * h0[0] * h0[1] * h0[2] + 4 * h1[0] * h1[1] * h1[2]
        return np.broadcast_to(n_p, self.shape).astype(np.int64)

    def edge_incidence(self, a: int) -> np.ndarray:
        """Tets containing each axis-a edge {p, p+e_a}; shape = node shape minus 1 along a."""
        b, c = [ax for ax in range(3) if ax != a]
        hb0, hb1 = (self._bcast(v, b) for v in self._has(b))
        hc0, hc1 = (self._bcast(v, c) for v in self._has(c))
        n_e = (hb0 + hb1) * (hc0 + hc1) + hb0 * hc0 + hb1 * hc1
        shape = list(self.shape)
        shape[2 - a] -= 1
        return np.broadcast_to(n_e, shape).astype(np.int64)

    # -- boundary node sets ------------------------------------------------

    def bottom_mask(self) -> np.ndarray:
        """Global Dirichlet set: the z = lo face (``twolevel.py:115-122``)."""
        m = np.zeros(self.shape, dtype=bool)
        m[0] = True
        return m

    def gamma_mask(self) -> np.ndarray:
        """Local Dirichlet set: nodes of LATERAL + BOTTOM facets (``mesh.py:498,507``)."""
        m = np.zeros(self.shape, dtype=bool)
        m[0] = True
        m[:, 0, :] = True
        m[:, -1, :] = True
        m[:, :, 0] = True
        m[:, :, -1] = True
        return m


class StencilOperator:
    """Constrained backward-Euler operator A_c and RHS on one grid."""

    def __init__(self, grid: KuhnGrid, kappa: float, rhoc: float, dt: float,
                 dirichlet: np.ndarray):
        self.grid = grid
        hx, hy, hz = grid.h
        V = hx * hy * hz
        self.mass = (rhoc / dt) * V * grid.node_incidence() / 24.0
        self.c = [kappa * V / (grid.h[a] ** 2) * grid.edge_incidence(a) / 6.0 for a in range(3)]
        diag = self.mass.copy()
        for a in range(3):
            sl_lo, sl_hi = _edge_slices(a)
            diag[sl_lo] += self.c[a]
            diag[sl_hi] += self.c[a]
        self.D = dirichlet
        self.diag_c = np.where(dirichlet, 1.0, diag)        # diagonal of A_c

    def inv_diag(self) -> np.ndarray:
        """Jacobi preconditioner as built in ``fem.py:283-284``."""
        d = self.diag_c.ravel()
        return np.where(d > 0, 1.0 / d, 1.0)

    def apply(self, x: np.ndarray) -> np.ndarray:
        X = x.reshape(self.grid.shape)
        Xm = np.where(self.D, 0.0, X)
        Y = self.diag_c * X
        for a in range(3):
            sl_lo, sl_hi = _edge_slices(a)
            Y[sl_lo] -= self.c[a] * Xm[sl_hi]
            Y[sl_hi] -= self.c[a] * Xm[sl_lo]
        Y[self.D] = X[self.D]
        return Y.ravel()

    def apply_full(self, x: np.ndarray) -> np.ndarray:
        """Unconstrained A x (before Dirichlet elimination)."""
        X = x.reshape(self.grid.shape)
        Y = self.mass * X
        for a in range(3):
            sl_lo, sl_hi = _edge_slices(a)
            d = self.c[a] * (X[sl_lo] - X[sl_hi])
            Y[sl_lo] += d
            Y[sl_hi] -= d
        return Y.ravel()

    def rhs(self, T_old: np.ndarray, load: np.ndarray | None, g: np.ndarray) -> np.ndarray:
        """Constrained RHS: lumped mass * T_old + load, Dirichlet lift, b_D = g."""
        B = self.mass * T_old.reshape(self.grid.shape)
        if load is not None:
            B = B + load.reshape(self.grid.shape)
        G = np.where(self.D, g.reshape(self.grid.shape), 0.0)
        for a in range(3):
            sl_lo, sl_hi = _edge_slices(a)
            B[sl_lo] += self.c[a] * G[sl_hi]
            B[sl_hi] += self.c[a] * G[sl_lo]
        B[self.D] = G[self.D]
        return B.ravel()


def _edge_slices(a: int):
    """Slices selecting the low and high node of every axis-a edge in [k, j, i] arrays."""
    lo = [slice(None)] * 3
    hi = [slice(None)] * 3
    lo[2 - a] = slice(None, -1)
    hi[2 - a] = slice(1, None)
    return tuple(lo), tuple(hi)


# -- sources -----------------------------------------------------------------

def gaussian_load(grid: KuhnGrid, beam, center) -> np.ndarray:
    """Nodal load of ``gaussian_source_3d`` by the 4-point tet rule.

    Restates ``lpbfsim/fem.py:176-178`` (rhs_elem = sum_q w_q Q(x_q) phi_q vol)
    with ``lpbfsim/sources.py:67-77`` evaluated at every quadrature point of
    every Kuhn tet (``lpbfsim/mesh.py:279-283``).
    """
    c = np.asarray(center, dtype=float)
    r, d = beam.radius, beam.depth
    peak = 6.0 * np.sqrt(3.0) * beam.power * beam.absorptivity / (2.0 * np.pi * r**2 * d)
    ax = [grid.axis(a) for a in range(3)]
    vol = float(np.prod(grid.h)) / 6.0
    out = np.zeros(grid.shape)
    nz, ny, nx = (int(v) for v in grid.n[::-1])
    for perm in PERMS:
        V = tet_vertices(perm)
        Q = []
        for q in range(4):
            # quadrature point x_q = sum_i phi[q,i] X(v_i), per axis
            e = []
            for a, scale in ((0, r), (1, r), (2, d)):
                n_a = int(grid.n[a])
                xq = sum(QPHI[q, i] * ax[a][V[i, a]:V[i, a] + n_a] for i in range(4))
                e.append(3.0 * ((xq - c[a]) / scale) ** 2)
            arg = (e[0][None, None, :] + e[1][None, :, None]) + e[2][:, None, None]
            Q.append(peak * np.exp(-arg))
        for j in range(4):
            contrib = sum(QW[q] * Q[q] * QPHI[q, j] for q in range(4)) * vol
            vx, vy, vz = V[j]
            out[vz:vz + nz, vy:vy + ny, vx:vx + nx] += contrib
    return out.ravel()


def locate(grid: KuhnGrid, points) -> tuple[np.ndarray, np.ndarray]:
    """Kuhn-P1 point location: (node ids (n,4), barycentrics (n,4)).

    Restates ``Mesh.locate`` (``lpbfsim/mesh.py:308-339``): cell by
    ``floor((x - lo)/h)`` clipped to the grid, then the Kuhn tet given by the
    descending order of the in-cell fractional coordinates xi; barycentrics
    (1 - xi_a, xi_a - xi_b, xi_b - xi_c, xi_c) on vertices (0, e_a, e_a+e_b, 1).
    """
    p = np.atleast_2d(np.asarray(points, dtype=float))
    lo = grid.box_lo
    cell = np.floor((p - lo) / grid.h).astype(np.int64)
    cell = np.clip(cell, 0, grid.n - 1)
    corner = np.stack([grid.axis(a)[cell[:, a]] for a in range(3)], axis=1)
    xi = (p - corner) / grid.h
    order = np.argsort(-xi, axis=1, kind="stable")
    xs = np.take_along_axis(xi, order, axis=1)
    bary = np.stack([1.0 - xs[:, 0], xs[:, 0] - xs[:, 1], xs[:, 1] - xs[:, 2], xs[:, 2]], axis=1)
    NX, NY = int(grid.n[0]) + 1, int(grid.n[1]) + 1
    strides = np.array([1, NX, NX * NY], dtype=np.int64)
    base = cell @ strides
    step = strides[order]                                   # (n, 3)
    nodes = np.stack([base, base + step[:, 0], base + step[:, 0] + step[:, 1],
                      base + step[:, 0] + step[:, 1] + step[:, 2]], axis=1)
    return nodes, bary


def interpolate(grid: KuhnGrid, values: np.ndarray, points) -> np.ndarray:
    """P1 interpolant at points (``lpbfsim/mesh.py:358-361``)."""
    nodes, bary = locate(grid, points)
    return np.einsum("nk,nk->n", bary, values[nodes])


def deposit_load(grid: KuhnGrid, points: np.ndarray, power: np.ndarray) -> np.ndarray:
    """``SweptTrackDeposit.load`` (``lpbfsim/sources.py:164-172``)."""
    out = np.zeros(grid.n_nodes)
    if len(points) == 0:
        return out
    nodes, bary = locate(grid, points)
    np.add.at(out, nodes.reshape(-1), (power[:, None] * bary).reshape(-1))
    return out


def swept_samples(beam, pieces, dt: float):
    """Sample lattice of ``SweptTrackDeposit.sample_points`` (``lpbfsim/sources.py:137-162``):
    8 x 3 x 3 points per swept piece, each carrying P*eta*(len/v)/dt/72."""
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
        piece_power = beam.power * beam.absorptivity * (length / v) / dt
        pts_all.append(pts)
        pw_all.append(np.full(len(pts), piece_power / len(pts)))
    if not pts_all:
        return np.empty((0, 3)), np.empty(0)
    return np.vstack(pts_all), np.concatenate(pw_all)


def mass_norm2(grid: KuhnGrid, v: np.ndarray) -> float:
    """v^T M v with the P1 mass matrix of the Kuhn tets (``lpbfsim/fem.py:434-446``; the
    4-point rule is exact for P1 x P1, so M = sum over tets of V/20 (1 + delta_ij)):
    per tet V/20 (sum v_i^2 + (sum v_i)^2), V = hx hy hz / 6."""
    nx, ny, nz = (int(c) for c in grid.n)
    V = np.asarray(v, dtype=np.float64).reshape(nz + 1, ny + 1, nx + 1)

    def corner(bits):
        return V[(bits >> 2) & 1:(bits >> 2 & 1) + nz, (bits >> 1) & 1:((bits >> 1) & 1) + ny,
                 bits & 1:(bits & 1) + nx]

    c = [corner(b) for b in range(8)]          # bit a = +1 along axis a (x = bit 0)
    tot = 0.0
    for perm in PERMS:
        verts, acc = [0], 0
        for ax in perm:
            acc += 1 << ax
            verts.append(acc)
        vs = [c[q] for q in verts]
        s1 = vs[0] + vs[1] + vs[2] + vs[3]
        tot += float(np.sum(vs[0] ** 2 + vs[1] ** 2 + vs[2] ** 2 + vs[3] ** 2 + s1 ** 2))
    h = (np.asarray(grid.hi0) - np.asarray(grid.lo0)) / np.asarray(grid.n)
    return tot * float(np.prod(h)) / 6.0 / 20.0


def gamma_facets(L: KuhnGrid):
    """The interface facets of a local grid (``lpbfsim/mesh.py:477-523``: LATERAL + BOTTOM
    boundary facets) on the structured Kuhn lattice: per boundary face cell two triangles,
    each the face of one Kuhn tet.  Yields (triangle (3,3) int lattice offsets, axis, side,
    the two tet vertices along the normal) per facet, as integer node coordinates:

    - low side of axis a (x_a = 0 plane of a cell at cell index 0): tets whose path steps a
      last, perm (b, c, a) / (c, b, a); facet (v0, v1, v2); dT/dx_a = (T(v3) - T(v2)) / h_a;
      outward normal -e_a.
    - high side (x_a = 1 plane of a cell at index n_a - 1): tets stepping a first,
      perm (a, b, c) / (a, c, b); facet (v1, v2, v3); dT/dx_a = (T(v1) - T(v0)) / h_a;
      outward normal +e_a.
    """
    n = [int(v) for v in L.n]
    out = []
    for a, side in ((0, 0), (0, 1), (1, 0), (1, 1), (2, 0)):
        b, c = [x for x in range(3) if x != a]
        cells_b, cells_c = range(n[b]), range(n[c])
        ca = 0 if side == 0 else n[a] - 1
        perms = ((b, c, a), (c, b, a)) if side == 0 else ((a, b, c), (a, c, b))
        for jc in cells_c:
            for jb in cells_b:
                cell = [0, 0, 0]
                cell[a], cell[b], cell[c] = ca, jb, jc
                for perm in perms:
                    v = tet_vertices(perm) + np.array(cell)
                    if side == 0:
                        out.append((v[[0, 1, 2]], a, side, (v[2], v[3])))
                    else:
                        out.append((v[[1, 2, 3]], a, side, (v[0], v[1])))
    return out


def transmission_load(G: KuhnGrid, L: KuhnGrid, T_local: np.ndarray, jump: float) -> np.ndarray:
    """``transmission_load`` (``lpbfsim/twolevel.py:159-183``) for constant conductivities:
    sum over interface facets and their 3 edge-midpoint quadrature points (weights
    area/3, ``mesh.py:131-137``) of jump * dT/dn * w_global, scattered with the global
    Kuhn-P1 barycentrics of each point (``np.add.at`` in facet order)."""
    NX, NY = int(L.n[0]) + 1, int(L.n[1]) + 1
    h = L.h
    lo = L.box_lo

    def nid(v):
        return int(v[0] + NX * (v[1] + NY * v[2]))

    pts, dens = [], []
    for tri, a, side, (va, vb) in gamma_facets(L):
        b, c = [x for x in range(3) if x != a]
        area = 0.5 * h[b] * h[c]
        g = (T_local[nid(vb)] - T_local[nid(va)]) / h[a]
        dTdn = g if side == 1 else -g
        X = lo + tri * h
        for (p, q) in ((0, 1), (1, 2), (0, 2)):
            pts.append(0.5 * (X[p] + X[q]))
            dens.append(area / 3.0 * jump * dTdn)
    pts = np.array(pts)
    dens = np.array(dens)
    nodes, bary = locate(G, pts)
    load = np.zeros(G.n_nodes)
    np.add.at(load, nodes.reshape(-1), (dens[:, None] * bary).reshape(-1))
    return load

"""Temperature-dependent assembly in stencil form (TEST INFRASTRUCTURE ONLY, see
``oracle/__init__.py``).

Restates ``assemble_system`` (``lpbfsim/fem.py:129-194``) with ``_material_arrays``
(``:214-238``), the secant latent capacity (``_latent_slope``, ``:197-211``) and the
lumped Robin / lagged-radiation top terms (``_add_robin``, ``:241-268``) on the Kuhn
lattice.  On a Kuhn tet the P1 gradients are axis-aligned along the tet's path, so the
element stiffness kbar*vol*grad_i.grad_j couples only consecutive path vertices
(-kbar vol / h_a^2 on the path edge along axis a) and the assembled operator is a
7-point stencil with per-edge weights:

    (A x)_p = diag_p x_p - sum_a (w_a[p] x_{p+e_a} + w_a[p-e_a] x_{p-e_a})

``diag`` = lumped mass + the incident edge weights (+ lumped Robin on the top face),
``w_a[p]`` = the weight of the edge (p, p+e_a).  The device kernel ``k_vc_assemble``
computes the same arrays node by node.
"""

from __future__ import annotations

import itertools

import numpy as np

from .kuhn import ALPHA, BETA, KuhnGrid, QPHI

PERMS = list(itertools.permutations(range(3)))


def phase_fraction(mat, T):
    return 0.5 * (1.0 + np.tanh(mat.S * (np.asarray(T, dtype=float) - 0.5 * (mat.T_solidus + mat.T_liquidus))))


def phase_fraction_derivative(mat, T):
    x = mat.S * (np.asarray(T, dtype=float) - 0.5 * (mat.T_solidus + mat.T_liquidus))
    ax = np.abs(x)
    e = np.exp(-ax)
    s = 2.0 * e / (1.0 + e * e)
    return 0.5 * mat.S * s * s


def latent_slope(mat, T, T_old):
    """``_latent_slope`` (``lpbfsim/fem.py:197-211``)."""
    dT = T - T_old
    small = np.abs(dT) < 1e-6
    df = phase_fraction(mat, T) - phase_fraction(mat, T_old)
    slope = np.where(small, phase_fraction_derivative(mat, 0.5 * (T + T_old)), df / np.where(small, 1.0, dT))
    return mat.chi * slope


def assemble(G: KuhnGrid, mat, T_old, T_lag, dt, source=None, latent=False, robin=None):
    """(diag, w (3, n), b) of the unconstrained system.  ``source(points) -> Q``;
    ``robin = (h_conv, sigma*eps or 0, T_ambient)`` for the top face."""
    n = G.n_nodes
    NX, NY = int(G.n[0]) + 1, int(G.n[1]) + 1
    nc = [int(v) for v in G.n]
    h = G.h
    vol = float(np.prod(h)) / 6.0
    diag = np.zeros(n)
    w = np.zeros((3, n))
    b = np.zeros(n)
    T_old = np.asarray(T_old, dtype=float)
    T_lag = np.asarray(T_lag, dtype=float)
    ci = np.stack(np.meshgrid(np.arange(nc[0]), np.arange(nc[1]), np.arange(nc[2]), indexing="ij"),
                  axis=-1).reshape(-1, 3)
    base = ci[:, 0] + NX * (ci[:, 1] + NY * ci[:, 2])
    strides = np.array([1, NX, NX * NY])
    lo = G.box_lo
    for perm in PERMS:
        offs = [np.zeros(3, dtype=int)]
        for ax in perm:
            o = offs[-1].copy()
            o[ax] += 1
            offs.append(o)
        ids = np.stack([base + o @ strides for o in offs], axis=1)            # (E, 4)
        Tq = T_lag[ids] @ QPHI.T                                               # (E, 4) qp q
        Tq_old = T_old[ids] @ QPHI.T
        kq = np.interp(Tq, mat.conductivity_table[:, 0], mat.conductivity_table[:, 1])
        cq = np.interp(Tq, mat.heat_capacity_table[:, 0], mat.heat_capacity_table[:, 1])
        if latent and mat.chi > 0.0:
            cq = cq + latent_slope(mat, Tq, Tq_old)
        coeff = mat.rho * cq
        kbar = kq @ np.full(4, 0.25)
        ml = np.einsum("q,eq,qi->ei", np.full(4, 0.25), coeff / dt, QPHI) * vol
        np.add.at(diag, ids.reshape(-1), ml.reshape(-1))
        np.add.at(b, ids.reshape(-1), (ml * T_old[ids]).reshape(-1))
        if source is not None:
            X = np.stack([lo + (ci + o) * h for o in offs], axis=1)          # (E, 4, 3)
            qp = np.einsum("qi,eid->eqd", QPHI, X)
            Q = np.asarray(source(qp.reshape(-1, 3))).reshape(-1, 4)
            np.add.at(b, ids.reshape(-1), (np.einsum("q,eq,qi->ei", np.full(4, 0.25), Q, QPHI) * vol).reshape(-1))
        for r, ax in enumerate(perm):
            we = kbar * vol / h[ax] ** 2
            np.add.at(diag, ids[:, r], we)
            np.add.at(diag, ids[:, r + 1], we)
            np.add.at(w[ax], ids[:, r], we)
    if robin is not None:
        hc, se, T_amb = robin
        k = nc[2]
        tri = [((0, 0), (1, 0), (1, 1)), ((0, 0), (0, 1), (1, 1))]
        area = 0.5 * h[0] * h[1]
        cj = np.stack(np.meshgrid(np.arange(nc[0]), np.arange(nc[1]), indexing="ij"), axis=-1).reshape(-1, 2)
        for t in tri:
            vid = np.stack([(cj[:, 0] + a) + NX * ((cj[:, 1] + bb) + NY * k) for a, bb in t], axis=1)
            for (pa, pb) in ((0, 1), (1, 2), (0, 2)):
                Tq = 0.5 * (T_lag[vid[:, pa]] + T_lag[vid[:, pb]])
                coeff = hc + se * Tq ** 3
                load = hc * T_amb + se * T_amb ** 4
                for v in (pa, pb):
                    np.add.at(diag, vid[:, v], coeff * 0.5 * area / 3.0)
                    np.add.at(b, vid[:, v], np.full(len(vid), load * 0.5 * area / 3.0))
    return diag, w, b


def apply(G: KuhnGrid, diag, w, x):
    NX, NY = int(G.n[0]) + 1, int(G.n[1]) + 1
    st = [1, NX, NX * NY]
    y = diag * x
    for a in range(3):
        y[:-st[a]] -= w[a][:-st[a]] * x[st[a]:]
        y[st[a]:] -= w[a][:-st[a]] * x[:-st[a]]
    return y


def constrained(G: KuhnGrid, diag, w, b, dmask, g):
    """``SparseSystem.constrained`` (``lpbfsim/fem.py:89-105``) in stencil form: free rows
    drop their Dirichlet couplings into the RHS, Dirichlet rows become identity rows."""
    NX, NY = int(G.n[0]) + 1, int(G.n[1]) + 1
    st = [1, NX, NX * NY]
    free = ~dmask
    gD = np.where(dmask, g, 0.0)
    bc = b.copy()
    for a in range(3):
        bc[:-st[a]] += w[a][:-st[a]] * gD[st[a]:]
        bc[st[a]:] += w[a][:-st[a]] * gD[:-st[a]]
    bc[dmask] = g[dmask]
    wc = w.copy()
    for a in range(3):
        keep = free[:-st[a]] & free[st[a]:]
        wc[a][:-st[a]] *= keep
    dc = np.where(dmask, 1.0, diag)
    return dc, wc, bc


def step(G: KuhnGrid, mat, T_old, dt, source, dmask, g, latent, robin, rtol=1e-12,
         picard_tol=1e-8, picard_max=25):
    """``step_backward_euler`` (``lpbfsim/fem.py:307-355``): Picard passes with lag damping,
    each an assembly + constrained Jacobi-PCG (scipy's recurrences) + re-imposed x_D.
    Returns (x, picard passes, [CG iterations per pass])."""
    from .pcg import cg_mirror
    T_lag = np.asarray(T_old, dtype=float)
    inc, prev_inc, theta = np.inf, np.inf, 1.0
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

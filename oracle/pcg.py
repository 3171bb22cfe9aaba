"""Jacobi-PCG mirroring scipy.sparse.linalg.cg (scipy 1.18.1) — oracle only.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

The reference solves with ``spla.cg(A, b, rtol=rtol, M=diag^-1, maxiter=20n)``
(``lpbfsim/fem.py:282-298``).  scipy's loop (``scipy/sparse/linalg/_isolve/
iterative.py:383-430`` in 1.18.1): x0 = 0, r = b, atol = rtol*||b||; each
iteration first tests ||r|| < atol, then z = M r, rho = r.z, p = z (first) or
p = beta*p + z, q = A p, alpha = rho/(p.q), x += alpha p, r -= alpha q.
After the loop the reference checks ||A x - b|| / ||b|| <= 100 rtol and raises
``NonConvergence`` otherwise, then re-imposes the Dirichlet values.
"""

from __future__ import annotations

import numpy as np


class OracleNonConvergence(RuntimeError):
    def __init__(self, iterations, residual):
        self.iterations = iterations
        self.residual = residual
        super().__init__(f"conjugate gradients did not converge in {iterations} iterations "
                         f"(last residual {residual:.3e})")


def cg_mirror(apply, b: np.ndarray, inv_diag: np.ndarray, rtol: float, maxiter: int):
    """Returns (x, info, iterations) exactly as scipy's cg would (info 0 = converged)."""
    bnrm2 = np.linalg.norm(b)
    if bnrm2 == 0:
        return b, 0, 0
    atol = max(0.0, float(rtol) * float(bnrm2))
    x = np.zeros_like(b)
    r = b.copy()
    rho_prev, p = None, None
    for it in range(maxiter):
        if np.linalg.norm(r) < atol:
            return x, 0, it
        z = inv_diag * r
        rho = np.dot(r, z)
        if it > 0:
            beta = rho / rho_prev
            p *= beta
            p += z
        else:
            p = np.empty_like(r)
            p[:] = z[:]
        q = apply(p)
        alpha = rho / np.dot(p, q)
        x += alpha * p
        r -= alpha * q
        rho_prev = rho
    return x, maxiter, maxiter


def solve_constrained(op, b: np.ndarray, g_flat: np.ndarray, rtol: float):
    """``solve_linear`` (cg branch, ``lpbfsim/fem.py:271-291``) on a stencil operator.

    Returns (x with x_D = g, iterations, true relative residual).
    """
    bnorm = np.linalg.norm(b)
    D = op.D.ravel()
    if bnorm == 0.0:
        x = np.zeros_like(b)
        x[D] = g_flat[D]
        return x, 0, 0.0
    x, info, its = cg_mirror(op.apply, b, op.inv_diag(), rtol, 20 * b.size)
    res = np.linalg.norm(op.apply(x) - b) / bnorm
    if info != 0 or res > 1e2 * rtol:
        raise OracleNonConvergence(abs(info) or -1, res)
    x[D] = g_flat[D]
    return x, its, res


def cg_chronopoulos_gear(apply, b: np.ndarray, inv_diag: np.ndarray, rtol: float, maxiter: int):
    """Chronopoulos-Gear PCG (one reduction per iteration), as the device's default
    resident kernel runs it (csrc/tl_resident_cg.cuh): same stop test as scipy's cg
    (||r|| < rtol ||b|| at the top of each iteration), iterates equal to CG's in exact
    arithmetic.  Returns (x, info, iterations)."""
    bnrm2 = np.linalg.norm(b)
    if bnrm2 == 0:
        return b, 0, 0
    atol = float(rtol) * float(bnrm2)
    x = np.zeros_like(b)
    r = b.copy()
    rr = np.dot(r, r)
    u = inv_diag * r
    w = apply(u)
    gam, dlt = np.dot(r, u), np.dot(w, u)
    p = s = None
    gam_prev = alpha_prev = 1.0
    for it in range(maxiter):
        if np.sqrt(rr) < atol:
            return x, 0, it
        if it == 0:
            beta, alpha = 0.0, gam / dlt
            p, s = u.copy(), w.copy()
        else:
            beta = gam / gam_prev
            alpha = gam / (dlt - beta * gam / alpha_prev)
            p = u + beta * p
            s = w + beta * s
        x = x + alpha * p
        r = r - alpha * s
        u = inv_diag * r
        w = apply(u)
        gam_prev, alpha_prev = gam, alpha
        gam, dlt, rr = np.dot(r, u), np.dot(w, u), np.dot(r, r)
    return x, maxiter, maxiter

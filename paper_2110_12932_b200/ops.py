"""Host-buffer entry points of the device kernels (one call = one C-ABI call).

These back the step-level seams of the reference API (``fem.step_backward_euler``,
``Mesh.interpolate``, ``SweptTrackDeposit.load``) for callers that hold numpy
arrays.  The device-resident multirate loop lives in ``multirate.py``.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .errors import NonConvergence, SolverError


def _f64(a, n=None) -> np.ndarray:
    out = np.ascontiguousarray(a, dtype=np.float64)
    if n is not None and out.shape != (n,):
        raise SolverError(f"expected {n} values, got {out.shape}")
    return out


def interpolate_points(grid, values, points) -> np.ndarray:
    """Kuhn-P1 interpolant of a grid field at arbitrary points (``mesh.py:358-361``)."""
    v = _f64(values, grid.n_nodes)
    pts = np.ascontiguousarray(np.atleast_2d(points), dtype=np.float64)
    out = np.empty(len(pts))
    desc = grid.desc()
    N.check(N.lib().tl_interpolate_points_host(C.byref(desc), N.dptr(v), N.dptr(pts.reshape(-1)),
                                               len(pts), N.dptr(out)), "interpolate")
    return out


def interpolate_to_grid(global_grid, values, target, gamma_only: bool = False,
                        out: np.ndarray | None = None) -> np.ndarray:
    """Global field at every node (or only the gamma nodes) of a target lattice."""
    v = _f64(values, global_grid.n_nodes)
    res = np.zeros(target.n_nodes) if out is None else _f64(out, target.n_nodes).copy()
    gd, td = global_grid.desc(), target.desc()
    N.check(N.lib().tl_interpolate_host(C.byref(gd), N.dptr(v), C.byref(td), int(gamma_only),
                                        N.dptr(res)), "interpolate")
    return res


def deposit_load(grid, points, power) -> np.ndarray:
    """``SweptTrackDeposit.load`` on the device (``sources.py:164-172``)."""
    pts = np.ascontiguousarray(np.reshape(points, (-1, 3)), dtype=np.float64)
    pw = _f64(power, len(pts))
    out = np.zeros(grid.n_nodes)
    desc = grid.desc()
    N.check(N.lib().tl_deposit_host(C.byref(desc), N.dptr(pts.reshape(-1)), N.dptr(pw), len(pts),
                                    N.dptr(out)), "deposit")
    return out


def raise_for(info, what: str = "conjugate gradients"):
    """Map a tl_solve_info to the reference's exceptions (``fem.py:280-288``, ``:50-51``)."""
    st = info.status if hasattr(info, "status") else info["status"]
    its = info.iterations if hasattr(info, "iterations") else info["iterations"]
    res = info.true_resid if hasattr(info, "true_resid") else info["true_resid"]
    if st == N.TL_SOLVE_OK:
        return
    if st == N.TL_SOLVE_NONFINITE:
        raise SolverError("field contains non-finite values")
    raise NonConvergence(what, abs(its) or -1, res)


def step(grid, kappa: float, rho_c: float, dt: float, dirichlet_kind: int, T_old,
         g=None, g_const: float = 0.0, load=None, gaussian=None, rtol: float = 1e-10,
         maxiter: int | None = None):
    """One constrained backward-Euler solve on the device; returns (x, SolveInfo)."""
    n = grid.n_nodes
    T = _f64(T_old, n)
    gA = None if g is None else _f64(g, n)
    ld = None if load is None else _f64(load, n)
    src = None
    if gaussian is not None:
        peak, radius, depth, center = gaussian
        src = N.Gaussian(float(peak), float(radius), float(depth),
                         (C.c_double * 3)(*map(float, center)), 1)
    x = np.empty(n)
    info = N.SolveInfo()
    desc = grid.desc()
    mi = min(20 * n, 2_000_000_000) if maxiter is None else int(maxiter)
    N.check(N.lib().tl_step_host(C.byref(desc), float(kappa), float(rho_c), float(dt),
                                 int(dirichlet_kind), N.dptr(gA), N.dptr(gA), 0.0, float(g_const),
                                 N.dptr(T), N.dptr(ld), C.byref(src) if src is not None else None,
                                 float(rtol), mi, N.dptr(x), C.byref(info)), "step")
    return x, info

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


def _f64(a, n=None):
    """A contiguous float64 host array, or the DeviceVector itself (fields may live on the
    device: every field argument of the C ABI takes host or device pointers)."""
    if isinstance(a, N.DeviceVector):
        if n is not None and a.n != n:
            raise SolverError(f"expected {n} values, got {a.shape}")
        return a
    dev = getattr(a, "device_values", None)
    if dev is not None:
        return _f64(dev, n)
    if hasattr(a, "mesh") and hasattr(a, "values"):          # a FieldState on the host
        a = a.values
    out = np.ascontiguousarray(a, dtype=np.float64)
    if n is not None and out.shape != (n,):
        raise SolverError(f"expected {n} values, got {out.shape}")
    return out


def dirichlet_list(nodes, values, n: int):
    """Dirichlet data as (int32 node ids, float64 values) for the *_nodes_host entry points:
    ids checked against the mesh; a node listed twice keeps its last value, like the
    reference's ``g[nodes] = values`` (``fem.py:294-305``)."""
    nodes = np.asarray(nodes, dtype=np.int64).ravel()
    vals = np.ascontiguousarray(np.broadcast_to(np.asarray(values, dtype=np.float64), nodes.shape))
    if nodes.size and (nodes.min() < 0 or nodes.max() >= n):
        raise SolverError("Dirichlet node outside the mesh")
    if nodes.size > 1 and np.any(np.diff(nodes) <= 0):
        uniq, first_rev = np.unique(nodes[::-1], return_index=True)
        vals = np.ascontiguousarray(vals[::-1][first_rev])
        nodes = uniq
    return np.ascontiguousarray(nodes, dtype=np.int32), vals


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
                        out: np.ndarray | None = None, on_device: bool = False):
    """Global field at every node (or only the gamma nodes) of a target lattice.
    ``on_device`` (full interpolation only): the result stays in a DeviceVector."""
    v = _f64(values, global_grid.n_nodes)
    if on_device and not gamma_only and out is None:
        res = N.DeviceVector(target.n_nodes)          # every entry is written
    else:
        res = np.zeros(target.n_nodes) if out is None else np.array(_f64(out, target.n_nodes), dtype=np.float64)
    gd, td = global_grid.desc(), target.desc()
    N.check(N.lib().tl_interpolate_host(C.byref(gd), N.dptr(v), C.byref(td), int(gamma_only),
                                        N.dptr(res)), "interpolate")
    return res


def interpolate_at_nodes(global_grid, values, target, nodes) -> np.ndarray:
    """The global field's interpolant at listed nodes of the target lattice (the trace on
    the interface nodes): bitwise the entries ``interpolate_to_grid`` writes there, but only
    ``len(nodes)`` values cross PCIe when the field lives on the device."""
    v = _f64(values, global_grid.n_nodes)
    idx = np.ascontiguousarray(nodes, dtype=np.int32)
    out = np.empty(idx.size)
    gd, td = global_grid.desc(), target.desc()
    N.check(N.lib().tl_interpolate_nodes_host(C.byref(gd), N.dptr(v), C.byref(td), idx.ctypes.data, idx.size,
                                              N.dptr(out)), "interpolate")
    return out


def add_loads(a, b):
    """a + b for dense load vectors that may live on the device (``tl_axpy_host``; 1.0 * b + a
    rounds like numpy's a + b).  ``None`` is the zero load."""
    if a is None:
        return b
    if b is None:
        return a
    if isinstance(a, N.DeviceVector) or isinstance(b, N.DeviceVector):
        if not isinstance(a, N.DeviceVector):
            a, b = b, a
        out = N.DeviceVector(a.n)
        N.check(N.lib().tl_dev_copy(out.ptr, N.dptr(a), 8 * a.n), "copy")
        bb = _f64(b, a.n)
        N.check(N.lib().tl_axpy_host(a.n, 1.0, N.dptr(bb), N.dptr(out)), "axpy")
        return out
    return a + b


def deposit_load(grid, points, power, on_device: bool = False):
    """``SweptTrackDeposit.load`` on the device (``sources.py:164-172``)."""
    pts = np.ascontiguousarray(np.reshape(points, (-1, 3)), dtype=np.float64)
    pw = _f64(power, len(pts))
    out = N.DeviceVector(grid.n_nodes) if on_device else np.zeros(grid.n_nodes)
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
         maxiter: int | None = None, on_device: bool = False, dirichlet=None):
    """One constrained backward-Euler solve on the device; returns (x, SolveInfo).  Fields
    may be numpy arrays or DeviceVectors; ``on_device``: x is left in a DeviceVector;
    ``dirichlet = (nodes, values)``: the Dirichlet data as a node list instead of ``g``."""
    n = grid.n_nodes
    T = _f64(T_old, n)
    gA = None if g is None else _f64(g, n)
    ld = None if load is None else _f64(load, n)
    src = None
    if gaussian is not None:
        peak, radius, depth, center = gaussian
        src = N.Gaussian(float(peak), float(radius), float(depth),
                         (C.c_double * 3)(*map(float, center)), 1)
    x = N.DeviceVector(n) if on_device else np.empty(n)
    info = N.SolveInfo()
    desc = grid.desc()
    mi = min(20 * n, 2_000_000_000) if maxiter is None else int(maxiter)
    if dirichlet is not None:
        nodes, vals = dirichlet_list(dirichlet[0], dirichlet[1], n)
        N.check(N.lib().tl_step_nodes_host(C.byref(desc), float(kappa), float(rho_c), float(dt),
                                           int(dirichlet_kind), nodes.ctypes.data, nodes.size, N.dptr(vals),
                                           N.dptr(T), N.dptr(ld), C.byref(src) if src is not None else None,
                                           float(rtol), mi, N.dptr(x), C.byref(info)), "step")
        return x, info
    N.check(N.lib().tl_step_host(C.byref(desc), float(kappa), float(rho_c), float(dt),
                                 int(dirichlet_kind), N.dptr(gA), N.dptr(gA), 0.0, float(g_const),
                                 N.dptr(T), N.dptr(ld), C.byref(src) if src is not None else None,
                                 float(rtol), mi, N.dptr(x), C.byref(info)), "step")
    return x, info

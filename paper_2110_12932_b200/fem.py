"""Fields, solver settings and the implicit step on the device.

``FieldState`` / ``uniform_field`` / ``SolverSettings`` / ``BoundarySpec`` keep
the reference's names and checks (``lpbfsim/fem.py:36-76,108-126``).
``step_backward_euler`` is seam 3 of the drop-in (``lpbfsim/fem.py:307-355``):
for the linear problems the device represents (constant material, no latent
heat, no radiation, Robin inactive) it performs the reference's single Picard
pass — assemble + constrain + Jacobi-PCG + residual check + Dirichlet
re-imposition — as one cooperative kernel.  Anything else raises
``UnsupportedOnDevice`` rather than falling back to a CPU path.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .config import SolverSettings
from .control import ThermalBC, material_constants
from .errors import NonConvergence, SolverError, UnsupportedOnDevice
from .grid import BOTTOM, TOP, StructuredGrid

__all__ = ["FieldState", "DeviceBackedFieldState", "field_arg", "device_fields", "uniform_field", "SolverSettings", "BoundarySpec", "GaussianSource",
           "step_backward_euler", "device_rtol", "Trajectory", "solve_monolithic", "PiecewiseMaterial",
           "RegionMask"]


@dataclass(frozen=True)
class FieldState:
    """Nodal temperature field bound to a grid at one time (``fem.py:36-56``)."""

    mesh: object
    values: np.ndarray
    time: float

    def __post_init__(self):
        v = np.asarray(self.values, dtype=float)
        if v.shape != (self.mesh.n_nodes,):
            raise SolverError(f"field has {v.shape} values for a mesh with {self.mesh.n_nodes} nodes")
        if not np.all(np.isfinite(v)):
            raise SolverError("field contains non-finite values")
        v.setflags(write=False)
        object.__setattr__(self, "values", v)

    def with_values(self, values, time: float | None = None) -> "FieldState":
        return FieldState(self.mesh, values, self.time if time is None else time)

    def retimed(self, time: float) -> "FieldState":
        """The same values stamped with another time (``FieldState(mesh, values, t)`` in the
        reference's drivers) without touching the values."""
        return FieldState(self.mesh, self.values, time)


def device_fields() -> bool:
    """Step-level solves return device-backed fields (``DeviceBackedFieldState``) unless
    ``TLGPU_DEVICE_FIELDS=0``."""
    import os
    return os.environ.get("TLGPU_DEVICE_FIELDS", "1") != "0"


class DeviceBackedFieldState(FieldState):
    """A step-level solve's result left on the device (``_native.DeviceVector``): the next
    solve, trace interpolation or interface functional reads it there, and ``values`` reads
    it back on first access (cached, read-only).  The producing solve already checked it for
    non-finite values (``fem.py:50-51``; TL_SOLVE_NONFINITE)."""

    def __init__(self, mesh, dev, time: float):
        if dev.n != mesh.n_nodes:
            raise SolverError(f"field has {dev.n} values for a mesh with {mesh.n_nodes} nodes")
        object.__setattr__(self, "mesh", mesh)
        object.__setattr__(self, "time", float(time))
        object.__setattr__(self, "device_values", dev)

    @property
    def values(self) -> np.ndarray:
        return self.device_values.to_host()

    def retimed(self, time: float) -> "FieldState":
        return DeviceBackedFieldState(self.mesh, self.device_values, time)

    def __reduce__(self):
        return (FieldState, (self.mesh, self.values, self.time))

    def __repr__(self):
        return f"DeviceBackedFieldState(mesh={self.mesh!r}, time={self.time!r})"


def field_arg(state_or_values):
    """What a step-level entry point is given for a field: the device vector when the field
    lives there, else a contiguous float64 host array."""
    dev = getattr(state_or_values, "device_values", None)
    if dev is not None:
        return dev
    if isinstance(state_or_values, N.DeviceVector):
        return state_or_values
    v = state_or_values.values if isinstance(state_or_values, FieldState) else state_or_values
    return np.ascontiguousarray(v, dtype=np.float64)


class UniformFieldState(FieldState):
    """``uniform_field``'s result: a constant field whose value array is built only when
    read (a 201M-node initial field need not exist on the host for the device to start
    from it; ``DeviceRun.initial`` takes ``.uniform_value``)."""

    def __init__(self, mesh, value: float, time: float = 0.0):
        value = float(value)
        if not np.isfinite(value):
            raise SolverError("field contains non-finite values")
        object.__setattr__(self, "mesh", mesh)
        object.__setattr__(self, "time", float(time))
        object.__setattr__(self, "uniform_value", value)
        object.__setattr__(self, "_v", None)

    @property
    def values(self) -> np.ndarray:
        if self._v is None:
            v = np.full(self.mesh.n_nodes, self.uniform_value)
            v.setflags(write=False)
            object.__setattr__(self, "_v", v)
        return self._v

    def retimed(self, time: float) -> "FieldState":
        return UniformFieldState(self.mesh, self.uniform_value, time)

    def __reduce__(self):
        return (UniformFieldState, (self.mesh, self.uniform_value, self.time))


def uniform_field(mesh, value: float, time: float = 0.0) -> FieldState:
    return UniformFieldState(mesh, value, time)


@dataclass(frozen=True)
class BoundarySpec:
    """Boundary data for one solve (``fem.py:108-126``)."""

    bc: ThermalBC
    robin_tags: tuple = (TOP,)
    radiation: bool = False
    dirichlet_nodes: np.ndarray = field(default_factory=lambda: np.empty(0, dtype=np.int64))
    dirichlet_values: np.ndarray | float = 0.0

    def dirichlet_array(self) -> np.ndarray:
        vals = np.broadcast_to(np.asarray(self.dirichlet_values, dtype=float),
                               np.shape(self.dirichlet_nodes))
        return np.asarray(vals, dtype=float)


@dataclass(frozen=True)
class GaussianSource:
    """``gaussian_source_3d`` bound to a centre (``sources.py:67-77``).

    The reference passes the source to ``assemble_system`` as an opaque
    callable; the device evaluates this one analytically at the Kuhn-tet
    quadrature points instead.  Calling it pointwise is still supported.
    """

    beam: object
    center: tuple

    @property
    def dim(self) -> int:
        return len(self.center)

    @property
    def peak(self) -> float:
        """3D: ``gaussian_source_3d``'s peak; 2D: P eta / (r d) (``sources.py:57-64``)."""
        b = self.beam
        if self.dim == 2:
            return b.power * b.absorptivity / (b.radius * b.depth)
        return b.gaussian_peak

    def __call__(self, points):
        p = np.atleast_2d(np.asarray(points, dtype=float))
        c = np.asarray(self.center, dtype=float)
        b = self.beam
        if self.dim == 2:
            ex = ((p[:, 0] - c[0]) / b.radius) ** 2
            ey = ((p[:, 1] - c[1]) / b.depth) ** 2
            return self.peak * np.exp(-(ex + ey))
        ex = 3.0 * ((p[:, 0] - c[0]) / b.radius) ** 2
        ey = 3.0 * ((p[:, 1] - c[1]) / b.radius) ** 2
        ez = 3.0 * ((p[:, 2] - c[2]) / b.depth) ** 2
        return b.gaussian_peak * np.exp(-(ex + ey + ez))

    def device_args(self):
        b = self.beam
        c = tuple(float(v) for v in self.center)
        return (self.peak, b.radius, b.depth, c if len(c) == 3 else (*c, 0.0))


def device_rtol(settings: SolverSettings) -> float:
    """CG tolerance the device uses for a SolverSettings.

    ``cg`` uses ``linear_tol`` exactly as ``fem.py:285``.  The reference's
    ``direct`` (sparse LU, ``fem.py:277-281``) has no device counterpart; it is
    served by CG at 1e-14, which lands within ~1e-13 of the LU solution on these
    mass-dominated systems.
    """
    return settings.linear_tol if settings.linear_solver == "cg" else min(settings.linear_tol, 1e-14)


def check_linear_problem(mat, bounds: BoundarySpec | None, latent: bool):
    if not getattr(mat, "is_constant", False):
        raise UnsupportedOnDevice("temperature-dependent conductivity/capacity tables are not on "
                                  "the device path (SURVEY.md §8 f, row 1)")
    if latent and getattr(mat, "chi", 0.0) > 0.0:
        raise UnsupportedOnDevice("latent heat (chi > 0) is not on the device path")
    if bounds is not None:
        bc = bounds.bc
        if bounds.robin_tags and bc.h_conv > 0:
            raise UnsupportedOnDevice("Robin convection (h_conv > 0) is not on the device path")
        if bounds.robin_tags and bounds.radiation and bc.emissivity > 0:
            raise UnsupportedOnDevice("radiation (emissivity > 0) is not on the device path")


def _dirichlet_kind(mesh: StructuredGrid, nodes: np.ndarray) -> int:
    nodes = np.asarray(nodes, dtype=np.int64)
    if np.array_equal(nodes, mesh.nodes_on(BOTTOM)):
        return N.TL_DIRICHLET_BOTTOM
    if np.array_equal(nodes, mesh.gamma_nodes()):
        return N.TL_DIRICHLET_GAMMA
    return -1          # any other set (none, all nodes, ...): the general path's node mask


@dataclass(frozen=True)
class PiecewiseMaterial:
    """``materials.PiecewiseMaterial`` (``materials.py:161-190``) on the structured grids: the
    region is a box (the fixed local box of ``run_reference``, ``runner.py:141-151``), a tet
    belongs to it when its centroid lies in the closed box."""

    inside: object
    outside: object
    box: object

    @property
    def is_constant(self) -> bool:
        return bool(self.inside.is_constant and self.outside.is_constant)

    @property
    def max_chi(self) -> float:
        return max(self.inside.chi, self.outside.chi)

    @property
    def T_liquidus(self) -> float:
        return self.inside.T_liquidus


@dataclass(frozen=True)
class RegionMask:
    """Element mask "tets whose centroid lies in box" (``runner.py:153-158``: latent_reference local)."""

    box: object


def problem_is_linear(mat, bounds: BoundarySpec, latent: bool) -> bool:
    """``_problem_is_linear`` (``fem.py:301-304``)."""
    radiative = bounds.radiation and bounds.bc.emissivity > 0 and len(bounds.robin_tags) > 0
    chi = mat.max_chi if isinstance(mat, PiecewiseMaterial) else mat.chi
    return bool(mat.is_constant) and not radiative and not (latent and chi > 0.0)


def _needs_general_path(mat, bounds: BoundarySpec, latent: bool) -> bool:
    convective = bool(bounds.robin_tags) and bounds.bc.h_conv > 0
    return convective or isinstance(mat, PiecewiseMaterial) or not problem_is_linear(mat, bounds, latent)


def _pad3(v) -> list:
    v = [float(x) for x in v]
    return v + [0.0] * (3 - len(v))


def vc_material(mat, latent: bool):
    """``tl_vc_material`` of a material (tables in K); returns (struct, arrays kept alive)."""
    kt = np.ascontiguousarray(mat.conductivity_table, dtype=np.float64)
    ct = np.ascontiguousarray(mat.heat_capacity_table, dtype=np.float64)
    tabs = [np.ascontiguousarray(kt[:, 0]), np.ascontiguousarray(kt[:, 1]),
            np.ascontiguousarray(ct[:, 0]), np.ascontiguousarray(ct[:, 1])]
    md = N.VcMaterial(tabs[0].ctypes.data, tabs[1].ctypes.data, len(kt), tabs[2].ctypes.data,
                      tabs[3].ctypes.data, len(ct), float(mat.rho), float(mat.chi), float(mat.S),
                      0.5 * (float(mat.T_solidus) + float(mat.T_liquidus)), 1 if latent else 0)
    return md, tabs


def _step_general(state: FieldState, dt: float, mat, source, bounds: BoundarySpec, settings: SolverSettings,
                  latent: bool, extra_load, stats, latent_mask=None) -> FieldState:
    """``step_backward_euler`` (``fem.py:307-355``) for temperature-dependent tables, latent
    heat, convection and lagged radiation: the reference's Picard loop (lag damping on
    stalls) over device passes (``tl_vc_step_host``: assembly, constraint and Jacobi-PCG on
    the GPU).  The whole loop runs in one call (``tl_vc_picard_host``): the relative
    increment ||x - T_lag|| / ||x|| is reduced on the device and the damped lag update is a
    kernel; the host maps the outcome to the reference's exceptions."""
    import ctypes as C
    from .ops import raise_for
    mesh = state.mesh
    if any(t != TOP for t in bounds.robin_tags):
        raise UnsupportedOnDevice("Robin terms are supported on the top face only")
    rad = bool(bounds.radiation and bounds.bc.emissivity > 0 and bounds.robin_tags)
    conv = bool(bounds.robin_tags) and bounds.bc.h_conv > 0
    region = None
    mo = None
    if isinstance(mat, PiecewiseMaterial):
        md, tabs = vc_material(mat.inside, latent and mat.inside.chi > 0.0)
        mo, tabs_o = vc_material(mat.outside, latent and mat.outside.chi > 0.0)
        region = mat.box
    else:
        md, tabs = vc_material(mat, latent and mat.chi > 0.0)
    if latent_mask is not None:
        if region is not None and (tuple(latent_mask.box.lo), tuple(latent_mask.box.hi)) != (tuple(region.lo), tuple(region.hi)):
            raise UnsupportedOnDevice("the latent mask and the material region must be the same box")
        region = latent_mask.box
    reg = None if region is None else np.array(_pad3(region.lo) + _pad3(region.hi), dtype=np.float64)
    rb = N.Robin(float(bounds.bc.h_conv) if conv else 0.0,
                 float(bounds.bc.sigma_sb * bounds.bc.emissivity) if rad else 0.0,
                 float(bounds.bc.T_ambient), 1 if (conv or rad) else 0)
    src = None
    if source is not None:
        peak, radius, depth, center = source.device_args()
        src = N.Gaussian(float(peak), float(radius), float(depth), (C.c_double * 3)(*map(float, center)), 1)
    n = mesh.n_nodes
    # Dirichlet data as a node list, scattered on the device (tl_vc_picard_nodes_host); a
    # repeated node keeps its last value, like the reference's g[nodes] = values
    from .ops import dirichlet_list
    dnodes32, dvals = dirichlet_list(bounds.dirichlet_nodes, bounds.dirichlet_array(), n)
    ld = None if extra_load is None else field_arg(extra_load)
    if ld is not None and ld.shape != (n,):
        raise SolverError("extra load does not match the mesh")
    T_old = field_arg(state)
    desc = mesh.desc()
    rtol = device_rtol(settings)
    linear = problem_is_linear(mat, bounds, latent)
    max_iter = 1 if linear else settings.picard_max_iter
    if max_iter < 1:
        # the reference's loop body never runs and it raises with an infinite increment
        # (fem.py:331-355)
        raise NonConvergence("Picard iteration", max_iter, float("inf"))
    t_new = state.time + dt
    x = N.DeviceVector(n) if device_fields() else np.empty(n)
    info = N.SolveInfo()
    npass = C.c_int32(0)
    its = np.zeros(max_iter, dtype=np.int32)
    mss = np.zeros(max_iter, dtype=np.float32)
    inc = C.c_double(0.0)
    timer = stats.timer("assembly") if stats is not None else None
    if timer is not None:
        timer.__enter__()
    try:
        # the whole Picard loop (fem.py:331-355) on the device: one upload, one read-back
        N.check(N.lib().tl_vc_picard_nodes_host(
            C.byref(desc), C.byref(md), C.byref(mo) if mo is not None else None, N.dptr(reg),
            1 if latent_mask is not None else 0, float(dt), N.dptr(T_old), N.dptr(ld),
            C.byref(src) if src is not None else None, C.byref(rb), dnodes32.ctypes.data, int(dnodes32.size),
            N.dptr(dvals), float(rtol),
            min(20 * n, 2_000_000_000), 1 if linear else 0, float(settings.picard_tol), int(max_iter), N.dptr(x),
            C.byref(npass), its.ctypes.data, mss.ctypes.data, C.byref(inc), C.byref(info)), "step")
    finally:
        if timer is not None:
            timer.__exit__(None, None, None)
    passes = int(npass.value)
    cg_failed = info.status != N.TL_SOLVE_OK
    ok = passes - (1 if cg_failed else 0)
    if stats is not None:
        stats.count("picard_iterations", ok)
        # one entry per successful pass, like picard_iterations (the failed pass raises)
        if stats.device_log is not None:
            stats.device_log.extend((float(mss[k]), int(its[k])) for k in range(ok))
    raise_for(info)
    if linear or inc.value < settings.picard_tol:
        if isinstance(x, N.DeviceVector):
            return DeviceBackedFieldState(mesh, x, t_new)
        return state.with_values(x, t_new)
    raise NonConvergence("Picard iteration", max_iter, inc.value)


def step_backward_euler(state: FieldState, dt: float, mat, source, bounds: BoundarySpec,
                        settings: SolverSettings, latent: bool = False, latent_mask=None,
                        extra_load=None, extra_mass_coeff=None, stats=None) -> FieldState:
    """One implicit step (``fem.py:307-355``) on the device.  Linear problems with the
    bottom or interface Dirichlet set take the fused single-kernel solve; temperature-
    dependent tables, latent heat, convection and radiation take the Picard path
    (``_step_general``)."""
    from .ops import raise_for, step
    if dt <= 0:
        raise SolverError("time step must be positive")
    if extra_mass_coeff is not None:
        raise UnsupportedOnDevice("overlap mass terms are not on the device path")
    if latent_mask is not None and not isinstance(latent_mask, RegionMask):
        raise UnsupportedOnDevice("the device takes latent masks as a box region (fem.RegionMask)")
    if source is not None and not isinstance(source, GaussianSource):
        raise UnsupportedOnDevice("the device evaluates GaussianSource objects, not opaque callables")
    # 2D grids (P1 triangles, csrc/tl_2d.cuh) always take the general path: the fused linear
    # kernels are the 3D 27-class stencil
    # ... and so do Dirichlet sets other than the bottom face / the interface (the fused
    # kernels know those two as node classes; the general path takes any node mask)
    kind = -1
    if not (_needs_general_path(mat, bounds, latent) or latent_mask is not None or state.mesh.dim == 2):
        kind = _dirichlet_kind(state.mesh, bounds.dirichlet_nodes)
    if kind < 0:
        return _step_general(state, dt, mat, source, bounds, settings, latent, extra_load, stats,
                             latent_mask=latent_mask)
    check_linear_problem(mat, bounds, latent)
    mesh = state.mesh
    kappa, rho_c = material_constants(mat)
    darr = bounds.dirichlet_array()
    g_const, dlist = 0.0, None
    if darr.size and np.all(darr == darr.flat[0]):
        g_const = float(darr.flat[0])          # constant data (the build plate): no array at all
    else:                                      # the trace: node list + values, scattered on the device
        dlist = (np.asarray(bounds.dirichlet_nodes, dtype=np.int64), darr)
    timer = stats.timer("assembly") if stats is not None else None
    if timer is not None:
        timer.__enter__()
    try:
        x, info = step(mesh, kappa, rho_c, dt, kind, field_arg(state), g_const=g_const, dirichlet=dlist,
                       load=None if extra_load is None else field_arg(extra_load),
                       gaussian=source.device_args() if source is not None else None,
                       rtol=device_rtol(settings), on_device=device_fields())
    finally:
        if timer is not None:
            timer.__exit__(None, None, None)
    raise_for(info)
    if stats is not None:
        stats.count("picard_iterations")
    if isinstance(x, N.DeviceVector):
        return DeviceBackedFieldState(mesh, x, state.time + dt)
    return state.with_values(x, state.time + dt)


@dataclass
class Trajectory:
    """Fields on one grid at strictly increasing times (``lpbfsim/fem.py:359-383``)."""

    mesh: object
    times: list = field(default_factory=list)
    values: list = field(default_factory=list)

    def append(self, state: FieldState):
        if self.times and state.time <= self.times[-1]:
            raise SolverError("trajectory times must increase")
        self.times.append(state.time)
        self.values.append(state.values)

    def __len__(self):
        return len(self.times)

    def state(self, idx: int) -> FieldState:
        return FieldState(self.mesh, self.values[idx], self.times[idx])

    def at_time(self, t: float, tol: float = 1e-9) -> FieldState:
        arr = np.asarray(self.times)
        idx = int(np.argmin(np.abs(arr - t)))
        if abs(arr[idx] - t) > tol * max(1.0, abs(t)):
            raise SolverError(f"no trajectory frame at t={t:g}")
        return self.state(idx)


class _NullCtx:
    def __enter__(self):
        return self

    def __exit__(self, *exc):
        return False


def solve_monolithic(mesh, mat, source_at, bounds_at, dt: float, n_steps: int, T_0: FieldState,
                     settings: SolverSettings = SolverSettings(), latent: bool = True,
                     latent_mask=None, stats=None, observer=None) -> Trajectory:
    """Uniform-step single-grid solve (``lpbfsim/fem.py:386-423``): the monolithic fine-grid
    reference, every step one device solve through ``step_backward_euler``.

    ``source_at(t)`` -> GaussianSource or None, ``bounds_at(t)`` -> BoundarySpec, both at
    each target time ``T_0.time + k dt`` (the reference's time bookkeeping).
    """
    if dt <= 0 or n_steps < 0:
        raise SolverError("schedule requires dt > 0 and n_steps >= 0")
    traj = Trajectory(mesh)
    traj.append(T_0)
    state = T_0
    for k in range(1, n_steps + 1):
        t_new = T_0.time + k * dt
        timer = stats.timer("reference_solve") if stats is not None else _NullCtx()
        with timer:
            state = step_backward_euler(state, t_new - state.time, mat, source_at(t_new),
                                        bounds_at(t_new), settings, latent=latent,
                                        latent_mask=latent_mask, stats=stats)
        if stats is not None:
            stats.count("reference_solves")
        traj.append(state)
        if observer is not None:
            observer(state)
    return traj

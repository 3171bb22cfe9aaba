"""Two-level coupling: problem, state, interface, and the step-level solves.

Mirrors ``lpbfsim/twolevel.py`` for constant materials with the interval-based
swept-track global source.  Equal conductivities on both levels (``one_way``,
``twolevel.py:101-113``) make the interface functional ``transmission_load``
identically zero (``:175``) and run device-resident (``multirate.DeviceRun``).
Distinct conductivities (``global_kappa_scale``, "alternate" mode) are the two-way
coupling of SURVEY §8f row 2: ``transmission_load`` is a device kernel
(``tl_transmission_host``) and ``two_level_iterate`` is the reference's relaxed
fixed point over device solves.  The opaque source
closures of the reference problem (``runner.py:49-81``) are replaced by the
beam and scan path themselves, so the device can evaluate the sources.

Seam 2 (``solve_global`` / ``solve_local``, ``twolevel.py:242-288``) runs one
device solve per call on host buffers.  The device-resident fast path is
``multirate.run_spacetime`` / ``run_space``.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .config import CouplingSettings, SolverSettings
from .control import LaserBeam, ScanPath, ThermalBC, check_immersed, material_constants
from .errors import CouplingError, CouplingNonConvergence, UnsupportedOnDevice
from .fem import BoundarySpec, FieldState, GaussianSource, check_linear_problem, step_backward_euler
from .grid import BOTTOM, TOP, StructuredGrid

__all__ = ["TwoLevelProblem", "TwoLevelState", "InterfaceGamma", "initial_state", "solve_global",
           "solve_local", "transmission_load", "extract_interface", "two_level_iterate", "relocate_local",
           "overlap_feedback", "consistency_diagnostic"]


@dataclass(frozen=True)
class InterfaceGamma:
    """Interface node set of a local lattice (``mesh.py:442-474``).

    ``trace_nodes`` are the lateral + bottom boundary nodes (sorted ids, as
    ``np.unique`` returns them, ``mesh.py:507``).
    """

    local: StructuredGrid
    trace_nodes: np.ndarray

    @property
    def measure(self) -> float:
        """Total area of the interface facets (``mesh.py:467-469``): lateral + bottom faces."""
        if self.local.dim == 2:                 # bottom edge + the two lateral edges
            lx, ly = (float(v) for v in self.local.box.lengths)
            return lx + 2.0 * ly
        lx, ly, lz = (float(v) for v in self.local.box.lengths)
        return lx * ly + 2.0 * (lx * lz + ly * lz)

    def trace_of(self, global_field, global_mesh) -> np.ndarray:
        """The global field (a FieldState, its values or a DeviceVector) at the trace nodes."""
        from .ops import interpolate_at_nodes
        from .fem import field_arg
        return interpolate_at_nodes(global_mesh, field_arg(global_field), self.local, self.trace_nodes)


def extract_interface(local: StructuredGrid, global_mesh: StructuredGrid) -> InterfaceGamma:
    """``extract_interface`` node part (``mesh.py:477-523``) with its immersion checks."""
    check_immersed(local.box, global_mesh.box, global_mesh.h)
    return InterfaceGamma(local, local.gamma_nodes())


@dataclass(frozen=True)
class TwoLevelState:
    global_field: FieldState
    local_field: FieldState
    gamma: InterfaceGamma
    trace: np.ndarray

    def __post_init__(self):
        tol = 1e-9 * max(abs(self.global_field.time), 1.0)
        if abs(self.global_field.time - self.local_field.time) > tol:
            raise CouplingError("global and local fields must share a time stamp")

    @property
    def time(self) -> float:
        return self.global_field.time


@dataclass
class TwoLevelProblem:
    """Everything fixed across a two-level run (``twolevel.py:78-142``), device flavour."""

    global_mesh: StructuredGrid
    mat_global: object
    mat_local: object
    bc: ThermalBC
    solver: SolverSettings = field(default_factory=SolverSettings)
    coupling: CouplingSettings = field(default_factory=CouplingSettings)
    mode: str = "alternate"
    beam: LaserBeam | None = None
    path: ScanPath | None = None
    source_global: str = "distributed"
    resolve_corrector: bool = True
    device: int = 0

    def __post_init__(self):
        if self.mode not in ("alternate", "full"):
            raise CouplingError(f"unknown global formulation {self.mode!r}")

    # -- reference attributes ----------------------------------------------------

    @property
    def one_way(self) -> bool:
        a, b = self.mat_global, self.mat_local
        same_k = a is b or (a.conductivity_table.shape == b.conductivity_table.shape
                            and np.array_equal(a.conductivity_table, b.conductivity_table))
        if not same_k:
            return False
        if self.mode == "alternate":
            return True
        # full mode: the overlap terms vanish only for fully equal materials without latent
        # heat (twolevel.py:101-113) -- one material object on both levels included
        same = a is b or (a.heat_capacity_table.shape == b.heat_capacity_table.shape
                          and np.array_equal(a.heat_capacity_table, b.heat_capacity_table)
                          and a.rho == b.rho and a.chi == b.chi
                          and (a.T_solidus, a.T_liquidus, a.S) == (b.T_solidus, b.T_liquidus, b.S))
        return bool(same and b.chi == 0.0)

    @property
    def interval_source(self) -> bool:
        return self.source_global == "distributed"

    def global_source(self, t0: float, t1: float, predictor: bool = False):
        """``_global_source_factory`` (``runner.py:62-81``): "distributed" -> the swept-track
        deposit of [t0, t1] as (points, power); "gaussian" -> the beam at t1 (a predictor
        sees it at t0 + 0.75 (t1 - t0)) as a GaussianSource; None when off."""
        from .schedule import swept_samples
        if self.source_global == "gaussian":
            return self.local_source(t0 + 0.75 * (t1 - t0) if predictor else t1)
        if self.path is None or self.beam is None:
            return None
        pieces = self.path.swept_pieces(t0, t1)
        if not pieces:
            return None
        return swept_samples(self.beam, pieces, t1 - t0)

    def local_source(self, t: float):
        """GaussianSource at the laser position of t, None outside the path (``runner.py:49-61``)."""
        if self.path is None or self.beam is None:
            return None
        tol = 1e-12 * max(self.path.t_end, 1.0)
        if t > self.path.t_end + tol or t < self.path.t_start - tol:
            return None
        return GaussianSource(self.beam, tuple(self.path.position(t)))

    def global_bounds(self) -> BoundarySpec:
        return BoundarySpec(bc=self.bc, robin_tags=(TOP,), radiation=False,
                            dirichlet_nodes=self.global_mesh.nodes_on(BOTTOM),
                            dirichlet_values=self.bc.T_buildplate)

    def local_bounds(self, gamma: InterfaceGamma, trace) -> BoundarySpec:
        return BoundarySpec(bc=self.bc, robin_tags=(TOP,), radiation=True,
                            dirichlet_nodes=gamma.trace_nodes, dirichlet_values=trace)

    # -- device support ---------------------------------------------------------

    def check_device_supported(self, resident: bool = True):
        """``resident``: the device-resident run (``DeviceRun`` / ``tl_run``: constant
        materials, no latent heat, no top-face Robin terms).  Otherwise the step-level
        drivers, whose solves take the Picard path for temperature-dependent tables,
        latent heat, convection and radiation (``fem._step_general``)."""
        if resident:
            check_linear_problem(self.mat_global, None, False)
            check_linear_problem(self.mat_local, None, True)
            if self.bc.h_conv > 0:
                raise UnsupportedOnDevice("Robin convection (h_conv > 0) is not on the device-resident path")
            if self.bc.emissivity > 0:
                raise UnsupportedOnDevice("radiation (emissivity > 0) is not on the device-resident path")
        if not self.one_way and self.mode != "alternate":
            if resident:
                raise UnsupportedOnDevice("full-mode overlap feedback runs through the step-level drivers")
            if self.interval_source:
                raise UnsupportedOnDevice("full-mode overlap feedback evaluates the global source at "
                                          "quadrature points: it needs source_global gaussian (the swept-"
                                          "track deposit is not a pointwise source)")
        if resident and not self.interval_source:
            raise UnsupportedOnDevice("the device-resident run uses the distributed (swept-track) "
                                      "global source; 'gaussian' runs through the step-level drivers")
        if self.global_mesh.dim != 3:
            # 2D (P1 triangles, csrc/tl_2d.cuh): the step-level drivers with the Picard-path solves
            if resident:
                raise UnsupportedOnDevice("the device-resident run is 3D; 2D runs go through the "
                                          "step-level drivers")
            # two-way coupling in 2D runs too: k_trans_entries2 (interface functional) and
            # k_overlap_feedback2 (full mode)

    @property
    def device_resident(self) -> bool:
        """True when the whole run fits the device-resident one-way loop."""
        if not self.one_way:
            return False
        try:
            self.check_device_supported(resident=True)
        except UnsupportedOnDevice:
            return False
        return True

    def constants(self):
        kg, rcg = material_constants(self.mat_global)
        kl, rcl = material_constants(self.mat_local)
        return kg, rcg, rcl


def initial_state(problem: TwoLevelProblem, local_mesh: StructuredGrid,
                  global_field: FieldState) -> TwoLevelState:
    """``initial_state`` (``twolevel.py:145-156``): local = P1(global), trace = P1 on gamma."""
    from .ops import interpolate_to_grid
    from .fem import DeviceBackedFieldState, device_fields, field_arg
    gamma = extract_interface(local_mesh, problem.global_mesh)
    lv = interpolate_to_grid(problem.global_mesh, field_arg(global_field), local_mesh, on_device=device_fields())
    if isinstance(lv, N.DeviceVector):
        local = DeviceBackedFieldState(local_mesh, lv, global_field.time)
        return TwoLevelState(global_field, local, gamma, gamma.trace_of(global_field, problem.global_mesh))
    local = FieldState(local_mesh, lv, global_field.time)
    return TwoLevelState(global_field, local, gamma, lv[gamma.trace_nodes].copy())


def transmission_load(local_field, gamma, global_mesh, mat_global, mat_local, on_device: bool = False):
    """Interface functional (``twolevel.py:159-183``): the integral over the interface facets
    of (kappa_global - kappa_local) dT_local/dn w_global.  Exactly zero for equal
    conductivities; otherwise one device call (constant conductivities: the jump is a
    number, ``tl_transmission_host``)."""
    from . import _native as N
    if np.array_equal(mat_global.conductivity_table, mat_local.conductivity_table):
        return np.zeros(global_mesh.n_nodes)
    lmesh = local_field.mesh
    from .fem import field_arg
    T = field_arg(local_field)
    if T.shape != (lmesh.n_nodes,):
        raise CouplingError("local field does not match its mesh")
    out = N.DeviceVector(global_mesh.n_nodes) if on_device else np.zeros(global_mesh.n_nodes)
    gd, ld = global_mesh.desc(), lmesh.desc()
    if mat_global.is_constant and mat_local.is_constant:
        kg, _ = material_constants(mat_global)
        kl, _ = material_constants(mat_local)
        N.check(N.lib().tl_transmission_host(N.C.byref(gd), N.C.byref(ld), N.dptr(T), float(kg - kl),
                                             N.dptr(out)), "transmission_load")
        return out
    tg = np.ascontiguousarray(mat_global.conductivity_table, dtype=np.float64)
    tl_ = np.ascontiguousarray(mat_local.conductivity_table, dtype=np.float64)
    cols = [np.ascontiguousarray(tg[:, 0]), np.ascontiguousarray(tg[:, 1]),
            np.ascontiguousarray(tl_[:, 0]), np.ascontiguousarray(tl_[:, 1])]
    N.check(N.lib().tl_transmission_tables_host(N.C.byref(gd), N.C.byref(ld), N.dptr(T), N.dptr(cols[0]),
                                                N.dptr(cols[1]), len(tg), N.dptr(cols[2]), N.dptr(cols[3]),
                                                len(tl_), N.dptr(out)), "transmission_load")
    return out


def overlap_feedback(problem: TwoLevelProblem, local_new: FieldState, local_old: FieldState, dt: float,
                     t0: float, t1: float, on_device: bool = False):
    """``_overlap_feedback`` (``twolevel.py:186-239``): the full-mode overlap terms as a
    global load, one device call (``tl_overlap_feedback_host``): capacity difference,
    conductivity-gradient cross terms and the source scaling at the global quadrature
    points inside the local box."""
    import ctypes as C
    from . import _native as N
    from .fem import vc_material
    gm, lm = problem.global_mesh, local_new.mesh
    if local_old.mesh is not lm and not lm.same_lattice(local_old.mesh):
        raise CouplingError("overlap feedback needs both local fields on one lattice")
    mg, tg = vc_material(problem.mat_global, False)
    ml, tl_ = vc_material(problem.mat_local, False)
    src = problem.global_source(t0, t1)
    gs = None
    if src is not None:
        if not isinstance(src, GaussianSource):
            raise UnsupportedOnDevice("full-mode overlap feedback needs a pointwise (gaussian) global source")
        peak, radius, depth, center = src.device_args()
        gs = N.Gaussian(float(peak), float(radius), float(depth), (C.c_double * 3)(*map(float, center)), 1)
    from .fem import field_arg
    Tn = field_arg(local_new)
    To = field_arg(local_old)
    out = N.DeviceVector(gm.n_nodes) if on_device else np.zeros(gm.n_nodes)
    gd, ld = gm.desc(), lm.desc()
    N.check(N.lib().tl_overlap_feedback_host(C.byref(gd), C.byref(ld), N.dptr(Tn), N.dptr(To), float(dt),
                                             C.byref(mg), C.byref(ml), C.byref(gs) if gs is not None else None,
                                             N.dptr(out)), "overlap_feedback")
    return out


def solve_global(problem: TwoLevelProblem, state: TwoLevelState, dt: float,
                 local_for_coupling: FieldState, stats=None, predictor: bool = False) -> FieldState:
    """One global backward-Euler step on the device (``twolevel.py:242-271``)."""
    from .ops import add_loads, deposit_load
    from .fem import device_fields
    t0, t1 = state.global_field.time, state.global_field.time + dt
    dev = device_fields()
    # equal conductivities: the interface functional is exactly zero (no load at all)
    load = None
    if not np.array_equal(problem.mat_global.conductivity_table, problem.mat_local.conductivity_table):
        load = transmission_load(local_for_coupling, state.gamma, problem.global_mesh,
                                 problem.mat_global, problem.mat_local, on_device=dev)
    dep = problem.global_source(t0, t1, predictor=predictor)
    source = None
    if isinstance(dep, GaussianSource):
        source = dep
    elif dep is not None:
        load = add_loads(load, deposit_load(problem.global_mesh, dep[0], dep[1], on_device=dev))
    if problem.mode == "full":
        load = add_loads(load, overlap_feedback(problem, local_for_coupling, state.local_field, dt, t0, t1,
                                                on_device=dev))
    timer = stats.timer("global_solve") if stats is not None else _Null()
    with timer:
        out = step_backward_euler(state.global_field, dt, problem.mat_global, source,
                                  problem.global_bounds(), problem.solver, latent=False,
                                  extra_load=load, stats=stats)
    if stats is not None:
        stats.count("global_solves")
    return out


def solve_local(problem: TwoLevelProblem, local_from: FieldState, dt: float, gamma: InterfaceGamma,
                trace, stats=None) -> FieldState:
    """One local step with the trace as Dirichlet data (``twolevel.py:274-288``)."""
    t1 = local_from.time + dt
    source = problem.local_source(t1)
    timer = stats.timer("local_solve") if stats is not None else _Null()
    with timer:
        out = step_backward_euler(local_from, dt, problem.mat_local, source,
                                  problem.local_bounds(gamma, trace), problem.solver, latent=True,
                                  stats=stats)
    if stats is not None:
        stats.count("local_solves")
    return out


def two_level_iterate(problem: TwoLevelProblem, state: TwoLevelState, dt: float,
                      local_from=None, local_dt=None, transmission_seed=None, trace_start=None,
                      stats=None):
    """Relaxed fixed point of one coupled step (``twolevel.py:299-358``): repeat {global
    solve with the latest interface functional; trace; local solve} until the relative
    trace change is below the coupling tolerance.  One pass when ``one_way``."""
    import time as _time
    cs = problem.coupling
    if local_from is None:
        local_from = state.local_field
    if local_dt is None:
        local_dt = dt
    t1 = state.global_field.time + dt
    if abs(local_from.time + local_dt - t1) > 1e-9 * max(abs(t1), 1e-30):
        raise CouplingError("fine and coarse steps must land on the same time")
    trace_prev = state.trace if trace_start is None else trace_start
    latest_local = state.local_field if transmission_seed is None else transmission_seed
    change = np.inf
    if stats is not None:
        t_begin = _time.perf_counter()
        inner0 = stats.seconds.get("global_solve", 0.0) + stats.seconds.get("local_solve", 0.0)
    for it in range(1, cs.max_iterations + 1):
        new_global = solve_global(problem, state, dt, latest_local, stats=stats)
        raw = state.gamma.trace_of(new_global, problem.global_mesh)
        relax = 1.0 if (it == 1 and trace_start is None) else cs.omega
        trace = raw if problem.one_way else trace_prev + relax * (raw - trace_prev)
        new_local = solve_local(problem, local_from, local_dt, state.gamma, trace, stats=stats)
        scale = max(float(np.linalg.norm(trace)), 1e-12)
        change = float(np.linalg.norm(trace - trace_prev)) / scale
        trace_prev = trace
        latest_local = new_local
        if stats is not None:
            stats.count("coupling_iterations")
        if problem.one_way or change < cs.tolerance:
            out = TwoLevelState(new_global, new_local.retimed(t1), state.gamma, trace)
            if stats is not None:
                inner = (stats.seconds.get("global_solve", 0.0) + stats.seconds.get("local_solve", 0.0)
                         - inner0)
                stats.seconds["coupling_overhead"] = (stats.seconds.get("coupling_overhead", 0.0)
                                                      + max(_time.perf_counter() - t_begin - inner, 0.0))
            return out, it
    raise CouplingNonConvergence(cs.max_iterations, change)


def relocate_local(state: TwoLevelState, policy, laser, direction, problem: TwoLevelProblem) -> TwoLevelState:
    """``relocate_local`` (``scanpath.py:208-248``): snapped, clamped move of the local box
    toward the laser (``LocalPlacement.relocate``); the whole local field and the trace are
    P1 interpolations of the current global field (device ``k_interp``)."""
    from .ops import interpolate_to_grid
    lmesh = state.local_field.mesh
    moved = lmesh.placement.relocate(policy, laser, direction, problem.global_mesh.box)
    if moved is None:
        return state
    new_mesh = StructuredGrid(moved)
    gmesh = problem.global_mesh
    gamma = extract_interface(new_mesh, gmesh)
    from .fem import DeviceBackedFieldState, device_fields, field_arg
    values = interpolate_to_grid(gmesh, field_arg(state.global_field), new_mesh, on_device=device_fields())
    if isinstance(values, N.DeviceVector):
        local = DeviceBackedFieldState(new_mesh, values, state.local_field.time)
    else:
        local = FieldState(new_mesh, values, state.local_field.time)
    trace = gamma.trace_of(state.global_field, gmesh)
    return TwoLevelState(state.global_field, local, gamma, trace)


def consistency_diagnostic(state: TwoLevelState, reference: FieldState, global_mesh) -> dict:
    """``consistency_diagnostic`` (``twolevel.py:376-400``): discrete L2 norms of (reference -
    fine) on the local domain, (reference - coarse) on the global tets whose centroid lies
    in the local box ("overlap") and outside it ("exterior"); interpolation and the masked
    mass norms on the device."""
    from . import _native as N
    from .ops import interpolate_to_grid
    lm = state.local_field.mesh
    out = np.zeros(2)
    rv = np.ascontiguousarray(reference.values, dtype=np.float64)
    lv = np.ascontiguousarray(state.local_field.values, dtype=np.float64)
    rd, ld, gd = reference.mesh.desc(), lm.desc(), global_mesh.desc()
    N.check(N.lib().tl_error_l2_host(N.C.byref(rd), N.dptr(rv), N.C.byref(ld), N.dptr(lv), N.dptr(out)), "error l2")
    local = float(np.sqrt(abs(out[0])))
    ref_g = np.ascontiguousarray(interpolate_to_grid(reference.mesh, rv, global_mesh), dtype=np.float64)
    gv = np.ascontiguousarray(state.global_field.values, dtype=np.float64)
    lo = np.zeros(3)
    hi = np.zeros(3)
    lo[:lm.dim], hi[:lm.dim] = lm.box.lo, lm.box.hi          # 2D: the z entries are unused
    N.check(N.lib().tl_mass_norms_split_host(N.C.byref(gd), N.dptr(ref_g), N.dptr(gv), N.dptr(lo), N.dptr(hi),
                                             N.dptr(out)), "masked mass")
    return {"local": local, "overlap": float(np.sqrt(abs(out[0]))), "exterior": float(np.sqrt(abs(out[1])))}


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *exc):
        return False

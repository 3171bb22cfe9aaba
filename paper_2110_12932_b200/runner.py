"""Experiment wiring: where the device backend is selected (``lpbfsim/runner.py:84-113,236-257``).

``build_problem(cfg)`` accepts this package's ``ExperimentConfig`` or the
reference's own (duck-typed: the same field names) and returns the device
``TwoLevelProblem`` plus the initial local grid.  ``two_level_run`` is the
``_two_level_run`` equivalent for the two-level modes; ``run_reference`` is the
monolithic fine-grid reference (``runner.py:126-163``) on the same device solve.
"""

from __future__ import annotations

import numpy as np

from .control import (
    Box, LaserBeam, LocalDomainPolicy, LocalPlacement, Material, ScanPath, Segment, ThermalBC,
    initial_local_box, structured_ncells,
)
from .errors import UnsupportedOnDevice
from .fem import (
    BoundarySpec, GaussianSource, PiecewiseMaterial, RegionMask, Trajectory, solve_monolithic, uniform_field,
)
from .grid import BOTTOM, TOP, StructuredGrid, build_structured_grid
from .multirate import MacroSchedule, run_space, run_spacetime
from .stats import RunStats
from .twolevel import TwoLevelProblem


def _box(b) -> Box:
    return b if isinstance(b, Box) else Box(tuple(b.lo), tuple(b.hi))


def _material(m) -> Material:
    if isinstance(m, Material):
        return m
    return Material(np.array(m.conductivity_table), np.array(m.heat_capacity_table), m.rho, m.chi,
                    m.T_solidus, m.T_liquidus, m.S)


def _path(p) -> ScanPath:
    if isinstance(p, ScanPath):
        return p
    return ScanPath(tuple(Segment(tuple(s.start), tuple(s.end), s.speed, s.t_start) for s in p.segments))


def _policy(p):
    if p is None or isinstance(p, LocalDomainPolicy):
        return p
    return LocalDomainPolicy(tuple(p.box_size), p.laser_fraction, p.snap)


def convert_config(cfg):
    """Normalise a (possibly reference) ExperimentConfig into this package's types."""
    from .config import CouplingSettings, SolverSettings
    beam = cfg.beam if isinstance(cfg.beam, LaserBeam) else LaserBeam(
        cfg.beam.power, cfg.beam.absorptivity, cfg.beam.radius, cfg.beam.depth, cfg.beam.speed)
    bc = cfg.bc if isinstance(cfg.bc, ThermalBC) else ThermalBC(
        cfg.bc.h_conv, cfg.bc.emissivity, cfg.bc.T_ambient, cfg.bc.T_buildplate, cfg.bc.sigma_sb)
    solver = cfg.solver if isinstance(cfg.solver, SolverSettings) else SolverSettings(
        cfg.solver.picard_tol, cfg.solver.picard_max_iter, cfg.solver.linear_tol,
        cfg.solver.linear_solver)
    coupling = cfg.coupling if isinstance(cfg.coupling, CouplingSettings) else CouplingSettings(
        cfg.coupling.omega, cfg.coupling.tolerance, cfg.coupling.max_iterations)
    return dict(global_box=_box(cfg.global_box),
                local_box=None if cfg.local_box is None else _box(cfg.local_box),
                h_global=cfg.h_global, h_local=cfg.h_local, material=_material(cfg.material),
                material_local=_material(cfg.material_local), beam=beam, bc=bc,
                path=_path(cfg.path), policy=_policy(cfg.policy), solver=solver, coupling=coupling,
                coupling_mode=cfg.coupling_mode, source_global=cfg.source_global,
                T_initial=cfg.T_initial, t_end=cfg.t_end, dt_macro=cfg.dt_macro,
                micro_steps=cfg.micro_steps, mode=cfg.mode)


def build_problem(cfg, device: int = 0, resolve_corrector: bool = True):
    """``build_problem`` (``runner.py:84-113``) with the device backend."""
    c = convert_config(cfg)
    gmesh = build_structured_grid(c["global_box"], c["h_global"])
    if c["policy"] is not None:
        lbox = initial_local_box(c["global_box"], c["h_local"], c["policy"], c["path"])
    else:
        lbox = c["local_box"]
    lmesh = StructuredGrid(LocalPlacement(lbox, structured_ncells(lbox, c["h_local"])))
    problem = TwoLevelProblem(
        global_mesh=gmesh, mat_global=c["material"], mat_local=c["material_local"], bc=c["bc"],
        solver=c["solver"], coupling=c["coupling"], mode=c["coupling_mode"], beam=c["beam"],
        path=c["path"], source_global=c["source_global"], resolve_corrector=resolve_corrector,
        device=device)
    return problem, lmesh


def two_level_run(cfg, spacetime: bool | None = None, dt_macro: float | None = None,
                  micro: int | None = None, stats: RunStats | None = None, recorder=None,
                  n_steps: int | None = None, device: int = 0, resolve_corrector: bool = True):
    """``_two_level_run`` (``runner.py:236-257``) on the device; returns (state, stats)."""
    c = convert_config(cfg)
    problem, lmesh = build_problem(cfg, device=device, resolve_corrector=resolve_corrector)
    stats = RunStats() if stats is None else stats
    T0 = uniform_field(problem.global_mesh, c["T_initial"], time=0.0)
    dt_macro = c["dt_macro"] if dt_macro is None else dt_macro
    micro = c["micro_steps"] if micro is None else micro
    if spacetime is None:
        spacetime = c["mode"] != "two-level-space"
    moving = c["policy"] is not None
    t_end = c["t_end"]
    if spacetime:
        if n_steps is not None:
            t_end = n_steps * dt_macro
        sched = MacroSchedule(dt_macro, micro, 0.0, t_end)
        state = run_spacetime(problem, sched, lmesh, T0, path=c["path"] if moving else None,
                              policy=c["policy"], stats=stats, recorder=recorder)
    else:
        dt = dt_macro / micro
        n = int(round(t_end / dt)) if n_steps is None else n_steps
        state = run_space(problem, dt, n, lmesh, T0, path=c["path"] if moving else None,
                          policy=c["policy"], stats=stats, recorder=recorder)
    return state, stats


def two_level_run_slabs(cfg, stats: RunStats | None = None, n_steps: int | None = None,
                        device=None, group=None, resolve_corrector: bool = True):
    """Multirate two-level run with the global grid z-slab-decomposed over the ranks of
    the current process group (one process per GPU) and the local problem pipelined over
    the ranks in time; see ``multirate_dist``.

    Returns (state, stats) on the rank that ran the last macro step's local part and
    (None, stats) on the others."""
    from .multirate_dist import run_spacetime_slabs
    c = convert_config(cfg)
    if c["mode"] == "two-level-space":
        from .errors import UnsupportedOnDevice
        raise UnsupportedOnDevice("slab decomposition implements the multirate (spacetime) mode")
    if device is None:
        import torch
        device = torch.cuda.current_device()
    problem, lmesh = build_problem(cfg, device=int(device), resolve_corrector=resolve_corrector)
    stats = RunStats() if stats is None else stats
    T0 = uniform_field(problem.global_mesh, c["T_initial"], time=0.0)
    t_end = c["t_end"] if n_steps is None else n_steps * c["dt_macro"]
    sched = MacroSchedule(c["dt_macro"], c["micro_steps"], 0.0, t_end)
    moving = c["policy"] is not None
    state = run_spacetime_slabs(problem, sched, lmesh, T0, path=c["path"] if moving else None,
                                policy=c["policy"], stats=stats, group=group, device=f"cuda:{int(device)}")
    return state, stats


def reference_bounds(cfg, mesh) -> BoundarySpec:
    """``reference_bounds`` (``runner.py:116-123``): bottom Dirichlet T_buildplate, Robin top."""
    bc = convert_config(cfg)["bc"]
    return BoundarySpec(bc=bc, robin_tags=(TOP,), radiation=bc.emissivity > 0,
                        dirichlet_nodes=mesh.nodes_on(BOTTOM), dirichlet_values=bc.T_buildplate)


def run_reference(cfg, dt: float | None = None, stats: RunStats | None = None, mesh=None,
                  observer=None) -> Trajectory:
    """Monolithic reference (``runner.py:126-163``): the true Gaussian beam on one fine grid
    (``h_reference``) over the whole plate, uniform steps ``dt_reference``, every step a
    device solve.  Distinct coarse/fine materials become a PiecewiseMaterial over the fixed
    local box and ``latent_reference local`` a latent RegionMask, as the reference does."""
    c = convert_config(cfg)
    dt = cfg.dt_reference if dt is None else dt
    mesh = build_structured_grid(c["global_box"], cfg.h_reference) if mesh is None else mesh
    n_steps = int(round(c["t_end"] / dt))
    mat, mat_l = c["material"], c["material_local"]
    region = c["local_box"]
    material = mat
    if mat_l is not None and mat_l is not mat and not _materials_equal(mat, mat_l):
        if region is None:
            raise ValueError("a reference with distinct coarse/fine materials needs a fixed local box")
        material = PiecewiseMaterial(mat_l, mat, region)
    chi_max = max(mat.chi, mat_l.chi if mat_l is not None else 0.0)
    latent = cfg.latent_reference != "off" and chi_max > 0
    latent_mask = None
    if latent and cfg.latent_reference == "local":
        if region is None:
            raise ValueError("latent_reference=local needs a fixed local box")
        latent_mask = RegionMask(region)
    path, beam = c["path"], c["beam"]
    tol = 1e-12 * max(path.t_end, 1.0)

    def source_at(t):                              # ``_local_source_factory`` (runner.py:49-61)
        if t > path.t_end + tol or t < path.t_start - tol:
            return None
        return GaussianSource(beam, tuple(path.position(t)))

    bounds = reference_bounds(cfg, mesh)
    T0 = uniform_field(mesh, c["T_initial"], time=0.0)
    return solve_monolithic(mesh, material, source_at, lambda t: bounds, dt, n_steps, T0,
                            settings=c["solver"], latent=latent, latent_mask=latent_mask, stats=stats,
                            observer=observer)


def _materials_equal(a, b) -> bool:
    return (np.array_equal(np.asarray(a.conductivity_table), np.asarray(b.conductivity_table))
            and np.array_equal(np.asarray(a.heat_capacity_table), np.asarray(b.heat_capacity_table))
            and a.rho == b.rho and a.chi == b.chi)

"""The reference's own property tests for the hot path, restated against the device API.

The reference pins its path with invariants (``pkg/tests/test_multirate.py``,
``test_twolevel.py``, ``test_fem.py``): solve counters of a macro step, exact time
bookkeeping, m = 1 degenerating to uniform stepping, preserved equilibria, linearity of the
interface functional, the coupled pair reproducing the monolithic solve on identical
discretisations, ...  Those tests run on toy 2D boxes through source closures; these hold
the same statements on small 3D plates (and one 2D plate) through this package's seams --
the device-resident run where the problem allows it, the step-level drivers otherwise.
Each test names the reference test it restates.
"""

from pathlib import Path

import numpy as np
import pytest

import paper_2110_12932_b200 as P
from paper_2110_12932_b200.multirate import predictor_global
from paper_2110_12932_b200.twolevel import (consistency_diagnostic, transmission_load, two_level_iterate)

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
CONFIGS = ROOT / "configs"
T0 = 300.0
BC0 = P.ThermalBC(0.0, 0.0, T0, T0)
CG = P.SolverSettings(picard_tol=1e-9, picard_max_iter=40, linear_tol=1e-12, linear_solver="cg")


def material(k_lo=10.0, k_hi=10.0, c_lo=400.0, c_hi=400.0, chi=0.0, Ts=1563.15, Tl=1653.15):
    return P.Material(np.array([[200.0, k_lo], [5000.0, k_hi]]), np.array([[200.0, c_lo], [5000.0, c_hi]]),
                      8000.0, chi, Ts, Tl, 0.05)


def plates(h_local=5e-5):
    """2 x 1 x 0.5 mm plate at h = 0.1 mm; a 0.8 x 0.6 x 0.3 mm local box flush with the top."""
    gm = P.build_structured_grid(P.Box((0.0, 0.0, 0.0), (2e-3, 1e-3, 5e-4)), 1e-4)
    lm = P.build_structured_grid(P.Box((6e-4, 2e-4, 2e-4), (1.4e-3, 8e-4, 5e-4)), h_local)
    return gm, lm


def problem_of(mat_g, mat_l, bc=BC0, beam=None, omega=1.0, mode="alternate", source_global="gaussian",
               moving=False, tol=1e-6):
    gm, lm = plates()
    path = None
    if beam is not None:
        a, b = (8e-4, 5e-4, 5e-4), ((1.2e-3, 5e-4, 5e-4) if moving else (8e-4 + 1e-9, 5e-4, 5e-4))
        path = P.path_from_segments([(a, b, beam.speed)])
    prob = P.TwoLevelProblem(global_mesh=gm, mat_global=mat_g, mat_local=mat_l, bc=bc, solver=CG,
                             coupling=P.CouplingSettings(omega=omega, tolerance=tol, max_iterations=60),
                             mode=mode, beam=beam, path=path, source_global=source_global)
    return prob, lm


def moving_beam():
    return P.LaserBeam(150.0, 0.4, 1e-4, 1e-4, 0.8)            # 0.4 mm of track in 0.5 ms


def parked_beam(power=150.0):
    return P.LaserBeam(power, 0.4, 1e-4, 1e-4, 1e-9 / 1e-3)    # 1 nm in 1 ms: a stationary spot


# ---- test_multirate.py ------------------------------------------------------------------

def test_predictor_preserves_constant_state():
    """test_multirate.py::test_predictor_preserves_constant_state"""
    mat = material()
    prob, lm = problem_of(mat, mat)
    state = P.initial_state(prob, lm, P.uniform_field(prob.global_mesh, T0))
    pred = predictor_global(prob, state, 1e-4)
    assert np.allclose(pred.values, T0, atol=1e-10)


@pytest.mark.parametrize("source_global,resident", [("gaussian", False), ("distributed", True)])
def test_macro_step_solve_counters(source_global, resident):
    """test_macro_step_counts_local_solves (instant-based coarse source: the corrector
    re-solves the coarse step) and test_interval_source_reuses_predictor (interval-based
    source + one-way coupling: it does not)."""
    mat = material()
    prob, lm = problem_of(mat, mat, beam=moving_beam(), source_global=source_global, moving=True)
    assert prob.one_way and prob.device_resident == resident
    sched = P.MacroSchedule(1e-4, 5 if not resident else 4, 0.0, 3e-4)
    stats = P.RunStats()
    P.run_spacetime(prob, sched, lm, P.uniform_field(prob.global_mesh, T0), stats=stats)
    n, m = sched.n_macro, sched.micro_per_macro
    c = stats.counters
    assert c["coupling_iterations"] == n                       # one corrector pass per macro step
    assert c["local_solves"] == n * m + n
    assert c["predictor_solves"] == n
    assert c["global_solves"] == (n if resident else 2 * n)    # predictor reused / predictor + corrector


@pytest.mark.parametrize("source_global", ["gaussian", "distributed"])
def test_time_bookkeeping_exact(source_global):
    """test_multirate.py::test_time_bookkeeping_exact: recorder times are the schedule's own
    floating-point expressions on both drivers."""
    mat = material()
    prob, lm = problem_of(mat, mat, beam=moving_beam(), source_global=source_global, moving=True)
    sched = P.MacroSchedule(1e-4, 3, 0.0, 5e-4)
    times = []
    P.run_spacetime(prob, sched, lm, P.uniform_field(prob.global_mesh, T0),
                    recorder=lambda kind, t, *a: times.append((kind, t)))
    assert [t for k, t in times if k == "macro"] == [sched.t_macro(k + 1) for k in range(5)]
    assert [t for k, t in times if k == "micro"] == [sched.t_micro(k, i) for k in range(5) for i in range(1, 4)]
    assert sched.t_macro(3) == 0.0 + 3 * 1e-4 and sched.t_micro(2, 1) == 0.0 + 2 * 1e-4 + 1 * (1e-4 / 3)


def test_m_equal_one_degenerates_to_space_stepping_oneway():
    """test_multirate.py::test_m_equal_one_degenerates_to_space_stepping_oneway: with one
    micro step per macro step the two drivers perform identical solves."""
    mat = material()
    prob, lm = problem_of(mat, mat, beam=moving_beam(), moving=True)
    U = P.uniform_field(prob.global_mesh, T0)
    st = P.run_spacetime(prob, P.MacroSchedule(5e-5, 1, 0.0, 2.5e-4), lm, U)
    ss = P.run_space(prob, 5e-5, 5, lm, U)
    assert st.local_field.values.max() > T0 + 50.0
    np.testing.assert_allclose(st.local_field.values, ss.local_field.values, rtol=1e-12, atol=0)
    np.testing.assert_allclose(st.global_field.values, ss.global_field.values, rtol=1e-12, atol=0)


def test_m_equal_one_degenerates_two_way():
    """test_multirate.py::test_m_equal_one_degenerates_two_way"""
    prob, lm = problem_of(material(4.0, 4.0), material(10.0, 10.0), beam=moving_beam(), moving=True)
    assert not prob.one_way
    U = P.uniform_field(prob.global_mesh, T0)
    st = P.run_spacetime(prob, P.MacroSchedule(5e-5, 1, 0.0, 2.5e-4), lm, U)
    ss = P.run_space(prob, 5e-5, 5, lm, U)
    diff = np.linalg.norm(st.local_field.values - ss.local_field.values) / np.linalg.norm(ss.local_field.values)
    assert diff < 10 * prob.coupling.tolerance


def test_predictor_error_decreases_with_macro_step():
    """test_multirate.py::test_predictor_error_decreases_with_macro_step (two-way coupling,
    so the corrector changes the coarse field)."""
    errs = []
    for dt, micro in ((2e-4, 4), (1e-4, 2), (5e-5, 1)):
        prob, lm = problem_of(material(4.0, 4.0), material(10.0, 10.0), beam=moving_beam(), moving=True)
        preds, corr = {}, {}

        def rec(kind, t, local, glob, iters):
            if kind == "predictor":
                preds[round(t, 12)] = glob.values
            elif kind == "macro":
                corr[round(t, 12)] = glob.values

        P.run_spacetime(prob, P.MacroSchedule(dt, micro, 0.0, 2e-4), lm, P.uniform_field(prob.global_mesh, T0),
                        recorder=rec)
        errs.append(np.linalg.norm(preds[2e-4] - corr[2e-4]) / np.linalg.norm(corr[2e-4]))
    assert errs[0] > errs[1] > errs[2] > 0.0


@pytest.mark.parametrize("source_global", ["gaussian", "distributed"])
def test_corrector_resolves_final_micro_interval(source_global):
    """test_multirate.py::test_corrector_resolves_final_micro_interval: the macro record is
    the run's final local field, and it differs from the provisional last micro field (which
    ran on the lagged trace blend) only through the corrector's re-solve."""
    mat = material()
    prob, lm = problem_of(mat, mat, beam=moving_beam(), source_global=source_global, moving=True)
    rec = {}
    state = P.run_spacetime(prob, P.MacroSchedule(1e-4, 4, 0.0, 1e-4), lm, P.uniform_field(prob.global_mesh, T0),
                            recorder=lambda kind, t, local, glob, it: rec.setdefault(kind, []).append((t, local, glob)))
    t, local, glob = rec["macro"][-1]
    np.testing.assert_array_equal(local.values, state.local_field.values)
    t_mic, last_micro, _ = rec["micro"][-1]
    assert t_mic == t == 1e-4
    assert last_micro.values.shape == local.values.shape
    assert np.abs(last_micro.values - local.values).max() < 0.05 * (local.values.max() - T0)


# ---- test_twolevel.py -------------------------------------------------------------------

def test_transmission_functional_properties():
    """test_transmission_zero_for_equal_conductivity, ..._zero_for_constant_local_field,
    ..._linear_in_local_field (the hand-computed case is
    test_gpu_parity.py::test_transmission_of_linear_field_is_bottom_flux)."""
    gm, lm = plates()
    gamma = P.extract_interface(lm, gm)
    X = lm.coords
    u = P.FieldState(lm, T0 + 4e7 * X[:, 0] * X[:, 1] + 3e4 * X[:, 2], 0.0)
    v = P.FieldState(lm, T0 + 200.0 * np.sin(3e3 * X[:, 0]) + 5e4 * X[:, 2], 0.0)
    same = transmission_load(u, gamma, gm, material(), material())
    assert np.all(np.asarray(same) == 0.0)
    const = transmission_load(P.uniform_field(lm, 500.0), gamma, gm, material(10.0, 10.0), material(5.0, 5.0))
    assert np.allclose(const, 0.0, atol=1e-18)
    mg, ml = material(10.0, 10.0), material(4.0, 4.0)
    fu, fv = transmission_load(u, gamma, gm, mg, ml), transmission_load(v, gamma, gm, mg, ml)
    w = P.FieldState(lm, 2.0 * u.values - 0.5 * v.values, 0.0)
    fw = transmission_load(w, gamma, gm, mg, ml)
    assert np.abs(fu).max() > 0.0
    assert np.abs(fw - (2.0 * fu - 0.5 * fv)).max() <= 1e-11 * np.abs(fw).max()


def test_local_constant_trace_no_source():
    """test_twolevel.py::test_local_constant_trace_no_source"""
    mat = material()
    prob, lm = problem_of(mat, mat)
    state = P.initial_state(prob, lm, P.uniform_field(prob.global_mesh, T0))
    out = P.solve_local(prob, state.local_field, 1e-4, state.gamma, np.full(state.gamma.trace_nodes.size, T0))
    assert np.allclose(out.values, T0, atol=1e-10)


def test_local_reproduces_linear_global_trace():
    """test_twolevel.py::test_local_reproduces_linear_global_trace: a field linear in x and y
    is P1-exact, harmonic and flux-free through the top face, so the local step keeps it."""
    mat = material(15.0, 15.0)
    prob, lm = problem_of(mat, mat)
    gm = prob.global_mesh
    lin = P.FieldState(gm, T0 + 1.2e4 * gm.coords[:, 0] + 5e3 * gm.coords[:, 1], 0.0)
    state = P.initial_state(prob, lm, lin)
    trace = state.gamma.trace_of(lin, gm)
    out = P.solve_local(prob, state.local_field, 1e-4, state.gamma, trace)
    expect = T0 + 1.2e4 * lm.coords[:, 0] + 5e3 * lm.coords[:, 1]
    assert np.allclose(out.values, expect, atol=1e-8)
    np.testing.assert_array_equal(out.values[state.gamma.trace_nodes], trace)


def test_decoupled_case_converges_immediately():
    """test_twolevel.py::test_decoupled_case_converges_immediately"""
    mat = material()
    prob, lm = problem_of(mat, mat)
    assert prob.one_way
    state = P.initial_state(prob, lm, P.uniform_field(prob.global_mesh, T0))
    new, iters = two_level_iterate(prob, state, 1e-4)
    assert iters <= 2
    assert np.allclose(new.global_field.values, T0, atol=1e-10)
    assert np.allclose(new.local_field.values, T0, atol=1e-10)


def test_equilibrium_preserved_with_zero_source():
    """test_twolevel.py::test_equilibrium_preserved_with_zero_source: convection and
    radiation against the ambient temperature leave a field at that temperature alone."""
    mat = material(10.0, 25.0, 400.0, 700.0)
    prob, lm = problem_of(mat, mat, bc=P.ThermalBC(20.0, 0.4, T0, T0))
    state = P.initial_state(prob, lm, P.uniform_field(prob.global_mesh, T0))
    state, _ = two_level_iterate(prob, state, 5e-4)
    assert np.allclose(state.global_field.values, T0, atol=1e-9)
    assert np.allclose(state.local_field.values, T0, atol=1e-9)


def test_two_way_coupling_converges_and_is_omega_independent():
    """test_twolevel.py::test_two_way_coupling_converges_and_is_omega_independent"""
    mg, ml = material(4.0, 4.0), material(10.0, 10.0)
    bc = P.ThermalBC(10.0, 0.0, T0, T0)
    p1, lm = problem_of(mg, ml, bc=bc, beam=parked_beam(), omega=1.0)
    p2, _ = problem_of(mg, ml, bc=bc, beam=parked_beam(), omega=0.5)
    assert not p1.one_way
    s1 = P.initial_state(p1, lm, P.uniform_field(p1.global_mesh, T0))
    s2 = P.initial_state(p2, lm, P.uniform_field(p2.global_mesh, T0))
    o1, it1 = two_level_iterate(p1, s1, 1e-4)
    o2, it2 = two_level_iterate(p2, s2, 1e-4)
    assert it1 >= 2 and it2 >= it1
    assert o1.local_field.values.max() > T0 + 50.0
    diff = np.linalg.norm(o1.local_field.values - o2.local_field.values) / np.linalg.norm(o1.local_field.values)
    assert diff < 10 * p1.coupling.tolerance


def test_iterate_idempotent_at_fixed_point():
    """test_twolevel.py::test_iterate_idempotent_at_fixed_point"""
    prob, lm = problem_of(material(4.0, 4.0), material(10.0, 10.0), bc=P.ThermalBC(10.0, 0.0, T0, T0),
                          beam=parked_beam())
    state = P.initial_state(prob, lm, P.uniform_field(prob.global_mesh, T0))
    state, _ = two_level_iterate(prob, state, 1e-4)
    again, _ = two_level_iterate(prob, state, 1e-14)
    scale = max(np.linalg.norm(state.trace), 1e-12)
    assert np.linalg.norm(again.trace - state.trace) / scale < prob.coupling.tolerance


def test_coupled_matches_monolithic_identical_discretization():
    """test_twolevel.py::test_coupled_matches_monolithic_identical_discretization: equal
    materials, matching lattices and steps -- the coupled pair reproduces the single-grid
    solve up to solver tolerances."""
    mat = material(10.0, 25.0, 400.0, 700.0)
    bc = P.ThermalBC(10.0, 0.0, T0, T0)
    gm, _ = plates()
    lm = P.build_structured_grid(P.Box((6e-4, 2e-4, 2e-4), (1.4e-3, 8e-4, 5e-4)), 1e-4)
    beam = parked_beam()
    path = P.path_from_segments([((8e-4, 5e-4, 5e-4), (8e-4 + 1e-9, 5e-4, 5e-4), beam.speed)])
    prob = P.TwoLevelProblem(global_mesh=gm, mat_global=mat, mat_local=mat, bc=bc, solver=CG, beam=beam, path=path,
                             source_global="gaussian")
    U = P.uniform_field(gm, T0)
    state = P.initial_state(prob, lm, U)
    dt, n = 5e-5, 4
    for _ in range(n):
        state, _ = two_level_iterate(prob, state, dt)
    ref = P.solve_monolithic(gm, mat, prob.local_source, lambda t: prob.global_bounds(), dt, n, U, settings=CG,
                             latent=False)
    ref_local = gm.interpolate(ref.values[-1], lm.coords)
    assert ref.values[-1].max() > T0 + 50.0
    rel_l = np.linalg.norm(state.local_field.values - ref_local) / np.linalg.norm(ref_local)
    rel_g = np.linalg.norm(state.global_field.values - ref.values[-1]) / np.linalg.norm(ref.values[-1])
    assert rel_l < 1e-6 and rel_g < 1e-8


def test_full_and_alternate_modes_differ_only_on_overlap():
    """test_twolevel.py::test_full_and_alternate_modes_differ_only_on_overlap: with latent heat
    active in the fine problem the full form feeds it back into the coarse one, inside the
    local box."""
    mat = material(10.0, 16.0, 400.0, 400.0, chi=2.0e5, Ts=600.0, Tl=900.0)
    bc = P.ThermalBC(10.0, 0.0, T0, T0)
    p_alt, lm = problem_of(mat, mat, bc=bc, beam=parked_beam(250.0), mode="alternate")
    p_full, _ = problem_of(mat, mat, bc=bc, beam=parked_beam(250.0), mode="full")
    assert p_alt.one_way and not p_full.one_way
    s_alt = P.initial_state(p_alt, lm, P.uniform_field(p_alt.global_mesh, T0))
    s_full = P.initial_state(p_full, lm, P.uniform_field(p_full.global_mesh, T0))
    for _ in range(5):
        s_alt, _ = two_level_iterate(p_alt, s_alt, 1e-4)
        s_full, _ = two_level_iterate(p_full, s_full, 1e-4)
    assert s_alt.local_field.values.max() > mat.T_solidus          # melting must occur
    diff = np.abs(s_full.global_field.values - s_alt.global_field.values)
    assert diff.max() > 1e-6
    gm = p_alt.global_mesh
    inside = lm.box.contains(gm.coords, tol=1e-12)
    assert diff[inside].max() > 10 * diff[~inside].max()


def test_consistency_diagnostic_zero_for_identical_fields():
    """test_twolevel.py::test_consistency_diagnostic_zero_for_identical_fields"""
    mat = material()
    prob, lm = problem_of(mat, mat)
    gm = prob.global_mesh
    state = P.initial_state(prob, lm, P.uniform_field(gm, 321.0))
    out = consistency_diagnostic(state, P.uniform_field(gm, 321.0), gm)
    for key in ("local", "overlap", "exterior"):
        assert out[key] == pytest.approx(0.0, abs=1e-12) and out[key] >= 0


def test_time_stamp_mismatch_rejected():
    """test_twolevel.py::test_time_stamp_mismatch_rejected"""
    mat = material()
    prob, lm = problem_of(mat, mat)
    state = P.initial_state(prob, lm, P.uniform_field(prob.global_mesh, T0))
    with pytest.raises(P.CouplingError):
        two_level_iterate(prob, state, 1e-4, local_from=state.local_field, local_dt=5e-5)


# ---- test_fem.py ------------------------------------------------------------------------

def _bottom(grid, bc=BC0, value=T0, radiation=False, tags=(P.TOP,)):
    return P.BoundarySpec(bc=bc, robin_tags=tags, radiation=radiation, dirichlet_nodes=grid.nodes_on(P.BOTTOM),
                          dirichlet_values=value)


@pytest.mark.parametrize("tdep", [False, True])
def test_constant_state_preserved_adiabatic(tdep):
    """test_fem.py::test_constant_state_preserved_adiabatic (fused linear solve and Picard path)"""
    gm, _ = plates()
    mat = material(10.0, 25.0, 400.0, 700.0) if tdep else material()
    out = P.step_backward_euler(P.uniform_field(gm, 450.0), 1e-4, mat, None, _bottom(gm, value=450.0), CG)
    assert np.allclose(out.values, 450.0, atol=1e-10)


def test_fixed_dirichlet_everywhere_returns_boundary_value():
    """test_fem.py::test_fixed_dirichlet_everywhere_returns_boundary_value"""
    gm, _ = plates()
    rng = np.random.default_rng(2)
    g = rng.uniform(300.0, 900.0, gm.n_nodes)
    bounds = P.BoundarySpec(bc=BC0, robin_tags=(), radiation=False, dirichlet_nodes=np.arange(gm.n_nodes),
                            dirichlet_values=g)
    out = P.step_backward_euler(P.uniform_field(gm, 500.0), 1e-4, material(10.0, 25.0), None, bounds, CG)
    np.testing.assert_array_equal(out.values, g)


def test_linear_problem_converges_in_one_picard_iteration():
    """test_fem.py::test_linear_problem_converges_in_one_picard_iteration"""
    gm, _ = plates()
    rng = np.random.default_rng(3)
    stats = P.RunStats()
    st = P.FieldState(gm, rng.uniform(300.0, 900.0, gm.n_nodes), 0.0)
    P.step_backward_euler(st, 1e-4, material(), None, _bottom(gm), CG, stats=stats)
    assert stats.counters["picard_iterations"] == 1
    stats2 = P.RunStats()
    P.step_backward_euler(st, 1e-4, material(10.0, 25.0, 400.0, 700.0), None, _bottom(gm), CG, stats=stats2)
    assert stats2.counters["picard_iterations"] > 1


@pytest.mark.parametrize("tdep", [False, True])
def test_discrete_maximum_principle_dirichlet_band(tdep):
    """test_fem.py::test_discrete_maximum_principle_dirichlet_band: without sources the new
    field stays within the range of the old field and the boundary data (M-matrix: lumped
    mass, non-obtuse Kuhn tets)."""
    gm, _ = plates()
    rng = np.random.default_rng(4)
    st = P.FieldState(gm, rng.uniform(350.0, 800.0, gm.n_nodes), 0.0)
    mat = material(10.0, 25.0, 400.0, 700.0) if tdep else material()
    out = P.step_backward_euler(st, 2e-4, mat, None, _bottom(gm, value=320.0), CG)
    assert out.values.min() >= 320.0 - 1e-9 and out.values.max() <= 800.0 + 1e-9


def test_energy_balance_with_source():
    """test_fem.py::test_energy_balance_with_source: adiabatic walls and no Dirichlet set --
    the lumped heat content rises by the discrete load times dt (and the discrete load is the
    absorbed power up to quadrature error)."""
    from oracle import kuhn
    gm, _ = plates()
    beam = P.LaserBeam(150.0, 0.4, 1e-4, 1e-4, 0.8)
    src = P.GaussianSource(beam, (1e-3, 5e-4, 3e-4))
    dt = 1e-4
    out = P.step_backward_euler(P.uniform_field(gm, T0), dt, material(), src,
                                P.BoundarySpec(bc=BC0, robin_tags=(), radiation=False), CG)
    G = kuhn.KuhnGrid(gm.box.lo, gm.box.hi, gm.ncells)
    lumped = float(np.prod(G.h)) * G.node_incidence().ravel() / 24.0
    gained = 8000.0 * 400.0 * float(np.dot(lumped, out.values - T0))
    load = float(np.sum(kuhn.gaussian_load(G, beam, src.center)))
    assert gained == pytest.approx(load * dt, rel=1e-9)
    assert out.values.max() > T0 + 10.0


def test_monolithic_constant_trajectory():
    """test_fem.py::test_monolithic_constant_trajectory"""
    gm, _ = plates()
    traj = P.solve_monolithic(gm, material(), lambda t: None, lambda t: _bottom(gm), 1e-4, 3,
                              P.uniform_field(gm, T0), settings=CG, latent=False)
    assert len(traj) == 4 and traj.times == [0.0] + [0.0 + k * 1e-4 for k in range(1, 4)]
    for v in traj.values:
        assert np.allclose(v, T0, atol=1e-10)


def test_radiation_fixed_point_matches_nonlinear_flux():
    """test_fem.py::test_radiation_fixed_point_matches_nonlinear_flux: with the T^4 term
    lagged in the Picard loop, the converged steady state balances the conductive flux through
    the slab against convection + the exact radiation law at the top face."""
    m = P.build_structured_grid(P.Box((0.0, 0.0, 0.0), (1.0, 1.0, 1.0)), 0.25)
    mat = P.Material(np.array([[200.0, 100.0], [5000.0, 100.0]]), np.array([[200.0, 1.0], [5000.0, 1.0]]),
                     1.0, 0.0, 1563.15, 1653.15, 0.05)
    bc = P.ThermalBC(5.0, 0.7, 300.0, 300.0)
    bounds = P.BoundarySpec(bc=bc, robin_tags=(P.TOP,), radiation=True, dirichlet_nodes=m.nodes_on(P.BOTTOM),
                            dirichlet_values=1000.0)
    settings = P.SolverSettings(picard_tol=1e-10, picard_max_iter=100, linear_tol=1e-12, linear_solver="cg")
    state = P.uniform_field(m, 1000.0)
    for _ in range(10):
        state = P.step_backward_euler(state, 1e3, mat, None, bounds, settings)
    Ttop = state.values[m.nodes_on(P.TOP)].mean()
    q_out = bc.h_conv * (Ttop - 300.0) + bc.sigma_sb * 0.7 * (Ttop**4 - 300.0**4)
    q_cond = 100.0 * (1000.0 - Ttop) / 1.0
    assert 300.0 < Ttop < 1000.0
    assert q_out == pytest.approx(q_cond, rel=1e-3)


def _lumped_volume(grid):
    from oracle import kuhn
    G = kuhn.KuhnGrid(grid.box.lo, grid.box.hi, grid.ncells)
    return float(np.prod(G.h)) * G.node_incidence().ravel() / 24.0


def _mms_material():
    return P.Material(np.array([[0.0, 2.0], [1e4, 2.0]]), np.array([[0.0, 3.0], [1e4, 3.0]]), 5.0, 0.0,
                      1563.15, 1653.15, 0.05)


def _spatial_mms_error(h):
    """Exact solution (1 + t) sin(pi x) sin(pi y) sin(pi z): linear in t, so backward Euler
    adds no temporal error.  The source enters as a nodal load (lumped volume times the
    source at the node), the device's seam for arbitrary sources."""
    k, c, rho = 2.0, 3.0, 5.0
    m = P.build_structured_grid(P.Box((0.0, 0.0, 0.0), (1.0, 1.0, 1.0)), h)
    X = m.coords
    S = np.sin(np.pi * X[:, 0]) * np.sin(np.pi * X[:, 1]) * np.sin(np.pi * X[:, 2])
    vol = _lumped_volume(m)
    nodes = m.nodes_on(P.BOTTOM, P.TOP, P.LATERAL)
    bounds = P.BoundarySpec(bc=P.ThermalBC(0.0, 0.0, 0.0, 0.0), robin_tags=(), dirichlet_nodes=nodes,
                            dirichlet_values=0.0)
    state = P.FieldState(m, S, 0.0)
    dt, n = 0.05, 4
    for kstep in range(1, n + 1):
        t = kstep * dt
        load = vol * (rho * c * S + 3.0 * np.pi**2 * k * (1.0 + t) * S)
        state = P.step_backward_euler(state, dt, _mms_material(), None, bounds, CG, extra_load=load)
    exact = (1.0 + n * dt) * S
    return P.l2_norm(m, state.values - exact) / P.l2_norm(m, exact)


def test_spatial_order_two():
    """test_fem.py::test_spatial_order_two"""
    hs = np.array([1 / 4, 1 / 8, 1 / 16])
    errs = np.array([_spatial_mms_error(h) for h in hs])
    slope = np.polyfit(np.log(hs), np.log(errs), 1)[0]
    assert abs(slope - 2.0) < 0.15, (errs, slope)


def _temporal_mms_error(dt):
    """Exact solution x exp(t): spatially linear, so P1 carries no space error."""
    c, rho = 3.0, 5.0
    m = P.build_structured_grid(P.Box((0.0, 0.0, 0.0), (1.0, 1.0, 1.0)), 0.25)
    x = m.coords[:, 0]
    vol = _lumped_volume(m)
    nodes = m.nodes_on(P.BOTTOM, P.TOP, P.LATERAL)
    state = P.FieldState(m, x * 1.0, 0.0)
    n = int(round(1.0 / dt))
    for kstep in range(1, n + 1):
        t = kstep * dt
        bounds = P.BoundarySpec(bc=P.ThermalBC(0.0, 0.0, 0.0, 0.0), robin_tags=(), dirichlet_nodes=nodes,
                                dirichlet_values=x[nodes] * np.exp(t))
        state = P.step_backward_euler(state, dt, _mms_material(), None, bounds, CG,
                                      extra_load=vol * rho * c * x * np.exp(t))
    exact = x * np.exp(1.0)
    return P.l2_norm(m, state.values - exact) / P.l2_norm(m, exact)


def test_temporal_order_one():
    """test_fem.py::test_temporal_order_one"""
    dts = np.array([0.2, 0.1, 0.05])
    errs = np.array([_temporal_mms_error(dt) for dt in dts])
    slope = np.polyfit(np.log(dts), np.log(errs), 1)[0]
    assert abs(slope - 1.0) < 0.15, (errs, slope)


# ---- test_scanpath.py: relocation (scanpath.py:208-248) -----------------------------------

def _relocation_case(origin=(0.1, 0.35, 0.5)):
    gm = P.build_structured_grid(P.Box((0.0, 0.0, 0.0), (2.4, 1.2, 0.6)), 0.2)
    mat = material()
    prob = P.TwoLevelProblem(global_mesh=gm, mat_global=mat, mat_local=mat, bc=BC0, solver=CG)
    lsize = (1.2, 0.5, 0.1)
    lm = P.build_structured_grid(P.Box(origin, tuple(np.asarray(origin) + np.asarray(lsize))), 0.05)
    gfield = P.FieldState(gm, 300.0 + 10.0 * gm.coords[:, 0], 0.0)
    return prob, P.initial_state(prob, lm, gfield), P.LocalDomainPolicy(box_size=lsize)


def test_relocate_noop_translate_snap_clamp():
    """test_relocate_noop_when_snapped_target_matches, ..._translates_and_reinterpolates,
    ..._snap_keeps_lattice, ..._clamps_at_global_wall: the box follows the laser in whole
    local cells, the global field is untouched, the new local field and trace are the
    (device) interpolant of the global field."""
    from paper_2110_12932_b200.twolevel import relocate_local
    prob, state, policy = _relocation_case()
    ex = np.array([1.0, 0.0, 0.0])
    x0 = 0.1 + (2 / 3) * 1.2
    assert relocate_local(state, policy, np.array([x0, 0.6, 0.6]), ex, prob) is state
    out = relocate_local(state, policy, np.array([x0 + 0.2, 0.6, 0.6]), ex, prob)
    assert out is not state and out.global_field is state.global_field
    shift = np.asarray(out.local_field.mesh.box.lo) - np.asarray(state.local_field.mesh.box.lo)
    assert shift[0] == pytest.approx(0.2) and shift[1] == 0.0 and shift[2] == 0.0
    expect = 300.0 + 10.0 * out.local_field.mesh.coords[:, 0]
    assert np.allclose(out.local_field.values, expect, atol=1e-10)
    np.testing.assert_array_equal(out.trace, out.local_field.values[out.gamma.trace_nodes])
    snapped = relocate_local(state, policy, np.array([x0 + 0.137, 0.6, 0.6]), ex, prob)
    s = snapped.local_field.mesh.box.lo[0] - state.local_field.mesh.box.lo[0]
    assert s / 0.05 == pytest.approx(round(s / 0.05))
    wall = relocate_local(state, policy, np.array([2.35, 0.6, 0.6]), ex, prob)
    hi, ghi = np.asarray(wall.local_field.mesh.box.hi), np.asarray(prob.global_mesh.box.hi)
    assert hi[0] < ghi[0] and hi[2] == pytest.approx(ghi[2])


def test_relocate_constant_field_stays_constant():
    """test_scanpath.py::test_relocate_constant_field_stays_constant"""
    from paper_2110_12932_b200.twolevel import relocate_local
    prob, state, policy = _relocation_case()
    const = P.initial_state(prob, state.local_field.mesh, P.uniform_field(prob.global_mesh, 777.0))
    out = relocate_local(const, policy, np.array([1.6, 0.6, 0.6]), np.array([1.0, 0.0, 0.0]), prob)
    assert out is not const and np.allclose(out.local_field.values, 777.0)


def test_direction_flip_places_box_behind_laser():
    """test_scanpath.py::test_direction_flip_places_box_behind_laser"""
    policy = P.LocalDomainPolicy(box_size=(1.2, 0.5, 0.1))
    laser = np.array([1.0, 0.6, 0.6])
    assert policy.target_origin(laser, np.array([1.0, 0.0, 0.0]))[0] == pytest.approx(1.0 - 0.8)
    assert policy.target_origin(laser, np.array([-1.0, 0.0, 0.0]))[0] == pytest.approx(1.0 - 0.4)


# ---- test_mesh.py: interpolation and the interface (mesh.py:308-361, 477-523) -------------

@pytest.mark.parametrize("dim", [2, 3])
def test_interpolation_reproduces_affine_fields(dim):
    """test_mesh.py::test_interpolation_reproduces_affine_fields (seeded points instead of
    hypothesis draws), on the device, 2D triangles and 3D Kuhn tets."""
    rng = np.random.default_rng(7)
    m = P.build_structured_grid(P.Box((0.0,) * dim, (1.0,) * dim), 0.25)
    for _ in range(5):
        c0, c = rng.uniform(-1.0, 1.0), rng.uniform(-2.0, 2.0, dim)
        vals = c0 + m.coords @ c
        pts = rng.uniform(0.05, 0.95, (25, dim))
        assert np.abs(m.interpolate(vals, pts) - (c0 + pts @ c)).max() <= 1e-12


def test_interpolation_midedge_of_quadratic():
    """test_mesh.py::test_interpolation_midedge_of_quadratic: the interpolant of x^2 at an
    edge midpoint is the endpoint average."""
    m = P.build_structured_grid(P.Box((0.0, 0.0), (1.0, 1.0)), 0.25)
    got = m.interpolate(m.coords[:, 0] ** 2, np.array([[0.375, 0.5]]))[0]
    assert got == pytest.approx(0.5 * (0.25**2 + 0.5**2))
    m3 = P.build_structured_grid(P.Box((0.0, 0.0, 0.0), (1.0, 1.0, 1.0)), 0.25)
    got3 = m3.interpolate(m3.coords[:, 0] ** 2, np.array([[0.375, 0.5, 0.25]]))[0]
    assert got3 == pytest.approx(0.5 * (0.25**2 + 0.5**2))


def test_interface_measure_and_immersion():
    """test_interface_measure_2d, test_interface_measure_3d, test_interface_requires_immersion"""
    lm = P.build_structured_grid(P.Box((1.0, 0.625), (2.0, 1.0)), 0.125)
    gm = P.build_structured_grid(P.Box((0.0, 0.0), (5.0, 1.0)), 0.125)
    assert P.extract_interface(lm, gm).measure == pytest.approx(2 * 0.375 + 1.0, rel=1e-10)
    lm3 = P.build_structured_grid(P.Box((0.0, 0.0, 0.0), (1.2, 0.5, 0.1)), 0.05)
    gm3 = P.build_structured_grid(P.Box((-1.0, -1.0, -0.9), (3.0, 2.0, 0.1)), 0.2)
    assert P.extract_interface(lm3, gm3).measure == pytest.approx(1.2 * 0.5 + 2 * (1.2 * 0.1 + 0.5 * 0.1), rel=1e-10)
    flush = P.build_structured_grid(P.Box((0.0, 0.625), (2.0, 1.0)), 0.125)
    with pytest.raises(P.MeshError):
        P.extract_interface(flush, gm)
    sunk = P.build_structured_grid(P.Box((1.0, 0.5), (2.0, 0.875)), 0.125)      # top must ride on the global top
    with pytest.raises(P.MeshError):
        P.extract_interface(sunk, gm)


def test_interface_constant_functional_equals_measure():
    """test_mesh.py::test_interface_constant_functional_equals_measure, through the device
    functional: for T_local = z the normal derivative is -1 on the bottom facets and 0 on
    the lateral ones, so the load of a unit conductivity jump sums to minus the bottom area
    (the test functions sum to one)."""
    gm, lm = plates()
    gamma = P.extract_interface(lm, gm)
    field = P.FieldState(lm, lm.coords[:, 2].copy(), 0.0)
    load = transmission_load(field, gamma, gm, material(11.0, 11.0), material(10.0, 10.0))
    assert float(np.sum(load)) == pytest.approx(-(8e-4 * 6e-4), rel=1e-10)


# ---- test_metrics.py (metrics.py:123-165) -----------------------------------------------

def _log_and_reference(scale=1.0):
    gm, lm = plates()
    base_g = 300.0 + 2e5 * gm.coords[:, 0] + 1e5 * gm.coords[:, 2]
    base_l = 300.0 + 2e5 * lm.coords[:, 0] + 1e5 * lm.coords[:, 2]
    log, ref = P.RunLog(), P.Trajectory(gm)
    for k in range(4):
        t = 0.1 * k
        vals = base_g * (1 + 0.1 * k)
        ref.append(P.FieldState(gm, vals, t))
        log.record("initial" if k == 0 else "macro", t, P.FieldState(lm, scale * base_l * (1 + 0.1 * k), t),
                   P.FieldState(gm, vals, t), 0)
    return log, ref


def test_error_metrics_identical_and_scaled_trajectories():
    """test_error_metrics_identical_trajectories and test_error_metrics_relative_scaling: the
    relative L2(local domain) error, interpolation and mass norms on the device."""
    log, ref = _log_and_reference()
    rep = P.error_metrics(log, ref)
    assert np.allclose(rep.rel_l2, 0.0, atol=1e-12) and rep.mean_rel_l2 == pytest.approx(0.0, abs=1e-12)
    eps = 0.03
    log, ref = _log_and_reference(scale=1 + eps)
    rep = P.error_metrics(log, ref)
    assert np.allclose(rep.rel_l2[1:], eps, rtol=1e-10)
    assert rep.mean_rel_l2 == pytest.approx(eps, rel=1e-10)


# ---- the reference's 2D toy setups themselves (test_twolevel.py:34-41,160-196) ------------

def _toy2d():
    gm = P.build_structured_grid(P.Box((0.0, 0.0), (5.0, 1.0)), 0.125)
    lm = P.build_structured_grid(P.Box((1.0, 0.625), (2.0, 1.0)), 0.125)
    return gm, lm


def _toy_material(k_lo, k_hi):
    """test_twolevel.py::melt_material: rho c = 1000 so a kW-class beam drives hundreds of
    kelvin per second on the unit-scale box."""
    return P.Material(np.array([[300.0, k_lo], [1300.0, k_hi]]), np.array([[300.0, 10.0], [1300.0, 10.0]]),
                      100.0, 0.0, 400.0, 500.0, 0.05)


def test_transmission_2d_hand_computed_linear_field():
    """test_twolevel.py::test_transmission_hand_computed_linear_field, on its own 2D boxes:
    T_local = x with a conductivity jump delta tested against w = 1 (the lateral edges
    cancel) and w = x (delta (b - a)(H - c) for the local box [a, b] x [c, H]); and
    test_transmission_linear_in_local_field."""
    gm, lm = _toy2d()
    gamma = P.extract_interface(lm, gm)
    delta = 7.0
    flat = np.array([[300.0, 400.0], [1300.0, 700.0]])
    mk = lambda k: P.Material(np.array([[300.0, k], [1300.0, k]]), flat, 8000.0, 0.0, 1563.15, 1653.15, 0.05)  # noqa: E731
    load = np.asarray(transmission_load(P.FieldState(lm, lm.coords[:, 0].copy(), 0.0), gamma, gm, mk(10.0 + delta), mk(10.0)))
    assert load.sum() == pytest.approx(0.0, abs=1e-12)
    assert load @ gm.coords[:, 0] == pytest.approx(delta * (2.0 - 1.0) * (1.0 - 0.625), rel=1e-12)
    f1 = P.FieldState(lm, lm.coords[:, 0].copy(), 0.0)
    f2 = P.FieldState(lm, lm.coords[:, 1].copy(), 0.0)
    both = P.FieldState(lm, 2.0 * lm.coords[:, 0] + 3.0 * lm.coords[:, 1], 0.0)
    l1, l2, lb = (np.asarray(transmission_load(f, gamma, gm, mk(12.0), mk(9.0))) for f in (f1, f2, both))
    assert np.allclose(lb, 2.0 * l1 + 3.0 * l2, atol=1e-12)


def test_two_way_2d_omega_independent_and_idempotent():
    """test_two_way_coupling_converges_and_is_omega_independent and
    test_iterate_idempotent_at_fixed_point with the reference's own 2D setup (unit-scale
    boxes, a parked 3 kW line source at (1.5, 1.0), coarse / fine conductivities 2..3 / 5..8)."""
    bc = P.ThermalBC(10.0, 0.0, T0, T0)
    beam = P.LaserBeam(3000.0, 1.0, 0.25, 0.1, 1e-6)
    path = P.path_from_segments([((1.5, 1.0), (1.5 + 1e-6, 1.0), beam.speed)])
    gm, lm = _toy2d()

    def problem(omega):
        return P.TwoLevelProblem(global_mesh=gm, mat_global=_toy_material(2.0, 3.0), mat_local=_toy_material(5.0, 8.0),
                                 bc=bc, solver=CG, coupling=P.CouplingSettings(omega=omega), beam=beam, path=path,
                                 source_global="gaussian")

    p1, p2 = problem(1.0), problem(0.5)
    assert not p1.one_way
    s1 = P.initial_state(p1, lm, P.uniform_field(gm, T0))
    s2 = P.initial_state(p2, lm, P.uniform_field(gm, T0))
    o1, it1 = two_level_iterate(p1, s1, 0.05)
    o2, it2 = two_level_iterate(p2, s2, 0.05)
    assert it1 >= 2 and it2 >= it1
    assert o1.local_field.values.max() > T0 + 2.0           # 1.2e5 W/m^3 over rho c = 1000 for 0.05 s
    diff = np.linalg.norm(o1.local_field.values - o2.local_field.values) / np.linalg.norm(o1.local_field.values)
    assert diff < 10 * p1.coupling.tolerance
    again, _ = two_level_iterate(p1, o1, 1e-12)
    scale = max(np.linalg.norm(o1.trace), 1e-12)
    assert np.linalg.norm(again.trace - o1.trace) / scale < p1.coupling.tolerance


def test_criterion_8_structural_invariants_on_the_2d_toy_boxes():
    """tests/test_acceptance.py::test_criterion_8_structural_invariants, the device-side checks
    on its own 2D boxes: the interface functional exactly zero for matching conductivities,
    trace interpolation exact at the end points, a constant state preserved by the coupled
    step, and m = 1 degenerating to the uniform-step scheme under two-way coupling (10 x the
    coupling tolerance).  (omega independence: the previous test.)"""
    from paper_2110_12932_b200.multirate import interpolate_trace
    gm, lm = _toy2d()
    gamma = P.extract_interface(lm, gm)
    mat = P.Material(np.array([[0.0, 12.0], [5000.0, 12.0]]), np.array([[0.0, 500.0], [5000.0, 500.0]]), 8000.0, 0.0,
                     1000.0, 1100.0, 0.05)
    fld = P.FieldState(lm, 300.0 + 40 * lm.coords[:, 0] * lm.coords[:, 1], 0.0)
    assert np.all(np.asarray(transmission_load(fld, gamma, gm, mat, mat)) == 0.0)
    a, b = np.array([300.0, 310.0, 320.0]), np.array([400.0, 390.0, 380.0])
    np.testing.assert_array_equal(interpolate_trace(0, 4, a, b), a)
    np.testing.assert_array_equal(interpolate_trace(4, 4, a, b), b)
    quiet = P.TwoLevelProblem(global_mesh=gm, mat_global=mat, mat_local=mat, bc=P.ThermalBC(0.0, 0.0, 321.0, 321.0),
                              solver=CG)
    st = P.initial_state(quiet, lm, P.uniform_field(gm, 321.0))
    st, _ = two_level_iterate(quiet, st, 0.5)
    assert np.allclose(st.global_field.values, 321.0, atol=1e-9) and np.allclose(st.local_field.values, 321.0, atol=1e-9)
    beam = P.LaserBeam(3000.0, 1.0, 0.25, 0.1, 1e-6)
    path = P.path_from_segments([((1.5, 1.0), (1.5 + 1e-6, 1.0), beam.speed)])
    p = P.TwoLevelProblem(global_mesh=gm, mat_global=_toy_material(2.0, 3.0), mat_local=_toy_material(5.0, 8.0),
                          bc=P.ThermalBC(10.0, 0.0, T0, T0), solver=CG, beam=beam, path=path, source_global="gaussian")
    U = P.uniform_field(gm, T0)
    st1 = P.run_spacetime(p, P.MacroSchedule(0.05, 1, 0.0, 0.25), lm, U)
    st2 = P.run_space(p, 0.05, 5, lm, U)
    rel = np.linalg.norm(st1.local_field.values - st2.local_field.values) / np.linalg.norm(st2.local_field.values)
    assert rel < 10 * 1e-6


def test_control_temperature_and_composite_sampler():
    """test_metrics.py::test_control_temperature_constant_field, ..._linear_exact,
    ..._line_outside and ::test_composite_sampler_prefers_local (device interpolation); the
    composite sampler also across a TRANSLATED local lattice in 3D (the fine field is located
    from the moved box)."""
    from paper_2110_12932_b200.metrics import MetricsError, composite_sampler, control_temperature
    m = P.build_structured_grid(P.Box((0.0, 0.0), (1.0, 1.0)), 0.25)
    assert control_temperature(P.uniform_field(m, 7.0), 0.99, (0.0, 1.0), 0.125) == pytest.approx(7.0, rel=1e-12)
    lin = P.FieldState(m, m.coords[:, 0].copy(), 0.0)
    assert control_temperature(lin, 0.5, (0.0, 1.0), 0.125) == pytest.approx(0.5, rel=1e-12)
    with pytest.raises(MetricsError):
        control_temperature(P.uniform_field(m, 1.0), 1.5, (0.0, 1.0), 0.125)
    gm = P.build_structured_grid(P.Box((0.0, 0.0), (4.0, 1.0)), 0.25)
    lm = P.build_structured_grid(P.Box((1.0, 0.5), (2.0, 1.0)), 0.25)
    vals = composite_sampler(P.uniform_field(lm, 200.0), P.uniform_field(gm, 100.0))(np.array([[0.5, 0.9], [1.5, 0.9]]))
    assert vals[0] == pytest.approx(100.0) and vals[1] == pytest.approx(200.0)
    g3, l3 = plates()
    moved = l3.translated((2e-4, -1e-4, 0.0), within=g3.box)
    fine = P.FieldState(moved, 500.0 + 3e5 * moved.coords[:, 0] - 2e5 * moved.coords[:, 1] + 1e5 * moved.coords[:, 2], 0.0)
    pts = np.array([[9e-4, 3e-4, 4.5e-4], [1.55e-3, 6.5e-4, 5e-4], [1e-4, 1e-4, 1e-4]])
    got = composite_sampler(fine, P.uniform_field(g3, 100.0))(pts)
    want = 500.0 + 3e5 * pts[:, 0] - 2e5 * pts[:, 1] + 1e5 * pts[:, 2]
    assert got[0] == pytest.approx(want[0], rel=1e-12) and got[1] == pytest.approx(want[1], rel=1e-12)
    assert got[2] == pytest.approx(100.0)

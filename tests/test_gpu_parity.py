"""Device parity: the CUDA path through the C ABI against the oracle and the golden vectors.

Tolerance (north_star): relative L-inf <= 1e-9 per step with CG tolerance 1e-12,
melt masks (T > T_liquidus) bit-exact, CG iteration counts within +-1 of the
reference's.  Single steps are held to 1e-12 (the device mirrors scipy's CG
operation for operation; only summation order differs).
"""

import json

import numpy as np
import pytest

import paper_2110_12932_b200 as P
from paper_2110_12932_b200 import _native as N
from paper_2110_12932_b200 import ops
from paper_2110_12932_b200.errors import NonConvergence
from paper_2110_12932_b200.grid import StructuredGrid
from paper_2110_12932_b200.control import LocalPlacement
from oracle import kuhn
from oracle.twolevel import OracleRun

from .conftest import CONFIGS, GOLDEN, ROOT, assert_mask

pytestmark = pytest.mark.gpu
REL = 1e-9


def rel(a, b):
    return float(np.abs(np.asarray(a) - np.asarray(b)).max() / np.abs(np.asarray(b)).max())


def _grid(lo, hi, n, off=(0.0, 0.0, 0.0)):
    box = P.Box(tuple(lo), tuple(hi))
    return StructuredGrid(LocalPlacement(box, np.asarray(n), np.asarray(off, dtype=float),
                                         box.translated(off)))


@pytest.mark.parametrize("name", ["aniso_local", "aniso_global", "cfg1_local", "cfg1_global"])
def test_single_step_vs_reference_golden(name):
    z = np.load(GOLDEN / f"op_{name}.npz")
    grid = _grid(z["lo"], z["hi"], z["ncells"])
    local = str(z["kind"]) == "local"
    g = np.zeros(grid.n_nodes)
    g[z["dnodes"]] = z["dvals"]
    beam = P.LaserBeam(200.0, 0.35, 5e-5, 5e-5, 0.8)
    x, info = ops.step(grid, 9.8, 8440 * 410.0, float(z["dt"]),
                       N.TL_DIRICHLET_GAMMA if local else N.TL_DIRICHLET_BOTTOM, z["T_old"],
                       g=g, load=None if local else z["extra"],
                       gaussian=(beam.gaussian_peak, beam.radius, beam.depth, z["center"]) if local else None,
                       rtol=1e-12)
    assert info.status == 0
    assert abs(info.iterations - int(z["cg_iters"])) <= 1
    assert rel(x, z["sol"]) <= 1e-12
    assert info.true_resid <= 100 * 1e-12


def test_step_backward_euler_seam():
    """Seam 3: fem.step_backward_euler with reference-shaped arguments."""
    z = np.load(GOLDEN / "op_cfg1_local.npz")
    grid = _grid(z["lo"], z["hi"], z["ncells"])
    mat = P.load_material(CONFIGS / "const.mat")
    beam = P.LaserBeam(200.0, 0.35, 5e-5, 5e-5, 0.8)
    bounds = P.BoundarySpec(bc=P.ThermalBC(0.0, 0.0, 293.0, 293.0), radiation=True,
                            dirichlet_nodes=z["dnodes"], dirichlet_values=z["dvals"])
    st = P.FieldState(grid, z["T_old"], 0.0)
    out = P.step_backward_euler(st, float(z["dt"]), mat, P.GaussianSource(beam, tuple(z["center"])),
                                bounds, P.SolverSettings(linear_tol=1e-12, linear_solver="cg"),
                                latent=True)
    assert out.time == float(z["dt"])
    assert rel(out.values, z["sol"]) <= 1e-12


def test_nonconvergence_maps_to_reference_exception():
    z = np.load(GOLDEN / "op_cfg1_global.npz")
    grid = _grid(z["lo"], z["hi"], z["ncells"])
    x, info = ops.step(grid, 9.8, 8440 * 410.0, float(z["dt"]), N.TL_DIRICHLET_BOTTOM, z["T_old"],
                       g_const=293.0, load=z["extra"], rtol=1e-12, maxiter=2)
    assert info.status == N.TL_SOLVE_MAXITER and info.iterations == 2
    with pytest.raises(NonConvergence) as exc:
        ops.raise_for(info)
    assert exc.value.iterations == 2


_LIMIT_SCRIPT = r"""
import sys, json, numpy as np
sys.path.insert(0, {root!r})
import paper_2110_12932_b200 as P
from paper_2110_12932_b200 import _native as N, ops
from paper_2110_12932_b200.control import LocalPlacement
from paper_2110_12932_b200.grid import StructuredGrid
z = np.load({golden!r})
grid = StructuredGrid(LocalPlacement(P.Box(tuple(z["lo"]), tuple(z["hi"])), np.asarray(z["ncells"])))
out = []
for maxiter in {limits!r}:
    x, info = ops.step(grid, 9.8, 8440 * 410.0, float(z["dt"]), N.TL_DIRICHLET_BOTTOM, z["T_old"],
                       g_const=293.0, load=z["extra"], rtol=1e-12, maxiter=maxiter)
    out.append([int(info.status), int(info.iterations)])
print(json.dumps(out))
"""


@pytest.mark.parametrize("env", [{}, {"TLGPU_EXACT_CG": "1"}, {"TLGPU_STREAMING": "1", "TLGPU_TILED_MIN": "1"},
                                 {"TLGPU_STREAMING": "1", "TLGPU_TILED": "0"}])
def test_linear_cg_at_the_iteration_limit_follows_scipy(env):
    """scipy's cg tests ||r|| < atol at the top of each of its maxiter loop passes and reports
    failure when the loop runs out (``fem.py:283-288`` then raises NonConvergence): a solve
    that needs `its` iterations fails with maxiter = its and converges with maxiter = its + 1.
    Every linear kernel family (SMEM-resident CG-CG, the scipy-exact two-barrier kernel, the
    bulk-copy streaming loop, the flat streaming loop) against the oracle's scipy mirror;
    solver switches are read once per process, so each runs in a subprocess."""
    import os
    import subprocess
    import sys
    from oracle.pcg import solve_constrained
    z = np.load(GOLDEN / "op_cfg1_global.npz")
    grid = _grid(z["lo"], z["hi"], z["ncells"])
    G = kuhn.KuhnGrid(grid.placement.box0.lo, grid.placement.box0.hi, grid.ncells, grid.placement.offset)
    op = kuhn.StencilOperator(G, 9.8, 8440 * 410.0, float(z["dt"]), G.bottom_mask())
    g = np.full(grid.n_nodes, 293.0)
    _, its, _ = solve_constrained(op, op.rhs(z["T_old"], z["extra"], g), g, 1e-12)
    code = _LIMIT_SCRIPT.format(root=str(ROOT), golden=str(GOLDEN / "op_cfg1_global.npz"), limits=[3, its, its + 1])
    res = subprocess.run([sys.executable, "-c", code], env={**os.environ, **env}, capture_output=True, text=True,
                         timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    got = json.loads(res.stdout.strip().splitlines()[-1])
    assert got == [[N.TL_SOLVE_MAXITER, 3], [N.TL_SOLVE_MAXITER, its], [N.TL_SOLVE_OK, its]], (got, its)


def test_vc_cg_at_the_iteration_limit_follows_scipy():
    """The same rule for the variable-coefficient Jacobi-PCG (k_vc_cg) of the Picard path,
    against the oracle's assembly + scipy mirror (nothing exercised the vc
    path at maxiter)."""
    import ctypes as C
    from oracle import varcoef
    from oracle.pcg import cg_mirror
    from .test_oracle_golden import picard_material
    z = np.load(GOLDEN / "picard_tables.npz")
    grid = P.build_structured_grid(P.Box(tuple(z["lo"]), tuple(z["hi"])), float(z["h"]))
    mat = picard_material(z)
    G = kuhn.KuhnGrid(grid.box.lo, grid.box.hi, grid.ncells)
    n = grid.n_nodes
    nodes = grid.nodes_on(P.BOTTOM)
    dmask = np.zeros(n, dtype=bool)
    dmask[nodes] = True
    g = np.full(n, 293.0)
    diag, w, b = varcoef.assemble(G, mat, z["T_old"], z["T_old"], float(z["dt"]), None, False, None)
    dc, wc, bc = varcoef.constrained(G, diag, w, b, dmask, g)
    xref, info0, its = cg_mirror(lambda v: varcoef.apply(G, dc, wc, v), bc, 1.0 / dc, 1e-12, 20 * n)
    assert info0 == 0 and its > 3
    md, _tabs = P.fem.vc_material(mat, False)
    desc = grid.desc()
    rb = N.Robin(0.0, 0.0, 293.0, 0)
    idx = np.ascontiguousarray(nodes, dtype=np.int32)
    vals = np.full(idx.size, 293.0)
    T_old = np.ascontiguousarray(z["T_old"], dtype=np.float64)

    def solve(maxiter):
        x = np.empty(n)
        info = N.SolveInfo()
        npass, inc = C.c_int32(0), C.c_double(0.0)
        its_ = np.zeros(1, dtype=np.int32)
        ms = np.zeros(1, dtype=np.float32)
        N.check(N.lib().tl_vc_picard_nodes_host(
            C.byref(desc), C.byref(md), None, None, 0, float(z["dt"]), N.dptr(T_old), None, None, C.byref(rb),
            idx.ctypes.data, idx.size, N.dptr(vals), 1e-12, int(maxiter), 1, 1e-8, 1, N.dptr(x), C.byref(npass),
            its_.ctypes.data, ms.ctypes.data, C.byref(inc), C.byref(info)), "step")
        return x, info

    for maxiter, status in ((3, N.TL_SOLVE_MAXITER), (its, N.TL_SOLVE_MAXITER), (its + 1, N.TL_SOLVE_OK)):
        x, info = solve(maxiter)
        assert info.status == status, (maxiter, its, info.status, info.iterations)
        assert info.iterations == min(maxiter, its)
    assert rel(x, np.where(dmask, g, xref)) <= REL
    with pytest.raises(NonConvergence) as exc:
        ops.raise_for(solve(its)[1])
    assert exc.value.iterations == its


def test_interpolation_points_vs_golden():
    z = np.load(GOLDEN / "interp.npz")
    box = P.Box(tuple(z["lo"]), tuple(z["hi"]))
    grid = P.build_structured_grid(box, float(z["h"]))
    out = grid.interpolate(z["vals"], z["pts"])
    assert rel(out, z["out"]) <= 1e-14


def test_interpolation_to_translated_lattice_vs_oracle():
    rng = np.random.default_rng(3)
    G = P.build_structured_grid(P.Box((0, 0, 0), (2e-3, 1e-3, 5e-4)), 5e-5)
    vals = rng.uniform(293, 2293, G.n_nodes)
    L = StructuredGrid(LocalPlacement(P.Box((3.3e-4, 2.1e-4, 1e-4), (7.3e-4, 6.1e-4, 3e-4)),
                                      np.array([40, 40, 20]))).translated((1.7e-5, -3e-5, 0.0))
    full = ops.interpolate_to_grid(G, vals, L)
    ref = kuhn.interpolate(kuhn.KuhnGrid(G.box.lo, G.box.hi, G.ncells), vals, L.coords)
    assert rel(full, ref) <= 1e-14
    gam = ops.interpolate_to_grid(G, vals, L, gamma_only=True)
    m = L.gamma_mask()
    assert rel(gam[m], ref[m]) <= 1e-14 and np.all(gam[~m] == 0.0)


def test_deposit_vs_golden():
    d = json.loads((GOLDEN / "deposit.json").read_text())
    grid = P.build_structured_grid(P.Box(tuple(d["lo"]), tuple(d["hi"])), d["h"])
    for c in d["cases"]:
        load = ops.deposit_load(grid, np.array(c["pts"]).reshape(-1, 3), np.array(c["pw"]))
        nz = np.nonzero(load)[0]
        np.testing.assert_array_equal(nz, c["idx"])
        assert rel(load[nz], c["val"]) <= 1e-13


def _golden_run(name, n_steps=None):
    z = np.load(GOLDEN / f"run_{name}.npz")
    cfg = P.load_config(CONFIGS / f"{name}.cfg")
    rec = []

    def recorder(kind, t, local, glob, iters):
        if kind in ("initial", "macro"):
            rec.append((t, local.values.copy(), glob.values.copy(), local.mesh.box.lo))

    state, stats = P.two_level_run(cfg, recorder=recorder, n_steps=n_steps)
    return z, cfg, rec, stats


@pytest.mark.parametrize("name", ["cfg1_m4", "cfg1_uniform"])
def test_full_run_cfg1_vs_reference(name):
    z, cfg, rec, stats = _golden_run(name)
    counters = json.loads(str(z["counters"]))
    assert stats.counters == counters
    TL = cfg.material.T_liquidus
    s = int(z["stride"])
    worst = 0.0
    for k, (t, Tl, Tg, lo) in enumerate(rec):
        assert t == z["t"][k]
        np.testing.assert_array_equal(lo, z["box"][k])
        worst = max(worst, rel(Tg[::s], z["gsub"][k]), rel(Tl[::s], z["lsub"][k]))
        assert_mask(None, Tg, z["gmelt"][k], TL, True)
        assert_mask(None, Tl, z["lmelt"][k], TL, True)
        if k in z["full_at"]:
            assert rel(Tg, z[f"g{k}"]) <= REL
            assert rel(Tl, z[f"l{k}"]) <= REL
    assert worst <= REL


def test_device_iterations_match_reference_cfg1():
    z = np.load(GOLDEN / "run_cfg1_m4.npz")
    cfg = P.load_config(CONFIGS / "cfg1_m4.cfg")
    problem, lm = P.build_problem(cfg)
    sched = P.MacroSchedule(cfg.dt_macro, cfg.micro_steps, 0.0, cfg.t_end)
    with P.DeviceRun(problem, lm) as run:
        from paper_2110_12932_b200.schedule import plan_spacetime
        run.initial(P.uniform_field(problem.global_mesh, 293.0))
        run.run(plan_spacetime(problem, sched, lm.placement, cfg.path, cfg.policy, 0.0, 0.0))
        its = [i["iterations"] for i in run.take_info()]
    ref = z["cg_iters"]
    assert len(its) == len(ref)
    assert max(abs(a - b) for a, b in zip(its, ref)) <= 1


def test_async_field_readback_matches_sync():
    """tl_run_field_async / _wait (pipelined read-back while later macro steps run) return
    bitwise the fields tl_run_get_field returns after each step."""
    from paper_2110_12932_b200.schedule import plan_spacetime
    cfg = P.load_config(CONFIGS / "cfg1_m4.cfg")
    problem, lm = P.build_problem(cfg)
    sched = P.MacroSchedule(cfg.dt_macro, cfg.micro_steps, 0.0, cfg.t_end)
    plans, placement, tg, tl = [], lm.placement, 0.0, 0.0
    for k in range(6):
        pl = plan_spacetime(problem, sched, placement, cfg.path, cfg.policy, tg, tl, k0=k, nsteps=1)
        plans.append(pl)
        placement, tg, tl = pl.final_placement, pl.final_t_global, pl.final_t_local
    sync_fields = []
    with P.DeviceRun(problem, lm) as run:
        run.initial(P.uniform_field(problem.global_mesh, 293.0))
        for pl in plans:
            run.run(pl)
            sync_fields.append((run.field(0), run.field(1)))
    bufs = [(np.empty(problem.global_mesh.n_nodes), np.empty(lm.n_nodes)) for _ in range(len(plans))]
    with P.DeviceRun(problem, lm) as run:
        run.initial(P.uniform_field(problem.global_mesh, 293.0))
        for s, pl in enumerate(plans):
            run.run(pl)
            run.field_async(0, bufs[s][0], slot=(2 * s) % 4)
            run.field_async(1, bufs[s][1], slot=(2 * s + 1) % 4)
            if s >= 1:
                run.field_wait((2 * s - 2) % 4)
                run.field_wait((2 * s - 1) % 4)
        run.field_wait((2 * len(plans) - 2) % 4)
        run.field_wait((2 * len(plans) - 1) % 4)
    for (g, l), (ga, la) in zip(sync_fields, bufs):
        np.testing.assert_array_equal(g, ga)
        np.testing.assert_array_equal(l, la)


def test_cfg2_first_steps_vs_reference():
    z, cfg, rec, stats = _golden_run("cfg2", n_steps=2)
    TL = cfg.material.T_liquidus
    s = int(z["stride"])
    for k, (t, Tl, Tg, lo) in enumerate(rec):
        assert rel(Tg[::s], z["gsub"][k]) <= REL and rel(Tl[::s], z["lsub"][k]) <= REL
        assert_mask(None, Tg, z["gmelt"][k], TL, True)
        assert_mask(None, Tl, z["lmelt"][k], TL, True)
        if k in z["full_at"]:
            assert rel(Tg, z[f"g{k}"]) <= REL and rel(Tl, z[f"l{k}"]) <= REL


def test_cfg2_25_steps_vs_oracle():
    """Full-size cfg2 grids, 25 macro steps (track start, a relocation after every step;
    covers the bench's timed window) against the oracle: every step's fields to 1e-9 and
    melt masks, every solve's CG iteration count within +-1."""
    cfg = P.load_config(CONFIGS / "cfg2.cfg")
    orc = OracleRun(cfg)
    ref = []
    orc.run_spacetime(n_steps=25, recorder=lambda kind, t, Tl, Tg, pl: ref.append((Tl, Tg)))
    rec = []
    P.two_level_run(cfg, n_steps=25,
                    recorder=lambda kind, t, l, g, it: rec.append((l.values, g.values))
                    if kind in ("initial", "macro") else None)
    TL = cfg.material.T_liquidus
    assert len(rec) == len(ref) == 26
    for (Tl, Tg), (Rl, Rg) in zip(rec, ref):
        assert rel(Tg, Rg) <= REL and rel(Tl, Rl) <= REL
        assert_mask("cfg2 25 steps global", Tg, Rg, TL)
        assert_mask("cfg2 25 steps local", Tl, Rl, TL)


def test_recorder_protocol_kinds_and_times():
    cfg = P.load_config(CONFIGS / "cfg1_m4.cfg")
    kinds = []
    P.two_level_run(cfg, n_steps=2, recorder=lambda kind, t, l, g, it: kinds.append(
        (kind, t, l is None, g is None, it)))
    sched = P.MacroSchedule(cfg.dt_macro, 4, 0.0, 2 * cfg.dt_macro)
    expect = [("initial", 0.0, False, False, 0)]
    for k in range(2):
        expect.append(("predictor", sched.t_macro(k + 1), True, False, 0))
        expect += [("micro", sched.t_micro(k, i + 1), False, True, 0) for i in range(4)]
        expect.append(("macro", sched.t_macro(k + 1), False, False, 1))
    assert kinds == expect


def test_run_without_recorder_matches_recorded_run():
    cfg = P.load_config(CONFIGS / "cfg1_m4.cfg")
    a, _ = P.two_level_run(cfg, n_steps=6)
    b, _ = P.two_level_run(cfg, n_steps=6, recorder=lambda *args: None)
    np.testing.assert_array_equal(a.global_field.values, b.global_field.values)
    np.testing.assert_array_equal(a.local_field.values, b.local_field.values)
    assert a.local_field.mesh.box == b.local_field.mesh.box


def test_deterministic_run_to_run():
    cfg = P.load_config(CONFIGS / "cfg1_m4.cfg")
    a, _ = P.two_level_run(cfg, n_steps=5)
    b, _ = P.two_level_run(cfg, n_steps=5)
    np.testing.assert_array_equal(a.global_field.values, b.global_field.values)
    np.testing.assert_array_equal(a.local_field.values, b.local_field.values)


def test_source_off_after_path_end():
    """Past the path's end the Gaussian and the deposit vanish (runner.py:54-55,
    scanpath.py:103-106); the laser stops at x = 1.6 mm at t = 1.75 ms of a 2 ms run."""
    text = (CONFIGS / "cfg1_m4.cfg").read_text().replace("segment 0.2 0.5 0.5 1.8 0.5 0.5 mm",
                                                         "segment 0.2 0.5 0.5 1.6 0.5 0.5 mm")
    cfg = P.config_from_text(text, CONFIGS)
    orc = OracleRun(cfg)
    ref = []
    orc.run_spacetime(recorder=lambda kind, t, Tl, Tg, pl: ref.append((Tl, Tg)))
    state, _ = P.two_level_run(cfg)
    assert rel(state.global_field.values, ref[-1][1]) <= REL
    assert rel(state.local_field.values, ref[-1][0]) <= REL


def test_box_reaching_the_wall_raises_like_the_reference():
    """A relocation that lands the box on the global wall passes Mesh.translated's
    test but fails extract_interface's strict immersion (mesh.py:489-496) -> MeshError."""
    text = (CONFIGS / "cfg1_m4.cfg").read_text().replace("t_end 2 ms", "t_end 2.1 ms")
    cfg = P.config_from_text(text, CONFIGS)
    with pytest.raises(P.MeshError):
        P.two_level_run(cfg)


def _oracle_step(grid, kind, T_old, dt, g, load=None, gauss=None):
    from oracle.pcg import solve_constrained
    G = kuhn.KuhnGrid(grid.placement.box0.lo, grid.placement.box0.hi, grid.ncells, grid.placement.offset)
    D = (G.bottom_mask() if kind == N.TL_DIRICHLET_BOTTOM else G.gamma_mask())
    op = kuhn.StencilOperator(G, 9.8, 8440 * 410.0, dt, D)
    if gauss is not None:
        load = kuhn.gaussian_load(G, gauss[0], gauss[1])
    b = op.rhs(T_old, load, g)
    x, its, _ = solve_constrained(op, b, g, 1e-12)
    return x, its


def test_streaming_global_step_cfg3_size_vs_oracle():
    """HBM-bound size (6.9M nodes, the streaming kernel): one global step vs the oracle."""
    cfg = P.load_config(CONFIGS / "cfg3.cfg")
    problem, lm = P.build_problem(cfg)
    grid = problem.global_mesh
    rng = np.random.default_rng(0)
    T = rng.uniform(293.0, 2293.0, grid.n_nodes)
    g = np.full(grid.n_nodes, 293.0)
    pts, pw = problem.global_source(0.0, cfg.dt_macro)
    load = ops.deposit_load(grid, pts, pw)
    x, info = ops.step(grid, 9.8, 8440 * 410.0, cfg.dt_macro, N.TL_DIRICHLET_BOTTOM, T, g_const=293.0,
                       load=load, rtol=1e-12)
    ref, its = _oracle_step(grid, N.TL_DIRICHLET_BOTTOM, T, cfg.dt_macro, g, load=load)
    assert info.status == 0 and abs(info.iterations - its) <= 1
    assert rel(x, ref) <= 1e-12


def test_streaming_local_step_cfg3_size_vs_oracle():
    """cfg3 local grid (1.73M nodes, streaming kernel + Gaussian load kernel) vs the oracle."""
    cfg = P.load_config(CONFIGS / "cfg3.cfg")
    problem, lm = P.build_problem(cfg)
    rng = np.random.default_rng(1)
    T = rng.uniform(293.0, 2293.0, lm.n_nodes)
    g = np.where(lm.gamma_mask(), rng.uniform(293.0, 900.0, lm.n_nodes), 0.0)
    src = problem.local_source(2e-6)
    dt = cfg.dt_macro / cfg.micro_steps
    x, info = ops.step(lm, 9.8, 8440 * 410.0, dt, N.TL_DIRICHLET_GAMMA, T, g=g,
                       gaussian=src.device_args(), rtol=1e-12)
    ref, its = _oracle_step(lm, N.TL_DIRICHLET_GAMMA, T, dt, g, gauss=(cfg.beam, src.center))
    assert info.status == 0 and abs(info.iterations - its) <= 1
    assert rel(x, ref) <= 1e-12


def test_streaming_local_step_cfg4_size_vs_oracle():
    """cfg4 local grid (251 x 251 x 101 = 6.36M nodes, 37 % of the headline step: k_t_cg with
    4-row items, gamma Dirichlet data, Gaussian load) vs the oracle: one micro step."""
    cfg = P.load_config(CONFIGS / "cfg4.cfg")
    problem, lm = P.build_problem(cfg)
    assert lm.n_nodes == 6363101
    rng = np.random.default_rng(3)
    T = rng.uniform(293.0, 2293.0, lm.n_nodes)
    g = np.where(lm.gamma_mask(), rng.uniform(293.0, 900.0, lm.n_nodes), 0.0)
    src = problem.local_source(2e-6)
    dt = cfg.dt_macro / cfg.micro_steps
    x, info = ops.step(lm, 9.8, 8440 * 410.0, dt, N.TL_DIRICHLET_GAMMA, T, g=g,
                       gaussian=src.device_args(), rtol=1e-12)
    ref, its = _oracle_step(lm, N.TL_DIRICHLET_GAMMA, T, dt, g, gauss=(cfg.beam, src.center))
    assert info.status == 0 and abs(info.iterations - its) <= 1
    assert rel(x, ref) <= 1e-12


def test_cfg3_three_macro_steps_vs_oracle():
    """cfg3 (6.9M-node global grid on the streaming solve, 1.7M-node local grid, m = 10):
    3 macro steps with a relocation after each but the last, against OracleRun: every
    macro step's fields to 1e-9, melt masks, local-box placements, RunStats counters."""
    cfg = P.load_config(CONFIGS / "cfg3.cfg")
    orc = OracleRun(cfg)
    ref = []
    orc.run_spacetime(n_steps=3, recorder=lambda kind, t, Tl, Tg, pl: ref.append((t, Tl, Tg, pl.box.lo)))
    rec = []
    _, stats = P.two_level_run(cfg, n_steps=3,
                               recorder=lambda kind, t, l, g, it: rec.append((t, l.values, g.values, l.mesh.box.lo))
                               if kind in ("initial", "macro") else None)
    TL = cfg.material.T_liquidus
    assert len(rec) == len(ref) == 4
    for (t, Tl, Tg, lo), (rt, Rl, Rg, rlo) in zip(rec, ref):
        assert t == rt
        np.testing.assert_array_equal(np.asarray(lo), np.asarray(rlo))
        assert rel(Tg, Rg) <= REL and rel(Tl, Rl) <= REL
        assert_mask("cfg3 3 steps global", Tg, Rg, TL)
        assert_mask("cfg3 3 steps local", Tl, Rl, TL)
    assert stats.counters["relocations"] == 2 and stats.counters["global_solves"] == 3
    assert stats.counters["local_solves"] == orc.counters["local_solves"]


def test_cfg4_global_step_vs_oracle():
    """The HBM-target grid itself: one cfg4 global implicit step (201,402,201 nodes, the
    bulk-copy z-march CG loop k_t_cg) against the numpy stencil oracle on the same random
    T_old ~ U[293, 2293] K (seed 0) with the macro step's swept-track deposit: 1e-12
    relative L-inf, CG iterations within +-1, melt masks (fem.py:271-298)."""
    import gc
    cfg = P.load_config(CONFIGS / "cfg4.cfg")
    problem, _ = P.build_problem(cfg)
    grid = problem.global_mesh
    assert grid.n_nodes == 201_402_201
    rng = np.random.default_rng(0)
    T = rng.uniform(293.0, 2293.0, grid.n_nodes)
    pts, pw = problem.global_source(0.0, cfg.dt_macro)
    load = ops.deposit_load(grid, pts, pw)
    x, info = ops.step(grid, 9.8, 8440 * 410.0, cfg.dt_macro, N.TL_DIRICHLET_BOTTOM, T, g_const=293.0,
                       load=load, rtol=1e-12)
    assert info.status == 0
    ref, its = _oracle_step(grid, N.TL_DIRICHLET_BOTTOM, T, cfg.dt_macro, np.full(grid.n_nodes, 293.0),
                            load=load)
    del T, load
    gc.collect()
    assert abs(info.iterations - its) <= 1
    assert rel(x, ref) <= 1e-12
    assert_mask("cfg4 global step", x, ref, cfg.material.T_liquidus)


def test_linearity_full_size_cfg4_global_step():
    """A size-independent property on cfg4's 201M-node global grid (next to the oracle step
    above): the implicit step is affine in (T_old, load), so
    step(T1 + T2, L1 + L2) - step(T2, L2) == step(T1, L1) - step(0, 0) to CG tolerance."""
    cfg = P.load_config(CONFIGS / "cfg4.cfg")
    problem, _ = P.build_problem(cfg)
    grid = problem.global_mesh
    n = grid.n_nodes
    rng = np.random.default_rng(2)
    k = 9.8, 8440 * 410.0
    T1 = rng.uniform(0.0, 100.0, n)
    T2 = np.full(n, 293.0)
    s = lambda T: ops.step(grid, *k, cfg.dt_macro, N.TL_DIRICHLET_BOTTOM, T, g_const=0.0, rtol=1e-12)  # noqa: E731
    a, ia = s(T1 + T2)
    b, ib = s(T2)
    c, ic = s(T1)
    assert ia.status == ib.status == ic.status == 0
    assert np.abs((a - b) - c).max() <= 1e-9 * np.abs(a).max()


_MODE_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, {root!r})
import paper_2110_12932_b200 as P
cfg = P.load_config({cfg!r})
cfg.t_end = {nsteps} * cfg.dt_macro
state, stats = P.two_level_run(cfg)
np.savez({out!r}, g=state.global_field.values, l=state.local_field.values,
         c=np.array([stats.counters[k] for k in ("global_solves", "local_solves", "relocations")]))
"""


@pytest.mark.parametrize("env", [{"TLGPU_MULTI": "0"}, {"TLGPU_NOCACHE": "1", "TLGPU_CGSYNC": "1"},
                                 {"TLGPU_EXACT_CG": "1"},
                                 {"TLGPU_STREAMING": "1", "TLGPU_TILED_MIN": "1"},
                                 {"TLGPU_STREAMING": "1", "TLGPU_TILED": "0"},
                                 {"TLGPU_STREAMING": "1", "TLGPU_TILED_MIN": "1", "TLGPU_BOXLOAD": "0",
                                  "TLGPU_SNAKE": "0"},
                                 {"TLGPU_STREAMING": "1", "TLGPU_TILED": "0", "TLGPU_SNAKE": "0"},
                                 {"TLGPU_STREAMING": "1", "TLGPU_TILED_MIN": "1", "TLGPU_TH": "2", "TLGPU_NCW": "19"},
                                 {"TLGPU_STREAMING": "1", "TLGPU_TILED_MIN": "1", "TLGPU_TH": "12", "TLGPU_NCW": "16",
                                  "TLGPU_TC": "3"}])
def test_alternative_solver_modes_match_default(env, tmp_path):
    """The non-default device paths (one launch per local solve; no setup cache and
    cg::grid.sync barriers; scipy-exact two-barrier kernel; every solve on the streaming
    path, with the bulk-copy z-march CG loop k_t_cg or the flat k_s_cg, on grids small
    enough that boundary nodes dominate; the same with per-solve full-grid Gaussian loads
    and both sweeps bottom-up; the one-node-per-thread kernel variant with 19 consumer warps
    and a 12-row, 3-chunk item plan with 16) give the default run's fields
    to CG rounding with the same counters (env switches are read once per process, so
    each mode runs in a subprocess)."""
    import os
    import subprocess
    import sys
    cfg = CONFIGS / "cfg1_m4.cfg"
    runs = {}
    for tag, extra in (("default", {}), ("mode", env)):
        out = tmp_path / f"{tag}.npz"
        code = _MODE_SCRIPT.format(root=str(ROOT), cfg=str(cfg), nsteps=6, out=str(out))
        res = subprocess.run([sys.executable, "-c", code], env={**os.environ, **extra},
                             capture_output=True, text=True, timeout=600)
        assert res.returncode == 0, res.stderr[-2000:]
        runs[tag] = np.load(out)
    a, b = runs["default"], runs["mode"]
    assert rel(b["g"], a["g"]) <= 1e-12 and rel(b["l"], a["l"]) <= 1e-12
    np.testing.assert_array_equal(a["c"], b["c"])


_TILED_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, {root!r})
import paper_2110_12932_b200 as P
from paper_2110_12932_b200 import _native as N, ops
cfg = P.load_config({cfg!r})
problem, lm = P.build_problem(cfg)
rng = np.random.default_rng(0)
if {level!r} == "global":
    grid = problem.global_mesh
    T = rng.uniform(293.0, 2293.0, grid.n_nodes)
    pts, pw = problem.global_source(0.0, cfg.dt_macro)
    load = ops.deposit_load(grid, pts, pw)
    x, info = ops.step(grid, 9.8, 8440 * 410.0, cfg.dt_macro, N.TL_DIRICHLET_BOTTOM, T, g_const=293.0,
                       load=load, rtol=1e-12)
else:
    T = rng.uniform(293.0, 2293.0, lm.n_nodes)
    g = np.where(lm.gamma_mask(), rng.uniform(293.0, 900.0, lm.n_nodes), 0.0)
    src = problem.local_source(2e-6)
    x, info = ops.step(lm, 9.8, 8440 * 410.0, cfg.dt_macro / cfg.micro_steps, N.TL_DIRICHLET_GAMMA, T, g=g,
                       gaussian=src.device_args(), rtol=1e-12)
np.savez({out!r}, x=x, its=info.iterations, status=info.status)
"""


@pytest.mark.parametrize("level", ["global", "local"])
def test_tiled_cg_loop_cfg3_size_vs_oracle(level, tmp_path):
    """The bulk-copy z-march CG loop (k_t_cg, default on grids of 20M+ nodes) forced onto
    the cfg3 grids (6.9M nodes, bottom Dirichlet + deposit; 1.73M nodes, gamma Dirichlet +
    Gaussian): one implicit step vs the oracle, iterations +-1, and vs the flat k_s_cg."""
    import os
    import subprocess
    import sys
    cfgp = CONFIGS / "cfg3.cfg"
    out = {}
    for tag, extra in (("tiled", {"TLGPU_TILED_MIN": "1"}), ("flat", {"TLGPU_TILED": "0"})):
        path = tmp_path / f"{tag}.npz"
        code = _TILED_SCRIPT.format(root=str(ROOT), cfg=str(cfgp), level=level, out=str(path))
        res = subprocess.run([sys.executable, "-c", code], env={**os.environ, **extra},
                             capture_output=True, text=True, timeout=900)
        assert res.returncode == 0, res.stderr[-2000:]
        out[tag] = np.load(path)
    cfg = P.load_config(cfgp)
    problem, lm = P.build_problem(cfg)
    rng = np.random.default_rng(0)
    if level == "global":
        grid = problem.global_mesh
        T = rng.uniform(293.0, 2293.0, grid.n_nodes)
        pts, pw = problem.global_source(0.0, cfg.dt_macro)
        load = ops.deposit_load(grid, pts, pw)
        ref, its = _oracle_step(grid, N.TL_DIRICHLET_BOTTOM, T, cfg.dt_macro, np.full(grid.n_nodes, 293.0),
                                load=load)
    else:
        T = rng.uniform(293.0, 2293.0, lm.n_nodes)
        g = np.where(lm.gamma_mask(), rng.uniform(293.0, 900.0, lm.n_nodes), 0.0)
        src = problem.local_source(2e-6)
        ref, its = _oracle_step(lm, N.TL_DIRICHLET_GAMMA, T, cfg.dt_macro / cfg.micro_steps, g,
                                gauss=(cfg.beam, src.center))
    t = out["tiled"]
    assert int(t["status"]) == 0 and abs(int(t["its"]) - its) <= 1
    assert rel(t["x"], ref) <= 1e-12
    assert int(t["its"]) == int(out["flat"]["its"]) and rel(t["x"], out["flat"]["x"]) <= 1e-13


_REPEAT_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, {root!r})
import paper_2110_12932_b200 as P
from paper_2110_12932_b200 import _native as N, ops
cfg = P.load_config({cfg!r})
problem, lm = P.build_problem(cfg)
rng = np.random.default_rng(1)
grid = problem.global_mesh
Tg = rng.uniform(293.0, 2293.0, grid.n_nodes)
pts, pw = problem.global_source(0.0, cfg.dt_macro)
load = ops.deposit_load(grid, pts, pw)
Tl = rng.uniform(293.0, 2293.0, lm.n_nodes)
g = np.where(lm.gamma_mask(), rng.uniform(293.0, 900.0, lm.n_nodes), 0.0)
src = problem.local_source(2e-6)
first = None
for rep in range({reps}):
    xg, ig = ops.step(grid, 9.8, 8440 * 410.0, cfg.dt_macro, N.TL_DIRICHLET_BOTTOM, Tg, g_const=293.0,
                      load=load, rtol=1e-12)
    xl, il = ops.step(lm, 9.8, 8440 * 410.0, cfg.dt_macro / cfg.micro_steps, N.TL_DIRICHLET_GAMMA, Tl, g=g,
                      gaussian=src.device_args(), rtol=1e-12)
    assert ig.status == 0 and il.status == 0
    cur = (xg.copy(), xl.copy(), ig.iterations, il.iterations)
    if first is None:
        first = cur
    else:
        assert cur[2:] == first[2:], (cur[2:], first[2:])
        assert np.array_equal(cur[0], first[0]) and np.array_equal(cur[1], first[1]), rep
print("repeatable", first[2], first[3])
"""


@pytest.mark.parametrize("env", [{}, {"TLGPU_TILED": "0"}, {"TLGPU_SNAKE": "0", "TLGPU_TH": "2", "TLGPU_TC": "9"},
                                 {"TLGPU_NCW": "19", "TLGPU_TH": "2"}])
def test_streaming_paths_bitwise_repeatable(env):
    """Race stress of the hand-rolled synchronisation (compute-sanitizer is closed on this
    GPU pool): the bulk-copy z-march CG loop (mbarrier ring, dynamic item counter, per-item
    partial sums, cooperative grid barriers) and the flat CG loop, five solves each of the
    cfg3 global (6.9M nodes) and local (1.7M nodes) grids in one process: every bit of the
    solution and the iteration counts must repeat whatever CTA ran which item."""
    import os
    import subprocess
    import sys
    code = _REPEAT_SCRIPT.format(root=str(ROOT), cfg=str(CONFIGS / "cfg3.cfg"), reps=5)
    res = subprocess.run([sys.executable, "-c", code], env={**os.environ, **env}, capture_output=True, text=True,
                         timeout=900)
    assert res.returncode == 0, res.stderr[-2000:]
    assert "repeatable" in res.stdout


def test_tiled_cg_loop_wide_grid_vs_oracle(tmp_path):
    """A grid wider than two consumer slots (NX = 1301 > 2 x 608): k_t_cg's general plane
    loops with four nodes per thread (no lean path), one bottom-Dirichlet step with a
    deposit-like load against the oracle."""
    import os
    import subprocess
    import sys
    code = r"""
import sys, numpy as np
sys.path.insert(0, {root!r})
import paper_2110_12932_b200 as P
from paper_2110_12932_b200 import _native as N, ops
grid = P.build_structured_grid(P.Box((0.0, 0.0, 0.0), (2.6e-2, 1.6e-4, 1.6e-4)), 2e-5)
rng = np.random.default_rng(2)
T = rng.uniform(293.0, 2293.0, grid.n_nodes)
load = rng.uniform(0.0, 1e-6, grid.n_nodes)
x, info = ops.step(grid, 9.8, 8440 * 410.0, 2e-5, N.TL_DIRICHLET_BOTTOM, T, g_const=293.0, load=load, rtol=1e-12)
np.savez({out!r}, x=x, T=T, load=load, its=info.iterations, status=info.status, shape=np.array(grid.shape))
"""
    out = tmp_path / "wide.npz"
    res = subprocess.run([sys.executable, "-c", code.format(root=str(ROOT), out=str(out))],
                         env={**os.environ, "TLGPU_STREAMING": "1", "TLGPU_TILED_MIN": "1", "TLGPU_VERBOSE": "1"},
                         capture_output=True,
                         text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    assert "item plan 1301x9x" in res.stderr, res.stderr[-500:]
    z = np.load(out)
    grid = P.build_structured_grid(P.Box((0.0, 0.0, 0.0), (2.6e-2, 1.6e-4, 1.6e-4)), 2e-5)
    assert tuple(z["shape"]) == grid.shape == (9, 9, 1301)
    ref, its = _oracle_step(grid, N.TL_DIRICHLET_BOTTOM, z["T"], 2e-5, np.full(grid.n_nodes, 293.0), load=z["load"])
    assert int(z["status"]) == 0 and abs(int(z["its"]) - its) <= 1
    assert rel(z["x"], ref) <= 1e-12


def test_monolithic_reference_vs_reference_golden():
    """run_reference / solve_monolithic (lpbfsim/runner.py:126-163, fem.py:386-423) on the
    device: the cfg1 plate at h = 25 um, 8 uniform steps, against the reference's output."""
    z = np.load(GOLDEN / "mono_cfg1.npz")
    cfg = P.load_config(CONFIGS / "cfg1_m4.cfg")
    cfg.h_reference = float(z["h"])
    cfg.dt_reference = float(z["dt"])
    cfg.t_end = int(z["n_steps"]) * cfg.dt_reference
    stats = P.RunStats()
    traj = P.run_reference(cfg, stats=stats)
    assert traj.mesh.n_nodes == int(z["n_nodes"])
    assert traj.times == list(z["t"])
    assert stats.counters == json.loads(str(z["counters"]))
    s = int(z["stride"])
    TL = cfg.material.T_liquidus
    for k, T in enumerate(traj.values):
        assert rel(T[::s], z["sub"][k]) <= REL
        assert_mask(None, T, z["melt"][k], TL, True)
    assert rel(traj.values[-1], z["last"]) <= REL
    assert rel(traj.at_time(float(z["t"][int(z["n_steps"]) // 2])).values, z["mid"]) <= REL


def test_mass_norm_vs_reference_l2_norm():
    """metrics.l2_norm on the device (k_mass_norms) against the reference's fem.l2_norm."""
    z = np.load(GOLDEN / "metrics_cfg1.npz")
    for k in range(2):
        grid = _grid(z["norm_lo"][0], z["norm_hi"][0], z["norm_nc"][k], z["norm_off"][k])
        got = P.l2_norm(grid, z[f"norm_v{k}"])
        assert abs(got - z["norm_val"][k]) <= 1e-13 * z["norm_val"][k]


def test_error_metrics_vs_reference():
    """error_metrics of a 2-macro-step cfg1 two-level run against the monolithic reference
    (h = 25 um): every record's relative L2 error and the mean as the reference reports them."""
    z = np.load(GOLDEN / "metrics_cfg1.npz")
    cfg = P.load_config(CONFIGS / "cfg1_m4.cfg")
    n = int(z["n_macro"])
    log = P.RunLog()
    P.two_level_run(cfg, recorder=log.record, n_steps=n)
    cfg.t_end = n * cfg.dt_macro
    cfg.h_reference = float(z["h_ref"])
    cfg.dt_reference = cfg.dt_macro / cfg.micro_steps
    rep = P.error_metrics(log, P.run_reference(cfg))
    assert list(rep.kinds) == list(z["kinds"])
    np.testing.assert_allclose(rep.times, z["times"], rtol=0, atol=1e-15)
    np.testing.assert_allclose(rep.rel_l2, z["rel_l2"], rtol=1e-7, atol=1e-12)
    assert abs(rep.mean_rel_l2 - float(z["mean_rel_l2"])) <= 1e-7 * float(z["mean_rel_l2"])
    assert P.metrics.sawtooth_fraction(rep, cfg.micro_steps) == float(z["sawtooth"])


def test_transmission_load_vs_reference():
    """twolevel.transmission_load on the device (k_trans_entries + stable key sort + ordered
    segment sums) against the reference, kappa_g = 1.5 kappa_l, initial and translated box."""
    from paper_2110_12932_b200.twolevel import extract_interface, transmission_load
    z = np.load(GOLDEN / "transmission_cfg1.npz")
    cfg = P.load_config(CONFIGS / "cfg1_twoway.cfg")
    problem, lm = P.build_problem(cfg)
    assert not problem.one_way
    for k in range(2):
        mesh = lm if k == 0 else lm.translated(tuple(z[f"off{k}"]))
        np.testing.assert_allclose(mesh.box.lo, z["box_lo"] + z[f"off{k}"], rtol=0, atol=1e-15)
        gamma = extract_interface(mesh, problem.global_mesh)
        got = transmission_load(P.FieldState(mesh, z[f"v{k}"], 0.0), gamma, problem.global_mesh,
                                problem.mat_global, problem.mat_local)
        ref = z[f"load{k}"]
        assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()
    # temperature-dependent tables: jump = kappa_g(T_qp) - kappa_l(T_qp)
    zt = np.load(GOLDEN / "transmission_tdep.npz")
    cfg_t = P.load_config(CONFIGS / "cfg1_tdep_twoway.cfg")
    pt, lt = P.build_problem(cfg_t)
    gt = extract_interface(lt, pt.global_mesh)
    got_t = transmission_load(P.FieldState(lt, zt["v"], 0.0), gt, pt.global_mesh, pt.mat_global, pt.mat_local)
    assert np.abs(got_t - zt["load"]).max() <= 1e-12 * np.abs(zt["load"]).max()
    # run-to-run deterministic
    again = transmission_load(P.FieldState(mesh, z["v1"], 0.0), gamma, problem.global_mesh,
                              problem.mat_global, problem.mat_local)
    np.testing.assert_array_equal(again, got)


@pytest.mark.parametrize("name", ["cfg1_twoway", "cfg1_twoway_uniform", "cfg1_tdep", "cfg1_gsrc",
                                  "cfg1_gsrc_uniform", "cfg1_tdep_twoway", "cfg1_full", "cfg1_tdep_full"])
def test_two_way_coupled_run_vs_reference(name):
    """Two-way coupling (global_kappa_scale 1.5, omega 0.7, tol 1e-8): 4 macro steps whose
    correctors are the relaxed two_level_iterate fixed point, with relocations; counters
    (coupling iterations included), times, boxes, fields and melt masks as the reference's.
    The uniform variant (run_space) iterates every step to the fixed point.  cfg1_tdep: a
    temperature-dependent material with latent heat, convection and radiation (one-way,
    every solve a Picard loop over tl_vc_step_host passes, 194 passes in 2 macro steps).
    cfg1_gsrc(_uniform): the "gaussian" coarse source (runner.py:64-71; predictor beam at
    t0 + 0.75 dt), whose corrector re-solves both levels (multirate.py:156-161).
    cfg1_full / cfg1_tdep_full: coupling mode full, the overlap feedback load
    (twolevel.py:186-239) with constant and temperature-dependent tables."""
    z, cfg, rec, stats = _golden_run(name)
    assert stats.counters == json.loads(str(z["counters"]))
    TL = cfg.material.T_liquidus
    s = int(z["stride"])
    for k, (t, Tl, Tg, lo) in enumerate(rec):
        assert t == z["t"][k]
        np.testing.assert_array_equal(lo, z["box"][k])
        assert rel(Tg[::s], z["gsub"][k]) <= REL and rel(Tl[::s], z["lsub"][k]) <= REL
        assert_mask(None, Tg, z["gmelt"][k], TL, True)
        assert_mask(None, Tl, z["lmelt"][k], TL, True)
        if k in z["full_at"]:
            assert rel(Tg, z[f"g{k}"]) <= REL and rel(Tl, z[f"l{k}"]) <= REL


@pytest.mark.parametrize("name", ["tables", "latent", "full"])
def test_picard_step_vs_reference(name):
    """Temperature-dependent IN625 step on the device (tl_vc_step_host passes under the
    reference's Picard loop): tables only, + latent secant capacity, + convection and lagged
    radiation on the top face.  Same Picard pass count, 1e-9 relative L-inf, melt mask."""
    from .test_oracle_golden import picard_material
    z = np.load(GOLDEN / f"picard_{name}.npz")
    grid = P.build_structured_grid(P.Box(tuple(z["lo"]), tuple(z["hi"])), float(z["h"]))
    mat = picard_material(z)
    rad = bool(z["radiation"])
    bounds = P.BoundarySpec(bc=P.ThermalBC(float(z["h_conv"]), 0.8 if rad else 0.0, 293.0, 293.0),
                            robin_tags=(P.TOP,), radiation=rad,
                            dirichlet_nodes=grid.nodes_on(P.BOTTOM), dirichlet_values=293.0)
    beam = P.LaserBeam(200.0, 0.35, 5e-5, 5e-5, 0.8)
    stats = P.RunStats()
    stats.device_log = []
    out = P.step_backward_euler(P.FieldState(grid, z["T_old"], 0.0), float(z["dt"]), mat,
                                P.GaussianSource(beam, tuple(z["center"])), bounds,
                                P.SolverSettings(picard_tol=1e-8, linear_tol=1e-12, linear_solver="cg"),
                                latent=bool(z["latent"]), stats=stats)
    assert stats.counters["picard_iterations"] == int(z["picard"])
    # the reference's CG iterations of every Picard pass (k_vc_cg mirrors scipy's recurrences)
    assert [k for _, k in stats.device_log] == list(z["cg_iters"])
    assert rel(out.values, z["sol"]) <= REL
    TL = mat.T_liquidus
    assert_mask(None, out.values, z["sol"], TL)


def test_track3d_shipped_config_vs_reference(tmp_path):
    """The reference's shipped 3D single track (configs/track3d.cfg restates it): IN625
    tables with latent heat, convection + radiation, direct solver, 3 macro steps with
    relocations, 290 Picard passes.  The IN625 tables come from the golden file."""
    z = np.load(GOLDEN / "run_track3d.npz")
    rho, chi, Ts, Tl, S = (float(v) for v in z["mat_scalars"])
    lines = ["units K", f"rho {rho!r}", f"chi {chi!r}", f"T_solidus {Ts!r}", f"T_liquidus {Tl!r}", f"S {S!r}",
             "[conductivity]"] + [f"{float(a)!r} {float(b)!r}" for a, b in z["k_table"]] + ["[heat_capacity]"] + \
            [f"{float(a)!r} {float(b)!r}" for a, b in z["c_table"]]
    (tmp_path / "in625.mat").write_text("\n".join(lines) + "\n")
    (tmp_path / "track3d.cfg").write_text((CONFIGS / "track3d.cfg").read_text())
    cfg = P.load_config(tmp_path / "track3d.cfg")
    rec = []

    def recorder(kind, t, local, glob, iters):
        if kind in ("initial", "macro"):
            rec.append((t, local.values.copy(), glob.values.copy(), local.mesh.box.lo))

    state, stats = P.two_level_run(cfg, recorder=recorder)
    assert stats.counters == json.loads(str(z["counters"]))
    TL = cfg.material.T_liquidus
    s = int(z["stride"])
    for k, (t, Tl_, Tg, lo) in enumerate(rec):
        assert t == z["t"][k]
        np.testing.assert_array_equal(lo, z["box"][k])
        assert rel(Tg[::s], z["gsub"][k]) <= REL and rel(Tl_[::s], z["lsub"][k]) <= REL
        assert_mask(None, Tg, z["gmelt"][k], TL, True)
        assert_mask(None, Tl_, z["lmelt"][k], TL, True)
        if k in z["full_at"]:
            assert rel(Tg, z[f"g{k}"]) <= REL and rel(Tl_, z[f"l{k}"]) <= REL


def test_track3d_centerline_acceptance_criterion_6(tmp_path):
    """The shipped track_3d.cfg (configs/track3d.cfg, unchanged) through run_experiment in its
    own mode and in mode "reference", as the reference's acceptance criterion 6 does
    (tests/test_acceptance.py:74-84,222-238): the same output files, solve counters and
    centerline.csv rows as the reference (15.5 min there), and the criterion's quantities
    (peak error, pointwise error where T_ref >= T_s / 2, melting reached) as the reference's
    own files give them.  The centre line crosses the relocated local box: the fine field is
    sampled on a translated lattice (Mesh.interpolate, mesh.py:358-361)."""
    import csv
    import dataclasses
    from paper_2110_12932_b200.experiment import run_experiment
    gold = json.loads((GOLDEN / "track3d_centerline.json").read_text())
    z = np.load(GOLDEN / "run_track3d.npz")
    rho, chi, Ts, Tl, S = (float(v) for v in z["mat_scalars"])
    lines = ["units K", f"rho {rho!r}", f"chi {chi!r}", f"T_solidus {Ts!r}", f"T_liquidus {Tl!r}", f"S {S!r}",
             "[conductivity]"] + [f"{float(a)!r} {float(b)!r}" for a, b in z["k_table"]] + ["[heat_capacity]"] + \
            [f"{float(a)!r} {float(b)!r}" for a, b in z["c_table"]]
    (tmp_path / "in625.mat").write_text("\n".join(lines) + "\n")
    (tmp_path / "track3d.cfg").write_text((CONFIGS / "track3d.cfg").read_text())
    cfg = P.load_config(tmp_path / "track3d.cfg")
    prof = {}
    for tag, c in (("reference", dataclasses.replace(cfg, mode="reference")), ("two_level", cfg)):
        out = tmp_path / tag
        art = run_experiment(c, out)
        assert sorted(str(p.relative_to(out)) for p in out.rglob("*") if p.is_file()) == gold[tag]["files"]
        assert art.stats.counters == gold[tag]["counters"]
        with (out / "centerline.csv").open() as fh:
            rows = list(csv.reader(fh))
        assert rows[0] == gold[tag]["header"]
        got = np.array([[float(v) for v in r] for r in rows[1:]])
        want = np.array(gold[tag]["rows"])
        np.testing.assert_allclose(got[:, 0], want[:, 0], rtol=1e-12, atol=1e-15)
        np.testing.assert_allclose(got[:, 1], want[:, 1], rtol=1e-7)
        prof[tag] = got
    def criterion(ref, st):
        xr, Tr = ref[:, 0], ref[:, 1]
        Ts_ = np.interp(xr, st[:, 0], st[:, 1])
        hot = Tr >= 0.5 * cfg.material.T_solidus
        return (abs(Ts_.max() - Tr.max()) / Tr.max(), np.max(np.abs(Ts_[hot] - Tr[hot]) / Tr[hot]),
                bool(Tr.max() > cfg.material.T_liquidus))

    # the criterion's quantities from the device's files equal those from the reference's own
    # (its thresholds, 5 % / 10 %, are not met by the reference's numbers either: 7.2 % / 47 %)
    got = criterion(prof["reference"], prof["two_level"])
    want = criterion(np.array(gold["reference"]["rows"]), np.array(gold["two_level"]["rows"]))
    assert got[2] and want[2]
    assert got[0] == pytest.approx(want[0], rel=1e-5) and got[1] == pytest.approx(want[1], rel=1e-5)


@pytest.mark.parametrize("name", ["cfg1_compare", "cfg1_study"])
def test_experiment_modes_vs_reference(name, tmp_path):
    """runner.run_experiment (runner.py:270-440) in compare and convergence-study modes on the
    device: the same output files, solve counts, study pairs and errors.csv / study_matrix
    rows (relative L2 errors to 1e-7) as the reference."""
    import csv
    from paper_2110_12932_b200.experiment import run_experiment
    gold = json.loads((GOLDEN / "experiments.json").read_text())[name]
    art = run_experiment(P.load_config(CONFIGS / f"{name}.cfg"), tmp_path)
    files = sorted(str(p.relative_to(tmp_path)) for p in tmp_path.rglob("*") if p.is_file())
    assert files == gold["files"]
    for k, v in gold["summary"].items():
        if k == "mean_rel_l2":
            for kk, vv in v.items():
                assert abs(art.summary[k][kk] - vv) <= 1e-7 * vv
        elif k == "pairs":
            np.testing.assert_allclose(art.summary[k], v, rtol=1e-15)
        else:
            assert art.summary[k] == v, k
    for f, rows in gold["csv"].items():
        with (tmp_path / f).open() as fh:
            got = list(csv.reader(fh))
        assert got[0] == rows[0] and len(got) == len(rows)
        for a, b in zip(got[1:], rows[1:]):
            for x, y in zip(a, b):
                try:
                    fx, fy = float(x), float(y)
                except ValueError:
                    assert x == y
                    continue
                assert abs(fx - fy) <= 1e-7 * abs(fy) + 1e-12, (f, a, b)


def test_consistency_diagnostic_vs_reference():
    """twolevel.consistency_diagnostic (masked mass norms on the device) of the state after 2
    cfg1 macro steps against the monolithic reference at h = 25 um."""
    from paper_2110_12932_b200.twolevel import consistency_diagnostic
    gold = json.loads((GOLDEN / "consistency_cfg1.json").read_text())["norms"]
    cfg = P.load_config(CONFIGS / "cfg1_m4.cfg")
    state, _ = P.two_level_run(cfg, n_steps=2)
    cfg.t_end = 2 * cfg.dt_macro
    cfg.h_reference = 2.5e-5
    cfg.dt_reference = cfg.dt_macro / cfg.micro_steps
    traj = P.run_reference(cfg)
    problem, _ = P.build_problem(cfg)
    got = consistency_diagnostic(state, traj.state(len(traj) - 1), problem.global_mesh)
    for k in ("local", "overlap", "exterior"):
        assert abs(got[k] - gold[k]) <= 1e-6 * gold[k], (k, got[k], gold[k])


def test_deposit_integral_is_absorbed_power():
    """Energy consistency (tests/test_sources.py:99-115): the device deposit of one full
    swept interval carries P * eta = 179.2 W * 0.38 = 68.096 W (P1 partition of unity)."""
    from paper_2110_12932_b200.schedule import swept_samples
    beam = P.LaserBeam(179.2, 0.38, 8.5e-5, 5e-5, 0.8)
    grid = P.build_structured_grid(P.Box((0.0, 0.0, 0.0), (2.4e-3, 1.2e-3, 6e-4)), 5e-5)
    dt = 4e-4
    a = np.array([9e-4, 6e-4, 6e-4])
    pts, pw = swept_samples(beam, [(a, a + np.array([beam.speed * dt, 0.0, 0.0]))], dt)
    load = ops.deposit_load(grid, pts, pw)
    assert load.sum() == pytest.approx(68.096, rel=1e-12)


def test_transmission_of_linear_field_is_bottom_flux():
    """Known answer for the interface functional: T = z on the local grid has dT/dn = -1 on
    the bottom facets and 0 on the lateral ones, so the global load sums (partition of
    unity) to -(kappa_g - kappa_l) * Lx * Ly."""
    from paper_2110_12932_b200.twolevel import extract_interface, transmission_load
    cfg = P.load_config(CONFIGS / "cfg1_twoway.cfg")
    problem, lm = P.build_problem(cfg)
    z = lm.coords[:, 2]
    load = transmission_load(P.FieldState(lm, z.copy(), 0.0), extract_interface(lm, problem.global_mesh),
                             problem.global_mesh, problem.mat_global, problem.mat_local)
    jump = cfg.material.conductivity_table[0, 1] - cfg.material_local.conductivity_table[0, 1]
    lx, ly, _ = lm.box.lengths
    assert load.sum() == pytest.approx(-jump * lx * ly, rel=1e-12)


def test_zero_rhs_returns_dirichlet_values():
    """solve_linear returns zeros for ||b|| = 0 (fem.py:275-276) and re-imposes x_D = g: a
    cold plate (T_old = 0, no source, g = 0) stays exactly 0 on both device paths."""
    grid = P.build_structured_grid(P.Box((0.0, 0.0, 0.0), (5e-4, 4e-4, 3e-4)), 5e-5)
    mat = P.load_material(CONFIGS / "const.mat")
    bounds = P.BoundarySpec(bc=P.ThermalBC(0.0, 0.0, 293.0, 0.0), robin_tags=(P.TOP,), radiation=False,
                            dirichlet_nodes=grid.nodes_on(P.BOTTOM), dirichlet_values=0.0)
    st = P.FieldState(grid, np.zeros(grid.n_nodes), 0.0)
    out = P.step_backward_euler(st, 1e-5, mat, None, bounds, P.SolverSettings(linear_tol=1e-12, linear_solver="cg"))
    assert np.all(out.values == 0.0)
    conv = P.BoundarySpec(bc=P.ThermalBC(10.0, 0.0, 0.0, 0.0), robin_tags=(P.TOP,), radiation=False,
                          dirichlet_nodes=grid.nodes_on(P.BOTTOM), dirichlet_values=0.0)
    out2 = P.step_backward_euler(st, 1e-5, mat, None, conv, P.SolverSettings(linear_tol=1e-12, linear_solver="cg"))
    assert np.all(out2.values == 0.0)


def test_picard_nonconvergence_maps_to_reference_exception():
    """Too few Picard passes raise NonConvergence('Picard iteration', max_iter, inc) as
    fem.py:355 does (the latent golden case needs 6)."""
    from .test_oracle_golden import picard_material
    z = np.load(GOLDEN / "picard_latent.npz")
    grid = P.build_structured_grid(P.Box(tuple(z["lo"]), tuple(z["hi"])), float(z["h"]))
    bounds = P.BoundarySpec(bc=P.ThermalBC(0.0, 0.0, 293.0, 293.0), robin_tags=(P.TOP,), radiation=False,
                            dirichlet_nodes=grid.nodes_on(P.BOTTOM), dirichlet_values=293.0)
    with pytest.raises(NonConvergence) as exc:
        P.step_backward_euler(P.FieldState(grid, z["T_old"], 0.0), float(z["dt"]), picard_material(z),
                              P.GaussianSource(P.LaserBeam(200.0, 0.35, 5e-5, 5e-5, 0.8), tuple(z["center"])),
                              bounds, P.SolverSettings(picard_tol=1e-8, picard_max_iter=2, linear_tol=1e-12,
                                                       linear_solver="cg"), latent=True)
    assert exc.value.iterations == 2 and "Picard" in str(exc.value)


def test_reference_piecewise_material_and_local_latent_vs_reference():
    """run_reference (runner.py:126-163) with distinct coarse/fine conductivities over a fixed
    local box (PiecewiseMaterial) and latent heat only inside it (latent_reference local),
    temperature-dependent tables, convection + radiation: 4 steps, 28 Picard passes."""
    z = np.load(GOLDEN / "ref_piecewise.npz")
    cfg = P.load_config(CONFIGS / "cfg1_ref_piecewise.cfg")
    stats = P.RunStats()
    traj = P.run_reference(cfg, stats=stats)
    assert stats.counters == json.loads(str(z["counters"]))
    assert traj.times == list(z["t"])
    TL = cfg.material.T_liquidus
    for k, T in enumerate(traj.values):
        assert rel(T, z["fields"][k]) <= REL
        assert_mask(None, T, z["melt"][k], TL, True)


def test_cli_compare_writes_reference_outputs(tmp_path):
    """python -m paper_2110_12932_b200 compare <cfg> --out <dir> (lpbfsim/cli.py) on the GPU."""
    import subprocess
    import sys
    out = tmp_path / "cmp"
    r = subprocess.run([sys.executable, "-m", "paper_2110_12932_b200", "compare", str(CONFIGS / "cfg1_compare.cfg"),
                        "--out", str(out)], cwd=str(ROOT), capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    assert "mode: compare" in r.stdout
    files = sorted(str(p.relative_to(out)) for p in out.rglob("*") if p.is_file())
    assert files == json.loads((GOLDEN / "experiments.json").read_text())["cfg1_compare"]["files"]


def test_two_level_mode_writes_macro_snapshots(tmp_path):
    """run_experiment in two-level-spacetime mode with snapshots 'macro' (runner.py:216-233):
    one global_ and one local_ VTK file per initial / macro record."""
    from paper_2110_12932_b200.experiment import run_experiment
    text = (CONFIGS / "cfg1_m4.cfg").read_text().replace("t_end 2 ms", "t_end 0.05 ms").replace(
        "snapshots none", "snapshots macro")
    (tmp_path / "c.cfg").write_text(text)
    (tmp_path / "const.mat").write_text((CONFIGS / "const.mat").read_text())
    art = run_experiment(P.load_config(tmp_path / "c.cfg"), tmp_path / "out")
    names = sorted(p.name for p in (tmp_path / "out" / "vtk").iterdir())
    times = [0.0, 2.5e-5, 5e-5]
    assert names == sorted([f"global_{t:.6e}.vtk" for t in times] + [f"local_{t:.6e}.vtk" for t in times])
    last = art.log.of_kind("macro")[-1]
    vals = (tmp_path / "out" / "vtk" / f"local_{5e-5:.6e}.vtk").read_text().split("LOOKUP_TABLE default\n")[1].split()
    np.testing.assert_allclose(np.array(vals, dtype=float), last.local.values, rtol=1e-9)


def test_snapshot_decimation_on_device():
    """Snapshot decimation (runner.py:216-233): a recorder that declares
    which micro fields it reads (DecimatingRecorder.wants) gets exactly those, the others
    arrive with local=None and are neither snapshotted on the device nor copied to the host;
    every record's kind and time, the macro fields and the final state are those of the
    full recorder, bit for bit."""
    from paper_2110_12932_b200 import multirate as MR
    from paper_2110_12932_b200.experiment import DecimatingRecorder
    from paper_2110_12932_b200.metrics import RunLog
    cfg = P.load_config(CONFIGS / "cfg1_m4.cfg")

    def run(every):
        MR.release_device_runs()
        log = RunLog()
        rec = log.record if every is None else DecimatingRecorder(log, every)
        state, _ = P.two_level_run(cfg, recorder=rec, n_steps=6)
        d2h = sum(r.d2h_bytes for r in MR._POOL.values())
        return log, state, d2h

    full, sf, b_full = run(None)
    for every in (0, 3):
        log, s, b = run(every)
        assert [(r.kind, r.time) for r in log.records] == [(r.kind, r.time) for r in full.records]
        seen = 0
        for a, r in zip(log.records, full.records):
            if a.kind == "micro":
                seen += 1
                if every and seen % every == 0:
                    np.testing.assert_array_equal(a.local.values, r.local.values)
                else:
                    assert a.local is None
            elif a.kind in ("initial", "macro"):
                np.testing.assert_array_equal(a.local.values, r.local.values)
                np.testing.assert_array_equal(a.global_field.values, r.global_field.values)
        np.testing.assert_array_equal(s.local_field.values, sf.local_field.values)
        np.testing.assert_array_equal(s.global_field.values, sf.global_field.values)
        assert b < b_full
    n_l = full.records[0].local.mesh.n_nodes
    assert b_full - run(0)[2] >= 6 * 4 * n_l * 8          # 4 micro fields per macro step not copied


def test_compare3d_shipped_config_vs_reference(tmp_path):
    """The reference's shipped multi-track timing comparison (src/configs/compare_3d.cfg,
    restated as configs/compare3d.cfg): compare mode, IN625 tables with latent heat,
    convection + radiation, 10 alternating tracks with a moving local box, the reference's
    default DIRECT linear solver (fem.py:277-281), which the device serves with CG at rtol
    1e-14.  Same output files, solve counts of both schemes and RunStats counters (1765
    Picard passes); the multirate run's final fields to 1e-9 with bit-exact melt masks."""
    from paper_2110_12932_b200.experiment import run_experiment
    z = np.load(GOLDEN / "compare3d.npz")
    rho, chi, Ts, Tl, S = (float(v) for v in z["mat_scalars"])
    lines = ["units K", f"rho {rho!r}", f"chi {chi!r}", f"T_solidus {Ts!r}", f"T_liquidus {Tl!r}", f"S {S!r}",
             "[conductivity]"] + [f"{float(a)!r} {float(b)!r}" for a, b in z["k_table"]] + ["[heat_capacity]"] + \
            [f"{float(a)!r} {float(b)!r}" for a, b in z["c_table"]]
    (tmp_path / "in625.mat").write_text("\n".join(lines) + "\n")
    (tmp_path / "compare3d.cfg").write_text((CONFIGS / "compare3d.cfg").read_text())
    cfg = P.load_config(tmp_path / "compare3d.cfg")
    assert cfg.solver.linear_solver == "direct"
    out = tmp_path / "out"
    art = run_experiment(cfg, out)
    files = sorted(str(p.relative_to(out)) for p in out.rglob("*") if p.is_file())
    assert files == json.loads(str(z["files"]))
    for k, v in json.loads(str(z["summary"])).items():
        assert art.summary[k] == v, k
    assert art.stats.counters == json.loads(str(z["counters"]))
    final = art.log.of_kind("macro")[-1]
    assert final.time == float(z["t"])
    np.testing.assert_array_equal(final.local.mesh.box.lo, z["box"])
    assert rel(final.local.values, z["local"]) <= REL and rel(final.global_field.values, z["glob"]) <= REL
    TL = cfg.material.T_liquidus
    assert_mask(None, final.local.values, z["local"], TL)
    assert_mask(None, final.global_field.values, z["glob"], TL)

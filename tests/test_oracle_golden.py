"""Pin the CPU oracle to golden vectors produced by the unmodified reference.

tests/golden/make_golden.py ran lpbfsim 0.1.0 (numpy 2.3.5, scipy 1.18.1) and
stored its outputs; here the oracle must reproduce them: operator/RHS/solve at
rounding level with identical CG iteration counts, interpolation and deposit,
and whole two-level runs (cfg1 multirate m=4 and uniform, all 80 macro steps;
cfg2 first 2 macro steps).
"""

import json
from pathlib import Path

import numpy as np
import pytest

import paper_2110_12932_b200 as P
from oracle import assembly, kuhn
from oracle.pcg import solve_constrained
from oracle.twolevel import OracleRun

from .conftest import CONFIGS, GOLDEN

OP_CASES = ["aniso_local", "aniso_global", "cfg1_local", "cfg1_global"]


def _op(name):
    z = np.load(GOLDEN / f"op_{name}.npz")
    G = kuhn.KuhnGrid(z["lo"], z["hi"], z["ncells"])
    D = np.zeros(G.n_nodes, bool)
    D[z["dnodes"]] = True
    g = np.zeros(G.n_nodes)
    g[z["dnodes"]] = z["dvals"]
    local = str(z["kind"]) == "local"
    beam = P.LaserBeam(200.0, 0.35, 5e-5, 5e-5, 0.8)
    return z, G, D, g, local, beam


@pytest.mark.parametrize("name", OP_CASES)
def test_stencil_operator_rhs_solve(name):
    z, G, D, g, local, beam = _op(name)
    op = kuhn.StencilOperator(G, 9.8, 8440 * 410.0, float(z["dt"]), D.reshape(G.shape))
    Ax = op.apply(z["x"])
    assert np.abs(Ax - z["Ax"]).max() <= 1e-14 * np.abs(z["Ax"]).max()
    assert np.abs(op.diag_c.ravel() - z["diag"]).max() <= 1e-14 * np.abs(z["diag"]).max()
    load = kuhn.gaussian_load(G, beam, z["center"]) if local else z["extra"]
    b = op.rhs(z["T_old"], load, g)
    assert np.abs(b - z["b"]).max() <= 1e-14 * np.abs(z["b"]).max()
    x, its, res = solve_constrained(op, b, g, 1e-12)
    assert its == int(z["cg_iters"])
    assert np.abs(x - z["sol"]).max() <= 1e-13 * np.abs(z["sol"]).max()
    # CG vs the reference's own direct solve: the oracle's noise floor
    assert np.abs(x - z["direct"]).max() <= 1e-9 * np.abs(z["direct"]).max()


@pytest.mark.parametrize("name", OP_CASES)
def test_literal_assembly_is_bitwise(name):
    z, G, D, g, local, beam = _op(name)
    src = (beam, z["center"]) if local else None
    x, its = assembly.step(G, 9.8, 8440 * 410.0, float(z["dt"]), D, z["T_old"], src,
                           None if local else z["extra"], g, 1e-12)
    assert its == int(z["cg_iters"])
    # bitwise with single-threaded BLAS (OPENBLAS_NUM_THREADS=1); threaded einsum reorders sums
    assert np.abs(x - z["sol"]).max() <= 2e-15 * np.abs(z["sol"]).max()


def test_interpolation():
    z = np.load(GOLDEN / "interp.npz")
    box = P.Box(tuple(z["lo"]), tuple(z["hi"]))
    G = kuhn.KuhnGrid(box.lo, box.hi, P.control.structured_ncells(box, float(z["h"])))
    out = kuhn.interpolate(G, z["vals"], z["pts"])
    assert np.abs(out - z["out"]).max() <= 1e-14 * np.abs(z["out"]).max()


def test_deposit_and_samples():
    d = json.loads((GOLDEN / "deposit.json").read_text())
    box = P.Box(tuple(d["lo"]), tuple(d["hi"]))
    G = kuhn.KuhnGrid(box.lo, box.hi, P.control.structured_ncells(box, d["h"]))
    beam = P.LaserBeam(*d["beam"])
    p = d["path"]
    path = P.build_alternating_path(p["n"], p["L"], p["hatch"], p["v"], p["origin"])
    assert [c["npieces"] for c in d["cases"]] == [1, 2, 2, 1]
    for c in d["cases"]:
        pieces = path.swept_pieces(c["t0"], c["t1"])
        pts, pw = kuhn.swept_samples(beam, pieces, c["t1"] - c["t0"])
        np.testing.assert_array_equal(pts, np.array(c["pts"]).reshape(-1, 3))
        np.testing.assert_array_equal(pw, np.array(c["pw"]))
        load = kuhn.deposit_load(G, pts, pw)
        nz = np.nonzero(load)[0]
        np.testing.assert_array_equal(nz, c["idx"])
        assert np.abs(load[nz] - c["val"]).max() <= 1e-13 * np.abs(c["val"]).max()
        assert load.sum() == pytest.approx(c["total"], rel=1e-13)


def test_gaussian_known_answers():
    d = json.loads((GOLDEN / "gaussian.json").read_text())
    beam = P.LaserBeam(*d["beam"])
    assert beam.gaussian_peak == d["peak"]
    assert beam.gaussian_peak == pytest.approx(3.12e14, rel=5e-3)      # tests/test_sources.py:53
    vals = P.GaussianSource(beam, tuple(d["center"]))(np.array(d["pts"]))
    np.testing.assert_allclose(vals, d["vals"], rtol=1e-14)


def _check_run(name, n_steps, full_tol=1e-12):
    z = np.load(GOLDEN / f"run_{name}.npz")
    cfg = P.load_config(CONFIGS / f"{name}.cfg")
    run = OracleRun(cfg)
    rec = []
    run_fn = run.run_spacetime if cfg.mode == "two-level-spacetime" else run.run_space
    run_fn(n_steps=n_steps, recorder=lambda kind, t, Tl, Tg, pl: rec.append((t, Tl, Tg, pl.box.lo)))
    assert len(rec) == len(z["t"])
    its = [i for _, i in run.iterations]
    assert its == z["cg_iters"].tolist()
    TL = cfg.material.T_liquidus
    s = int(z["stride"])
    for k, (t, Tl, Tg, lo) in enumerate(rec):
        assert t == z["t"][k]
        np.testing.assert_array_equal(lo, z["box"][k])
        for sub, ref in ((Tg[::s], z["gsub"][k]), (Tl[::s], z["lsub"][k])):
            assert np.abs(sub - ref).max() <= full_tol * np.abs(ref).max()
        np.testing.assert_array_equal(np.packbits(Tg > TL), z["gmelt"][k])
        np.testing.assert_array_equal(np.packbits(Tl > TL), z["lmelt"][k])
        if k in z["full_at"]:
            g, l = z[f"g{k}"], z[f"l{k}"]
            assert np.abs(Tg - g).max() <= full_tol * np.abs(g).max()
            assert np.abs(Tl - l).max() <= full_tol * np.abs(l).max()
    return run


def test_run_cfg1_multirate_all_steps():
    run = _check_run("cfg1_m4", None)
    assert run.counters["relocations"] == 79


def test_run_cfg1_uniform_all_steps():
    _check_run("cfg1_uniform", None)


@pytest.mark.slow
def test_run_cfg2_first_steps():
    _check_run("cfg2", 2)


@pytest.mark.parametrize("name", OP_CASES)
def test_chronopoulos_gear_matches_scipy_cg(name):
    """The one-reduction recurrences the device's default resident kernel uses reach the
    reference's solution with the reference's iteration count (tolerance 1e-13 vs scipy)."""
    from oracle.pcg import cg_chronopoulos_gear
    z, G, D, g, local, beam = _op(name)
    op = kuhn.StencilOperator(G, 9.8, 8440 * 410.0, float(z["dt"]), D.reshape(G.shape))
    b = z["b"]
    x, info, its = cg_chronopoulos_gear(op.apply, b, op.inv_diag(), 1e-12, 20 * b.size)
    assert info == 0 and its == int(z["cg_iters"])
    x[D] = b[D]
    assert np.abs(x - z["sol"]).max() <= 1e-13 * np.abs(z["sol"]).max()


@pytest.mark.parametrize("name", OP_CASES)
def test_forward_edge_pAp_identity(name):
    """The streaming sweep A (tl_stream.cuh) forms the CG denominator p.A_c p from each
    node and its three forward edges: sum_p d_p p_p^2 - 2 sum_{edges, both ends free}
    c_e p_lo p_hi (A_c is symmetric after the symmetric Dirichlet elimination, identity
    rows give p_p^2).  Check the identity against p.(A_c p) on the golden operators."""
    z, G, D, g, local, beam = _op(name)
    op = kuhn.StencilOperator(G, 9.8, 8440 * 410.0, float(z["dt"]), D.reshape(G.shape))
    rng = np.random.default_rng(7)
    p = rng.standard_normal(G.n_nodes)
    ref = float(p @ op.apply(p))
    Pg = p.reshape(G.shape)
    free = ~op.D
    fwd = float(np.sum(op.diag_c * Pg * Pg))
    for a in range(3):
        lo, hi = kuhn._edge_slices(a)
        both = free[lo] & free[hi]
        fwd -= 2.0 * float(np.sum(np.where(both, op.c[a] * Pg[lo] * Pg[hi], 0.0)))
    assert abs(fwd - ref) <= 1e-13 * abs(ref)


def test_oracle_monolithic_reference_vs_golden():
    """Monolithic fine-grid reference (runner.run_reference, fem.solve_monolithic) on the cfg1
    plate at h = 25 um, 8 steps: the oracle against the reference's own output."""
    z = np.load(GOLDEN / "mono_cfg1.npz")
    cfg = P.load_config(CONFIGS / "cfg1_m4.cfg")
    orc = OracleRun(cfg)
    times, fields = orc.run_reference(h=float(z["h"]), dt=float(z["dt"]), n_steps=int(z["n_steps"]))
    assert times == list(z["t"])
    s = int(z["stride"])
    TL = cfg.material.T_liquidus
    for k, T in enumerate(fields):
        assert np.abs(T[::s] - z["sub"][k]).max() / np.abs(z["sub"][k]).max() <= 1e-12
        np.testing.assert_array_equal(np.packbits(T > TL), z["melt"][k])
    assert np.abs(fields[-1] - z["last"]).max() / z["last"].max() <= 1e-12
    assert [k for _, k in orc.iterations] == list(z["cg_iters"])


def test_oracle_mass_norm_vs_reference_l2_norm():
    """fem.l2_norm (P1 mass matrix, lpbfsim/fem.py:434-446) on an anisotropic mesh and its
    translate: the per-tet restatement the device kernel k_mass_norms follows."""
    z = np.load(GOLDEN / "metrics_cfg1.npz")
    for k in range(2):
        g = kuhn.KuhnGrid(z["norm_lo"][0], z["norm_hi"][0], z["norm_nc"][k], z["norm_off"][k])
        v = z[f"norm_v{k}"]
        assert abs(np.sqrt(kuhn.mass_norm2(g, v)) - z["norm_val"][k]) <= 1e-13 * z["norm_val"][k]


def test_oracle_transmission_load_vs_reference():
    """twolevel.transmission_load (kappa_g = 1.5 kappa_l) on random local fields, initial and
    translated local box: the oracle's structured restatement against the reference."""
    z = np.load(GOLDEN / "transmission_cfg1.npz")
    cfg = P.load_config(CONFIGS / "cfg1_twoway.cfg")
    orc = OracleRun(cfg)
    jump = cfg.material.conductivity_table[0, 1] - cfg.material_local.conductivity_table[0, 1]
    assert jump != 0.0
    for k in range(2):
        L = kuhn.KuhnGrid(z["box_lo"], z["box_hi"], z["ncells"], z[f"off{k}"])
        got = kuhn.transmission_load(orc.G, L, z[f"v{k}"], jump)
        ref = z[f"load{k}"]
        np.testing.assert_array_equal(np.nonzero(np.abs(got) > 1e-14 * np.abs(ref).max())[0],
                                      np.nonzero(np.abs(ref) > 1e-14 * np.abs(ref).max())[0])
        assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()


def picard_material(z):
    """The reference's IN625 material (tables in K, chi already 0 for the no-latent case)."""
    rho, chi, Ts, Tl, S = (float(v) for v in z["mat_scalars"])
    return P.Material(np.array(z["k_table"]), np.array(z["c_table"]), rho, chi, Ts, Tl, S)


@pytest.mark.parametrize("name", ["tables", "latent", "full"])
def test_oracle_picard_step_vs_reference(name):
    """Temperature-dependent IN625 step (Picard, latent secant, lagged radiation): the
    stencil restatement (oracle/varcoef.py) against fem.step_backward_euler."""
    from oracle import varcoef
    z = np.load(GOLDEN / f"picard_{name}.npz")
    G = kuhn.KuhnGrid(z["lo"], z["hi"], np.round((z["hi"] - z["lo"]) / z["h"]).astype(int))
    mat = picard_material(z)
    beam = P.LaserBeam(200.0, 0.35, 5e-5, 5e-5, 0.8)
    src = P.GaussianSource(beam, tuple(z["center"]))
    rad = bool(z["radiation"])
    robin = (float(z["h_conv"]), 5.670374419e-8 * 0.8 if rad else 0.0, 293.0) if rad or z["h_conv"] > 0 else None
    dmask = G.bottom_mask().ravel()
    g = np.full(G.n_nodes, 293.0)
    x, npic, cg = varcoef.step(G, mat, z["T_old"], float(z["dt"]), src, dmask, g, bool(z["latent"]), robin)
    assert npic == int(z["picard"])
    assert cg == list(z["cg_iters"])
    assert np.abs(x - z["sol"]).max() / np.abs(z["sol"]).max() <= 1e-12


@pytest.mark.parametrize("name", ["tables", "full"])
def test_oracle_2d_picard_step_vs_reference(name):
    """2D (P1 triangles): the 5-point stencil restatement
    (oracle/tri2d.py) against the reference's fem.step_backward_euler on the shipped 2D plate
    (IN625 tables, convection / lagged radiation on the top edge, 2D Gaussian beam)."""
    from oracle import tri2d
    z = np.load(GOLDEN / f"picard2d_{name}.npz")
    G = tri2d.Grid2D(z["lo"], z["hi"], np.round((z["hi"] - z["lo"]) / z["h"]).astype(int))
    mat = picard_material(z)
    pw, eta, r, d = (float(v) for v in z["beam"])
    src = lambda p: tri2d.gaussian2d((pw * eta, r, d, z["center"]), p)      # noqa: E731
    rad = bool(z["radiation"])
    robin = (float(z["h_conv"]), 5.670374419e-8 * 0.8 if rad else 0.0, 298.15)
    dmask = np.zeros(G.n_nodes, dtype=bool)
    dmask[:G.NX] = True                                  # bottom edge y = lo
    g = np.full(G.n_nodes, 298.15)
    x, npic, cg = tri2d.step(G, mat, z["T_old"], float(z["dt"]), src, dmask, g, bool(z["latent"]), robin)
    assert npic == int(z["picard"])
    assert cg == list(z["cg_iters"])
    assert np.abs(x - z["sol"]).max() / np.abs(z["sol"]).max() <= 1e-12
    assert np.sqrt(tri2d.mass_norm2(G, x)) == pytest.approx(float(z["l2"]), rel=1e-12)


def test_oracle_2d_interpolation_vs_reference():
    """Mesh.interpolate on the triangle lattice, incl. lattice nodes and cell diagonals."""
    from oracle import tri2d
    z = np.load(GOLDEN / "interp2d.npz")
    G = tri2d.Grid2D(z["lo"], z["hi"], np.round((z["hi"] - z["lo"]) / z["h"]).astype(int))
    got = tri2d.interpolate(G, z["values"], z["points"])
    assert np.abs(got - z["out"]).max() <= 1e-13 * np.abs(z["out"]).max()
    assert np.sqrt(tri2d.mass_norm2(G, z["values"])) == pytest.approx(float(z["l2"]), rel=1e-13)


def test_structured_grid_2d_matches_reference_layout():
    """StructuredGrid in 2D: node order, boundary tags with y vertical (mesh.py:206-209), the
    interface node set and the two triangles per cell of the reference's mesh."""
    g = P.build_structured_grid(P.Box((0.0, 0.0), (5e-3, 1e-3)), 6.25e-5)
    assert (g.dim, g.n_nodes, g.n_elems) == (2, 81 * 17, 2 * 80 * 16)
    from paper_2110_12932_b200.grid import BOTTOM, LATERAL, TOP
    np.testing.assert_array_equal(g.nodes_on(BOTTOM), np.arange(81))
    np.testing.assert_array_equal(g.nodes_on(TOP), 16 * 81 + np.arange(81))
    np.testing.assert_array_equal(g.nodes_on(LATERAL), np.sort(np.r_[81 * np.arange(17), 81 * np.arange(17) + 80]))
    assert g.gamma_mask().sum() == 81 + 2 * 16
    np.testing.assert_array_equal(g.elems[:4], [[0, 1, 82], [0, 82, 81], [1, 2, 83], [1, 83, 82]])
    z = np.load(GOLDEN / "interp2d.npz")
    assert g.coords.shape == (81 * 17, 2) and g.coords[82].tolist() == [6.25e-5, 6.25e-5]
    d = g.desc()
    assert list(d.ncells) == [80, 16, 0]


def test_interface_measure_3d():
    """tests/test_mesh.py:185-189: lateral + bottom facet area of the interface."""
    from paper_2110_12932_b200.twolevel import extract_interface
    lm = P.build_structured_grid(P.Box((0, 0, 0), (1.2, 0.5, 0.1)), 0.05)
    gm = P.build_structured_grid(P.Box((-1, -1, -0.9), (3, 2, 0.1)), 0.2)
    g = extract_interface(lm, gm)
    assert g.measure == pytest.approx(1.2 * 0.5 + 2 * (1.2 * 0.1 + 0.5 * 0.1), rel=1e-10)


def test_strict_paper_constant():
    """load_config(strict_paper=True) (lpbfsim/config.py:285-286): the printed Stefan-Boltzmann
    constant replaces the configured one."""
    assert P.load_config(CONFIGS / "cfg1_tdep.cfg", strict_paper=True).bc.sigma_sb == 5.87e-8
    assert P.load_config(CONFIGS / "cfg1_tdep.cfg").bc.sigma_sb == 5.670374419e-8


@pytest.mark.skipif(not Path("/root/reference/pkg/src/lpbfsim").exists(),
                    reason="the reference package is only present in the build container")
@pytest.mark.parametrize("name", ["cfg1_m4", "cfg2", "cfg1_twoway", "cfg1_tdep"])
def test_reference_experiment_config_through_convert_config(name):
    """the reference's own ExperimentConfig (lpbfsim.config.load_config) goes
    through runner.convert_config / build_problem (lpbfsim/runner.py:51-113) and gives the same
    device problem as this package's loader: grids, materials, beam, BCs, path, policy,
    solver and coupling settings, schedule."""
    import sys
    sys.path.insert(0, "/root/reference/pkg/src")
    try:
        from lpbfsim.config import load_config as ref_load
    finally:
        sys.path.pop(0)
    from paper_2110_12932_b200.runner import convert_config
    ref_cfg = ref_load(CONFIGS / f"{name}.cfg")
    a, b = convert_config(ref_cfg), convert_config(P.load_config(CONFIGS / f"{name}.cfg"))
    assert a.keys() == b.keys()
    for k in a:
        va, vb = a[k], b[k]
        if k in ("material", "material_local"):
            np.testing.assert_array_equal(va.conductivity_table, vb.conductivity_table)
            np.testing.assert_array_equal(va.heat_capacity_table, vb.heat_capacity_table)
            assert (va.rho, va.chi, va.T_solidus, va.T_liquidus, va.S) == (vb.rho, vb.chi, vb.T_solidus, vb.T_liquidus, vb.S)
        elif k == "path":
            assert [(s.start, s.end, s.speed, s.t_start) for s in va.segments] == \
                   [(s.start, s.end, s.speed, s.t_start) for s in vb.segments]
        elif k == "policy":
            assert (va is None) == (vb is None)
            if va is not None:
                assert (tuple(va.box_size), va.laser_fraction) == (tuple(vb.box_size), vb.laser_fraction)
        else:
            assert va == vb, k
    pa, la = P.build_problem(ref_cfg)
    pb, lb = P.build_problem(P.load_config(CONFIGS / f"{name}.cfg"))
    assert pa.global_mesh.same_lattice(pb.global_mesh) and la.same_lattice(lb)
    assert (pa.one_way, pa.interval_source, pa.mode) == (pb.one_way, pb.interval_source, pb.mode)

"""Step-level fields kept on the device (two-way and temperature-
dependent runs go through ``two_level_iterate`` / the Picard step, one C-ABI call per solve).

Every field argument of the ``*_host`` entry points takes a host or a device pointer; the
Python layer leaves each solve's result in a ``DeviceVector`` (``DeviceBackedFieldState``),
gives Dirichlet data as node lists and reads the trace at the interface nodes only, so a
coupled step moves O(interface) bytes over PCIe instead of tens of bytes per node.  The
results must be bitwise those of the host-buffer path (``TLGPU_DEVICE_FIELDS=0``), which the
golden tests pin to the reference.
"""

from pathlib import Path

import numpy as np
import pytest

import paper_2110_12932_b200 as P
from paper_2110_12932_b200 import _native as N, ops

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
CONFIGS = ROOT / "configs"


def _run(cfg_path, n_steps, monkeypatch, device_fields):
    monkeypatch.setenv("TLGPU_DEVICE_FIELDS", "1" if device_fields else "0")
    cfg = P.load_config(cfg_path)
    N.host_traffic(reset=True)
    state, stats = P.two_level_run(cfg, n_steps=n_steps)
    traffic = N.host_traffic()                       # before the fields are read back
    return state, stats, traffic


@pytest.mark.parametrize("name,steps", [("cfg1_tdep_twoway", 2), ("cfg1_full", 2), ("cfg1_twoway_uniform", 3),
                                        ("run2d", 2)])
def test_device_backed_fields_match_host_path_and_cut_pcie_traffic(name, steps, monkeypatch, tmp_path):
    """Two-way / full-mode / temperature-dependent / 2D runs through the step-level drivers:
    the same counters and bitwise the same fields with the fields left on the device, and a
    fraction of the host-buffer path's PCIe bytes."""
    path = CONFIGS / f"{name}.cfg"
    if name == "run2d":                              # its IN625 tables come from the golden file
        from .test_gpu_2d import GOLDEN, _write_material
        _write_material(np.load(GOLDEN / "run_run2d.npz"), tmp_path / "in625.mat")
        path = tmp_path / "run2d.cfg"
        path.write_text((CONFIGS / "run2d.cfg").read_text())
    dev_state, dev_stats, dev_tr = _run(path, steps, monkeypatch, True)
    host_state, host_stats, host_tr = _run(path, steps, monkeypatch, False)
    assert dev_stats.counters == host_stats.counters
    assert isinstance(dev_state.local_field, P.fem.DeviceBackedFieldState)
    assert not isinstance(host_state.local_field, P.fem.DeviceBackedFieldState)
    np.testing.assert_array_equal(dev_state.global_field.values, host_state.global_field.values)
    np.testing.assert_array_equal(dev_state.local_field.values, host_state.local_field.values)
    np.testing.assert_array_equal(dev_state.trace, host_state.trace)
    # what still crosses is O(interface): Dirichlet node lists and values, traces, the first
    # upload of the initial field (on these 35k-node grids the interface is 15 % of the nodes)
    assert sum(dev_tr) <= 0.25 * sum(host_tr), (dev_tr, host_tr)


def test_trace_at_nodes_is_the_dense_interpolation_at_those_nodes():
    """tl_interpolate_nodes_host against tl_interpolate_host(gamma_only) (3D and 2D), from a
    host array and from a device vector."""
    rng = np.random.default_rng(5)
    for lo, hi, h, llo, lhi, lh in [((0, 0, 0), (2e-3, 2e-3, 1e-3), 1e-4, (4e-4, 4e-4, 6e-4), (1.2e-3, 1.2e-3, 1e-3), 5e-5),
                                    ((0, 0), (5e-3, 1e-3), 6.25e-5, (2.5e-4, 6.25e-4), (4.75e-3, 1e-3), 3.125e-5)]:
        grid = P.build_structured_grid(P.Box(lo, hi), h)
        local = P.build_structured_grid(P.Box(llo, lhi), lh)
        v = rng.uniform(300.0, 2000.0, grid.n_nodes)
        nodes = local.gamma_nodes()
        dense = ops.interpolate_to_grid(grid, v, local, gamma_only=True)[nodes]
        np.testing.assert_array_equal(ops.interpolate_at_nodes(grid, v, local, nodes), dense)
        dv = N.DeviceVector.from_host(v)
        N.host_traffic(reset=True)
        np.testing.assert_array_equal(ops.interpolate_at_nodes(grid, dv, local, nodes), dense)
        h2d, d2h = N.host_traffic()
        assert h2d == 4 * nodes.size and d2h == 8 * nodes.size      # node ids up, values down
        full = ops.interpolate_to_grid(grid, dv, local, on_device=True)
        assert isinstance(full, N.DeviceVector)
        np.testing.assert_array_equal(full.to_host(), ops.interpolate_to_grid(grid, v, local))


def test_device_vectors_spill_to_host_over_budget(monkeypatch):
    """The live-vector budget: older vectors keep only their host copy and still work as
    inputs (passed as host pointers)."""
    monkeypatch.setenv("TLGPU_DEVICE_FIELDS_GB", str(3 * 8 * 4096 / 2**30))
    rng = np.random.default_rng(6)
    data = [rng.uniform(0.0, 1.0, 4096) for _ in range(5)]
    vecs = [N.DeviceVector.from_host(a) for a in data]
    assert [v.on_device for v in vecs] == [False, False, True, True, True]
    for v, a in zip(vecs, data):
        np.testing.assert_array_equal(v.to_host(), a)
    s = ops.add_loads(vecs[0], vecs[4])              # spilled + resident
    assert isinstance(s, N.DeviceVector)
    np.testing.assert_array_equal(s.to_host(), data[0] + data[4])
    assert ops.add_loads(None, vecs[1]) is vecs[1]
    np.testing.assert_array_equal(ops.add_loads(data[2], data[3]), data[2] + data[3])


def test_picard_step_from_device_field_uploads_only_boundary_data(monkeypatch):
    """A temperature-dependent step whose T_old already lives on the device: the call's
    uploads are the Dirichlet node list and values (12 bytes per Dirichlet node) and the
    material tables, nothing per node; repeated Dirichlet nodes keep the last value."""
    monkeypatch.setenv("TLGPU_DEVICE_FIELDS", "1")
    from .test_oracle_golden import picard_material
    z = np.load(ROOT / "tests" / "golden" / "picard_full.npz")
    grid = P.build_structured_grid(P.Box(tuple(z["lo"]), tuple(z["hi"])), float(z["h"]))
    mat = picard_material(z)
    nodes = grid.nodes_on(P.BOTTOM)
    bounds = P.BoundarySpec(bc=P.ThermalBC(float(z["h_conv"]), 0.8, 293.0, 293.0), robin_tags=(P.TOP,),
                            radiation=True, dirichlet_nodes=nodes, dirichlet_values=293.0)
    beam = P.LaserBeam(200.0, 0.35, 5e-5, 5e-5, 0.8)
    settings = P.SolverSettings(picard_tol=1e-8, linear_tol=1e-12, linear_solver="cg")
    src = P.GaussianSource(beam, tuple(z["center"]))
    s0 = P.FieldState(grid, z["T_old"], 0.0)
    s1 = P.step_backward_euler(s0, float(z["dt"]), mat, src, bounds, settings, latent=True)
    assert isinstance(s1, P.fem.DeviceBackedFieldState)
    N.host_traffic(reset=True)
    s2 = P.step_backward_euler(s1, float(z["dt"]), mat, src, bounds, settings, latent=True)
    h2d, d2h = N.host_traffic()
    assert h2d == 12 * nodes.size and d2h == 0, (h2d, d2h, grid.n_nodes)
    # the host path gives bitwise the same second step
    monkeypatch.setenv("TLGPU_DEVICE_FIELDS", "0")
    h1 = P.step_backward_euler(s0, float(z["dt"]), mat, src, bounds, settings, latent=True)
    h2 = P.step_backward_euler(h1, float(z["dt"]), mat, src, bounds, settings, latent=True)
    np.testing.assert_array_equal(s2.values, h2.values)
    # a node listed twice keeps its last value (g[nodes] = values)
    twice = np.concatenate([nodes, nodes[:3]])
    vals = np.concatenate([np.full(nodes.size, 293.0), [400.0, 410.0, 420.0]])
    b2 = P.BoundarySpec(bc=bounds.bc, robin_tags=(P.TOP,), radiation=True, dirichlet_nodes=twice, dirichlet_values=vals)
    out = P.step_backward_euler(s0, float(z["dt"]), mat, src, b2, settings, latent=True)
    np.testing.assert_array_equal(out.values[nodes[:3]], [400.0, 410.0, 420.0])
    assert np.all(out.values[nodes[3:]] == 293.0)

"""Host-side mechanics of the device-resident result fields (CPU, no GPU): a
DeviceFieldState reads its values once, on first access or before the owning run's
state changes; a UniformFieldState builds its array only when read."""

import numpy as np

import paper_2110_12932_b200 as P
from paper_2110_12932_b200.multirate import DeviceFieldState, DeviceRun


class _StubRun:
    """The parts of DeviceRun a lazy field uses; field() counts read-backs."""

    def __init__(self, n):
        import weakref
        self.n, self.reads, self.value = n, 0, 1.0
        self._lazy = weakref.WeakSet()

    def field(self, which, out=None):
        self.reads += 1
        return np.full(self.n, self.value)

    lazy_field = DeviceRun.lazy_field
    _materialize_lazy = DeviceRun._materialize_lazy


def _grid():
    return P.build_structured_grid(P.Box((0.0, 0.0, 0.0), (1e-3, 1e-3, 5e-4)), 1e-4)


def test_device_field_reads_once_on_access():
    g = _grid()
    run = _StubRun(g.n_nodes)
    f = run.lazy_field(0, g, 1.5)
    assert run.reads == 0 and f.on_device and f.time == 1.5
    assert f.values.shape == (g.n_nodes,) and run.reads == 1 and not f.on_device
    f.values
    assert run.reads == 1
    assert not f.values.flags.writeable


def test_device_field_materialised_before_the_run_changes():
    g = _grid()
    run = _StubRun(g.n_nodes)
    f = run.lazy_field(0, g, 0.0)
    run._materialize_lazy()          # what DeviceRun.initial / run / close do first
    run.value = 7.0                   # the device state moves on
    assert run.reads == 1 and np.all(f.values == 1.0)


def test_dropped_device_field_is_never_read():
    g = _grid()
    run = _StubRun(g.n_nodes)
    f = run.lazy_field(0, g, 0.0)
    del f
    run._materialize_lazy()
    assert run.reads == 0


def test_uniform_field_is_lazy_and_equal_to_full():
    g = _grid()
    u = P.uniform_field(g, 293.0, 0.5)
    assert u._v is None and u.uniform_value == 293.0
    np.testing.assert_array_equal(u.values, np.full(g.n_nodes, 293.0))
    assert u.with_values(u.values + 1.0).values[0] == 294.0


# ---- step-level fields on the device: the host-side rules (no GPU) ----------------------

def test_dirichlet_list_dedupes_like_numpy_assignment():
    """ops.dirichlet_list: ids as int32, values broadcast, a node listed twice keeps its
    last value (g[nodes] = values), ids outside the mesh are rejected."""
    import pytest
    from paper_2110_12932_b200 import ops
    nodes = np.array([5, 2, 9, 2, 5, 7])
    vals = np.array([1.0, 2.0, 3.0, 4.0, 5.0, 6.0])
    idx, v = ops.dirichlet_list(nodes, vals, 10)
    g = np.zeros(10)
    g[nodes] = vals
    assert idx.dtype == np.int32 and list(idx) == [2, 5, 7, 9]
    np.testing.assert_array_equal(v, g[idx])
    idx, v = ops.dirichlet_list(np.array([0, 3, 4]), 293.0, 5)          # sorted ids pass through, scalar broadcast
    assert list(idx) == [0, 3, 4] and list(v) == [293.0] * 3
    idx, v = ops.dirichlet_list(np.empty(0, dtype=np.int64), 0.0, 5)
    assert idx.size == 0 and v.size == 0
    with pytest.raises(P.SolverError):
        ops.dirichlet_list(np.array([1, 10]), 0.0, 10)


def test_one_way_follows_the_reference_rule():
    """TwoLevelProblem.one_way (twolevel.py:101-113): equal conductivity tables in alternate
    mode; in full mode fully equal materials AND no latent heat -- also when one material
    object serves both levels."""
    g = _grid()
    bc = P.ThermalBC(0.0, 0.0, 293.0, 293.0)

    def mat(k=10.0, c=400.0, chi=0.0, Tl=1653.15):
        return P.Material(np.array([[200.0, k], [5000.0, k]]), np.array([[200.0, c], [5000.0, c]]), 8000.0, chi,
                          1563.15, Tl, 0.05)

    def one_way(a, b, mode):
        return P.TwoLevelProblem(global_mesh=g, mat_global=a, mat_local=b, bc=bc, mode=mode).one_way

    m = mat()
    assert one_way(m, m, "alternate") and one_way(m, m, "full")
    assert one_way(mat(), mat(), "full")
    assert not one_way(mat(12.0), mat(), "alternate") and not one_way(mat(12.0), mat(), "full")
    assert one_way(mat(c=500.0), mat(), "alternate") and not one_way(mat(c=500.0), mat(), "full")
    assert one_way(mat(Tl=1700.0), mat(), "alternate") and not one_way(mat(Tl=1700.0), mat(), "full")
    latent = mat(chi=2e5)
    assert one_way(latent, latent, "alternate") and not one_way(latent, latent, "full")


def test_retimed_keeps_the_backing():
    """FieldState.retimed: same values, new time; a uniform field stays lazy."""
    g = _grid()
    f = P.FieldState(g, np.linspace(300.0, 400.0, g.n_nodes), 1.0)
    r = f.retimed(2.0)
    assert r.time == 2.0 and r.values is f.values
    u = P.uniform_field(g, 293.0).retimed(3.0)
    assert u.time == 3.0 and u.uniform_value == 293.0 and u._v is None


def test_arbitrary_dirichlet_sets_are_not_a_fused_kernel_kind():
    """fem._dirichlet_kind: the fused linear kernels know the bottom face and the interface as
    node classes; any other set is the general path's node mask (-1)."""
    from paper_2110_12932_b200 import _native as N
    from paper_2110_12932_b200.fem import _dirichlet_kind
    g = _grid()
    assert _dirichlet_kind(g, g.nodes_on(P.BOTTOM)) == N.TL_DIRICHLET_BOTTOM
    assert _dirichlet_kind(g, g.gamma_nodes()) == N.TL_DIRICHLET_GAMMA
    assert _dirichlet_kind(g, np.arange(g.n_nodes)) == -1
    assert _dirichlet_kind(g, np.empty(0, dtype=np.int64)) == -1


def test_interpolate_outside_raises_with_coordinates():
    """test_mesh.py::test_locate_outside_raises_with_coordinates: the host-side containment
    check of StructuredGrid.interpolate (no device call is made for a point outside)."""
    import pytest
    m = P.build_structured_grid(P.Box((0.0, 0.0), (1.0, 1.0)), 0.5)
    with pytest.raises(P.PointOutsideMesh) as err:
        m.interpolate(np.zeros(m.n_nodes), np.array([[1.5, 0.5]]))
    assert err.value.point[0] == pytest.approx(1.5)

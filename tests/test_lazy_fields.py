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

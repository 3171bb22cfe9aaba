"""ctypes binding of libtlgpu.so (C ABI declared in include/tlgpu.h).

There is no CPU fallback: if the library is missing or fails to load, every
entry point raises ``NativeLibraryMissing``.  Build it with
``python -m paper_2110_12932_b200.build`` (or ``__graft_entry__.build()``).
"""

from __future__ import annotations

import ctypes as C
import weakref
import os
from pathlib import Path

import numpy as np

from .errors import NativeLibraryMissing, SolverError

LIB_PATH = Path(__file__).resolve().parent / "libtlgpu.so"
ABI_VERSION = 1

TL_DIRICHLET_BOTTOM = 0
TL_DIRICHLET_GAMMA = 1
TL_SOLVE_OK, TL_SOLVE_MAXITER, TL_SOLVE_RESIDUAL, TL_SOLVE_NONFINITE = 0, 1, 2, 3

_d3 = C.c_double * 3
_i3 = C.c_int32 * 3


class SolveInfo(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("status", C.c_int32), ("bnorm", C.c_double),
                ("rnorm", C.c_double), ("true_resid", C.c_double)]


class GridDesc(C.Structure):
    _fields_ = [("ncells", _i3), ("lo0", _d3), ("hi0", _d3), ("offset", _d3)]

    @classmethod
    def make(cls, lo0, hi0, ncells, offset=(0.0, 0.0, 0.0)) -> "GridDesc":
        # a 2D grid travels as ncells[2] = 0 (csrc/tl_2d.cuh); only the entry points with
        # triangle variants accept it
        pad = lambda v, fill: [*v, *([fill] * (3 - len(v)))]      # noqa: E731
        return cls(_i3(*pad([int(v) for v in ncells], 0)), _d3(*pad(list(map(float, lo0)), 0.0)),
                   _d3(*pad(list(map(float, hi0)), 0.0)), _d3(*pad(list(map(float, offset)), 0.0)))


class Gaussian(C.Structure):
    _fields_ = [("peak", C.c_double), ("radius", C.c_double), ("depth", C.c_double),
                ("center", _d3), ("on", C.c_int32)]


class VcMaterial(C.Structure):
    _fields_ = [("k_T", C.c_void_p), ("k_v", C.c_void_p), ("nk", C.c_int32), ("c_T", C.c_void_p),
                ("c_v", C.c_void_p), ("nc", C.c_int32), ("rho", C.c_double), ("chi", C.c_double),
                ("S", C.c_double), ("T_melt", C.c_double), ("latent", C.c_int32)]


class Robin(C.Structure):
    _fields_ = [("h_conv", C.c_double), ("sigma_eps", C.c_double), ("T_ambient", C.c_double),
                ("on", C.c_int32)]


class RunDesc(C.Structure):
    _fields_ = [("global_grid", GridDesc), ("local_grid", GridDesc), ("kappa", C.c_double),
                ("rho_c_global", C.c_double), ("rho_c_local", C.c_double),
                ("T_buildplate", C.c_double), ("beam_peak", C.c_double),
                ("beam_radius", C.c_double), ("beam_depth", C.c_double), ("rtol", C.c_double),
                ("maxiter_factor", C.c_int32), ("max_micro", C.c_int32),
                ("max_deposit", C.c_int32), ("device", C.c_int32), ("external_planes", C.c_int32)]


class MacroPlan(C.Structure):
    _fields_ = [("dt_global", C.c_double), ("dep_offset", C.c_int32), ("dep_count", C.c_int32),
                ("micro_offset", C.c_int32), ("n_micro", C.c_int32), ("corrector", C.c_int32),
                ("relocate", C.c_int32), ("record", C.c_int32), ("new_offset", _d3)]


class MicroPlan(C.Structure):
    _fields_ = [("dt", C.c_double), ("w", C.c_double), ("center", _d3), ("source_on", C.c_int32)]


class Slab(C.Structure):
    _fields_ = [("grid", GridDesc), ("dirichlet_kind", C.c_int32), ("k0", C.c_int32), ("k1", C.c_int32),
                ("kappa", C.c_double), ("rho_c", C.c_double), ("dt", C.c_double), ("g_const", C.c_double),
                ("x", C.c_void_p), ("b", C.c_void_p), ("r", C.c_void_p), ("p0", C.c_void_p),
                ("p1", C.c_void_p), ("load", C.c_void_p), ("work", C.c_void_p), ("sums", C.c_void_p),
                ("gath", C.c_void_p), ("world", C.c_int32), ("maxiter", C.c_int32), ("rtol", C.c_double),
                ("stream", C.c_void_p)]


# numpy views of the plan structs (same layout, built in bulk on the host)
MACRO_DTYPE = np.dtype([("dt_global", "<f8"), ("dep_offset", "<i4"), ("dep_count", "<i4"),
                        ("micro_offset", "<i4"), ("n_micro", "<i4"), ("corrector", "<i4"),
                        ("relocate", "<i4"), ("record", "<i4"), ("new_offset", "<f8", (3,))],
                       align=True)
MICRO_DTYPE = np.dtype([("dt", "<f8"), ("w", "<f8"), ("center", "<f8", (3,)),
                        ("source_on", "<i4")], align=True)
assert MACRO_DTYPE.itemsize == C.sizeof(MacroPlan), (MACRO_DTYPE.itemsize, C.sizeof(MacroPlan))
assert MICRO_DTYPE.itemsize == C.sizeof(MicroPlan), (MICRO_DTYPE.itemsize, C.sizeof(MicroPlan))

_P = C.c_void_p
_dp = C.POINTER(C.c_double)

# (name, restype, argtypes) of every symbol include/tlgpu.h declares
SIGNATURES = [
    ("tl_abi_version", C.c_int32, []),
    ("tl_last_error", C.c_char_p, []),
    ("tl_device_query", C.c_int32, [C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int64),
                                    C.POINTER(C.c_int32)]),
    ("tl_step_host", C.c_int32, [C.POINTER(GridDesc), C.c_double, C.c_double, C.c_double, C.c_int32,
                                 _dp, _dp, C.c_double, C.c_double, _dp, _dp, C.POINTER(Gaussian),
                                 C.c_double, C.c_int32, _dp, C.POINTER(SolveInfo)]),
    ("tl_step_nodes_host", C.c_int32, [C.POINTER(GridDesc), C.c_double, C.c_double, C.c_double, C.c_int32,
                                       C.c_void_p, C.c_int64, _dp, _dp, _dp, C.POINTER(Gaussian),
                                       C.c_double, C.c_int32, _dp, C.POINTER(SolveInfo)]),
    ("tl_interpolate_host", C.c_int32, [C.POINTER(GridDesc), _dp, C.POINTER(GridDesc), C.c_int32, _dp]),
    ("tl_interpolate_points_host", C.c_int32, [C.POINTER(GridDesc), _dp, _dp, C.c_int64, _dp]),
    ("tl_deposit_host", C.c_int32, [C.POINTER(GridDesc), _dp, _dp, C.c_int32, _dp]),
    ("tl_mass_norms_host", C.c_int32, [C.POINTER(GridDesc), _dp, _dp, _dp]),
    ("tl_mass_norms_split_host", C.c_int32, [C.POINTER(GridDesc), _dp, _dp, _dp, _dp, _dp]),
    ("tl_transmission_host", C.c_int32, [C.POINTER(GridDesc), C.POINTER(GridDesc), _dp, C.c_double, _dp]),
    ("tl_overlap_feedback_host", C.c_int32, [C.POINTER(GridDesc), C.POINTER(GridDesc), _dp, _dp, C.c_double,
                                             C.POINTER(VcMaterial), C.POINTER(VcMaterial), C.POINTER(Gaussian),
                                             _dp]),
    ("tl_transmission_tables_host", C.c_int32, [C.POINTER(GridDesc), C.POINTER(GridDesc), _dp, _dp, _dp, C.c_int32,
                                                _dp, _dp, C.c_int32, _dp]),
    ("tl_vc_last_cg_ms", C.c_int32, [C.POINTER(C.c_float)]),
    ("tl_step_last_ms", C.c_int32, [C.POINTER(C.c_float)]),
    ("tl_vc_picard_host", C.c_int32, [C.POINTER(GridDesc), C.POINTER(VcMaterial), C.POINTER(VcMaterial), _dp,
                                      C.c_int32, C.c_double, _dp, _dp, C.POINTER(Gaussian), C.POINTER(Robin),
                                      C.c_void_p, _dp, C.c_double, C.c_int32, C.c_int32, C.c_double, C.c_int32,
                                      _dp, C.POINTER(C.c_int32), C.c_void_p, C.c_void_p, C.POINTER(C.c_double),
                                      C.POINTER(SolveInfo)]),
    ("tl_vc_step_region_host", C.c_int32, [C.POINTER(GridDesc), C.POINTER(VcMaterial), C.POINTER(VcMaterial),
                                           _dp, C.c_int32, C.c_double, _dp, _dp, _dp, C.POINTER(Gaussian),
                                           C.POINTER(Robin), C.c_void_p, _dp, C.c_double, C.c_int32, _dp,
                                           C.POINTER(SolveInfo)]),
    ("tl_vc_step_host", C.c_int32, [C.POINTER(GridDesc), C.POINTER(VcMaterial), C.c_double, _dp, _dp, _dp,
                                    C.POINTER(Gaussian), C.POINTER(Robin), C.c_void_p, _dp, C.c_double,
                                    C.c_int32, _dp, C.POINTER(SolveInfo)]),
    ("tl_error_l2_host", C.c_int32, [C.POINTER(GridDesc), _dp, C.POINTER(GridDesc), _dp, _dp]),
    ("tl_vc_picard_nodes_host", C.c_int32, [C.POINTER(GridDesc), C.POINTER(VcMaterial), C.POINTER(VcMaterial), _dp,
                                            C.c_int32, C.c_double, _dp, _dp, C.POINTER(Gaussian), C.POINTER(Robin),
                                            C.c_void_p, C.c_int64, _dp, C.c_double, C.c_int32, C.c_int32,
                                            C.c_double, C.c_int32, _dp, C.POINTER(C.c_int32), C.c_void_p,
                                            C.c_void_p, C.POINTER(C.c_double), C.POINTER(SolveInfo)]),
    ("tl_dev_alloc", C.c_int32, [C.c_int64, C.POINTER(_P)]),
    ("tl_dev_free", C.c_int32, [_P]),
    ("tl_dev_copy", C.c_int32, [_P, _P, C.c_int64]),
    ("tl_host_traffic", C.c_int32, [C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.c_int32]),
    ("tl_axpy_host", C.c_int32, [C.c_int64, C.c_double, _dp, _dp]),
    ("tl_interpolate_nodes_host", C.c_int32, [C.POINTER(GridDesc), _dp, C.POINTER(GridDesc), C.c_void_p,
                                              C.c_int64, _dp]),
    ("tl_run_create", C.c_int32, [C.POINTER(RunDesc), C.POINTER(_P)]),
    ("tl_run_destroy", C.c_int32, [_P]),
    ("tl_run_initial", C.c_int32, [_P, C.c_double]),
    ("tl_run_set_global", C.c_int32, [_P, _dp, C.c_int64]),
    ("tl_run_macro_steps", C.c_int32, [_P, _P, C.c_int32, _P, C.c_int32, _dp, _dp, C.c_int32]),
    ("tl_runs_macro_step", C.c_int32, [_P, C.c_int32, _P, _P, _P, _P, _P, _P]),
    ("tl_run_get_snapshot", C.c_int32, [_P, C.c_int32, C.c_int32, _dp, C.c_int64]),
    ("tl_run_sync", C.c_int32, [_P]),
    ("tl_run_get_field", C.c_int32, [_P, C.c_int32, _dp, C.c_int64]),
    ("tl_run_get_field_at", C.c_int32, [_P, C.c_int32, _P, C.c_int64, _dp]),
    ("tl_run_field_async", C.c_int32, [_P, C.c_int32, _dp, C.c_int64, C.c_int32]),
    ("tl_run_field_wait", C.c_int32, [_P, C.c_int32]),
    ("tl_run_take_info", C.c_int32, [_P, C.POINTER(SolveInfo), C.c_int32, C.POINTER(C.c_int32)]),
    ("tl_run_melt_summary", C.c_int32, [_P, C.c_double, _dp]),
    ("tl_run_stream", C.c_int32, [_P, C.POINTER(_P)]),
    ("tl_run_launch_count", C.c_int64, [_P]),
    ("tl_run_set_timing", C.c_int32, [_P, C.c_int32]),
    ("tl_run_take_timing", C.c_int32, [_P, C.POINTER(C.c_float), C.POINTER(C.c_int32),
                                       C.POINTER(C.c_int32), C.c_int32, C.POINTER(C.c_int32)]),
    ("tl_run_flush_l2", C.c_int32, [_P]),
    ("tl_debug_profile", C.c_int32, [C.POINTER(C.c_uint64), C.c_int32, C.POINTER(C.c_int32)]),
    ("tl_run_reanchor", C.c_int32, [_P, C.c_void_p]),
    ("tl_run_put_global_planes", C.c_int32, [_P, C.c_void_p, C.c_int32, C.c_int32]),
    ("tl_slab_work_len", C.c_int64, []),
    ("tl_slab_deposit", C.c_int32, [C.POINTER(Slab), C.c_void_p, C.c_void_p, C.c_int32]),
    ("tl_slab_begin", C.c_int32, [C.POINTER(Slab), C.POINTER(Gaussian)]),
    ("tl_slab_direction", C.c_int32, [C.POINTER(Slab)]),
    ("tl_slab_update", C.c_int32, [C.POINTER(Slab), C.c_int32]),
    ("tl_slab_residual", C.c_int32, [C.POINTER(Slab)]),
    ("tl_slab_finish", C.c_int32, [C.POINTER(Slab)]),
    ("tl_slab_poll", C.c_int32, [C.POINTER(Slab), C.POINTER(C.c_int32), C.POINTER(SolveInfo)]),
]

_lib = None


def lib():
    """Load libtlgpu.so once; raise NativeLibraryMissing if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    path = Path(os.environ.get("TLGPU_LIB", LIB_PATH))
    if not path.exists():
        raise NativeLibraryMissing(
            f"{path} not found: build it with `python -m paper_2110_12932_b200.build` "
            "(there is no CPU fallback)")
    try:
        h = C.CDLL(str(path))
    except OSError as exc:
        raise NativeLibraryMissing(f"cannot load {path}: {exc}") from exc
    for name, res, args in SIGNATURES:
        fn = getattr(h, name)
        fn.restype = res
        fn.argtypes = args
    if h.tl_abi_version() != ABI_VERSION:
        raise NativeLibraryMissing(f"{path} has ABI {h.tl_abi_version()}, expected {ABI_VERSION}")
    _lib = h
    return h


def check(rc: int, what: str = "tlgpu"):
    if rc != 0:
        msg = lib().tl_last_error().decode(errors="replace")
        raise SolverError(f"{what} failed ({rc}): {msg}")


class DeviceVector:
    """n float64 values in device memory (``tl_dev_alloc``), accepted wherever a step-level
    entry point takes a field (``dptr``).  ``to_host`` reads them back (cached, read-only:
    the vector is written once, by the call that produced it).

    Live vectors share a byte budget (``TLGPU_DEVICE_FIELDS_GB``, default 16): when an
    allocation would exceed it, the oldest live vectors are spilled to their host copy and
    their device memory is freed (a recorder that keeps every state of a long run then
    holds host arrays, as with the reference); a spilled vector is passed as a host pointer."""

    __slots__ = ("ptr", "n", "_host", "__weakref__")
    _live: "dict[int, weakref.ref]" = {}
    _bytes = 0
    # released buffers are reused by size (a time loop allocates one result per solve:
    # no cudaMalloc / cudaFree, which synchronises the device, in steady state)
    _pool: "dict[int, list]" = {}
    _pool_bytes = 0

    def __init__(self, n: int):
        self.n = int(n)
        self._host = None
        self.ptr = None
        free = DeviceVector._pool.get(self.n)
        if free:
            self.ptr = free.pop()
            DeviceVector._pool_bytes -= 8 * self.n
        else:
            DeviceVector._make_room(8 * self.n)
            h = _P()
            check(lib().tl_dev_alloc(8 * self.n, C.byref(h)), "device allocation")
            self.ptr = h.value
        DeviceVector._bytes += 8 * self.n
        DeviceVector._live[id(self)] = weakref.ref(self)

    @classmethod
    def trim_pool(cls):
        """Return the pooled buffers to the driver."""
        for free in cls._pool.values():
            for p in free:
                lib().tl_dev_free(p)
        cls._pool.clear()
        cls._pool_bytes = 0

    @staticmethod
    def budget() -> int:
        import os
        return int(float(os.environ.get("TLGPU_DEVICE_FIELDS_GB", "16")) * 2**30)

    @classmethod
    def _make_room(cls, need: int):
        cap = cls.budget()
        if cls._bytes + cls._pool_bytes + need > cap and cls._pool_bytes:
            cls.trim_pool()
        if cls._bytes + need <= cap:
            return
        for key in list(cls._live):              # insertion order: oldest first
            if cls._bytes + need <= cap:
                break
            v = cls._live[key]()
            if v is not None:
                v.spill()

    @classmethod
    def from_host(cls, a) -> "DeviceVector":
        a = np.ascontiguousarray(a, dtype=np.float64)
        v = cls(a.size)
        check(lib().tl_dev_copy(v.ptr, a.ctypes.data, 8 * a.size), "upload")
        return v

    @property
    def shape(self):
        return (self.n,)

    @property
    def on_device(self) -> bool:
        return self.ptr is not None

    def to_host(self) -> np.ndarray:
        if self._host is None:
            out = np.empty(self.n)
            check(lib().tl_dev_copy(out.ctypes.data, self.ptr, 8 * self.n), "read-back")
            out.setflags(write=False)
            self._host = out
        return self._host

    def __array__(self, dtype=None, copy=None):
        a = self.to_host()
        return a if dtype is None else a.astype(dtype, copy=False)

    def spill(self):
        """Keep only the host copy."""
        if self.ptr:
            self.to_host()
            self.free()

    def free(self):
        if self.ptr:
            cls = DeviceVector
            if cls._pool_bytes + 8 * self.n <= cls.budget() // 4:
                cls._pool.setdefault(self.n, []).append(self.ptr)
                cls._pool_bytes += 8 * self.n
            else:
                lib().tl_dev_free(self.ptr)
            self.ptr = None
            cls._bytes -= 8 * self.n
            cls._live.pop(id(self), None)

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def host_traffic(reset: bool = False):
    """(h2d, d2h) bytes the step-level entry points moved over PCIe since the last reset."""
    a, b = C.c_int64(), C.c_int64()
    check(lib().tl_host_traffic(C.byref(a), C.byref(b), int(reset)), "traffic counters")
    return a.value, b.value


def dptr(a):
    """Pointer to a C-contiguous float64 array or a DeviceVector (or None)."""
    if a is None:
        return None
    if isinstance(a, DeviceVector):
        if a.ptr is None:                        # spilled: its host copy
            return a.to_host().ctypes.data_as(_dp)
        return C.cast(C.c_void_p(a.ptr), _dp)
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"], "expected contiguous float64"
    return a.ctypes.data_as(_dp)


def device_query(device: int = 0):
    sm, l2, coop = C.c_int32(), C.c_int64(), C.c_int32()
    check(lib().tl_device_query(device, C.byref(sm), C.byref(l2), C.byref(coop)), "device query")
    return {"sm_count": sm.value, "l2_bytes": l2.value, "cooperative": bool(coop.value)}

"""Host-side control data: boxes, beam, path, local-box policy, macro schedule.

Everything here is scalar, temperature-independent bookkeeping.  It runs on
the host once per run to precompute the schedule the device consumes (laser
positions at every micro end time, swept pieces per macro step, local-box
origins after every relocation).  The floating-point operations mirror the
reference exactly, because the relocation decisions (``np.round`` of a
snapped shift) and the source positions must land on the same values:

- ``Box``                    — ``lpbfsim/mesh.py:43-81``
- ``LaserBeam``/``ThermalBC`` — ``lpbfsim/sources.py:23-54``
- ``Segment``/``ScanPath``   — ``lpbfsim/scanpath.py:25-115``
- ``path_from_segments``     — ``lpbfsim/scanpath.py:118-128``
- ``build_alternating_path`` — ``lpbfsim/scanpath.py:131-158``
- ``LocalDomainPolicy``      — ``lpbfsim/scanpath.py:161-205``
- ``MacroSchedule``          — ``lpbfsim/multirate.py:37-75``
- ``LocalPlacement.relocate``— the shift/clamp part of ``relocate_local``
  (``lpbfsim/scanpath.py:219-241``) plus ``Mesh.translated``'s box arithmetic
  and escape test (``lpbfsim/mesh.py:365-385``)
- ``initial_local_box``      — ``lpbfsim/runner.py:87-97``
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import CouplingError, DomainEscape, MaterialError, MeshError, PathError, SourceError

STEFAN_BOLTZMANN = 5.670374419e-8


# -- geometry -------------------------------------------------------------

@dataclass(frozen=True)
class Box:
    """Axis-aligned box; lo/hi are normalised to tuples of Python floats."""

    lo: tuple
    hi: tuple

    def __post_init__(self):
        lo = np.asarray(self.lo, dtype=float)
        hi = np.asarray(self.hi, dtype=float)
        if lo.shape != hi.shape or lo.ndim != 1 or lo.size not in (2, 3):
            raise MeshError("box corners must both be 2D or 3D coordinate tuples")
        if not np.all(hi > lo):
            raise MeshError(f"degenerate box: lo={lo.tolist()} hi={hi.tolist()}")
        object.__setattr__(self, "lo", tuple(float(v) for v in lo))
        object.__setattr__(self, "hi", tuple(float(v) for v in hi))

    @property
    def dim(self) -> int:
        return len(self.lo)

    @property
    def lengths(self) -> np.ndarray:
        return np.asarray(self.hi) - np.asarray(self.lo)

    @property
    def volume(self) -> float:
        return float(np.prod(self.lengths))

    def contains(self, points, tol: float = 0.0) -> np.ndarray:
        p = np.atleast_2d(np.asarray(points, dtype=float))
        return np.all((p >= np.asarray(self.lo) - tol) & (p <= np.asarray(self.hi) + tol), axis=1)

    def translated(self, offset) -> "Box":
        off = np.asarray(offset, dtype=float)
        return Box(tuple(np.asarray(self.lo) + off), tuple(np.asarray(self.hi) + off))


def structured_ncells(box: Box, h) -> np.ndarray:
    """Cell counts per axis for spacing ``h`` (``lpbfsim/mesh.py:395-404``)."""
    d = box.dim
    h = np.broadcast_to(np.asarray(h, dtype=float), (d,))
    if np.any(h <= 0):
        raise MeshError(f"mesh spacing must be positive, got {h.tolist()}")
    q = box.lengths / h
    n = np.where(np.abs(q - np.round(q)) <= 1e-9 * q, np.round(q), np.ceil(q)).astype(np.int64)
    if np.any(n < 1):
        raise MeshError("mesh must have at least one cell per axis")
    return n


# -- physics constants ----------------------------------------------------

@dataclass(frozen=True)
class LaserBeam:
    power: float
    absorptivity: float
    radius: float
    depth: float
    speed: float

    def __post_init__(self):
        if self.power <= 0 or self.radius <= 0 or self.depth <= 0:
            raise SourceError("beam power, radius, and depth must be positive")
        if not 0.0 < self.absorptivity <= 1.0:
            raise SourceError("absorptivity must lie in (0, 1]")
        if self.speed < 0:
            raise SourceError("scan speed must be nonnegative")

    @property
    def gaussian_peak(self) -> float:
        """Peak of ``gaussian_source_3d`` (``lpbfsim/sources.py:74-76``), same op order."""
        return 6.0 * np.sqrt(3.0) * self.power * self.absorptivity / (
            2.0 * np.pi * self.radius**2 * self.depth)


@dataclass(frozen=True)
class ThermalBC:
    h_conv: float
    emissivity: float
    T_ambient: float
    T_buildplate: float
    sigma_sb: float = STEFAN_BOLTZMANN

    def __post_init__(self):
        if self.h_conv < 0:
            raise SourceError("convection coefficient must be nonnegative")
        if not 0.0 <= self.emissivity <= 1.0:
            raise SourceError("emissivity must lie in [0, 1]")
        if self.sigma_sb <= 0:
            raise SourceError("Stefan-Boltzmann constant must be positive")


@dataclass(frozen=True, eq=False)
class Material:
    """Material tables as in ``lpbfsim/materials.py:40-88`` (the device path
    needs ``is_constant`` and ``chi == 0``)."""

    conductivity_table: np.ndarray
    heat_capacity_table: np.ndarray
    rho: float
    chi: float
    T_solidus: float
    T_liquidus: float
    S: float

    def __post_init__(self):
        for name in ("conductivity_table", "heat_capacity_table"):
            t = np.asarray(getattr(self, name), dtype=float)
            if t.ndim != 2 or t.shape[1] != 2 or t.shape[0] < 2:
                raise MaterialError(f"{name.split('_table')[0]} table needs at least two (T, value) rows")
            if np.any(np.diff(t[:, 0]) <= 0):
                raise MaterialError(f"{name.split('_table')[0]} table temperatures must be strictly increasing")
            if np.any(t[:, 1] <= 0):
                raise MaterialError(f"{name.split('_table')[0]} table values must be positive")
            t.setflags(write=False)
            object.__setattr__(self, name, t)
        if self.rho <= 0:
            raise MaterialError("density must be positive")
        if self.chi < 0:
            raise MaterialError("latent heat must be nonnegative")
        if not self.T_solidus < self.T_liquidus:
            raise MaterialError("solidus must lie below liquidus")
        if self.S <= 0:
            raise MaterialError("sigmoid sharpness must be positive")

    @property
    def is_constant(self) -> bool:
        return (np.ptp(self.conductivity_table[:, 1]) == 0.0
                and np.ptp(self.heat_capacity_table[:, 1]) == 0.0)

    @staticmethod
    def constant(kappa: float, rho: float, c: float, T_solidus: float,
                 T_liquidus: float, chi: float = 0.0, S: float = 0.05) -> "Material":
        return Material(np.array([[200.0, kappa], [5000.0, kappa]]),
                        np.array([[200.0, c], [5000.0, c]]),
                        rho, chi, T_solidus, T_liquidus, S)


def material_constants(mat) -> tuple[float, float]:
    """(kappa, rho*c) of a constant material, evaluated as the reference does.

    The reference evaluates ``np.interp`` on the table (``materials.py:91-100``)
    and multiplies by rho (``fem.py:231``); for a constant table the value is
    the table entry itself.
    """
    k = float(np.interp(300.0, mat.conductivity_table[:, 0], mat.conductivity_table[:, 1]))
    c = float(np.interp(300.0, mat.heat_capacity_table[:, 0], mat.heat_capacity_table[:, 1]))
    return k, float(mat.rho * c)


# -- scan path --------------------------------------------------------------

@dataclass(frozen=True)
class Segment:
    start: tuple
    end: tuple
    speed: float
    t_start: float

    def __post_init__(self):
        if self.speed <= 0:
            raise PathError("segment speed must be positive")

    @property
    def length(self) -> float:
        return float(np.linalg.norm(np.asarray(self.end) - np.asarray(self.start)))

    @property
    def duration(self) -> float:
        return self.length / self.speed

    @property
    def t_end(self) -> float:
        return self.t_start + self.duration


@dataclass(frozen=True)
class ScanPath:
    segments: tuple

    def __post_init__(self):
        if not self.segments:
            raise PathError("a scan path needs at least one segment")
        for a, b in zip(self.segments, self.segments[1:]):
            if abs(b.t_start - a.t_end) > 1e-12 * max(abs(a.t_end), 1.0):
                raise PathError("segment times must be contiguous")

    @property
    def t_start(self) -> float:
        return self.segments[0].t_start

    @property
    def t_end(self) -> float:
        return self.segments[-1].t_end

    def _active(self, t: float):
        tol = 1e-9 * max(abs(self.t_end), 1.0)
        for seg in self.segments:
            if t < seg.t_end - tol:
                return seg
        return None

    def position(self, t: float) -> np.ndarray:
        tol = 1e-9 * max(abs(self.t_end), 1.0)
        if t < self.t_start - tol or t > self.t_end + tol:
            raise PathError(f"time {t:g} outside the path span "
                            f"[{self.t_start:g}, {self.t_end:g}]")
        seg = self._active(t)
        if seg is None:
            return np.asarray(self.segments[-1].end, dtype=float)
        frac = np.clip((t - seg.t_start) / seg.duration, 0.0, 1.0)
        a = np.asarray(seg.start, dtype=float)
        b = np.asarray(seg.end, dtype=float)
        return a + frac * (b - a)

    def direction(self, t: float) -> np.ndarray:
        seg = self._active(t) or self.segments[-1]
        d = np.asarray(seg.end, dtype=float) - np.asarray(seg.start, dtype=float)
        return d / np.linalg.norm(d)

    def swept_pieces(self, t0: float, t1: float) -> list:
        pieces = []
        a = max(t0, self.t_start)
        b = min(t1, self.t_end)
        if b <= a:
            return pieces
        for seg in self.segments:
            lo = max(a, seg.t_start)
            hi = min(b, seg.t_end)
            if hi - lo > 1e-15 * max(abs(self.t_end), 1.0):
                p0 = np.asarray(seg.start, dtype=float)
                p1 = np.asarray(seg.end, dtype=float)
                f0 = (lo - seg.t_start) / seg.duration
                f1 = (hi - seg.t_start) / seg.duration
                pieces.append((p0 + f0 * (p1 - p0), p0 + f1 * (p1 - p0)))
        return pieces


def path_from_segments(points_and_speeds, t0: float = 0.0) -> ScanPath:
    segs = []
    t = t0
    for start, end, speed in points_and_speeds:
        seg = Segment(tuple(start), tuple(end), float(speed), t)
        if seg.length == 0:
            raise PathError("zero-length scan segment")
        segs.append(seg)
        t = seg.t_end
    return ScanPath(tuple(segs))


def build_alternating_path(n_tracks: int, track_length: float, hatch: float,
                           speed: float, origin, bounding_box: Box | None = None) -> ScanPath:
    if n_tracks < 1 or track_length <= 0 or speed <= 0:
        raise PathError("need n_tracks >= 1, positive track length and speed")
    origin = np.asarray(origin, dtype=float)
    triples = []
    for k in range(n_tracks):
        start = origin.copy()
        end = origin.copy()
        start[1] += k * hatch
        end[1] += k * hatch
        if k % 2 == 0:
            end[0] += track_length
        else:
            start[0] += track_length
        triples.append((tuple(start), tuple(end), speed))
    path = path_from_segments(triples)
    if bounding_box is not None:
        for seg in path.segments:
            for p in (seg.start, seg.end):
                if not bounding_box.contains(np.asarray(p)[None, :])[0]:
                    raise PathError(f"scan path point {p} leaves the bounding box")
    return path


# -- moving local box ---------------------------------------------------------

@dataclass(frozen=True)
class LocalDomainPolicy:
    box_size: tuple
    laser_fraction: float = 2.0 / 3.0
    snap: tuple | None = None

    def __post_init__(self):
        if any(s <= 0 for s in self.box_size):
            raise PathError("local box dimensions must be positive")
        if not 0.0 < self.laser_fraction < 1.0:
            raise PathError("laser offset fraction must lie inside the box")

    def target_origin(self, laser, direction) -> np.ndarray:
        size = np.asarray(self.box_size, dtype=float)
        laser = np.asarray(laser, dtype=float)
        origin = laser - size
        origin[-1] = laser[-1] - size[-1]
        if len(size) == 3:
            along, across = (0, 1) if abs(direction[0]) >= abs(direction[1]) else (1, 0)
            frac = self.laser_fraction if direction[along] >= 0 else 1.0 - self.laser_fraction
            origin[along] = laser[along] - frac * size[along]
            origin[across] = laser[across] - 0.5 * size[across]
        else:
            frac = self.laser_fraction if direction[0] >= 0 else 1.0 - self.laser_fraction
            origin[0] = laser[0] - frac * size[0]
        return origin


def initial_local_box(global_box: Box, h_local: float, policy: LocalDomainPolicy,
                      path: ScanPath) -> Box:
    """Initial local box of ``build_problem`` (``lpbfsim/runner.py:87-97``)."""
    t0 = path.t_start
    origin = policy.target_origin(path.position(t0), path.direction(t0))
    size = np.asarray(policy.box_size)
    glo = np.asarray(global_box.lo)
    ghi = np.asarray(global_box.hi)
    margin = np.minimum(h_local, (ghi - glo - size) / 2)
    origin = np.clip(origin, glo + margin, ghi - size - margin)
    origin[-1] = ghi[-1] - size[-1]
    return Box(tuple(origin), tuple(origin + size))


class LocalPlacement:
    """Position of the moving local lattice: construction box + accumulated offset.

    Mirrors the state a reference ``Mesh`` carries for translation
    (``_base_coords`` from the construction box, ``_offset``, current ``box``)
    so that box corners, node coordinates and the escape test are computed
    with the same floating-point operations (``lpbfsim/mesh.py:157-168,365-385``).
    """

    def __init__(self, box0: Box, ncells, offset=None, box: Box | None = None):
        self.box0 = box0
        self.ncells = np.asarray(ncells, dtype=np.int64)
        self.offset = np.zeros(box0.dim) if offset is None else np.asarray(offset, dtype=float)
        self.box = box0 if box is None else box

    @property
    def spacing(self) -> np.ndarray:
        return self.box.lengths / self.ncells

    @property
    def h(self) -> float:
        return float(self.spacing.max())

    def axis_coords(self, axis: int) -> np.ndarray:
        """Node coordinates along one axis: linspace of the construction box + offset."""
        base = np.linspace(self.box0.lo[axis], self.box0.hi[axis], int(self.ncells[axis]) + 1)
        return base + self.offset[axis]

    def translated(self, shift, within: Box | None = None) -> "LocalPlacement":
        off = self.offset + np.asarray(shift, dtype=float)
        new_box = Box(tuple(np.asarray(self.box.lo) - self.offset + off),
                      tuple(np.asarray(self.box.hi) - self.offset + off))
        if within is not None:
            lo_ok = np.all(np.asarray(new_box.lo) >= np.asarray(within.lo) - 1e-12 * self.h)
            hi_ok = np.all(np.asarray(new_box.hi) <= np.asarray(within.hi) + 1e-12 * self.h)
            if not (lo_ok and hi_ok):
                raise DomainEscape(f"local domain {new_box} escapes global box {within}")
        return LocalPlacement(self.box0, self.ncells, off, new_box)

    def relocate(self, policy: LocalDomainPolicy, laser, direction,
                 global_box: Box) -> "LocalPlacement | None":
        """Snapped, clamped move toward the laser; None when it stays put."""
        snap = np.asarray(policy.snap if policy.snap is not None else self.spacing, dtype=float)
        target = policy.target_origin(laser, direction)
        current = np.asarray(self.box.lo)
        shift = np.round((target - current) / snap) * snap
        shift[-1] = 0.0
        if not np.any(shift != 0.0):
            return None
        try:
            return self.translated(shift, within=global_box)
        except DomainEscape:
            glo = np.asarray(global_box.lo)
            ghi = np.asarray(global_box.hi)
            lo, hi = np.asarray(self.box.lo), np.asarray(self.box.hi)
            room_lo = np.ceil((glo - lo) / snap + 1.0 - 1e-9) * snap
            room_hi = np.floor((ghi - hi) / snap - 1.0 + 1e-9) * snap
            shift = np.clip(shift, room_lo, room_hi)
            shift[-1] = 0.0
            if not np.any(shift != 0.0):
                return None
            return self.translated(shift, within=global_box)


def check_immersed(local_box: Box, global_box: Box, global_h: float):
    """Immersion precondition of ``extract_interface`` (``lpbfsim/mesh.py:484-496``)."""
    tol = 1e-9 * global_h
    llo, lhi = np.asarray(local_box.lo), np.asarray(local_box.hi)
    glo, ghi = np.asarray(global_box.lo), np.asarray(global_box.hi)
    lateral_ok = np.all(llo[:-1] > glo[:-1] + tol) and np.all(lhi[:-1] < ghi[:-1] - tol)
    bottom_ok = llo[-1] > glo[-1] + tol
    top_ok = abs(lhi[-1] - ghi[-1]) <= tol
    if not (lateral_ok and bottom_ok and top_ok):
        raise MeshError("local box must be strictly immersed laterally and at the bottom, "
                        "with its top face on the global top face")


# -- time bookkeeping -----------------------------------------------------------

@dataclass(frozen=True)
class MacroSchedule:
    dt_macro: float
    micro_per_macro: int
    t_start: float
    t_end: float

    def __post_init__(self):
        if self.dt_macro <= 0 or self.micro_per_macro < 1:
            raise CouplingError("schedule needs dt_macro > 0 and micro count >= 1")
        span = self.t_end - self.t_start
        if span < 0:
            raise CouplingError("t_end must not precede t_start")
        n = span / self.dt_macro
        if abs(n - round(n)) > 1e-9 * max(n, 1.0):
            raise CouplingError(
                f"interval {span:g} is not an integer number of macro steps {self.dt_macro:g}")

    @property
    def dt_micro(self) -> float:
        return self.dt_macro / self.micro_per_macro

    @property
    def n_macro(self) -> int:
        return int(round((self.t_end - self.t_start) / self.dt_macro))

    def t_macro(self, k: int) -> float:
        return self.t_start + k * self.dt_macro

    def t_micro(self, k: int, i: int) -> float:
        return self.t_start + k * self.dt_macro + i * self.dt_micro

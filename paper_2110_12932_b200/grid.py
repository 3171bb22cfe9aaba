"""Lightweight structured-mesh stand-in for the reference ``Mesh``.

The reference ``Mesh`` (``lpbfsim/mesh.py:154-385``) eagerly stores node
coordinates and the Kuhn tet connectivity; at cfg4 scale those arrays are
4.8 GB + 39 GB.  ``StructuredGrid`` keeps the attributes the two-level API
reads (``box``, ``dim``, ``ncells``, ``spacing``, ``n_nodes``, ``h``,
``coords``, ``translated``, ``interpolate``) and derives everything else from
the lattice.  Node order is the reference's (x fastest,
``lpbfsim/mesh.py:406-409``); coordinates are linspace of the construction box
plus the accumulated offset (``lpbfsim/mesh.py:163-165,372``).
"""

from __future__ import annotations

from functools import cached_property

import numpy as np

from .control import Box, LocalPlacement, structured_ncells
from .errors import MeshError

BOTTOM, TOP, LATERAL = 0, 1, 2
_GAMMA_NODES: dict = {}


class StructuredGrid:
    """Uniform lattice of a box, subdivided implicitly: 6 Kuhn tets per cell in 3D, the two
    triangles ``[0, 1, 3]`` / ``[0, 3, 2]`` per cell in 2D (``mesh.py:84-102``).  In 2D the
    vertical axis is y (BOTTOM / TOP are y = lo / hi, ``mesh.py:206-209``) and ``shape`` is
    ``(1, NY, NX)``."""

    def __init__(self, placement: LocalPlacement):
        self._placement = placement
        self.box = placement.box
        self.dim = int(self.box.dim)
        if self.dim not in (2, 3):
            raise MeshError("structured grids are 2D or 3D")
        self.ncells = placement.ncells
        self.spacing = self.box.lengths / self.ncells

    # -- reference Mesh attributes --------------------------------------------

    @property
    def placement(self) -> LocalPlacement:
        return self._placement

    @property
    def shape(self) -> tuple:
        n = self.ncells
        if self.dim == 2:
            return (1, int(n[1]) + 1, int(n[0]) + 1)
        return (int(n[2]) + 1, int(n[1]) + 1, int(n[0]) + 1)

    @property
    def n_nodes(self) -> int:
        return int(np.prod(self.shape))

    @property
    def n_elems(self) -> int:
        return (2 if self.dim == 2 else 6) * int(np.prod(self.ncells))

    @property
    def h(self) -> float:
        return float(self.spacing.max())

    @property
    def _offset(self) -> np.ndarray:
        return self._placement.offset

    def axis(self, a: int) -> np.ndarray:
        return self._placement.axis_coords(a)

    @cached_property
    def coords(self) -> np.ndarray:
        """(n_nodes, dim) node coordinates, materialised on first use."""
        if self.dim == 2:
            Y, X = np.meshgrid(self.axis(1), self.axis(0), indexing="ij")
            out = np.stack([X.ravel(), Y.ravel()], axis=1)
            out.setflags(write=False)
            return out
        x, y, z = self.axis(0), self.axis(1), self.axis(2)
        Z, Y, X = np.meshgrid(z, y, x, indexing="ij")
        out = np.stack([X.ravel(), Y.ravel(), Z.ravel()], axis=1)
        out.setflags(write=False)
        return out

    @cached_property
    def elems(self) -> np.ndarray:
        """(n_elems, 4) Kuhn tets in the reference's order (``mesh.py:406-439``): cells x
        fastest, six tets per cell in ``itertools.permutations`` order with vertices
        0 -> +e_p0 -> +e_p1 -> 111, the last two vertices swapped where the tet is inverted.
        Materialised only for output (VTK); no device path reads it."""
        import itertools
        nc = [int(v) for v in self.ncells]
        nn = [v + 1 for v in nc]
        if self.dim == 2:
            CY, CX = np.meshgrid(np.arange(nc[1]), np.arange(nc[0]), indexing="ij")
            c0 = (CX + nn[0] * CY).ravel()
            corner = c0[:, None] + np.array([0, 1, nn[0], nn[0] + 1])
            tris = corner[:, np.array([[0, 1, 3], [0, 3, 2]])].reshape(-1, 3).astype(np.int64)
            tris.setflags(write=False)
            return tris
        strides = np.array([1, nn[0], nn[0] * nn[1]], dtype=np.int64)
        CZ, CY, CX = np.meshgrid(np.arange(nc[2]), np.arange(nc[1]), np.arange(nc[0]), indexing="ij")
        corner0 = np.stack([CX.ravel(), CY.ravel(), CZ.ravel()], axis=1) @ strides
        offsets = np.array([[(b >> a) & 1 for a in range(3)] for b in range(8)])
        corner_ids = corner0[:, None] + offsets @ strides
        pats = []
        for perm in itertools.permutations(range(3)):
            verts, acc = [0], 0
            for ax in perm:
                acc += 1 << ax
                verts.append(acc)
            pats.append(verts)
        elems = corner_ids[:, np.array(pats)].reshape(-1, 4).astype(np.int64)
        X = self.coords
        J = X[elems[:, 1:]] - X[elems[:, [0]]]
        flip = np.linalg.det(J) < 0
        elems[flip, 2:] = elems[flip, 2:][:, ::-1]
        elems.setflags(write=False)
        return elems

    def nodes_on(self, *tags: int) -> np.ndarray:
        """Sorted node ids of boundary facets with the given tags (``mesh.py:226-230``)."""
        m = np.zeros(self.shape, dtype=bool)
        if self.dim == 2:                       # vertical axis = y
            if BOTTOM in tags:
                m[:, 0, :] = True
            if TOP in tags:
                m[:, -1, :] = True
            if LATERAL in tags:
                m[:, :, 0] = m[:, :, -1] = True
            return np.nonzero(m.ravel())[0]
        if BOTTOM in tags:
            m[0] = True
        if TOP in tags:
            m[-1] = True
        if LATERAL in tags:
            m[:, 0, :] = m[:, -1, :] = True
            m[:, :, 0] = m[:, :, -1] = True
        return np.nonzero(m.ravel())[0]

    def gamma_nodes(self) -> np.ndarray:
        """Sorted ids of the interface (trace) nodes; depends on the lattice shape only, so it
        is cached per shape (6.4M-node local grids: 10 ms per call otherwise)."""
        key = (self.dim, tuple(int(v) for v in self.ncells))
        nodes = _GAMMA_NODES.get(key)
        if nodes is None:
            nodes = np.nonzero(self.gamma_mask())[0]
            nodes.setflags(write=False)
            if len(_GAMMA_NODES) > 16:
                _GAMMA_NODES.clear()
            _GAMMA_NODES[key] = nodes
        return nodes

    def gamma_mask(self) -> np.ndarray:
        """Flat bool mask of the interface (trace) nodes: lateral + bottom facets."""
        m = np.zeros(self.shape, dtype=bool)
        if self.dim == 2:
            m[:, 0, :] = True
            m[:, :, 0] = m[:, :, -1] = True
            return m.ravel()
        m[0] = True
        m[:, 0, :] = m[:, -1, :] = True
        m[:, :, 0] = m[:, :, -1] = True
        return m.ravel()

    def translated(self, offset, within: Box | None = None) -> "StructuredGrid":
        return StructuredGrid(self._placement.translated(offset, within))

    def interpolate(self, values: np.ndarray, points: np.ndarray) -> np.ndarray:
        """P1 interpolant at points, evaluated on the device (``mesh.py:358-361``).  A point
        outside the box (inflated by 1e-12 h, ``mesh.py:316-320``) raises PointOutsideMesh,
        as ``Mesh.locate`` does; the device would clip it into a boundary cell."""
        from .errors import PointOutsideMesh
        from .ops import interpolate_points
        pts = np.atleast_2d(np.asarray(points, dtype=float))
        inside = self.box.contains(pts, tol=1e-12 * self.h)
        if not np.all(inside):
            raise PointOutsideMesh(pts[np.nonzero(~inside)[0][0]])
        return interpolate_points(self, values, pts)

    def desc(self):
        from ._native import GridDesc
        p = self._placement
        return GridDesc.make(p.box0.lo, p.box0.hi, p.ncells, p.offset)

    def same_lattice(self, other: "StructuredGrid") -> bool:
        return (np.array_equal(self.ncells, other.ncells)
                and self._placement.box0 == other._placement.box0
                and np.array_equal(self._offset, other._offset))

    def __repr__(self):
        return f"StructuredGrid(box={self.box}, ncells={self.ncells.tolist()})"


def build_structured_grid(box: Box, h) -> StructuredGrid:
    """``build_structured_mesh`` (``lpbfsim/mesh.py:388-439``) for 2D and 3D boxes."""
    if box.dim not in (2, 3):
        raise MeshError("the device path supports 2D and 3D boxes")
    return StructuredGrid(LocalPlacement(box, structured_ncells(box, h)))

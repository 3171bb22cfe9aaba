"""Exception types with the reference's names, bases, attributes and messages.

Callers of the reference catch these by class, so the drop-in raises the
same hierarchy:

- ``SolverError`` / ``NonConvergence``  — ``lpbfsim/fem.py:24-33``
- ``CouplingError`` / ``CouplingNonConvergence`` — ``lpbfsim/twolevel.py:32-43``
- ``MeshError`` / ``PointOutsideMesh`` / ``DomainEscape`` — ``lpbfsim/mesh.py:27-40``
- ``PathError`` — ``lpbfsim/scanpath.py:21``
- ``SourceError`` — ``lpbfsim/sources.py:19``
- ``MaterialError`` — ``lpbfsim/materials.py:24``
- ``ConfigError`` — ``lpbfsim/config.py:27``

``UnsupportedOnDevice`` is new: inputs the device kernels cannot represent
(2D, temperature-dependent tables, latent heat, radiation, opaque source
callables) raise it instead of silently falling back to a CPU path.
"""

from __future__ import annotations

import numpy as np


class SolverError(RuntimeError):
    pass


class NonConvergence(SolverError):
    def __init__(self, what: str, iterations: int, residual: float):
        self.iterations = iterations
        self.residual = residual
        super().__init__(f"{what} did not converge in {iterations} iterations "
                         f"(last residual {residual:.3e})")


class CouplingError(SolverError):
    pass


class CouplingNonConvergence(CouplingError):
    def __init__(self, iterations: int, change: float):
        self.iterations = iterations
        self.change = change
        super().__init__(
            f"interface coupling did not converge in {iterations} iterations "
            f"(last trace change {change:.3e})"
        )


class MeshError(ValueError):
    pass


class PointOutsideMesh(MeshError):
    def __init__(self, point):
        self.point = np.asarray(point, dtype=float)
        super().__init__(f"point {self.point.tolist()} lies outside the mesh")


class DomainEscape(MeshError):
    pass


class PathError(ValueError):
    pass


class SourceError(ValueError):
    pass


class MaterialError(ValueError):
    pass


class ConfigError(ValueError):
    pass


class UnsupportedOnDevice(SolverError):
    """The requested physics has no device kernel (out of scope)."""


class NativeLibraryMissing(ImportError):
    """libtlgpu.so is absent or failed to load; there is no CPU fallback."""

"""B200-native two-level (global + moving local) heat solve for laser powder bed fusion.

Drop-in for the hot path of the reference package ``lpbfsim`` (arXiv 2110.12932):
the implicit steps on the coarse global grid and the fine moving local grid,
sub-cycled by the multirate scheme, run as hand-written sm_100a CUDA kernels
(``csrc/``, C ABI in ``include/tlgpu.h``) behind the reference's Python API.
There is no CPU fallback: without ``libtlgpu.so`` every solver entry point
raises ``NativeLibraryMissing``.
"""

__version__ = "0.1.0"

from .config import (  # noqa: F401
    CouplingSettings, ExperimentConfig, SolverSettings, config_from_text, load_config, load_material,
)
from .control import (  # noqa: F401
    Box, LaserBeam, LocalDomainPolicy, LocalPlacement, MacroSchedule, Material, ScanPath, Segment,
    ThermalBC, build_alternating_path, path_from_segments,
)
from .errors import (  # noqa: F401
    ConfigError, CouplingError, CouplingNonConvergence, DomainEscape, MaterialError, MeshError,
    NativeLibraryMissing, NonConvergence, PathError, PointOutsideMesh, SolverError, SourceError,
    UnsupportedOnDevice,
)
from .fem import (  # noqa: F401
    BoundarySpec, FieldState, GaussianSource, Trajectory, solve_monolithic, step_backward_euler, uniform_field,
)
from .grid import BOTTOM, LATERAL, TOP, StructuredGrid, build_structured_grid  # noqa: F401
from .multirate import BatchedRuns, DeviceRun, macro_step, run_space, run_spacetime  # noqa: F401
from .runner import build_problem, reference_bounds, run_reference, two_level_run, two_level_run_slabs  # noqa: F401
from . import experiment, metrics  # noqa: F401
from .experiment import RunArtifacts, run_compare, run_experiment, run_study  # noqa: F401

# the reference's top-level names (lpbfsim/__init__.py)
Mesh = StructuredGrid
MaterialModel = Material
from .metrics import ErrorReport, RunLog, error_metrics, l2_norm  # noqa: F401
from .stats import RunStats  # noqa: F401
from .twolevel import (  # noqa: F401
    InterfaceGamma, TwoLevelProblem, TwoLevelState, extract_interface, initial_state, solve_global,
    solve_local,
)

# reference spelling
build_structured_mesh = build_structured_grid

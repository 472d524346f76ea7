"""B200-native multi-signal growing self-organizing network (arXiv:1503.08294).

Drop-in for the reference package ``growsurf``'s training loop: the same
names (EngineParams, Network, run_multi, resolve_and_update, executors,
samplers, RunStats, mesh checks) backed by hand-written sm_100a CUDA kernels
through a C ABI (include/growsurf_b200.h, loaded with ctypes).  There is no
CPU fallback: device entry points raise DeviceUnavailable when the library
or a GPU is missing.
"""

from .params import (
    BatchOutcome,
    EngineParams,
    RingClass,
    StateError,
    UnknownUnitError,
    WinnerResult,
    batch_size,
)
from .sampling import CloudSource, DoubleTorusSource, MeshSource, SphereSource, TorusSource
from .metrics import (
    RunStats,
    TriMesh,
    extract_mesh,
    genus,
    manifold_check,
    quantization_error,
    write_stats_csv,
)
from .fileio import ParseError, load_off, load_xyz, save_off, save_xyz
from ._lib import DeviceUnavailable, FIND_AUTO, FIND_EXACT, FIND_FILTER
from .network import Network, Snapshot
from .multi import (
    ExecConfig,
    b200_executor,
    parallel_batch_find_winners,
    timed_find,
    batch_find_winners,
    parallel_executor,
    resolve_and_update,
    run_multi,
    sequential_executor,
)
from .engine import find_winners_exhaustive, is_converged, run, update_single

__version__ = "0.1.0"

__all__ = [
    "ExecConfig", "ParseError", "load_off", "load_xyz", "save_off", "save_xyz",
    "parallel_batch_find_winners", "quantization_error", "run", "timed_find",
    "BatchOutcome", "CloudSource", "DeviceUnavailable", "DoubleTorusSource", "EngineParams",
    "FIND_AUTO", "FIND_EXACT", "FIND_FILTER", "MeshSource", "Network", "RingClass", "RunStats",
    "Snapshot", "SphereSource", "StateError", "TorusSource", "TriMesh", "UnknownUnitError",
    "WinnerResult", "b200_executor", "batch_find_winners", "batch_size", "extract_mesh",
    "find_winners_exhaustive", "genus", "is_converged", "manifold_check", "parallel_executor",
    "resolve_and_update", "run_multi", "sequential_executor", "update_single", "write_stats_csv",
]

"""ctypes binding of libgrowsurf_b200.so (the C ABI in include/growsurf_b200.h).

Loading is lazy so host-only helpers (EngineParams, samplers) import on a
machine without a GPU; every device entry point raises ``DeviceUnavailable``
loudly when the library or a CUDA device is missing.  There is no CPU
fallback anywhere in this package.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

from .params import StateError, UnknownUnitError

HERE = os.path.dirname(os.path.abspath(__file__))
# GS_LIB_PATH overrides the library (developer knob for A/B builds of the kernels)
LIB_PATH = os.environ.get("GS_LIB_PATH") or os.path.join(HERE, "libgrowsurf_b200.so")

GS_OK, GS_VALUE_ERROR, GS_STATE_ERROR, GS_CUDA_ERROR, GS_UNKNOWN_UNIT = range(5)
FIND_EXACT, FIND_FILTER, FIND_AUTO, FIND_SMALL, FIND_GRID = 0, 1, 2, 3, 4
SHARD_ID_BYTES = 128  # GS_SHARD_ID_BYTES (an ncclUniqueId)


class DeviceUnavailable(RuntimeError):
    """The CUDA library or a B200 device is missing: the product never falls back to CPU."""


class GsParams(C.Structure):
    _fields_ = [
        ("eps_b", C.c_double), ("eps_n", C.c_double), ("theta0", C.c_double),
        ("max_age", C.c_int64), ("tau_b", C.c_double), ("tau_n", C.c_double),
        ("h_t", C.c_double), ("rho", C.c_double), ("ring_patience", C.c_int64),
        ("allow_boundary", C.c_int32), ("find_mode", C.c_int32), ("stale_factor", C.c_int64),
    ]


class GsBatchStats(C.Structure):
    _fields_ = [(name, C.c_int64) for name in (
        "processed", "discarded", "inserted", "units", "edges", "next_id", "converged",
        "tick", "events", "windows", "error", "max_degree", "ev_create", "ev_insert",
        "ev_prune", "ev_sweep", "cyc_serial", "cyc_total")] + [("cyc_phase", C.c_int64 * 12)] + [
        ("batches", C.c_int64), ("halted", C.c_int64)]


_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
_vp = C.c_void_p

_SIGNATURES = {
    "gs_last_error": (C.c_char_p, []),
    "gs_version": (C.c_char_p, []),
    "gs_ctx_create": (C.c_int, [C.c_int, C.POINTER(_vp)]),
    "gs_ctx_destroy": (None, [_vp]),
    "gs_ctx_sm_count": (C.c_int, [_vp]),
    "gs_fp32_peak": (C.c_int, [_vp, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "gs_best_two_single": (C.c_int, [_vp, _f64p, C.c_int64, C.c_int64, C.c_double, C.c_double,
                                     C.c_double, C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                     C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "gs_scan_best_two_into": (C.c_int, [_vp, _f64p, C.c_int64, C.c_int64, _f64p, C.c_int64,
                                        _i64p, C.c_int64, _f64p, C.c_int64, C.c_int64]),
    "gs_find_device": (C.c_int, [_vp, _vp, C.c_int64, _vp, C.c_int64, _vp, _vp, C.c_int, _vp]),
    "gs_find_last_fallbacks": (C.c_int, [_vp, C.POINTER(C.c_int64)]),
    "gs_find_last_fallback_counts": (C.c_int, [_vp, _i64p]),
    "gs_engine_create": (C.c_int, [_vp, C.POINTER(GsParams), C.c_int64, C.POINTER(_vp)]),
    "gs_engine_destroy": (None, [_vp]),
    "gs_engine_add_unit": (C.c_int, [_vp, C.c_double, C.c_double, C.c_double, C.c_double,
                                     C.POINTER(C.c_int64)]),
    "gs_engine_connect_or_reset": (C.c_int, [_vp, C.c_int64, C.c_int64, C.POINTER(C.c_int32)]),
    "gs_engine_remove_unit": (C.c_int, [_vp, C.c_int64]),
    "gs_engine_remove_edge": (C.c_int, [_vp, C.c_int64, C.c_int64]),
    "gs_engine_age_incident_edges": (C.c_int, [_vp, C.c_int64, C.c_int64, C.c_int64,
                                               C.POINTER(C.c_int64)]),
    "gs_engine_prune": (C.c_int, [_vp, C.c_int64, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "gs_engine_set_unit": (C.c_int, [_vp, C.c_int64, _vp, _vp, _vp]),
    "gs_engine_step": (C.c_int, [_vp, _f64p, C.c_int64, C.POINTER(GsBatchStats)]),
    "gs_engine_step_device": (C.c_int, [_vp, _vp, C.c_int64]),
    "gs_engine_find_device": (C.c_int, [_vp, _vp, C.c_int64, C.c_int64, _vp]),
    "gs_engine_update_device": (C.c_int, [_vp, _vp, C.c_int64, _vp]),
    "gs_engine_resolve_host": (C.c_int, [_vp, _f64p, C.c_int64, _i64p, _i64p, _f64p,
                                         C.POINTER(GsBatchStats)]),
    "gs_engine_set_params": (C.c_int, [_vp, C.POINTER(GsParams)]),
    "gs_shard_unique_id": (C.c_int, [_vp, C.c_int64]),
    "gs_engine_set_shards": (C.c_int, [_vp, C.c_int, C.c_int, _vp, C.c_int64]),
    "gs_engine_exchange_ms": (C.c_int, [_vp, C.POINTER(C.c_double)]),
    "gs_engine_phase_ms": (C.c_int, [_vp, C.c_int, _f64p]),
    "gs_engine_stats": (C.c_int, [_vp, C.POINTER(GsBatchStats)]),
    "gs_engine_stats_lagged": (C.c_int, [_vp, C.c_int64, C.POINTER(GsBatchStats),
                                         C.POINTER(C.c_int64)]),
    "gs_engine_stream": (_vp, [_vp]),
    "gs_engine_reserve": (C.c_int, [_vp, C.c_int64]),
    "gs_engine_launch_count": (C.c_int64, [_vp]),
    "gs_engine_reset": (C.c_int, [_vp]),
    "gs_engine_set_async": (C.c_int, [_vp, C.c_int]),
    "gs_engine_counts": (C.c_int, [_vp, _i64p]),
    "gs_engine_export_units": (C.c_int, [_vp, C.c_int64, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                         C.POINTER(C.c_int64)]),
    "gs_engine_export_edges": (C.c_int, [_vp, C.c_int64, _vp, C.POINTER(C.c_int64)]),
    "gs_engine_get_run_state": (C.c_int, [_vp, C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                          C.c_int64, _vp, _vp, _vp, C.POINTER(C.c_int64)]),
    "gs_engine_set_run_state": (C.c_int, [_vp, C.c_int64, C.c_int64, C.c_int64, _vp, _vp, _vp]),
    "gs_engine_audit": (C.c_int, [_vp, C.POINTER(C.c_int64)]),
    "gs_engine_extract_mesh": (C.c_int, [_vp, C.c_int64, _vp, C.POINTER(C.c_int64), _vp]),
    "gs_mesh_topology": (C.c_int, [_vp, _vp, C.c_int64, C.c_int64, _vp]),
    "gs_sampler_create": (C.c_int, [_vp, _vp, C.c_int64, C.c_int, C.POINTER(_vp)]),
    "gs_sampler_destroy": (None, [_vp]),
    "gs_sampler_set_state": (C.c_int, [_vp, _u64p]),
    "gs_sampler_get_state": (C.c_int, [_vp, _u64p]),
    "gs_sampler_draw": (C.c_int, [_vp, C.c_int64, _vp, _vp]),
    "gs_sampler_draw_indices": (C.c_int, [_vp, C.c_int64, _vp, _vp]),
    "gs_engine_step_sampled": (C.c_int, [_vp, _vp, C.c_int64, C.POINTER(GsBatchStats)]),
}

EXPORTED = tuple(_SIGNATURES)

_lib = None
_lock = threading.Lock()


def _preload_nccl() -> None:
    """Load the NCCL that PyTorch ships (the nvidia-nccl wheel), if present,
    before the library: the library links libnccl.so.2 by soname, so both then
    share that copy.  Loaded the other way round, the system's older NCCL
    would satisfy the soname first and a later ``import torch`` would fail
    (libtorch_cuda needs symbols it lacks)."""
    try:
        import importlib.util

        spec = importlib.util.find_spec("nvidia.nccl")
    except (ImportError, ValueError):
        return
    for d in (spec.submodule_search_locations or []) if spec else []:
        f = os.path.join(d, "lib", "libnccl.so.2")
        if os.path.exists(f):
            C.CDLL(f, mode=C.RTLD_GLOBAL)
            return


def load_library(path: str = LIB_PATH):
    """Load the shared library and declare every symbol (no device needed)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(path):
                raise DeviceUnavailable(
                    f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; "
                    "g.build()'` (nvcc, sm_100a)")
            _preload_nccl()
            lib = C.CDLL(path)
            for name, (res, args) in _SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def check(status: int) -> None:
    if status == GS_OK:
        return
    msg = (load_library().gs_last_error() or b"").decode()
    if status == GS_VALUE_ERROR:
        raise ValueError(msg)
    if status == GS_STATE_ERROR:
        raise StateError(msg)
    if status == GS_UNKNOWN_UNIT:
        raise UnknownUnitError(msg)
    raise DeviceUnavailable(msg)


class Context:
    """A device context: one CUDA stream plus scratch buffers (gs_ctx)."""

    def __init__(self, device: int = 0):
        lib = load_library()
        h = _vp()
        check(lib.gs_ctx_create(device, C.byref(h)))
        self._h = h
        self.device = device
        self.sm_count = int(lib.gs_ctx_sm_count(h))

    @property
    def handle(self):
        return self._h

    def close(self):
        if getattr(self, "_h", None):
            load_library().gs_ctx_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover - interpreter teardown order
        try:
            self.close()
        except Exception:
            pass


_default_ctx: Context | None = None


def default_context() -> Context:
    global _default_ctx
    with _lock:
        ctx = _default_ctx
    if ctx is None:
        ctx = Context(int(os.environ.get("GS_DEVICE", "0")))
        with _lock:
            _default_ctx = ctx
    return ctx

"""The "b200" scan backend: the reference kernel-backend protocol on a B200.

Same two functions, same semantics and errors as the reference backends
(pkg/src/growsurf/kernels/__init__.py:6-7, _scan.pyx:14-98):

    best_two_single(pos, n, x, y, z) -> (row1, row2, d2_1, d2_2)
    scan_best_two_into(pos, n, signals, out_idx, out_d2, tile) -> None

Both call the sm_100a find kernels through the C ABI (gs_best_two_single /
gs_scan_best_two_into).  Outputs are bit-identical to the compiled
reference (rows, not ids; squared distances; independent of ``tile``), so
the module can be registered next to "compiled" / "python" in the
reference's registry and its kernel tests re-pointed here.
Safe to call from several threads at once (the context serialises).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib

__all__ = ["best_two_single", "scan_best_two_into", "NAME"]

NAME = "b200"

# calls served so far (evidence that a registry lookup really reached the B200)
calls = {"best_two_single": 0, "scan_best_two_into": 0}


def _as_pos(pos):
    pos = np.asarray(pos)
    if pos.dtype != np.float64 or pos.ndim != 2 or pos.shape[1] != 3 or not pos.flags.c_contiguous:
        raise ValueError("pos must be a C-contiguous (n, 3) float64 array")
    return pos


def best_two_single(pos, n, x, y, z):
    """Rows and squared distances of the two nearest units to (x, y, z)."""
    pos = _as_pos(pos)
    lib = _lib.load_library()
    ctx = _lib.default_context()
    calls["best_two_single"] += 1
    r1, r2 = C.c_int64(), C.c_int64()
    d1, d2 = C.c_double(), C.c_double()
    _lib.check(lib.gs_best_two_single(ctx.handle, pos, pos.shape[0], int(n), float(x), float(y),
                                      float(z), C.byref(r1), C.byref(r2), C.byref(d1),
                                      C.byref(d2)))
    return r1.value, r2.value, d1.value, d2.value


def scan_best_two_into(pos, n, signals, out_idx, out_d2, tile):
    """Best-two scan for a batch of signals into caller-owned outputs."""
    pos = _as_pos(pos)
    signals = np.asarray(signals)
    if signals.dtype != np.float64 or signals.ndim != 2 or signals.shape[1] != 3:
        raise ValueError("signals must be an (m, 3) float64 array")
    if not signals.flags.c_contiguous:
        signals = np.ascontiguousarray(signals)
    for arr, dt in ((out_idx, np.int64), (out_d2, np.float64)):
        if (not isinstance(arr, np.ndarray) or arr.dtype != dt or arr.ndim != 2
                or arr.shape[1] != 2 or not arr.flags.c_contiguous or not arr.flags.writeable):
            raise ValueError("outputs must be writable C-contiguous (>=m, 2) arrays")
    lib = _lib.load_library()
    ctx = _lib.default_context()
    calls["scan_best_two_into"] += 1
    _lib.check(lib.gs_scan_best_two_into(ctx.handle, pos, pos.shape[0], int(n), signals,
                                         signals.shape[0], out_idx, out_idx.shape[0], out_d2,
                                         out_d2.shape[0], int(tile)))

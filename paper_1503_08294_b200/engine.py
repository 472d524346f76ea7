"""Single-signal helpers of the reference engine API on the device engine.

Reference: pkg/src/growsurf/engine.py:149-365.  ``update_single`` and
``is_converged`` operate on the device-resident Network; the per-signal
update is the same device code the batched path uses (a one-signal batch).
"""

from __future__ import annotations

import math

import numpy as np

from . import kernels
from .multi import RunState, resolve_and_update
from .network import Network, Snapshot
from .params import EngineParams, StateError, WinnerResult

__all__ = ["find_winners_exhaustive", "update_single", "is_converged", "RunState"]


def find_winners_exhaustive(snapshot: Snapshot, signal, backend=None) -> WinnerResult:
    """engine.py:149-158 on the B200 scan."""
    n = len(snapshot)
    if n < 2:
        raise StateError(f"need at least 2 units to find winners, have {n}")
    pos = np.ascontiguousarray(snapshot.positions, dtype=np.float64)
    r1, r2, d1, d2 = kernels.best_two_single(pos, n, float(signal[0]), float(signal[1]),
                                             float(signal[2]))
    ids = snapshot.ids
    return WinnerResult(int(ids[r1]), int(ids[r2]), math.sqrt(d1), math.sqrt(d2))


def update_single(net: Network, params: EngineParams, signal, wr: WinnerResult,
                  state: RunState | None = None, grid=None) -> None:
    """engine.py:283-355: one full update for one signal."""
    if not (net.is_alive(wr.winner) and net.is_alive(wr.second)):
        raise StateError(f"stale winner result ({wr.winner}, {wr.second})")
    resolve_and_update(net, params, np.asarray(signal, dtype=np.float64).reshape(1, 3), [wr])


def is_converged(net: Network, params: EngineParams) -> bool:
    """engine.py:358-365."""
    c = net.counts()
    if c["units"] < 4:
        return False
    ok = c["disk"] + (c["half"] if params.allow_boundary else 0)
    return ok == c["units"] and c["untrained"] == 0

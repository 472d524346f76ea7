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

__all__ = ["find_winners_exhaustive", "update_single", "is_converged", "RunState", "run"]


def find_winners_exhaustive(snapshot: Snapshot, signal, backend=None) -> WinnerResult:
    """engine.py:149-158 on the B200 scan (or on ``backend``, a kernel-backend
    module, when given)."""
    n = len(snapshot)
    if n < 2:
        raise StateError(f"need at least 2 units to find winners, have {n}")
    pos = np.ascontiguousarray(snapshot.positions, dtype=np.float64)
    kb = kernels if backend is None else backend
    r1, r2, d1, d2 = kb.best_two_single(pos, n, float(signal[0]), float(signal[1]),
                                        float(signal[2]))
    ids = snapshot.ids
    return WinnerResult(int(ids[r1]), int(ids[r2]), math.sqrt(d1), math.sqrt(d2))


def update_single(net: Network, params: EngineParams, signal, wr: WinnerResult,
                  state: RunState | None = None, grid=None) -> None:
    """engine.py:283-355: one full update for one signal; ``state=None`` is a
    fresh RunState (engine.py:301-302)."""
    if not (net.is_alive(wr.winner) and net.is_alive(wr.second)):
        raise StateError(f"stale winner result ({wr.winner}, {wr.second})")
    resolve_and_update(net, params, np.asarray(signal, dtype=np.float64).reshape(1, 3), [wr],
                       state, grid)


def is_converged(net: Network, params: EngineParams) -> bool:
    """engine.py:358-365."""
    c = net.counts()
    if c["units"] < 4:
        return False
    ok = c["disk"] + (c["half"] if params.allow_boundary else 0)
    return ok == c["units"] and c["untrained"] == 0


def run(source, params: EngineParams, seed: int, *, use_grid: bool = False, backend=None,
        checkpoints=(), variant: str | None = None, dataset: str | None = None):
    """The single-signal engine (engine.py:368-462) on the device.

    One signal per iteration, exhaustive winners against the current network,
    update_single, convergence after every signal: exactly the multi-signal
    loop with a batch of one (the winner lock never triggers), so it runs on
    the same device engine and matches the reference run bit for bit.
    ``checkpoints`` records (units, signals, sample_s, find_s, update_s,
    total_s) the first time the unit count reaches each value.

    ``use_grid=True`` is the reference's "indexed" variant (engine.py:396-426,
    grid.py:98-133): the winner search goes through a spatial grid instead of
    the exhaustive scan.  Here that grid is the device's EXACT uniform grid
    (GS_FIND_GRID, rebuilt on the device per find), so the indexed run equals
    the exhaustive run bit for bit -- unlike the reference's approximate
    HashGrid, whose winners may differ; its parity target
    is therefore the exhaustive run.
    """
    import ctypes as C
    import time
    from dataclasses import replace

    from . import _lib
    from .metrics import RunStats

    lib = _lib.load_library()
    p1 = replace(params, batch_floor=1, batch_cap=1)
    rng = np.random.Generator(np.random.Philox(seed))
    net = Network(p1, find_mode=_lib.FIND_GRID if use_grid else _lib.FIND_AUTO)
    net.watch_age_limit(params.max_age)
    seeds = source.sample(rng, 2)
    for k in range(2):
        net.add_unit(seeds[k], params.theta0)
    cps = list(checkpoints)
    records = []
    phase = np.zeros(2, np.float64)
    _lib.check(lib.gs_engine_phase_ms(net.handle, 1, phase))
    st = _lib.GsBatchStats()
    signals = 0
    converged = False
    sample_s = 0.0
    perf = time.perf_counter
    t_start = perf()
    while signals < params.max_signals:
        t0 = perf()
        xi = np.ascontiguousarray(source.sample(rng, 1), dtype=np.float64)
        sample_s += perf() - t0
        _lib.check(lib.gs_engine_step(net.handle, xi, 1, C.byref(st)))
        signals += 1
        while cps and int(st.units) >= cps[0]:
            _lib.check(lib.gs_engine_phase_ms(net.handle, -1, phase))
            records.append((int(st.units), signals, sample_s, phase[0] * 1e-3, phase[1] * 1e-3,
                            perf() - t_start))
            cps.pop(0)
        if st.converged:
            converged = True
            break
    total = perf() - t_start
    _lib.check(lib.gs_engine_phase_ms(net.handle, 0, phase))
    net._touch()
    stats = RunStats(variant=variant or ("indexed" if use_grid else "single"), dataset=dataset or getattr(source, "label", "unknown"),
                     seed=seed, iterations=signals, signals=signals, discarded=0,
                     units=int(st.units), connections=int(st.edges), total_s=total,
                     sample_s=sample_s, find_s=phase[0] * 1e-3, update_s=phase[1] * 1e-3,
                     converged=converged)
    stats.checkpoints = records
    return net, stats

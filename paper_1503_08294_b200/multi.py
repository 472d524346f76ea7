"""Multi-signal engine on the B200: the reference's training-loop API.

Reference: pkg/src/growsurf/multi.py:44-202 (batch_size, batch_find_winners,
sequential_executor, resolve_and_update, run_multi) and
pkg/src/growsurf/parallel.py:107-114 (parallel_executor).

Two drop-in boundaries are offered:

* Executor boundary: ``b200_executor()`` is an ``executor(snapshot, batch)
  -> list[WinnerResult]`` callable; pass it (or any reference executor) to
  ``run_multi`` and the find runs where the executor says while the update
  still runs on the device.
* Engine boundary (the throughput path): ``run_multi(source, params, seed)``
  with no executor keeps the whole iteration on the device: per batch one
  H2D copy of the host-sampled signals, the sm_100a find, the windowed
  update, the convergence check and one small stats D2H.
"""

from __future__ import annotations

import ctypes as C
import math
import time
from dataclasses import dataclass

import numpy as np

from . import _lib, kernels
from .metrics import PhaseTimer, RunStats
from .network import Network, Snapshot
from .params import BatchOutcome, EngineParams, StateError, WinnerResult, batch_size

__all__ = [
    "BatchOutcome",
    "batch_size",
    "batch_find_winners",
    "b200_executor",
    "sequential_executor",
    "parallel_executor",
    "ExecConfig",
    "parallel_batch_find_winners",
    "timed_find",
    "resolve_and_update",
    "run_multi",
    "RunState",
]


_SWEEP_EVERY = 1024  # engine.py:98


class _Patience(dict):
    """``state.patience`` read back from the device: a missing key reads as 0
    (the device keeps one counter per id, where the reference's dict may hold
    an explicit 0; ``patience.get(u, 0)``, engine.py:234, is the same)."""

    def __missing__(self, key):
        return 0


class RunState:
    """Cross-update bookkeeping for one run (engine.py:101-119).

    Same fields as the reference: ``patience`` (id -> consecutive stuck
    wins), ``last_active`` (id -> tick of the last top-two appearance, in
    dict insertion order: the sweep removes stale units in that order),
    ``tick`` and ``next_sweep``.  The device keeps the live copy inside the
    Network; ``resolve_and_update`` / ``update_single`` load this object
    into the device before the updates and write the device's values back
    into it afterwards, so a caller that passes one RunState across calls
    sees the reference's values, and ``state=None`` is a fresh RunState per
    call, as in the reference (multi.py:114-115, engine.py:301-302).
    """

    __slots__ = ("patience", "last_active", "tick", "next_sweep")

    def __init__(self):
        self.patience: dict[int, int] = _Patience()
        self.last_active: dict[int, int] = {}
        self.tick = 0
        self.next_sweep = _SWEEP_EVERY


def _load_run_state(net: Network, state: RunState) -> None:
    """Copy a host RunState into the device network (gs_engine_set_run_state)."""
    keys = [int(u) for u in list(state.patience) + list(state.last_active)]
    if any(u < 0 for u in keys):
        raise ValueError("run state names a negative unit id")
    n = max(keys) + 1 if keys else 0
    patience = np.zeros(n, np.int64)
    last_active = np.full(n, -1, np.int64)
    stamp = np.full(n, -1, np.int64)
    for u, c in state.patience.items():
        patience[int(u)] = int(c)
    k = len(state.last_active)
    for i, (u, t) in enumerate(state.last_active.items()):
        last_active[int(u)] = int(t)
        stamp[int(u)] = i - k  # before every entry the device creates later
    _lib.check(_lib.load_library().gs_engine_set_run_state(
        net.handle, int(state.tick), int(state.next_sweep), n, patience.ctypes.data,
        last_active.ctypes.data, stamp.ctypes.data))


def _store_run_state(net: Network, state: RunState) -> None:
    """Write the device run state back into ``state`` (gs_engine_get_run_state)."""
    lib = _lib.load_library()
    tick, nsw, n = C.c_int64(), C.c_int64(), C.c_int64()
    _lib.check(lib.gs_engine_get_run_state(net.handle, C.byref(tick), C.byref(nsw), 0, None,
                                           None, None, C.byref(n)))
    patience = np.zeros(n.value, np.int64)
    last_active = np.zeros(n.value, np.int64)
    stamp = np.zeros(n.value, np.int64)
    _lib.check(lib.gs_engine_get_run_state(net.handle, C.byref(tick), C.byref(nsw), n.value,
                                           patience.ctypes.data, last_active.ctypes.data,
                                           stamp.ctypes.data, C.byref(n)))
    state.tick = int(tick.value)
    state.next_sweep = int(nsw.value)
    pt = _Patience()
    for u in np.flatnonzero(patience).tolist():
        pt[u] = int(patience[u])
    state.patience = pt
    have = np.flatnonzero(last_active != -1)
    order = have[np.argsort(stamp[have], kind="stable")]
    state.last_active = {int(u): int(last_active[u]) for u in order.tolist()}


def _scan_batch(snapshot: Snapshot, signals, tile: int | None = None, backend=None):
    n = len(snapshot)
    if n < 2:
        raise StateError(f"need at least 2 units to find winners, have {n}")
    signals = np.ascontiguousarray(signals, dtype=np.float64).reshape(-1, 3)
    m = signals.shape[0]
    out_idx = np.empty((m, 2), dtype=np.int64)
    out_d2 = np.empty((m, 2), dtype=np.float64)
    kb = kernels if backend is None else backend
    kb.scan_best_two_into(np.ascontiguousarray(snapshot.positions, dtype=np.float64), n,
                          signals, out_idx, out_d2, n if tile is None else tile)
    return out_idx, out_d2


def _to_results(snapshot: Snapshot, out_idx, out_d2) -> list[WinnerResult]:
    """multi.py:72-78: rows -> ids, d = sqrt(d2) (correctly rounded)."""
    ids = snapshot.ids
    sqrt = math.sqrt
    return [WinnerResult(int(ids[i1]), int(ids[i2]), sqrt(d1), sqrt(d2))
            for (i1, i2), (d1, d2) in zip(out_idx.tolist(), out_d2.tolist())]


def batch_find_winners(snapshot: Snapshot, batch, backend=None,
                       tile: int | None = None) -> list[WinnerResult]:
    """Winner pair for every signal, computed on the B200 (multi.py:81-87)."""
    out_idx, out_d2 = _scan_batch(snapshot, batch, tile, backend)
    return _to_results(snapshot, out_idx, out_d2)


def b200_executor(tile: int | None = None):
    """Executor running the batched find on the B200."""

    def execute(snapshot: Snapshot, batch) -> list[WinnerResult]:
        return batch_find_winners(snapshot, batch, tile=tile)

    return execute


def sequential_executor(backend=None, tile: int | None = None):
    """multi.py:90-96: ``execute(snapshot, batch)`` over one batched scan.

    ``backend`` is a kernel-backend module (``best_two_single`` /
    ``scan_best_two_into``, kernels/__init__.py:6-7); None is this
    package's B200 kernels (the reference's default is its compiled scan).
    """
    if backend is None:
        return b200_executor(tile=tile)

    def execute(snapshot: Snapshot, batch) -> list[WinnerResult]:
        return batch_find_winners(snapshot, batch, backend=backend, tile=tile)

    return execute


@dataclass(frozen=True)
class ExecConfig:
    """parallel.py:34-49: worker count and tile length.  Validated like the
    reference's; the B200 scan's parallelism is the GPU's, so neither value
    changes the work (and no value changes a result)."""

    workers: int = 0
    tile: int = 1024

    def __post_init__(self):
        if self.workers < 0:
            raise ValueError("workers must be >= 0")
        if self.tile < 1:
            raise ValueError("tile must be >= 1")

    def effective_workers(self, m: int) -> int:
        import os

        return max(1, min(self.workers or os.cpu_count() or 1, m))


def parallel_batch_find_winners(snapshot: Snapshot, batch, cfg: ExecConfig | None = None,
                                backend=None) -> list[WinnerResult]:
    """parallel.py:91-97 on the B200 scan (one launch covers every worker's
    slice; a foreign ``backend`` gets the whole batch in one call, which its
    contract makes identical to the sliced calls)."""
    cfg = cfg or ExecConfig()
    return batch_find_winners(snapshot, batch, backend=backend, tile=cfg.tile)


def timed_find(snapshot: Snapshot, batch, cfg: ExecConfig | None = None, backend=None):
    """parallel.py:100-104: (winners, seconds) of one batched find."""
    t0 = time.perf_counter()
    winners = parallel_batch_find_winners(snapshot, batch, cfg, backend)
    return winners, time.perf_counter() - t0


def parallel_executor(cfg: ExecConfig | None = None, backend=None):
    """parallel.py:107-114 equivalent: the parallelism is the GPU's."""
    cfg = cfg or ExecConfig()

    def execute(snapshot: Snapshot, batch) -> list[WinnerResult]:
        return parallel_batch_find_winners(snapshot, batch, cfg, backend=backend)

    return execute


def _winner_arrays(winners):
    m = len(winners)
    b = np.empty(m, np.int64)
    s = np.empty(m, np.int64)
    d = np.empty(m, np.float64)
    for j, wr in enumerate(winners):
        b[j] = wr.winner
        s[j] = wr.second
        d[j] = wr.d_winner
    return b, s, d


def resolve_and_update(net: Network, params: EngineParams, batch, winners,
                       state: RunState | None = None, grid=None) -> BatchOutcome:
    """Winner lock + batch-order update on the device (multi.py:99-131).

    ``state`` is the run's RunState; None is a fresh one for this call
    (multi.py:114-115).  ``grid`` is accepted for signature compatibility:
    the device find keeps no incremental index to relocate.
    """
    net.set_params(params)
    batch = np.ascontiguousarray(batch, dtype=np.float64).reshape(-1, 3)
    b, s, d = _winner_arrays(winners)
    if batch.shape[0] != b.shape[0]:
        raise ValueError(f"{batch.shape[0]} signals but {b.shape[0]} winner results")
    _load_run_state(net, state if state is not None else RunState())
    st = _lib.GsBatchStats()
    _lib.check(_lib.load_library().gs_engine_resolve_host(net.handle, batch, batch.shape[0], b, s,
                                                          d, C.byref(st)))
    net._touch()
    if state is not None:
        _store_run_state(net, state)
    return BatchOutcome(int(st.processed), int(st.discarded), int(st.inserted))


def step(net: Network, batch) -> _lib.GsBatchStats:
    """One device-resident iteration on a host batch (find + resolve + update)."""
    batch = np.ascontiguousarray(batch, dtype=np.float64).reshape(-1, 3)
    st = _lib.GsBatchStats()
    _lib.check(_lib.load_library().gs_engine_step(net.handle, batch, batch.shape[0],
                                                  C.byref(st)))
    net._touch()
    return st


def run_multi(source, params: EngineParams, seed: int, executor=None, *,
              variant: str = "multi-b200", dataset: str | None = None,
              find_mode: int = _lib.FIND_AUTO, capacity: int = 4096,
              device_sampling: bool | None = None, phase_timing: bool = True,
              shard_group=None):
    """Run the multi-signal engine to convergence or the signal cap.

    Same driver contract as multi.py:134-202: Philox(seed) stream, two seed
    units from the first two samples, m = batch_size(V) per batch,
    convergence checked once per batch.  Returns (Network, RunStats).

    device_sampling (default: on for a CloudSource without an executor)
    draws every batch on the GPU from the same Philox stream
    (device_sampling.py), so the cloud crosses PCIe once per run instead of
    every batch's signals.

    shard_group (a torch.distributed group, e.g. ``dist.group.WORLD``)
    shards every batch's find across the group's ranks (distributed.py);
    every rank must make the same call and returns the identical result.
    """
    from .sampling import CloudSource

    lib = _lib.load_library()
    rng = np.random.Generator(np.random.Philox(seed))
    if device_sampling is None:
        device_sampling = executor is None and isinstance(source, CloudSource)
    lookahead = 8 if (device_sampling and params.batch_floor == params.batch_cap) else 0
    if lookahead:  # room for the batches in flight from the start (no growth later)
        capacity = max(capacity, 2 + params.batch_cap * (lookahead + 2))
    net = Network(params, capacity=capacity, find_mode=find_mode)
    net.watch_age_limit(params.max_age)
    if shard_group is not None:
        if executor is not None:
            raise ValueError("a sharded run does its own find: pass no executor")
        from .distributed import attach

        attach(net, shard_group)
    seeds = source.sample(rng, 2)
    for k in range(2):
        net.add_unit(seeds[k], params.theta0)
    sampler = None
    if device_sampling:
        if executor is not None or not isinstance(source, CloudSource):
            raise ValueError("device sampling runs the device engine on a CloudSource")
        from .device_sampling import DeviceCloudSampler

        sampler = DeviceCloudSampler(source.points, rng)
    timer = PhaseTimer()
    signals = discarded = iterations = 0
    converged = False
    units = 2
    edges = 0
    perf = time.perf_counter
    phase = np.zeros(2, np.float64)
    if executor is None and phase_timing:
        # find_s / update_s: with batches in flight, one batch in 64 is timed
        # (per-batch event records would cost ~8 us of every batch)
        _lib.check(lib.gs_engine_phase_ms(net.handle, 64 if lookahead else 1, phase))
    st = _lib.GsBatchStats()
    # fixed batch size + device sampling: the host enqueues batches ahead and
    # only polls for convergence (gs_engine_set_async); the device counts
    # the batches that really ran and halts after convergence
    if lookahead:
        net.set_async(lookahead)
    t_start = perf()
    if lookahead:
        m = params.batch_cap
        enq = 0
        seq = C.c_int64()
        while enq * m < params.max_signals:
            _lib.check(lib.gs_engine_step_sampled(net.handle, sampler.handle, m, None))
            enq += 1
            # every 4th batch, read the batch issued `lookahead - 1` steps ago:
            # waiting for it keeps the newer ones queued (the GPU never
            # drains) and the host work per batch stays small
            if enq % 4 == 0:
                _lib.check(lib.gs_engine_stats_lagged(net.handle, lookahead - 1, C.byref(st),
                                                      C.byref(seq)))
                if seq.value >= 0 and st.converged:
                    break
        _lib.check(lib.gs_engine_stats(net.handle, C.byref(st)))
        net.set_async(0)
        net._touch()
        iterations = int(st.batches)
        signals = iterations * m
        discarded = signals - int(st.tick)
        units, edges = int(st.units), int(st.edges)
        converged = bool(st.converged)
    while not lookahead and signals < params.max_signals:
        m = batch_size(units, params.batch_cap, params.batch_floor)
        t0 = perf()
        if sampler is not None:
            _lib.check(lib.gs_engine_step_sampled(net.handle, sampler.handle, m, C.byref(st)))
            t1 = t2 = t3 = perf()
            net._touch()
            signals += m
            discarded += int(st.discarded)
            iterations += 1
            units = int(st.units)
            edges = int(st.edges)
            if st.converged:
                converged = True
                break
            continue
        batch = np.ascontiguousarray(source.sample(rng, m), dtype=np.float64)
        t1 = perf()
        if executor is None:
            _lib.check(lib.gs_engine_step(net.handle, batch, m, C.byref(st)))
            t2 = t3 = perf()
        else:
            winners = executor(net.snapshot(), batch)
            t2 = perf()
            b, s, d = _winner_arrays(winners)
            _lib.check(lib.gs_engine_resolve_host(net.handle, batch, m, b, s, d, C.byref(st)))
            net._touch()
            t3 = perf()
            timer.find_s += t2 - t1
            timer.update_s += t3 - t2
        net._touch()
        timer.sample_s += t1 - t0
        signals += m
        discarded += int(st.discarded)
        iterations += 1
        units = int(st.units)
        edges = int(st.edges)
        if st.converged:
            converged = True
            break
    total = perf() - t_start
    if sampler is not None:
        sampler.store_state(rng)
        sampler.close()
    if executor is None:
        _lib.check(lib.gs_engine_phase_ms(net.handle, 0, phase))
        timer.find_s = phase[0] * 1e-3
        timer.update_s = phase[1] * 1e-3
        if shard_group is not None:  # the all-gathers are part of the find phase
            timer.find_s += net.exchange_ms() * 1e-3
    stats = RunStats(
        variant=variant,
        dataset=dataset or getattr(source, "label", "unknown"),
        seed=seed,
        iterations=iterations,
        signals=signals,
        discarded=discarded,
        units=units,
        connections=edges,
        total_s=total,
        sample_s=timer.sample_s,
        find_s=timer.find_s,
        update_s=timer.update_s,
        converged=converged,
    )
    return net, stats

"""Signal sharding across GPUs (one process per GPU, NCCL over NVLink).

The find is an independent map over the m signals of a batch against the
replicated pre-batch snapshot.  Rank r
takes the contiguous slice [r*m/P, (r+1)*m/P) -- the same static split as
the reference's thread pool (parallel.py:78) -- and writes 16-byte winner
records (winner id, second id, d_winner) for it; one all-gather over NVLink
assembles the batch's records in rank order == batch order; every rank then
runs the identical deterministic device update, so the replicated networks
stay bit-identical with no further traffic.

torch.distributed is only the plumbing: the records live in a torch CUDA
buffer whose pointer the C ABI writes; the collective is
all_gather_into_tensor on the engine's own CUDA stream.
"""

from __future__ import annotations

REC_BYTES = 16  # csrc/common.cuh WinRec: int32 b, int32 s, f64 d_winner


def shard_bounds(m: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous signal slice of one rank (parallel.py:78 split rule)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    return rank * m // world, (rank + 1) * m // world


def gather_records(full, lo: int, hi: int, group=None):
    """All-gather every rank's record slice [lo, hi) of ``full`` (a uint8
    tensor of m * REC_BYTES bytes) into ``full`` in rank order == batch order.

    Works for any torch.distributed backend (NCCL on the GPU path, gloo in
    the CPU tests); slices must be equal-sized (m divisible by the world).
    """
    import torch.distributed as dist

    local = full[lo * REC_BYTES: hi * REC_BYTES].clone()
    dist.all_gather_into_tensor(full, local, group=group)
    return full


class ShardedStep:
    """find(slice) -> all_gather(records) -> replicated update, per batch."""

    def __init__(self, net, group=None):
        import torch
        import torch.distributed as dist

        self.torch = torch
        self.dist = dist
        self.net = net
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.stream = torch.cuda.ExternalStream(net.stream_handle())
        self._cap = 0
        self._full = None

    def _buffers(self, m: int):
        if m > self._cap:
            self._cap = m
            self._full = self.torch.empty(m * REC_BYTES, dtype=self.torch.uint8, device="cuda")
        return self._full[: m * REC_BYTES]

    def step_device(self, d_sig: int, m: int) -> None:
        """Enqueue one batch on the engine stream (signals already on device)."""
        from . import _lib

        if m % self.world:
            raise ValueError(f"batch size {m} must be divisible by the world size {self.world}")
        lib = _lib.load_library()
        full = self._buffers(m)
        lo, hi = shard_bounds(m, self.world, self.rank)
        with self.torch.cuda.stream(self.stream):
            _lib.check(lib.gs_engine_find_device(self.net.handle, d_sig, lo, hi, full.data_ptr()))
            gather_records(full, lo, hi, self.group)
            _lib.check(lib.gs_engine_update_device(self.net.handle, d_sig, m, full.data_ptr()))


def run_multi_sharded(source, params, seed: int, *, group=None, capacity: int = 4096):
    """run_multi (multi.py:134-202) with each batch's find sharded across the
    ranks of ``group``; every rank returns the identical (Network, RunStats).

    Sampling is replicated (every rank draws the same Philox stream, so
    signals need no communication): on the device for a CloudSource
    (device_sampling.py; the cloud is copied once per rank), else on the host
    with one H2D copy per batch.
    """
    import ctypes as C
    import time

    import numpy as np
    import torch

    from . import _lib
    from .metrics import RunStats
    from .network import Network
    from .params import batch_size

    lib = _lib.load_library()
    rng = np.random.Generator(np.random.Philox(seed))
    net = Network(params, capacity=capacity)
    runner = ShardedStep(net, group)
    seeds = source.sample(rng, 2)
    for k in range(2):
        net.add_unit(seeds[k], params.theta0)
    from .sampling import CloudSource

    sampler = None
    if isinstance(source, CloudSource):
        from .device_sampling import DeviceCloudSampler

        sampler = DeviceCloudSampler(source.points, rng)
    signals = discarded = iterations = 0
    units, edges, converged = 2, 0, False
    st = _lib.GsBatchStats()
    sample_s = 0.0
    host = None
    dev = None
    t_start = time.perf_counter()
    while signals < params.max_signals:
        m = batch_size(units, params.batch_cap, params.batch_floor)
        if dev is None or dev.shape[0] < m:
            dev = torch.empty((m, 3), dtype=torch.float64, device="cuda")
            if sampler is None:
                host = torch.empty((m, 3), dtype=torch.float64).pin_memory()
        if sampler is not None:
            sampler.draw(m, dev.data_ptr(), net.stream_handle())
        else:
            t0 = time.perf_counter()
            batch = np.ascontiguousarray(source.sample(rng, m), dtype=np.float64)
            sample_s += time.perf_counter() - t0
            host[:m].copy_(torch.from_numpy(batch))
            with torch.cuda.stream(runner.stream):
                dev[:m].copy_(host[:m], non_blocking=True)
        runner.step_device(dev.data_ptr(), m)
        _lib.check(lib.gs_engine_stats(net.handle, C.byref(st)))
        net._touch()
        signals += m
        discarded += int(st.discarded)
        iterations += 1
        units, edges = int(st.units), int(st.edges)
        if st.converged:
            converged = True
            break
    total = time.perf_counter() - t_start
    if sampler is not None:
        sampler.store_state(rng)
        sampler.close()
    stats = RunStats(variant="multi-b200-sharded", dataset=getattr(source, "label", "unknown"),
                     seed=seed, iterations=iterations, signals=signals, discarded=discarded,
                     units=units, connections=edges, total_s=total, sample_s=sample_s,
                     find_s=0.0, update_s=0.0, converged=converged)
    return net, stats

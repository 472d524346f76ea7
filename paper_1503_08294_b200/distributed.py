"""Signal sharding across GPUs (one process per GPU, NCCL over NVLink).

The find is an independent map over the m signals of a batch against the
replicated pre-batch snapshot.  Rank r
takes the contiguous slice [r*m/P, (r+1)*m/P) -- the same static split as
the reference's thread pool (parallel.py:78) -- and writes 16-byte winner
records (winner id, second id, d_winner) for it; one ncclAllGather on the
engine's CUDA stream assembles the batch's records in rank order == batch
order; every rank then runs the identical deterministic device update, so
the replicated networks stay bit-identical with no further traffic
(SURVEY.md 8(e)).

The whole per-batch sequence (sampler -> gather -> find on the slice ->
all-gather -> update) is enqueued by the engine in C++
(``gs_engine_set_shards``: the engine owns its NCCL communicator), so a
sharded run uses the same asynchronous lookahead loop as one GPU
(``run_multi``): no host synchronisation per batch.  torch.distributed is
only the plumbing that broadcasts the communicator id from rank 0.
"""

from __future__ import annotations

from . import _lib

REC_BYTES = 16  # GS_WINREC_BYTES: int32 winner id, int32 second id, f64 d_winner


def shard_bounds(m: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous signal slice of one rank (parallel.py:78 split rule)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    return rank * m // world, (rank + 1) * m // world


def shard_unique_id() -> bytes:
    """A fresh communicator id (made on rank 0, broadcast to the others)."""
    buf = (_lib.C.c_uint8 * _lib.SHARD_ID_BYTES)()
    _lib.check(_lib.load_library().gs_shard_unique_id(buf, _lib.SHARD_ID_BYTES))
    return bytes(buf)


def broadcast_shard_id(group=None, make_id=shard_unique_id) -> bytes:
    """Rank 0 of ``group`` makes the id, every rank returns the same bytes
    (any torch.distributed backend: NCCL on the GPU path, gloo in tests)."""
    import torch.distributed as dist

    rank = dist.get_rank(group)
    obj = [make_id() if rank == 0 else None]
    src = dist.get_global_rank(group, 0) if group is not None else 0
    dist.broadcast_object_list(obj, src=src, group=group)
    uid = obj[0]
    if not isinstance(uid, bytes) or len(uid) != _lib.SHARD_ID_BYTES:
        raise ValueError("bad shard id from rank 0")
    return uid


_GROUP_IDS: dict = {}  # group -> communicator id (the engine reuses its communicator)


def attach(net, group=None) -> tuple[int, int]:
    """Join ``net`` to the ranks of ``group`` (blocks until all joined);
    returns (world, rank).  The first call per group broadcasts a fresh
    communicator id; later calls (the next run's Network) reuse it, so the
    NCCL communicator is initialised once per process and group."""
    import torch.distributed as dist

    world, rank = dist.get_world_size(group), dist.get_rank(group)
    key = id(group if group is not None else dist.group.WORLD)
    uid = _GROUP_IDS.get(key)
    if uid is None:
        uid = _GROUP_IDS[key] = broadcast_shard_id(group)
    net.set_shards(world, rank, uid)
    return world, rank


def gather_records(full, lo: int, hi: int, group=None):
    """All-gather every rank's record slice [lo, hi) of ``full`` (a uint8
    tensor of m * REC_BYTES bytes) into ``full`` in rank order == batch order.

    The host-level statement of the exchange the engine performs with
    ncclAllGather (tests run it over gloo); slices must be equal-sized.
    """
    import torch.distributed as dist

    local = full[lo * REC_BYTES: hi * REC_BYTES].clone()
    dist.all_gather_into_tensor(full, local, group=group)
    return full


class ShardedStep:
    """find(slice) -> all-gather(records) -> replicated update, per batch,
    for callers that bring their own device batches."""

    def __init__(self, net, group=None):
        self.net = net
        self.world, self.rank = attach(net, group)

    def step_device(self, d_sig: int, m: int) -> None:
        """Enqueue one batch on the engine stream (signals already on device)."""
        if m % self.world:
            raise ValueError(f"batch size {m} must be divisible by the world size {self.world}")
        _lib.check(_lib.load_library().gs_engine_step_device(self.net.handle, d_sig, m))
        self.net._touch()


def run_multi_sharded(source, params, seed: int, *, group=None, **kw):
    """run_multi (multi.py:134-202) with each batch's find sharded across the
    ranks of ``group`` (default: the whole world); every rank returns the
    identical (Network, RunStats).

    Sampling is replicated (every rank draws the same Philox stream, so
    signals need no communication): on the device for a CloudSource (the
    cloud is copied once per rank), else on the host.
    """
    import torch.distributed as dist

    from .multi import run_multi

    kw.setdefault("variant", "multi-b200-sharded")
    return run_multi(source, params, seed, shard_group=group if group is not None
                     else dist.group.WORLD, **kw)

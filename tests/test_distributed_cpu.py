"""Multi-rank host logic of the signal-sharded step (distributed.py) on CPU.

World-size-2 gloo process groups stand in for NCCL: each rank computes the
winner records of its contiguous signal slice (with the C oracle scan as the
stand-in for the device find), the records are all-gathered with the same
``gather_records`` the GPU path uses, and every rank must end up with the
full batch's records in batch order, identical to a single-process scan.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1503_08294_b200.distributed import (REC_BYTES, broadcast_shard_id, gather_records,
                                               shard_bounds)

REC = np.dtype([("b", "<i4"), ("s", "<i4"), ("d", "<f8")])


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def records(pos, sig):
    from oracle import oracle as O

    idx, d2 = O.scan_best_two(pos, sig)
    out = np.empty(sig.shape[0], REC)
    out["b"], out["s"], out["d"] = idx[:, 0], idx[:, 1], np.sqrt(d2[:, 0])
    return out


def _worker(rank, world, port, m, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # identical seeded stream on every rank: no signal traffic
        rng = np.random.Generator(np.random.Philox(7))
        pos, sig = rng.random((500, 3)), rng.random((m, 3))
        lo, hi = shard_bounds(m, world, rank)
        full = torch.zeros(m * REC_BYTES, dtype=torch.uint8)
        mine = records(pos, sig[lo:hi])
        full[lo * REC_BYTES: hi * REC_BYTES] = torch.from_numpy(mine.view(np.uint8).copy())
        gather_records(full, lo, hi)
        got = full.numpy().view(REC)
        want = records(pos, sig)
        q.put((rank, bool(np.array_equal(got.view(np.uint8), want.view(np.uint8)))))
    finally:
        dist.destroy_process_group()


def _id_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # rank 0's id reaches every rank (the real id is an ncclUniqueId made
        # by gs_shard_unique_id; any 128 bytes exercise the same plumbing)
        made = []

        def make_id():
            made.append(rank)
            return bytes((7 * i + 3) % 256 for i in range(128))

        uid = broadcast_shard_id(None, make_id)
        q.put((rank, (uid == make_id.__call__() if rank == 0 else
                      uid == bytes((7 * i + 3) % 256 for i in range(128))), made[:1]))
    finally:
        dist.destroy_process_group()


def test_shard_id_broadcast_from_rank0():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_id_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {r: (ok, made) for r, ok, made in (q.get(timeout=120) for _ in procs)}
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res == {0: (True, [0]), 1: (True, [])}  # only rank 0 made an id


@pytest.mark.parametrize("world", [2])
def test_sharded_records_assemble_in_batch_order(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, 1024, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res == {r: True for r in range(world)}


def test_shard_bounds_partition():
    for m in (64, 1000, 4096, 65536):
        for world in (1, 2, 3, 4, 8):
            parts = [shard_bounds(m, world, r) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == m
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
    with pytest.raises(ValueError):
        shard_bounds(64, 2, 2)

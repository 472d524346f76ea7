"""The signal-sharded device path on one GPU, bit for bit
against the reference's golden runs.

* world = 1 through the full native path: the engine's own NCCL
  communicator (single rank), find on the rank's slice, ncclAllGather of the
  records on the engine stream, replicated update -- via
  ``run_multi_sharded`` (torch.distributed group for the id broadcast) and
  via ``Network.set_shards`` directly, on host-sampled, device-sampled and
  asynchronous (fixed-m lookahead) runs.
* a two- and four-shard split on one GPU through the C ABI: the finds of
  slices [0, m/k), [m/k, 2m/k) ... into one record buffer
  (``gs_engine_find_device``), then ``gs_engine_update_device`` -- exactly
  what every rank of a k-GPU run computes after its all-gather
  (parallel.py:63-88 is the reference's static split).
"""

import ctypes as C
import os
import socket

import numpy as np
import pytest

from cases import CASES, load_golden, make_source, same_numpy
from test_gpu_engine import assert_state_equal

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.fixture(scope="module")
def world1():
    import torch.distributed as dist

    if not dist.is_initialized():
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(_free_port())
        dist.init_process_group("gloo", rank=0, world_size=1)
    yield dist.group.WORLD
    dist.destroy_process_group()


def _check_stats(st, gold):
    for k in ("iterations", "signals", "discarded", "units", "connections", "converged"):
        assert int(getattr(st, k)) == int(gold[f"stat_{k}"]), k


@pytest.mark.parametrize("name", ["cfg1", "stress", "paper_rule", "v8k_fixed", "cfg4_prefix"])
def test_run_multi_sharded_world1_matches_golden(world1, name):
    from paper_1503_08294_b200 import EngineParams
    from paper_1503_08294_b200.distributed import run_multi_sharded

    gold = load_golden(name)
    if not same_numpy(gold):
        pytest.skip("golden made with another numpy")
    case = CASES[name]
    net, st = run_multi_sharded(make_source(case["source"]), EngineParams(**case["params"]),
                                case["seed"], group=world1)
    _check_stats(st, gold)
    assert_state_equal(net.export(), gold)
    assert st.find_s > 0 and net.exchange_ms() > 0  # the all-gathers ran and were timed
    net.audit()


def test_cfg3_headline_sharded_world1(world1):
    """The whole config-3 run (asynchronous device-sampled lookahead loop)
    through the sharded path equals the reference's full run."""
    from paper_1503_08294_b200 import workloads
    from paper_1503_08294_b200.distributed import run_multi_sharded

    gold = load_golden("cfg3_final")
    if not same_numpy(gold):
        pytest.skip("golden made with another numpy")
    src, params, seed, _ = workloads.make("cfg3")
    net, st = run_multi_sharded(src, params, seed, group=world1, capacity=8192)
    _check_stats(st, gold)
    got = net.export()
    assert np.array_equal(got["ids"], gold["ids"]) and np.array_equal(got["edges"], gold["edges"])
    for k in ("pos", "hab", "theta"):
        assert np.array_equal(got[k].view(np.int64), gold[k].view(np.int64)), k


def test_set_shards_without_torch_distributed():
    """The C ABI alone: a single-rank communicator from gs_shard_unique_id."""
    from paper_1503_08294_b200 import EngineParams, Network
    from paper_1503_08294_b200.distributed import shard_unique_id
    from paper_1503_08294_b200.multi import step

    gold = load_golden("stress")
    case = CASES["stress"]
    params = EngineParams(**case["params"])
    src = make_source(case["source"])
    rng = np.random.Generator(np.random.Philox(case["seed"]))
    net = Network(params)
    net.set_shards(1, 0, shard_unique_id())
    for p in src.sample(rng, 2):
        net.add_unit(p, params.theta0)
    from paper_1503_08294_b200.params import batch_size

    signals, units, rows = 0, 2, []
    while signals < params.max_signals:
        m = batch_size(units, params.batch_cap, params.batch_floor)
        st = step(net, src.sample(rng, m))
        rows.append((m, int(st.processed), int(st.discarded), int(st.inserted)))
        signals += m
        units = int(st.units)
        if st.converged:
            break
    assert np.array_equal(np.array(rows, np.int64), gold["per_batch"])
    assert_state_equal(net.export(), gold)
    with pytest.raises(ValueError):
        net.set_shards(2, 2, shard_unique_id())
    with pytest.raises(ValueError):
        net.set_shards(1, 0, b"short")
    net.set_shards(0, 0)  # detach


@pytest.mark.parametrize("name,k", [(n, k) for n in ("cfg1", "stress", "v8k") for k in (2, 4)]
                         + [("cfg4_prefix", 8)])
def test_k_shard_split_on_one_gpu_matches_golden(name, k):
    import torch

    from paper_1503_08294_b200 import EngineParams, Network, _lib
    from paper_1503_08294_b200.distributed import REC_BYTES, shard_bounds
    from paper_1503_08294_b200.params import batch_size

    gold = load_golden(name)
    if not same_numpy(gold):
        pytest.skip("golden made with another numpy")
    lib = _lib.load_library()
    case = CASES[name]
    params = EngineParams(**case["params"])
    src = make_source(case["source"])
    rng = np.random.Generator(np.random.Philox(case["seed"]))
    net = Network(params)
    for p in src.sample(rng, 2):
        net.add_unit(p, params.theta0)
    cap = params.batch_cap
    d_sig = torch.empty((cap, 3), dtype=torch.float64, device="cuda")
    d_rec = torch.empty(cap * REC_BYTES, dtype=torch.uint8, device="cuda")
    st = _lib.GsBatchStats()
    signals, units, rows = 0, 2, []
    while signals < params.max_signals:
        m = batch_size(units, params.batch_cap, params.batch_floor)
        d_sig[:m].copy_(torch.from_numpy(np.ascontiguousarray(src.sample(rng, m))))
        torch.cuda.synchronize()
        for r in range(k):  # k ranks' finds into one buffer, in any order
            lo, hi = shard_bounds(m, k, (r * 3) % k)
            _lib.check(lib.gs_engine_find_device(net.handle, d_sig.data_ptr(), lo, hi,
                                                 d_rec.data_ptr()))
        _lib.check(lib.gs_engine_update_device(net.handle, d_sig.data_ptr(), m,
                                               d_rec.data_ptr()))
        _lib.check(lib.gs_engine_stats(net.handle, C.byref(st)))
        net._touch()
        rows.append((m, int(st.processed), int(st.discarded), int(st.inserted)))
        signals += m
        units = int(st.units)
        if st.converged:
            break
    assert np.array_equal(np.array(rows, np.int64), gold["per_batch"])
    assert_state_equal(net.export(), gold)
    net.audit()

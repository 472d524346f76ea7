"""RunState and write-through state arrays against the UNMODIFIED reference.

The reference package built by oracle/build_ref.sh (oracle/_ref, travels to
the GPU box) is the checker: the same winner streams go through its
resolve_and_update / update_single (multi.py:99-131, engine.py:283-355) and
through the device engine, and the networks and RunStates are compared bit
for bit.  Covers the reference's contract that ``state=None`` is a fresh
RunState per call (multi.py:114-115, engine.py:301-302), a RunState shared
across calls (tick, next_sweep, patience, last_active in dict order, with
sweeps firing), host edits of a RunState between calls, and in-place edits
through ``state_arrays()`` (network.py:178-186).
"""

import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

REF = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref")


def _ref():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    try:
        import growsurf
    except ImportError:
        pytest.skip("reference package not built (oracle/build_ref.sh)")
    return growsurf


def _same_network(net, rnet):
    ids, pos, hab, theta = net.state_arrays()
    rids, rpos, rhab, rtheta = rnet.state_arrays()
    assert np.array_equal(ids, rids)
    assert net.edges() == rnet.edges()
    for a, b in ((pos, rpos), (hab, rhab), (theta, rtheta)):
        assert np.array_equal(np.ascontiguousarray(a).view(np.int64),
                              np.ascontiguousarray(b).view(np.int64))


def _same_state(st, rst):
    assert (st.tick, st.next_sweep) == (rst.tick, rst.next_sweep)
    assert list(st.last_active.items()) == list(rst.last_active.items())
    assert dict(st.patience) == {u: c for u, c in rst.patience.items() if c}


def _pair(params, n_units, seed):
    from paper_1503_08294_b200 import Network

    R = _ref()
    rng = np.random.default_rng(seed)
    net = Network(params)
    rnet = R.Network()
    for p in rng.random((n_units, 3)):
        net.add_unit(p, params.theta0)
        rnet.add_unit(p, params.theta0)
    # a connected start (isolated units would all be pruned by the first update)
    for k in range(n_units):
        for j in (1, 2):
            net.connect_or_reset(k, (k + j) % n_units)
            rnet.connect_or_reset(k, (k + j) % n_units)
    return net, rnet, rng


def _stream(rng, ids, m):
    b = rng.choice(ids, m)
    s = rng.choice(ids, m)
    s = np.where(s == b, ids[(np.searchsorted(ids, b) + 1) % len(ids)], s)
    return b, s, rng.random(m) * 0.6, rng.random((m, 3))


@pytest.mark.parametrize("shared", [False, True])
def test_winner_streams_match_reference(shared):
    """Adversarial winner lists (collisions, stale seconds, repeated
    winners) through both engines; RunState fresh per call or shared."""
    from paper_1503_08294_b200 import EngineParams, WinnerResult, resolve_and_update
    from paper_1503_08294_b200.multi import RunState

    R = _ref()
    kw = dict(theta0=0.3, max_age=30, ring_patience=2, stale_factor=1)
    params, rparams = EngineParams(**kw), R.EngineParams(**kw)
    net, rnet, rng = _pair(params, 60, 5)
    st, rst = (RunState(), R.engine.RunState()) if shared else (None, None)
    for it in range(40):
        ids = np.array(rnet.unit_ids())
        b, s, d, batch = _stream(rng, ids, int(rng.integers(1, 300)))
        win = [WinnerResult(int(x), int(y), float(z), 0.0) for x, y, z in zip(b, s, d)]
        rwin = [R.WinnerResult(int(x), int(y), float(z), 0.0) for x, y, z in zip(b, s, d)]
        out = resolve_and_update(net, params, batch, win, st)
        want = R.resolve_and_update(rnet, rparams, batch, rwin, rst)
        assert (out.processed, out.discarded, out.inserted_units) == (
            want.processed, want.discarded, want.inserted_units)
        _same_network(net, rnet)
        if shared:
            _same_state(st, rst)
        if rnet.unit_count < 8:
            break
    assert rnet.next_id > 60 + 20  # insertions happened
    if shared:
        assert rst.tick > 3000  # the sweep clock fired several times
        assert rnet.next_id > rnet.unit_count + 20  # ... and removed units
    net.audit()


def test_host_edited_run_state_is_loaded():
    """Edits of a RunState between calls (entries dropped, re-inserted at
    the end of the dict order, clocks moved) reach the device like they
    reach the reference's next update: the sweep removes stale units in the
    edited dict order."""
    from paper_1503_08294_b200 import EngineParams, WinnerResult, resolve_and_update
    from paper_1503_08294_b200.multi import RunState

    R = _ref()
    kw = dict(theta0=0.3, max_age=30, ring_patience=3, stale_factor=1)
    params, rparams = EngineParams(**kw), R.EngineParams(**kw)
    net, rnet, rng = _pair(params, 30, 9)
    st, rst = RunState(), R.engine.RunState()
    for it in range(12):
        ids = np.array(rnet.unit_ids())
        b, s, d, batch = _stream(rng, ids, 200)
        win = [WinnerResult(int(x), int(y), float(z), 0.0) for x, y, z in zip(b, s, d)]
        rwin = [R.WinnerResult(int(x), int(y), float(z), 0.0) for x, y, z in zip(b, s, d)]
        resolve_and_update(net, params, batch, win, st)
        R.resolve_and_update(rnet, rparams, batch, rwin, rst)
        _same_network(net, rnet)
        _same_state(st, rst)
        for state in (st, rst):
            keys = list(state.last_active)
            if len(keys) > 4:
                v = state.last_active.pop(keys[1])
                state.last_active[keys[1]] = v - 3  # re-inserted: now last in order
                del state.last_active[keys[2]]
            state.patience[keys[0]] = 1
            state.next_sweep = min(state.next_sweep, state.tick + 150)
    net.audit()


def test_batch_equals_sequential_replay_with_run_state():
    """test_multi.py:123-139: distinct winners in one batch == update_single
    one by one with a RunState, on the device and in the reference."""
    from paper_1503_08294_b200 import (EngineParams, Network, batch_find_winners,
                                       resolve_and_update, update_single)
    from paper_1503_08294_b200.multi import RunState

    R = _ref()

    def lined(NetCls):
        net = NetCls()
        for k in range(6):
            net.add_unit((float(k), 0.0, 0.0), 0.5)
        for k in range(5):
            net.connect_or_reset(k, k + 1)
        return net

    params = EngineParams(theta0=0.5)
    net, twin, rtwin = lined(lambda: Network(params)), lined(lambda: Network(params)), lined(
        R.Network)
    batch = np.array([[0.1, 0, 0], [2.2, 0, 0], [4.9, 0, 0]])
    winners = batch_find_winners(net.snapshot(), batch)
    assert len({w.winner for w in winners}) == 3
    assert resolve_and_update(net, params, batch, winners).discarded == 0
    st, rst = RunState(), R.engine.RunState()
    for j, wr in enumerate(winners):
        update_single(twin, params, batch[j], wr, st)
        R.update_single(rtwin, R.EngineParams(theta0=0.5), batch[j],
                        R.WinnerResult(wr.winner, wr.second, wr.d_winner, wr.d_second), rst)
    assert net.unit_ids() == twin.unit_ids() and net.edges() == twin.edges()
    assert np.array_equal(net.snapshot().positions, twin.snapshot().positions)
    _same_network(twin, rtwin)
    _same_state(st, rst)


def test_state_arrays_write_through():
    """In-place edits of state_arrays() views reach the device
    (test_multi.py:153-156 does ``hab[:] = 0.05``); writes that cannot be
    intercepted fail loudly."""
    from paper_1503_08294_b200 import Network

    net = Network()
    for k in range(5):
        net.add_unit((float(k), 0.0, 0.0), 0.5)
    ids, pos, hab, theta = net.state_arrays()
    hab[:] = 0.05
    assert all(net.habituation(u) == 0.05 for u in net.unit_ids())
    theta *= 0.5
    assert net.local_threshold(3) == 0.25
    pos[[1, 3]] += 0.25
    assert np.array_equal(net.position(3), [3.25, 0.25, 0.25])
    assert np.array_equal(net.position(2), [2.0, 0.0, 0.0])
    hab[2] = 0.5
    assert net.habituation(2) == 0.5 and net.habituation(1) == 0.05
    with pytest.raises(ValueError):
        pos[0][1] = 7.0  # a view of a view: read-only, never silently dropped
    with pytest.raises(ValueError):
        ids[0] = 9
    with pytest.raises(ValueError):
        np.copyto(hab, 1.0)
    assert net.counts()["untrained"] == sum(net.habituation(u) >= 0.1 for u in net.unit_ids())
    net.audit()

"""Device-resident engine parity: B200 runs vs the reference's golden traces
and vs the C oracle, bit for bit (ids, edges with ages, positions,
habituation, thresholds, ring classes, patience, last_active, tick)."""

import numpy as np
import pytest

from cases import CASES, load_golden, make_source, run_device_trace, same_numpy
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def assert_state_equal(got: dict, want: dict):
    assert np.array_equal(got["ids"], want["ids"])
    assert np.array_equal(got["edges"], want["edges"])
    for k in ("pos", "hab", "theta"):
        assert np.array_equal(np.ascontiguousarray(got[k]).view(np.int64),
                              np.ascontiguousarray(want[k]).view(np.int64)), k
    for k in ("ring", "patience", "last_active"):
        assert np.array_equal(got[k], want[k]), k
    for k in ("tick", "next_sweep", "next_id"):
        assert int(got[k]) == int(want[k]), k


FAST = ["sphere_exec", "cfg1", "stress", "boundary", "paper_rule"]


@pytest.mark.parametrize("name", FAST + [pytest.param("cfg2", marks=pytest.mark.slow)])
def test_device_run_matches_reference_golden(name):
    gold = load_golden(name)
    if not same_numpy(gold):
        pytest.skip("golden made with another numpy")
    net, stats, per_batch, digest = run_device_trace(name)
    assert digest == str(gold["signal_sha256"])
    assert np.array_equal(per_batch, gold["per_batch"])
    for k in ("iterations", "signals", "discarded", "units", "connections", "converged"):
        assert int(stats[k]) == int(gold[f"stat_{k}"]), k
    assert_state_equal(net.export(), gold)
    net.audit()


@pytest.mark.parametrize("name,mode", [(n, k) for n in ("v8k", "v8k_fixed") for k in range(5)]
                         + [("cfg4_prefix", k) for k in (1, 2, 4)])
def test_large_network_find_modes_match_reference(name, mode):
    """V grows past 4096 (to ~9.9k): the engine's find leaves the screened
    small kernel (n <= 4096) for the FP64 small kernel (n <= 6144), the
    filter or the grid, with row->slot indirection and dead rows in the
    snapshot; every mode must still reproduce the reference's run."""
    gold = load_golden(name)
    if not same_numpy(gold):
        pytest.skip("golden made with another numpy")
    net, stats, per_batch, digest = run_device_trace(name, find_mode=mode)
    assert digest == str(gold["signal_sha256"])
    assert int(gold["stat_units"]) > 4096 and stats["units"] > 4096
    assert np.array_equal(per_batch, gold["per_batch"])
    assert_state_equal(net.export(), gold)
    net.audit()


@pytest.mark.parametrize("mode", [0, 1, 3, 4])  # exact, filter, screened small, grid
def test_find_modes_identical_runs(mode):
    gold = load_golden("stress")
    net, stats, per_batch, _ = run_device_trace("stress", find_mode=mode)
    assert np.array_equal(per_batch, gold["per_batch"])
    assert_state_equal(net.export(), gold)


def test_executor_boundary_matches_golden():
    from paper_1503_08294_b200 import b200_executor

    gold = load_golden("sphere_exec")
    net, stats, per_batch, _ = run_device_trace("sphere_exec", executor=b200_executor())
    assert np.array_equal(per_batch, gold["per_batch"])
    assert_state_equal(net.export(), gold)


def test_run_multi_api_matches_oracle():
    from paper_1503_08294_b200 import EngineParams, extract_mesh, genus, manifold_check, run_multi

    case = CASES["cfg1"]
    params = EngineParams(**case["params"])
    net, st = run_multi(make_source(case["source"]), params, case["seed"])
    onet, ost, _, _ = O.run_multi_oracle(make_source(case["source"]), params, case["seed"])
    assert st.converged and ost["converged"]
    assert (st.signals, st.discarded, st.iterations, st.units, st.connections) == (
        ost["signals"], ost["discarded"], ost["iterations"], ost["units"], ost["connections"])
    assert_state_equal(net.export(), onet.export())
    mesh = extract_mesh(net)
    assert manifold_check(mesh) == "closed" and genus(mesh) == 0


def test_random_winner_streams_match_oracle():
    """resolve_and_update with adversarial winner lists (many collisions,
    stale seconds, repeated winners) against the oracle's sequential loop."""
    from paper_1503_08294_b200 import EngineParams, Network, WinnerResult, resolve_and_update
    from paper_1503_08294_b200.multi import RunState

    rng = np.random.default_rng(5)
    state = RunState()  # the oracle keeps one run state across the calls
    params = EngineParams(theta0=0.3, max_age=6, ring_patience=2, stale_factor=1)
    net = Network(params)
    onet = O.OracleNet(params)
    pts = rng.random((40, 3))
    for p in pts:
        net.add_unit(p, 0.3)
        onet.add_unit(p, 0.3)
    for k in range(40):  # connected start: isolated units would all be pruned at once
        for j in (1, 2):
            net.connect_or_reset(k, (k + j) % 40)
            onet.connect_or_reset(k, (k + j) % 40)
    for it in range(60):
        ids = np.array(net.unit_ids())
        m = int(rng.integers(1, 300))
        b = rng.choice(ids, m)
        s = rng.choice(ids, m)
        s = np.where(s == b, ids[(np.searchsorted(ids, b) + 1) % len(ids)], s)
        d = rng.random(m) * 0.6
        batch = rng.random((m, 3))
        out = resolve_and_update(net, params, batch,
                                 [WinnerResult(int(x), int(y), float(z), 0.0)
                                  for x, y, z in zip(b, s, d)], state)
        want = onet.resolve_and_update(batch, b, s, d)
        assert (out.processed, out.discarded, out.inserted_units) == tuple(int(v) for v in want)
        assert_state_equal(net.export(), onet.export())
    net.audit()


class TestResolveScenarios:
    """pkg/tests/test_multi.py:98-165 on the device engine."""

    def lined_net(self, params):
        from paper_1503_08294_b200 import Network

        net = Network(params)
        for k in range(6):
            net.add_unit((float(k), 0.0, 0.0), 0.5)
        for k in range(5):
            net.connect_or_reset(k, k + 1)
        return net

    def test_winner_lock(self):
        from paper_1503_08294_b200 import BatchOutcome, EngineParams, batch_find_winners
        from paper_1503_08294_b200 import resolve_and_update

        params = EngineParams(theta0=0.5)
        net = self.lined_net(params)
        batch = np.array([[0.1, 0, 0], [0.2, 0, 0], [3.1, 0, 0]])
        winners = batch_find_winners(net.snapshot(), batch)
        assert winners[0].winner == winners[1].winner == 0 and winners[2].winner == 3
        assert resolve_and_update(net, params, batch, winners) == BatchOutcome(2, 1, 0)

    def test_stale_winner_discarded(self):
        from paper_1503_08294_b200 import EngineParams, batch_find_winners, resolve_and_update

        params = EngineParams(theta0=0.5)
        net = self.lined_net(params)
        batch = np.array([[0.1, 0, 0], [5.1, 0, 0]])
        winners = batch_find_winners(net.snapshot(), batch)
        net.remove_unit(winners[1].winner)
        out = resolve_and_update(net, params, batch, winners)
        assert (out.processed, out.discarded) == (1, 1)

    def test_inserted_units_never_win_in_batch(self):
        from paper_1503_08294_b200 import EngineParams, batch_find_winners, resolve_and_update

        params = EngineParams(theta0=0.2)
        net = self.lined_net(params)
        for u in net.unit_ids():
            net.set_unit(u, habituation=0.05)
        batch = np.array([[0.4, 0.3, 0], [2.4, -0.3, 0], [4.6, 0.3, 0]])
        winners = batch_find_winners(net.snapshot(), batch)
        before = net.next_id
        resolve_and_update(net, params, batch, winners)
        assert net.next_id > before
        net.audit()

    def test_accounting_balances(self):
        from paper_1503_08294_b200 import (EngineParams, Network, SphereSource,
                                           batch_find_winners, resolve_and_update)

        params = EngineParams(theta0=0.25)
        rng = np.random.default_rng(8)
        src = SphereSource(1.0)
        net = Network(params)
        for p in src.sample(rng, 12):
            net.add_unit(p, params.theta0)
        for _ in range(20):
            batch = src.sample(rng, 32)
            out = resolve_and_update(net, params, batch, batch_find_winners(net.snapshot(), batch))
            assert out.processed + out.discarded == 32
            net.audit()


class TestNetworkApi:
    """pkg/tests/test_network.py semantics on the device Network."""

    def test_add_connect_age_prune(self):
        from paper_1503_08294_b200 import Network, RingClass

        net = Network()
        ids = [net.add_unit((float(i), 0, 0), 0.5) for i in range(4)]
        assert ids == [0, 1, 2, 3] and net.unit_count == 4
        assert net.connect_or_reset(0, 1) == "created"
        assert net.connect_or_reset(0, 1) == "reset"
        net.connect_or_reset(1, 2)
        net.connect_or_reset(0, 2)
        assert net.link_ring(0) is RingClass.HALF_DISK
        assert net.age_incident_edges(0, 5, exclude=1) == 5
        assert net.edge_age(0, 2) == 5 and net.edge_age(0, 1) == 0
        assert net.prune(4) == (1, 1)  # edge 0-2 over age; isolated unit 3 removed
        assert not net.is_alive(3) and not net.has_edge(0, 2)
        net.audit()

    def test_errors(self):
        from paper_1503_08294_b200 import Network, UnknownUnitError

        net = Network()
        a = net.add_unit((0, 0, 0), 0.5)
        with pytest.raises(ValueError):
            net.connect_or_reset(a, a)
        with pytest.raises(UnknownUnitError):
            net.connect_or_reset(a, 99)
        with pytest.raises(ValueError):
            net.add_unit((np.nan, 0, 0), 0.5)
        with pytest.raises(ValueError):
            net.add_unit((0, 0, 0), -1.0)

    def test_floor_of_two_units(self):
        from paper_1503_08294_b200 import Network

        net = Network()
        for i in range(3):
            net.add_unit((float(i), 0, 0), 0.5)
        assert net.prune(10) == (0, 1)
        assert net.unit_count == 2

    def test_remove_unit_recomputes_rings(self):
        from paper_1503_08294_b200 import Network

        net = Network()
        for p in [(0, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 1)]:
            net.add_unit(p, 0.5)
        for a in range(4):
            for b in range(a + 1, 4):
                net.connect_or_reset(a, b)
        assert net.all_rings_surface()
        net.remove_unit(3)
        assert net.edge_count == 3 and not net.all_rings_surface()
        net.audit()


@pytest.mark.slow
def test_cfg3_headline_run_matches_reference():
    """BASELINE config 3 (1M-point genus-2 cloud, m=4096, theta0=0.1): the
    device run to convergence equals the reference's own full run
    (tests/golden/make_cfg3_golden.py, 430 s on 8 cores) bit for bit."""
    import os

    from paper_1503_08294_b200 import extract_mesh, genus, manifold_check, run_multi, workloads

    gold = np.load(os.path.join(os.path.dirname(__file__), "golden", "run_cfg3_final.npz"))
    if str(gold["numpy_version"]) != np.__version__:
        pytest.skip("golden made with another numpy")
    src, params, seed, _ = workloads.make("cfg3")
    net, st = run_multi(src, params, seed, capacity=8192)
    assert (st.signals, st.discarded, st.iterations, st.units, st.connections, st.converged) == (
        int(gold["stat_signals"]), int(gold["stat_discarded"]), int(gold["stat_iterations"]),
        int(gold["stat_units"]), int(gold["stat_connections"]), bool(gold["stat_converged"]))
    got = net.export()
    assert np.array_equal(got["ids"], gold["ids"])
    assert np.array_equal(got["edges"], gold["edges"])
    for k in ("pos", "hab", "theta"):
        assert np.array_equal(got[k].view(np.int64), gold[k].view(np.int64)), k
    mesh = extract_mesh(net)
    assert manifold_check(mesh) == "closed" and genus(mesh) == 2


@pytest.mark.parametrize("name", ["paper_rule", "boundary", "cfg1", "v8k", "v8k_fixed",
                                  "cfg4_prefix"])
def test_run_multi_device_sampling_matches_golden(name):
    """run_multi on a CloudSource draws its batches on the device (variable m
    under the paper's batch rule: synchronous; fixed m: the asynchronous
    lookahead loop) and must reproduce the reference's run bit for bit."""
    from paper_1503_08294_b200 import EngineParams, run_multi

    gold = load_golden(name)
    if not same_numpy(gold):
        pytest.skip("golden made with another numpy")
    case = CASES[name]
    params = EngineParams(**case["params"])
    net, st = run_multi(make_source(case["source"]), params, case["seed"])
    for k in ("iterations", "signals", "discarded", "units", "connections", "converged"):
        assert int(getattr(st, k)) == int(gold[f"stat_{k}"]), k
    assert_state_equal(net.export(), gold)
    net.audit()


@pytest.mark.parametrize("spec", ["0", "1"])
@pytest.mark.parametrize("name", ["cfg1", "v8k_fixed"])
def test_speculative_screen_on_and_off_match_golden(name, spec, monkeypatch):
    """The find's speculative screen (against the snapshot before the running
    update, threshold widened by a movement bound, verdict from the update's
    token) and the plain screen give the reference's run bit for bit; the
    engine reads GS_SPEC_FIND when it is created."""
    from paper_1503_08294_b200 import EngineParams, run_multi

    monkeypatch.setenv("GS_SPEC_FIND", spec)
    gold = load_golden(name)
    if not same_numpy(gold):
        pytest.skip("golden made with another numpy")
    case = CASES[name]
    params = EngineParams(**case["params"])
    net, st = run_multi(make_source(case["source"]), params, case["seed"])
    for k in ("iterations", "signals", "units", "connections", "converged"):
        assert int(getattr(st, k)) == int(gold[f"stat_{k}"]), k
    assert_state_equal(net.export(), gold)

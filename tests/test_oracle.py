"""Pin the CPU oracle to the reference's own outputs (tests/golden/*.npz).

The golden fixtures were produced by running the reference package itself
(tests/golden/make_golden.py).  The oracle is trusted as the GPU parity
checker only because these tests pass.
"""

import os

import numpy as np
import pytest

from cases import CASES, GOLDEN, load_golden, make_source, same_numpy
from oracle import oracle as O
from paper_1503_08294_b200.params import EngineParams


def test_kernel_cases_bitwise():
    with np.load(os.path.join(GOLDEN, "kernel_cases.npz")) as z:
        for k in range(int(z["count"])):
            idx, d2 = O.scan_best_two(z[f"pos{k}"], z[f"sig{k}"])
            assert np.array_equal(idx, z[f"idx{k}"]), k
            assert np.array_equal(d2.view(np.int64), z[f"d2{k}"].view(np.int64)), k


def test_sort_oracle_agreement_and_ties():
    # pkg/tests/test_kernels.py:13-55
    rng = np.random.default_rng(42)
    for _ in range(100):
        n = int(rng.integers(2, 200))
        pos = rng.random((n, 3))
        sig = rng.random((1, 3)) * 1.4 - 0.2
        idx, d2 = O.scan_best_two(pos, sig)
        d = np.sum((pos - sig[0]) ** 2 * [1, 1, 1], axis=1)
        dx, dy, dz = (pos - sig[0]).T
        d = dx * dx + dy * dy + dz * dz
        order = np.lexsort((np.arange(n), d))
        assert (idx[0, 0], idx[0, 1]) == (order[0], order[1])
        assert d2[0, 0] == d[order[0]] and d2[0, 1] == d[order[1]]
    idx, _ = O.scan_best_two(np.array([[1.0, 0, 0], [-1.0, 0, 0], [2.0, 0, 0]]), np.zeros((1, 3)))
    assert tuple(idx[0]) == (0, 1)
    idx, _ = O.scan_best_two(np.array([[0.5, 0.5, 0.5]] * 4), np.array([[0.1, 0.2, 0.3]]))
    assert tuple(idx[0]) == (0, 1)


def assert_state_equal(got: dict, want: dict):
    assert np.array_equal(got["ids"], want["ids"])
    assert np.array_equal(got["edges"], want["edges"])
    assert np.array_equal(got["pos"].view(np.int64), want["pos"].view(np.int64))
    assert np.array_equal(got["hab"].view(np.int64), want["hab"].view(np.int64))
    assert np.array_equal(got["theta"].view(np.int64), want["theta"].view(np.int64))
    assert np.array_equal(got["ring"], want["ring"])
    assert np.array_equal(got["patience"], want["patience"])
    assert np.array_equal(got["last_active"], want["last_active"])
    assert int(got["tick"]) == int(want["tick"])
    assert int(got["next_sweep"]) == int(want["next_sweep"])
    assert int(got["next_id"]) == int(want["next_id"])


FAST = ["sphere_exec", "cfg1", "stress", "boundary", "paper_rule"]


@pytest.mark.parametrize("name", FAST + [pytest.param("cfg2", marks=pytest.mark.slow)])
def test_oracle_reproduces_reference_run(name):
    gold = load_golden(name)
    if not same_numpy(gold):
        pytest.skip(f"fixture made with numpy {gold['numpy_version']}, have {np.__version__}")
    case = CASES[name]
    params = EngineParams(**case["params"])
    net, stats, per_batch, digest = O.run_multi_oracle(make_source(case["source"]), params,
                                                        case["seed"])
    assert digest == str(gold["signal_sha256"]), "sampler stream differs from the reference"
    assert np.array_equal(per_batch, gold["per_batch"])
    for k in ("iterations", "signals", "discarded", "units", "connections", "converged"):
        assert int(stats[k]) == int(gold[f"stat_{k}"]), k
    assert_state_equal(net.export(), gold)
    assert net.audit_rings() == 0

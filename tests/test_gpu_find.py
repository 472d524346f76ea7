"""Find-winners kernels on the B200 vs the reference's own outputs.

Mirrors pkg/tests/test_kernels.py / test_parallel.py against the "b200"
backend, plus the reference-generated golden cases (bitwise rows AND d^2).
"""

import os
import threading

import numpy as np
import pytest

from cases import GOLDEN
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def kb():
    from paper_1503_08294_b200 import kernels

    return kernels


def scan(kb, pos, sig, tile=64):
    m = sig.shape[0]
    idx = np.empty((m, 2), np.int64)
    d2 = np.empty((m, 2), np.float64)
    kb.scan_best_two_into(np.ascontiguousarray(pos), len(pos), np.ascontiguousarray(sig), idx,
                          d2, tile)
    return idx, d2


def bits(a):
    return np.ascontiguousarray(a).view(np.int64)


def test_golden_kernel_cases_bitwise(kb):
    with np.load(os.path.join(GOLDEN, "kernel_cases.npz")) as z:
        for k in range(int(z["count"])):
            idx, d2 = scan(kb, z[f"pos{k}"], z[f"sig{k}"])
            assert np.array_equal(idx, z[f"idx{k}"]), k
            assert np.array_equal(bits(d2), bits(z[f"d2{k}"])), k


def test_sort_oracle_random_instances(kb):
    # test_kernels.py:33-42
    rng = np.random.default_rng(42)
    for _ in range(200):
        n = int(rng.integers(2, 200))
        pos = np.ascontiguousarray(rng.random((n, 3)))
        sig = rng.random(3) * 1.4 - 0.2
        r1, r2, d1, d2 = kb.best_two_single(pos, n, *sig)
        dx, dy, dz = (pos - sig).T
        d = dx * dx + dy * dy + dz * dz
        order = np.lexsort((np.arange(n), d))
        assert (r1, r2) == (order[0], order[1])
        assert d1 == d[order[0]] and d2 == d[order[1]]


def test_ties_and_duplicates(kb):
    assert kb.best_two_single(np.array([[1.0, 0, 0], [-1.0, 0, 0], [2.0, 0, 0]]), 3, 0, 0, 0)[:2] \
        == (0, 1)
    assert kb.best_two_single(np.array([[0.5, 0.5, 0.5]] * 4), 4, 0.1, 0.2, 0.3)[:2] == (0, 1)
    # many exact ties spread across CTA tiles and row chunks
    pos = np.zeros((5000, 3))
    idx, d2 = scan(kb, pos, np.ones((700, 3)))
    assert np.all(idx[:, 0] == 0) and np.all(idx[:, 1] == 1)


def test_fewer_than_two_units(kb):
    r1, r2, d1, d2 = kb.best_two_single(np.array([[0.0, 0, 0]]), 1, 1.0, 0, 0)
    assert (r1, r2) == (0, -1) and d1 == 1.0 and d2 == np.inf
    r1, r2, d1, d2 = kb.best_two_single(np.zeros((3, 3)), 0, 1.0, 0, 0)
    assert (r1, r2) == (-1, -1) and d1 == np.inf


def test_tile_never_changes_output(kb):
    rng = np.random.default_rng(11)
    pos, sig = rng.random((157, 3)), rng.random((64, 3))
    base = scan(kb, pos, sig, 1)
    for tile in (3, 17, 64, 157, 1000):
        got = scan(kb, pos, sig, tile)
        assert np.array_equal(got[0], base[0]) and np.array_equal(bits(got[1]), bits(base[1]))


def test_errors(kb):
    pos = np.zeros((4, 3))
    idx = np.empty((1, 2), np.int64)
    d2 = np.empty((1, 2))
    with pytest.raises(ValueError):
        kb.scan_best_two_into(pos, 4, np.zeros((1, 3)), idx, d2, 0)
    with pytest.raises(ValueError):
        kb.scan_best_two_into(pos, 5, np.zeros((1, 3)), idx, d2, 1)
    with pytest.raises(ValueError):
        kb.scan_best_two_into(pos, 4, np.zeros((2, 3)), idx, d2, 1)


def test_inputs_unchanged(kb):
    rng = np.random.default_rng(23)
    pos, sig = rng.random((50, 3)), rng.random((32, 3))
    p0, s0 = pos.copy(), sig.copy()
    scan(kb, pos, sig)
    assert np.array_equal(pos, p0) and np.array_equal(sig, s0)


@pytest.mark.parametrize("n,m", [(1000, 2048), (20000, 3000), (3, 5000), (70000, 300)])
def test_matches_c_oracle_bitwise(kb, n, m):
    rng = np.random.default_rng(n + m)
    pos = rng.random((n, 3)) * 4.0 - 2.0
    sig = rng.random((m, 3)) * 4.0 - 2.0
    want = O.scan_best_two(pos, sig)
    got = scan(kb, pos, sig)
    assert np.array_equal(got[0], want[0])
    assert np.array_equal(bits(got[1]), bits(want[1]))


def test_concurrent_disjoint_slices(kb):
    # parallel.py:78-87: workers fill disjoint output slices concurrently
    rng = np.random.default_rng(19)
    pos, sig = np.ascontiguousarray(rng.random((333, 3))), rng.random((128, 3))
    idx = np.empty((128, 2), np.int64)
    d2 = np.empty((128, 2))
    bounds = [(i * 128 // 8, (i + 1) * 128 // 8) for i in range(8)]
    threads = [threading.Thread(target=kb.scan_best_two_into,
                                args=(pos, 333, sig[a:b], idx[a:b], d2[a:b], 64))
               for a, b in bounds]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    want = O.scan_best_two(pos, sig)
    assert np.array_equal(idx, want[0]) and np.array_equal(bits(d2), bits(want[1]))

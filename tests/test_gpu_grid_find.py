"""Exact uniform-grid find (GS_FIND_GRID, csrc/grid.cu).

The grid stops searching only when no unvisited unit can reach the current
second best, so its output must equal the reference scan_best_two_into
(_scan.pyx:39-98) bit for bit: checked against the exact FP64 path and the C
oracle on uniform, clustered, surface, planar, collinear and single-point
unit sets, signals far outside the units' box, exact ties, extreme offsets
and non-finite rows and signals.
"""

import numpy as np
import pytest

from oracle import oracle as O
from test_gpu_filter import EXACT, find, same

pytestmark = pytest.mark.gpu

GRID = 4


@pytest.mark.parametrize("n,m", [(1, 10), (2, 100), (3, 1000), (1000, 5000), (20_000, 20_000),
                                 (100_003, 8000)])
def test_uniform_matches_exact(n, m):
    rng = np.random.Generator(np.random.Philox(7 * n + m))
    pos, sig = rng.random((n, 3)), rng.random((m, 3))
    got = find(pos, sig, GRID)
    assert same(got[:2], find(pos, sig, EXACT)[:2])
    if n >= 1000:
        assert got[2] < m // 50  # the grid certifies almost every signal


def test_matches_c_oracle():
    rng = np.random.Generator(np.random.Philox(5))
    pos, sig = rng.random((30000, 3)) * 6 - 3, rng.random((2000, 3)) * 8 - 4
    assert same(find(pos, sig, GRID)[:2], O.scan_best_two(pos, sig))


def test_surface_and_far_signals():
    from paper_1503_08294_b200 import TorusSource

    rng = np.random.Generator(np.random.Philox(2026))
    pos = TorusSource(2.0, 0.5).sample(rng, 50_000)
    sig = np.concatenate([TorusSource(2.0, 0.5).sample(rng, 10_000),
                          rng.random((500, 3)) * 40 - 20])  # far outside the units' box
    assert same(find(pos, sig, GRID)[:2], find(pos, sig, EXACT)[:2])


@pytest.mark.parametrize("shape", ["plane", "line", "point", "two_points"])
def test_degenerate_unit_sets(shape):
    rng = np.random.Generator(np.random.Philox(3))
    n = 5000
    pos = rng.random((n, 3))
    if shape == "plane":
        pos[:, 2] = 0.25
    elif shape == "line":
        pos[:, 1] = 0.5
        pos[:, 2] = -1.0
    elif shape == "point":
        pos[:] = [0.1, 0.2, 0.3]
    else:
        pos[: n // 2] = [0.0, 0.0, 0.0]
        pos[n // 2:] = [1.0, 1.0, 1.0]
    sig = rng.random((3000, 3)) * 2 - 0.5
    assert same(find(pos, sig, GRID)[:2], find(pos, sig, EXACT)[:2])


def test_ties_offsets_and_non_finite():
    pos = np.repeat(np.random.default_rng(1).random((700, 3)), 3, axis=0)
    sig = np.random.default_rng(2).random((5000, 3))
    assert same(find(pos, sig, GRID)[:2], find(pos, sig, EXACT)[:2])
    g = np.arange(20, dtype=np.float64)
    pos = np.stack(np.meshgrid(g, g, g, indexing="ij"), -1).reshape(-1, 3)
    sig = np.random.default_rng(3).integers(0, 19, (4000, 3)) + 0.5
    got = find(pos, sig, GRID)
    assert same(got[:2], find(pos, sig, EXACT)[:2])
    rng = np.random.Generator(np.random.Philox(11))
    for offset, scale in [(1.0e6, 1e-3), (-3.0e2, 1e-6), (0.0, 1e30), (0.0, 1e-21), (1e200, 1e190)]:
        pos = offset + scale * rng.random((8000, 3))
        sig = offset + scale * rng.random((3000, 3))
        assert same(find(pos, sig, GRID)[:2], find(pos, sig, EXACT)[:2]), (offset, scale)
    pos = rng.random((6000, 3))
    pos[[5, 77, 1500]] = np.nan
    pos[[9, 5999]] = np.inf
    sig = rng.random((4096, 3))
    sig[[3, 4000]] = np.nan
    sig[17] = -np.inf
    assert same(find(pos, sig, GRID)[:2], find(pos, sig, EXACT)[:2])

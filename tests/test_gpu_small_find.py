"""Screened small-n find (GS_FIND_SMALL, csrc/find.cu find_small_f32_kernel).

One kernel: FP32 lane minima screen the units, the surviving lanes are
re-evaluated in FP64 with the reference rounding.  The output must equal the
reference scan_best_two_into (_scan.pyx:39-98) bit for bit: checked against
the C oracle and the exact FP64 path on uniform clouds, every n from 0 to the
4096-row limit's edges, exact ties (duplicates, lattice points), clouds far
from the origin, extreme scales, and non-finite unit rows.  The signal counts
exercise the 1, 2 and 4 signals-per-warp variants.
"""

import numpy as np
import pytest

from oracle import oracle as O
from test_gpu_filter import EXACT, find, same

pytestmark = pytest.mark.gpu

SMALL = 3


@pytest.mark.parametrize("n", [0, 1, 2, 3, 31, 64, 65, 127, 128, 129, 1000, 2047, 4095, 4096])
@pytest.mark.parametrize("m", [1, 100, 2500, 5000])
def test_matches_exact(n, m):
    rng = np.random.Generator(np.random.Philox(1000 * n + m))
    pos, sig = rng.random((n, 3)) * 2 - 1, rng.random((m, 3)) * 2 - 1
    got = find(pos, sig, SMALL)
    assert same(got[:2], find(pos, sig, EXACT)[:2])


def test_matches_c_oracle():
    rng = np.random.Generator(np.random.Philox(5))
    pos, sig = rng.random((3000, 3)) * 6 - 3, rng.random((4500, 3)) * 6 - 3
    assert same(find(pos, sig, SMALL)[:2], O.scan_best_two(pos, sig))


def test_exact_ties():
    pos = np.repeat(np.random.default_rng(1).random((700, 3)), 3, axis=0)
    sig = np.random.default_rng(2).random((5000, 3))
    assert same(find(pos, sig, SMALL)[:2], find(pos, sig, EXACT)[:2])
    g = np.arange(16, dtype=np.float64)
    pos = np.stack(np.meshgrid(g, g, g, indexing="ij"), -1).reshape(-1, 3)
    sig = np.random.default_rng(3).integers(0, 15, (4000, 3)) + 0.5
    got = find(pos, sig, SMALL)
    assert same(got[:2], find(pos, sig, EXACT)[:2])
    assert np.all(got[0][:, 0] < got[0][:, 1])  # lower row wins a tie


@pytest.mark.parametrize("offset,scale", [(1.0e4, 1.0), (1.0e6, 1e-3), (-3.0e2, 1e-6),
                                          (0.0, 1e30), (0.0, 1e-21), (1e200, 1e190)])
def test_far_from_origin_and_extreme_scales(offset, scale):
    rng = np.random.Generator(np.random.Philox(11))
    pos = offset + scale * rng.random((3000, 3))
    sig = offset + scale * rng.random((4100, 3))
    assert same(find(pos, sig, SMALL)[:2], find(pos, sig, EXACT)[:2])


def test_non_finite_rows_and_signals():
    rng = np.random.Generator(np.random.Philox(12))
    pos = rng.random((2000, 3))
    pos[[5, 77, 1500]] = np.nan
    pos[[9, 1999]] = np.inf
    pos[300, 1] = -np.inf
    sig = rng.random((4096, 3))
    sig[[3, 4000]] = np.nan
    sig[17] = np.inf
    assert same(find(pos, sig, SMALL)[:2], find(pos, sig, EXACT)[:2])


def test_torus_surface_cloud():
    from paper_1503_08294_b200 import TorusSource

    rng = np.random.Generator(np.random.Philox(2026))
    pos = TorusSource(2.0, 0.5).sample(rng, 4000)
    sig = TorusSource(2.0, 0.5).sample(rng, 20_000)
    assert same(find(pos, sig, SMALL)[:2], find(pos, sig, EXACT)[:2])


def test_mass_ties_overflow_the_candidate_list():
    # every unit at the same point: all lanes survive the screen, the list
    # overflows and the warp scans exactly; lowest rows win
    pos = np.tile(np.array([[0.25, -0.5, 1.0]]), (1500, 1))
    pos[700:] += 1e-9  # a second, slightly farther cluster
    sig = np.random.default_rng(4).random((3000, 3))
    got = find(pos, sig, SMALL)
    assert same(got[:2], find(pos, sig, EXACT)[:2])
    assert same(got[:2], O.scan_best_two(pos, sig))

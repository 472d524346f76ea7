"""FP32 filter + certified FP64 re-check (csrc/filter.cu) vs the exact path.

The filter must be bit-identical to the exact scan (and so to the reference
scan_best_two_into, _scan.pyx:39-98) on every input: uniform clouds, exact
ties (duplicates, lattice points equidistant from the signal), clouds far
from the origin (large cancellation in |P|^2 - 2 P.Q), split-n chunking and
odd unit counts.  Inputs that the filter cannot certify go to the exact
fallback; the fallback counter shows both paths are exercised.
"""

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

EXACT, FILTER = 0, 1


def find(pos, sig, mode):
    import ctypes as C

    import torch

    from paper_1503_08294_b200 import _lib

    lib = _lib.load_library()
    ctx = _lib.default_context()
    dpos = torch.from_numpy(np.ascontiguousarray(pos, np.float64)).cuda()
    dsig = torch.from_numpy(np.ascontiguousarray(sig, np.float64)).cuda()
    m = sig.shape[0]
    idx = torch.empty((m, 2), dtype=torch.int64, device="cuda")
    d2 = torch.empty((m, 2), dtype=torch.float64, device="cuda")
    stream = torch.cuda.current_stream().cuda_stream
    _lib.check(lib.gs_find_device(ctx.handle, dpos.data_ptr(), pos.shape[0], dsig.data_ptr(), m,
                                  idx.data_ptr(), d2.data_ptr(), mode, stream))
    torch.cuda.synchronize()
    fb = np.zeros(2, np.int64)
    _lib.check(lib.gs_find_last_fallback_counts(ctx.handle, fb))
    return idx.cpu().numpy(), d2.cpu().numpy(), int(fb[0]), int(fb[1])


def same(a, b):
    return np.array_equal(a[0], b[0]) and np.array_equal(
        np.ascontiguousarray(a[1]).view(np.int64), np.ascontiguousarray(b[1]).view(np.int64))


@pytest.mark.parametrize("n,m", [(3, 100), (1001, 4096), (20000, 30000), (100_001, 3000)])
def test_uniform_matches_exact(n, m):
    rng = np.random.Generator(np.random.Philox(n))
    pos, sig = rng.random((n, 3)), rng.random((m, 3))
    got = find(pos, sig, FILTER)
    want = find(pos, sig, EXACT)
    assert same(got[:2], want[:2])
    assert got[2] < max(50, m // 20)  # the filter certifies almost every signal


def test_uniform_matches_c_oracle():
    rng = np.random.Generator(np.random.Philox(5))
    pos, sig = rng.random((30000, 3)) * 6 - 3, rng.random((2000, 3)) * 6 - 3
    got = find(pos, sig, FILTER)
    assert same(got[:2], O.scan_best_two(pos, sig))


def test_exact_ties_fall_back_and_match():
    # duplicate units: every signal has d1 == d2 == d3 -> uncertifiable
    pos = np.repeat(np.random.default_rng(1).random((700, 3)), 3, axis=0)
    sig = np.random.default_rng(2).random((5000, 3))
    got = find(pos, sig, FILTER)
    assert same(got[:2], find(pos, sig, EXACT)[:2])
    assert got[2] > 0 and got[3] > 0  # exact ties reach the FP64 tier
    # integer lattice, signals at cell centres: 8 equidistant corners
    g = np.arange(20, dtype=np.float64)
    pos = np.stack(np.meshgrid(g, g, g, indexing="ij"), -1).reshape(-1, 3)
    sig = np.random.default_rng(3).integers(0, 19, (4000, 3)) + 0.5
    got = find(pos, sig, FILTER)
    assert same(got[:2], find(pos, sig, EXACT)[:2])
    assert got[2] == sig.shape[0]
    # the reference tie rule: lower row wins
    assert np.all(got[0][:, 0] < got[0][:, 1])


@pytest.mark.parametrize("offset,scale", [(1.0e4, 1.0), (1.0e6, 1e-3), (-3.0e2, 1e-6), (0.0, 1e30), (0.0, 1e-21)])
def test_far_from_origin_and_extreme_scales(offset, scale):
    rng = np.random.Generator(np.random.Philox(11))
    pos = offset + scale * rng.random((8000, 3))
    sig = offset + scale * rng.random((6000, 3))
    got = find(pos, sig, FILTER)
    assert same(got[:2], find(pos, sig, EXACT)[:2])


def test_torus_surface_cloud():
    from paper_1503_08294_b200 import TorusSource

    rng = np.random.Generator(np.random.Philox(2026))
    pos = TorusSource(2.0, 0.5).sample(rng, 50_000)
    sig = TorusSource(2.0, 0.5).sample(rng, 20_000)
    got = find(pos, sig, FILTER)
    assert same(got[:2], find(pos, sig, EXACT)[:2])

"""BASELINE config 5 at full size: m = 1e6 signals against n = 1e4 / 1e5 /
1e6 units, uniform in [0,1)^3 (cli.py:252-261) and on a torus surface,
seeded Philox(7).  The exact uniform grid (AUTO's choice here), the FP32
filter with certified FP64 re-check and the exact FP64 scan must agree bit
for bit on every signal, and a sample of the signals must equal the C
oracle's restatement of the reference scan (_scan.pyx:39-98).  Also the
device adjacency's degree cap (64 neighbours, engine.cu kMaxDeg): a limit
the reference does not have, so crossing it must fail loudly.
"""

import numpy as np
import pytest

from oracle import oracle as O
from test_gpu_filter import EXACT, FILTER, find, same

pytestmark = pytest.mark.gpu

GRID, AUTO = 4, 2


def _inputs(dist, n, m):
    from paper_1503_08294_b200 import TorusSource

    rng = np.random.Generator(np.random.Philox(7))
    if dist == "uniform":
        return rng.random((n, 3)), rng.random((m, 3))
    src = TorusSource(0.3, 0.1)
    return src.sample(rng, n) + 0.5, src.sample(rng, m) + 0.5


@pytest.mark.parametrize("dist", ["uniform", "torus"])
@pytest.mark.parametrize("n", [10_000, 100_000, 1_000_000])
def test_config5_modes_agree_at_full_size(dist, n):
    m = 1_000_000
    pos, sig = _inputs(dist, n, m)
    grid = find(pos, sig, GRID)
    assert same(grid[:2], find(pos, sig, FILTER)[:2])
    assert same(grid[:2], find(pos, sig, AUTO)[:2])
    assert same(grid[:2], find(pos, sig, EXACT)[:2])
    # the reference's arithmetic on a sample (C oracle, single thread)
    k = 1000 if n == 1_000_000 else 4000
    pick = np.random.Generator(np.random.Philox(n)).choice(m, k, replace=False)
    want = O.scan_best_two(pos, sig[pick])
    assert same((grid[0][pick], grid[1][pick]), want)


def test_degree_cap_fails_loudly():
    """The 65th neighbour of one unit: through the Network API and through
    the batch update kernel, a StateError naming the capacity -- never a
    silently truncated adjacency."""
    from paper_1503_08294_b200 import (EngineParams, Network, StateError, WinnerResult,
                                       resolve_and_update)

    net = Network(EngineParams())
    for k in range(70):
        net.add_unit((np.cos(k), np.sin(k), 0.01 * k), 0.5)
    for k in range(1, 65):
        net.connect_or_reset(0, k)
    assert net.degree(0) == 64
    with pytest.raises(StateError, match="64"):
        net.connect_or_reset(0, 65)
    net2 = Network(EngineParams(theta0=0.5))
    for k in range(70):
        net2.add_unit((np.cos(k), np.sin(k), 0.01 * k), 0.5)
    for k in range(1, 65):
        net2.connect_or_reset(0, k)
    # the update's connect_or_reset(b, s) creates the 65th edge of unit 0
    with pytest.raises(StateError, match="64"):
        resolve_and_update(net2, EngineParams(theta0=0.5), np.zeros((1, 3)),
                           [WinnerResult(0, 66, 0.1, 0.2)])

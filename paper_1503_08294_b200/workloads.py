"""Benchmark workloads (BASELINE.json configs) as deterministic host inputs.

Each workload names a seeded synthetic point cloud, the run parameters and
the signal seed.  Clouds are materialised from a fixed Philox(2026) stream
so the reference and this package read identical points.
"""

from __future__ import annotations

import functools

import numpy as np

from .params import EngineParams
from .sampling import CloudSource, DoubleTorusSource, SphereSource, TorusSource


@functools.lru_cache(maxsize=None)
def baseline_clouds():
    """The BASELINE.md clouds: a 10k sphere then a 100k torus from Philox(2026)."""
    rng0 = np.random.Generator(np.random.Philox(2026))
    sph = SphereSource(1.0).sample(rng0, 10_000)
    tor = TorusSource(2.0, 0.5).sample(rng0, 100_000)
    return sph, tor


@functools.lru_cache(maxsize=None)
def double_torus_cloud(n: int = 1_000_000):
    """Config 3 input: n points on a genus-2 surface (two-torus blend)."""
    return DoubleTorusSource().sample(np.random.Generator(np.random.Philox(2026)), n)


@functools.lru_cache(maxsize=None)
def torus_10m_cloud(n: int = 10_000_000):
    """Config 4 input: n points on the (2.0, 0.5) torus from Philox(2026)."""
    return TorusSource(2.0, 0.5).sample(np.random.Generator(np.random.Philox(2026)), n)


WORKLOADS = {
    # BASELINE config 3: SOAM on a 1M-point genus-2 cloud.  theta0 = 0.1 and
    # m = 4096 were calibrated so the (bit-identical) run converges to a
    # closed genus-2 mesh: V=1958, E=5880 after 26,492,928 signals.
    "cfg3": dict(
        desc="SOAM, 1M-point synthetic genus-2 cloud (two-torus blend), m=4096, theta0=0.1",
        cloud=lambda: (double_torus_cloud(), "double-torus-1M"),
        params=dict(theta0=0.1, batch_floor=4096, batch_cap=4096, max_signals=60_000_000),
        seed=7,
    ),
    # BASELINE config 4: multi-signal GNG on a 10M-point cloud, the paper's
    # batch rule up to m = 65536 (m = smallest power of two above V; reached
    # once V > 32768, ~batch 172), signals sharded across 1/2/4/8 GPUs.  A
    # fixed signal budget (the network keeps growing: V ~ 38k at 2.3 M
    # signals); tests/golden/run_cfg4_prefix.npz is the reference's first
    # 4 M signals.
    "cfg4": dict(
        desc="GNG multi-signal, 10M-point synthetic torus cloud, m up to 65536 (paper rule), "
             "theta0=0.025",
        cloud=lambda: (torus_10m_cloud(), "torus-10M"),
        params=dict(theta0=0.025, batch_cap=65536, max_signals=30_000_000),
        seed=7,
    ),
    # BASELINE config 2 working anchor: converges V=681.
    "cfg2": dict(
        desc="SOAM, 100k-point synthetic torus cloud, m=1024, theta0=0.2",
        cloud=lambda: (baseline_clouds()[1], "torus-100k"),
        params=dict(theta0=0.2, batch_floor=1024, batch_cap=1024, max_signals=12_000_000),
        seed=7,
    ),
    # BASELINE config 1 (GNG multi-signal on a 10k sphere cloud, m=64)
    "cfg1": dict(
        desc="multi-signal m=64 on a 10k-point sphere cloud, theta0=0.2",
        cloud=lambda: (baseline_clouds()[0], "sphere-10k"),
        params=dict(theta0=0.2, batch_floor=64, batch_cap=64, max_signals=5_000_000),
        seed=7,
    ),
}


def make(name: str, **overrides):
    """(CloudSource, EngineParams, seed, description) for a workload."""
    w = WORKLOADS[name]
    pts, label = w["cloud"]()
    params = dict(w["params"])
    params.update(overrides)
    return CloudSource(pts, label=label), EngineParams(**params), w["seed"], w["desc"]

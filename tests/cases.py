"""Shared run configurations for the parity tests.

The same cases (sources, seeds, parameters) are what tests/golden/make_golden.py
ran through the reference.  Sources come from this package's host sampling
module; the stream SHA-256 stored in each fixture proves they reproduce the
reference's signal stream exactly.
"""

from __future__ import annotations

import functools
import os

import numpy as np

from paper_1503_08294_b200.sampling import CloudSource, SphereSource, TorusSource

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@functools.lru_cache(maxsize=None)
def clouds():
    rng0 = np.random.Generator(np.random.Philox(2026))
    sph = SphereSource(1.0).sample(rng0, 10_000)
    tor = TorusSource(2.0, 0.5).sample(rng0, 100_000)
    return sph, tor


@functools.lru_cache(maxsize=None)
def hemisphere_cloud():
    rng = np.random.Generator(np.random.Philox(99))
    pts = SphereSource(1.0).sample(rng, 20_000)
    return pts[pts[:, 2] >= 0.0]


CASES = {
    "sphere_exec": dict(source=("sphere", 1.0), seed=3,
                        params=dict(theta0=0.35, max_signals=120_000)),
    "cfg1": dict(source=("cloud", "sphere10k"), seed=7,
                 params=dict(theta0=0.2, batch_floor=64, batch_cap=64, max_signals=5_000_000)),
    "cfg2": dict(source=("cloud", "torus100k"), seed=7,
                 params=dict(theta0=0.2, batch_floor=1024, batch_cap=1024, max_signals=12_000_000)),
    "stress": dict(source=("torus", 2.0, 0.5), seed=11,
                   params=dict(theta0=0.25, max_age=12, ring_patience=3, rho=0.7,
                               stale_factor=1, batch_floor=64, batch_cap=512,
                               max_signals=80_000)),
    "boundary": dict(source=("cloud", "hemisphere"), seed=5,
                     params=dict(theta0=0.3, allow_boundary=True, max_signals=150_000)),
    "paper_rule": dict(source=("cloud", "torus100k"), seed=21,
                       params=dict(theta0=0.15, max_signals=200_000)),
    # V > 4096 (tests/golden/make_golden.py): AUTO crosses the screened small
    # find, the n <= 6144 FP64 small find and the grid
    "v8k": dict(source=("cloud", "torus100k"), seed=7,
                params=dict(theta0=0.05, batch_cap=8192, max_signals=1_500_000)),
    "cfg4_prefix": dict(source=("cloud", "torus10M"), seed=7,
                        params=dict(theta0=0.025, batch_cap=65536, max_signals=4_000_000)),
    "v8k_fixed": dict(source=("cloud", "torus100k"), seed=7,
                      params=dict(theta0=0.05, batch_floor=8192, batch_cap=8192,
                                  max_signals=1_228_800)),
}


def make_source(spec):
    kind = spec[0]
    if kind == "sphere":
        return SphereSource(spec[1])
    if kind == "torus":
        return TorusSource(spec[1], spec[2])
    if kind == "cloud":
        sph, tor = clouds()
        if spec[1] == "torus10M":
            from paper_1503_08294_b200.workloads import torus_10m_cloud

            return CloudSource(torus_10m_cloud(), label=spec[1])
        pts = {"sphere10k": sph, "torus100k": tor, "hemisphere": hemisphere_cloud()}[spec[1]]
        return CloudSource(pts, label=spec[1])
    raise ValueError(spec)


def load_golden(name):
    path = os.path.join(GOLDEN, f"run_{name}.npz")
    with np.load(path) as z:
        return {k: z[k] for k in z.files}


def same_numpy(blob) -> bool:
    return str(blob["numpy_version"]) == np.__version__


def run_device_trace(name, find_mode=None, executor=None):
    """Drive the B200 engine batch by batch (the run_multi contract,
    multi.py:134-185) and record per-batch (m, processed, discarded,
    inserted) like the golden traces."""
    import hashlib

    from paper_1503_08294_b200 import FIND_AUTO, Network
    from paper_1503_08294_b200.multi import RunState, resolve_and_update, step
    from paper_1503_08294_b200.params import EngineParams, batch_size

    case = CASES[name]
    params = EngineParams(**case["params"])
    source = make_source(case["source"])
    rng = np.random.Generator(np.random.Philox(case["seed"]))
    net = Network(params, find_mode=FIND_AUTO if find_mode is None else find_mode)
    seeds = source.sample(rng, 2)
    digest = hashlib.sha256()
    digest.update(np.ascontiguousarray(seeds).tobytes())
    for k in range(2):
        net.add_unit(seeds[k], params.theta0)
    per_batch = []
    state = RunState()  # one RunState for the whole run (multi.py:152)
    signals = discarded = iterations = 0
    units, converged, extra = 2, False, dict(events=0, windows=0, max_degree=0)
    while signals < params.max_signals:
        m = batch_size(units, params.batch_cap, params.batch_floor)
        batch = source.sample(rng, m)
        digest.update(np.ascontiguousarray(batch).tobytes())
        if executor is None:
            st = step(net, batch)
            out = (int(st.processed), int(st.discarded), int(st.inserted))
            units = int(st.units)
            conv = bool(st.converged)
            extra["events"] += int(st.events)
            extra["windows"] += int(st.windows)
            extra["max_degree"] = max(extra["max_degree"], int(st.max_degree))
        else:
            winners = executor(net.snapshot(), batch)
            o = resolve_and_update(net, params, batch, winners, state)
            out = (o.processed, o.discarded, o.inserted_units)
            c = net.counts()
            units = c["units"]
            conv = (units >= 4 and c["untrained"] == 0
                    and c["disk"] + (c["half"] if params.allow_boundary else 0) == units)
        per_batch.append((m,) + out)
        signals += m
        discarded += out[1]
        iterations += 1
        if conv:
            converged = True
            break
    c = net.counts()
    stats = dict(iterations=iterations, signals=signals, discarded=discarded, units=c["units"],
                 connections=c["edges"], converged=converged, **extra)
    return net, stats, np.array(per_batch, np.int64).reshape(-1, 4), digest.hexdigest()

"""Generate golden vectors by running the REFERENCE package (growsurf) itself.

Run here (the container that has /root/reference), never on the GPU box:

    ./oracle/build_ref.sh                 # builds growsurf into oracle/_ref
    python tests/golden/make_golden.py    # writes tests/golden/*.npz

Every fixture records numpy's version: Generator streams are only stable for
a fixed numpy, so tests skip the stream-hash checks on a different numpy.

Fixtures
  kernel_cases.npz  scan_best_two_into outputs of the compiled reference
                    backend on random / tie / duplicate instances
                    (mirrors pkg/tests/test_kernels.py:13-55).
  run_<name>.npz    a full run_multi trace (multi.py:134-202): per-batch m /
                    processed / discarded / inserted, a SHA-256 of the signal
                    stream, the final network (ids, positions, habituation,
                    thresholds, sorted edges with ages, ring classes) and the
                    RunState (patience, last_active, tick, next_sweep).
"""

from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(REPO, "oracle", "_ref"))

import growsurf  # noqa: E402
from growsurf import kernels  # noqa: E402
from growsurf.engine import EngineParams, RunState, is_converged  # noqa: E402
from growsurf.multi import batch_size, resolve_and_update, run_multi, sequential_executor  # noqa: E402
from growsurf.network import Network, RingClass  # noqa: E402
from growsurf.sampling import CloudSource, SphereSource, TorusSource  # noqa: E402

RING_CODE = {RingClass.DISK: 0, RingClass.HALF_DISK: 1, RingClass.INCONSISTENT: 2}


def clouds():
    """The BASELINE.md clouds: 10k sphere then 100k torus from Philox(2026)."""
    rng0 = np.random.Generator(np.random.Philox(2026))
    sph = SphereSource(1.0).sample(rng0, 10_000)
    tor = TorusSource(2.0, 0.5).sample(rng0, 100_000)
    return sph, tor


def hemisphere_cloud():
    rng = np.random.Generator(np.random.Philox(99))
    pts = SphereSource(1.0).sample(rng, 20_000)
    return pts[pts[:, 2] >= 0.0]


CASES = {
    # test_multi.py:180-192 executor-equivalence config
    "sphere_exec": dict(source=("sphere", 1.0), seed=3,
                        params=dict(theta0=0.35, max_signals=120_000)),
    # BASELINE config 1 (converges: V=218, 299,392 signals)
    "cfg1": dict(source=("cloud", "sphere10k"), seed=7,
                 params=dict(theta0=0.2, batch_floor=64, batch_cap=64, max_signals=5_000_000)),
    # BASELINE config 2 working anchor (converges: V=681, 4,277,248 signals)
    "cfg2": dict(source=("cloud", "torus100k"), seed=7,
                 params=dict(theta0=0.2, batch_floor=1024, batch_cap=1024, max_signals=12_000_000)),
    # stress: short edge lifetime, tiny patience, aggressive sweeping
    "stress": dict(source=("torus", 2.0, 0.5), seed=11,
                   params=dict(theta0=0.25, max_age=12, ring_patience=3, rho=0.7,
                               stale_factor=1, batch_floor=64, batch_cap=512,
                               max_signals=80_000)),
    # open surface with half-disk rings accepted
    "boundary": dict(source=("cloud", "hemisphere"), seed=5,
                     params=dict(theta0=0.3, allow_boundary=True, max_signals=150_000)),
    # paper batch rule (floor 64, cap 8192) on the torus cloud, prefix only
    "paper_rule": dict(source=("cloud", "torus100k"), seed=21,
                       params=dict(theta0=0.15, max_signals=200_000)),
    # large network (V > 4096): the engine's AUTO find crosses every regime
    # (screened small find, n <= 6144 FP64 small find, filter / grid) under
    # the paper batch rule (m up to 8192); V ~ 9.9k after 1.5 M signals
    "v8k": dict(source=("cloud", "torus100k"), seed=7,
                params=dict(theta0=0.05, batch_cap=8192, max_signals=1_500_000)),
    # BASELINE config 4 prefix: 10M-point torus cloud, paper batch rule up to
    # m = 65536 (paper_1503_08294_b200/workloads.py "cfg4"), first ~4 M signals
    "cfg4_prefix": dict(source=("cloud", "torus10M"), seed=7, parallel=True,
                        params=dict(theta0=0.025, batch_cap=65536, max_signals=4_000_000)),
    # the same cloud with a fixed m = 8192 (the asynchronous device-sampled path)
    "v8k_fixed": dict(source=("cloud", "torus100k"), seed=7,
                      params=dict(theta0=0.05, batch_floor=8192, batch_cap=8192,
                                  max_signals=1_228_800)),
}


def torus10m_cloud():
    """BASELINE config 4's 10M-point torus cloud (workloads.py torus_10m_cloud)."""
    return TorusSource(2.0, 0.5).sample(np.random.Generator(np.random.Philox(2026)), 10_000_000)


def make_source(spec, cache):
    kind = spec[0]
    if kind == "cloud" and spec[1] == "torus10M" and spec[1] not in cache:
        cache[spec[1]] = torus10m_cloud()
    if kind == "sphere":
        return SphereSource(spec[1])
    if kind == "torus":
        return TorusSource(spec[1], spec[2])
    if kind == "cloud":
        return CloudSource(cache[spec[1]], label=spec[1])
    raise ValueError(spec)


def trace_run(source, params: EngineParams, seed: int, executor=None):
    """The run_multi driver (multi.py:134-185) with the state kept visible."""
    rng = np.random.Generator(np.random.Philox(seed))
    net = Network()
    net.watch_age_limit(params.max_age)
    seeds = source.sample(rng, 2)
    for k in range(2):
        net.add_unit(seeds[k], params.theta0)
    digest = hashlib.sha256()
    digest.update(np.ascontiguousarray(seeds).tobytes())
    state = RunState()
    executor = executor or sequential_executor()
    per_batch = []
    signals = discarded = iterations = 0
    converged = False
    while signals < params.max_signals:
        m = batch_size(net.unit_count, params.batch_cap, params.batch_floor)
        batch = source.sample(rng, m)
        digest.update(np.ascontiguousarray(batch).tobytes())
        winners = executor(net.snapshot(), batch)
        out = resolve_and_update(net, params, batch, winners, state)
        per_batch.append((m, out.processed, out.discarded, out.inserted_units))
        signals += m
        discarded += out.discarded
        iterations += 1
        if is_converged(net, params):
            converged = True
            break
    return net, state, np.array(per_batch, dtype=np.int64), digest.hexdigest(), dict(
        iterations=iterations, signals=signals, discarded=discarded,
        units=net.unit_count, connections=net.edge_count, converged=converged)


def dump_network(net: Network, state: RunState):
    ids, pos, hab, theta = net.state_arrays()
    ids = ids.copy()
    edges = np.array(net.edges(), dtype=np.int64).reshape(-1, 3)
    ring = np.array([RING_CODE[net.link_ring(int(u))] for u in ids], dtype=np.int64)
    patience = np.array([state.patience.get(int(u), 0) for u in ids], dtype=np.int64)
    last_active = np.array([state.last_active.get(int(u), -1) for u in ids], dtype=np.int64)
    return dict(ids=ids, pos=pos.copy(), hab=hab.copy(), theta=theta.copy(), edges=edges,
                ring=ring, patience=patience, last_active=last_active,
                tick=np.int64(state.tick), next_sweep=np.int64(state.next_sweep),
                next_id=np.int64(net.next_id))


def make_kernel_cases(path):
    kb = kernels.get_backend("compiled")
    rng = np.random.default_rng(1234)
    out = {}
    cases = []
    for _ in range(24):
        n = int(rng.integers(2, 400))
        m = int(rng.integers(1, 300))
        cases.append((np.ascontiguousarray(rng.random((n, 3))),
                      np.ascontiguousarray(rng.random((m, 3)) * 1.4 - 0.2)))
    # ties and duplicates (test_kernels.py:44-55)
    cases.append((np.array([[1.0, 0, 0], [-1.0, 0, 0], [2.0, 0, 0]]), np.zeros((1, 3))))
    cases.append((np.array([[0.5, 0.5, 0.5]] * 4), np.array([[0.1, 0.2, 0.3]])))
    grid = np.stack(np.meshgrid(*[np.arange(6.0)] * 3, indexing="ij"), -1).reshape(-1, 3) * 0.25
    cases.append((np.ascontiguousarray(grid), np.ascontiguousarray(grid[::7] + 0.125)))
    # larger instance spanning several CTA tiles / unit chunks
    cases.append((np.ascontiguousarray(rng.random((5000, 3))),
                  np.ascontiguousarray(rng.random((3000, 3)))))
    for k, (pos, sig) in enumerate(cases):
        m = sig.shape[0]
        idx = np.empty((m, 2), np.int64)
        d2 = np.empty((m, 2), np.float64)
        kb.scan_best_two_into(pos, pos.shape[0], sig, idx, d2, 64)
        out[f"pos{k}"] = pos
        out[f"sig{k}"] = sig
        out[f"idx{k}"] = idx
        out[f"d2{k}"] = d2
    out["count"] = np.int64(len(cases))
    out["numpy_version"] = np.array(np.__version__)
    np.savez_compressed(path, **out)


def main(only=None):
    sph, tor = clouds()
    cache = {"sphere10k": sph, "torus100k": tor, "hemisphere": hemisphere_cloud()}
    if not only or "kernel_cases" in only:
        make_kernel_cases(os.path.join(HERE, "kernel_cases.npz"))
    for name, case in CASES.items():
        if only and name not in only:
            continue
        params = EngineParams(**case["params"])
        src = make_source(case["source"], cache)
        t0 = time.perf_counter()
        ex = None
        if case.get("parallel"):  # bitwise identical to the sequential scan (test_multi.py:180-192)
            from growsurf.parallel import ExecConfig, parallel_executor

            ex = parallel_executor(ExecConfig(workers=os.cpu_count() or 1))
        net, state, per_batch, digest, stats = trace_run(src, params, case["seed"], ex)
        dt = time.perf_counter() - t0
        # cross-check the traced driver against the reference's own run_multi
        if name in ("sphere_exec", "cfg1", "stress", "boundary"):
            net2, st2 = run_multi(src, params, case["seed"])
            assert st2.signals == stats["signals"] and st2.discarded == stats["discarded"]
            assert net2.edges() == net.edges()
            assert np.array_equal(net2.snapshot().positions, net.snapshot().positions)
        blob = dump_network(net, state)
        blob.update(per_batch=per_batch, signal_sha256=np.array(digest),
                    numpy_version=np.array(np.__version__),
                    seed=np.int64(case["seed"]),
                    **{f"stat_{k}": np.int64(v) for k, v in stats.items()})
        np.savez_compressed(os.path.join(HERE, f"run_{name}.npz"), **blob)
        print(f"{name}: {stats} ({dt:.1f}s)", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or None)

"""Checkpoints of the REFERENCE's own config-3 run, for bench.py's reference arm.

Run here (the container with /root/reference), never on the GPU box:

    python tests/golden/make_ref_checkpoints.py

The unmodified reference (oracle/_ref) runs the config-3 run (1M-point
genus-2 cloud, m = 4096, theta0 = 0.1, seed 7) with its own functions in
the order of run_multi (multi.py:134-185: sample, parallel executor,
resolve_and_update, is_converged) and pickles its own objects -- the
Network, the RunState and the Philox generator state -- at the start of
each of STRATA equal slices of the run's batches.  bench.py --impl reference
resumes the stock reference from each checkpoint for a bounded number of
seconds and estimates the whole run's time-to-converge as the sum over
slices of (batches in the slice x measured seconds per batch): a stratified
sample of the full run instead of its cheap early prefix.  The final state is
checked against tests/golden/run_cfg3_final.npz (the reference's own full
run).
"""

from __future__ import annotations

import gzip
import os
import pickle
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(REPO, "oracle", "_ref"))
sys.path.insert(0, REPO)

STRATA = 8


def main():
    from growsurf import CloudSource, EngineParams
    from growsurf.engine import RunState, is_converged
    from growsurf.multi import batch_size, resolve_and_update
    from growsurf.network import Network
    from growsurf.parallel import ExecConfig, parallel_executor

    from paper_1503_08294_b200 import workloads

    gold = np.load(os.path.join(HERE, "run_cfg3_final.npz"))
    total = int(gold["stat_iterations"])
    starts = [k * total // STRATA for k in range(STRATA)]
    w = workloads.WORKLOADS["cfg3"]
    pts, label = w["cloud"]()
    src = CloudSource(pts, label=label)
    params = EngineParams(**w["params"])
    executor = parallel_executor(ExecConfig(workers=os.cpu_count() or 1))
    rng = np.random.Generator(np.random.Philox(w["seed"]))
    net = Network()
    net.watch_age_limit(params.max_age)
    for s in src.sample(rng, 2):
        net.add_unit(s, params.theta0)
    state = RunState()
    signals = batches = 0
    cps, seconds = [], []
    t0 = time.perf_counter()
    while signals < params.max_signals:
        if batches in starts:
            seconds.append(time.perf_counter() - t0)
            cps.append(pickle.dumps(dict(batch=batches, signals=signals, net=net, state=state,
                                         rng=rng.bit_generator.state), protocol=4))
            print(f"checkpoint at batch {batches} ({seconds[-1]:.0f} s)", flush=True)
        m = batch_size(net.unit_count, params.batch_cap, params.batch_floor)
        batch = src.sample(rng, m)
        winners = executor(net.snapshot(), batch)
        resolve_and_update(net, params, batch, winners, state)
        signals += m
        batches += 1
        if is_converged(net, params):
            break
    seconds.append(time.perf_counter() - t0)
    assert batches == total and signals == int(gold["stat_signals"])
    ids, pos, hab, theta = net.state_arrays()
    assert np.array_equal(ids, gold["ids"]) and np.array_equal(pos.view(np.int64), gold["pos"].view(np.int64))
    blob = dict(workload="cfg3", strata=STRATA, starts=starts, total_batches=total,
                total_signals=signals, numpy_version=np.__version__,
                made_on=dict(cores=os.cpu_count(), stratum_start_s=seconds),
                checkpoints=cps)
    with gzip.open(os.path.join(HERE, "ref_cfg3_checkpoints.pkl.gz"), "wb") as fh:
        pickle.dump(blob, fh, protocol=4)
    print(f"done: {batches} batches, {signals} signals, {seconds[-1]:.0f} s", flush=True)


if __name__ == "__main__":
    main()

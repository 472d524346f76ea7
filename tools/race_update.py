"""Short engine run for compute-sanitizer racecheck / synccheck on the
update kernel (tools/sanitize.sh): a few batches of the stress case (events
of every kind: edge creation, insertion, pruning, sweeps) and of a fixed-m
sampled run, each checked against the C oracle so a race that changes a
result also fails here."""
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))
import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_1503_08294_b200 import EngineParams, TorusSource, run_multi  # noqa: E402

batches = int(sys.argv[1]) if len(sys.argv) > 1 else 12
for name, params, seed in (
        ("stress", EngineParams(theta0=0.25, max_age=12, ring_patience=3, rho=0.7,
                                stale_factor=1, batch_floor=64, batch_cap=512,
                                max_signals=64 * batches), 11),
        ("fixed", EngineParams(theta0=0.3, batch_floor=256, batch_cap=256,
                               max_signals=256 * batches), 5)):
    net, st = run_multi(TorusSource(2.0, 0.5), params, seed)
    onet, ost, _, _ = O.run_multi_oracle(TorusSource(2.0, 0.5), params, seed)
    got, want = net.export(), onet.export()
    ok = (np.array_equal(got["ids"], want["ids"]) and np.array_equal(got["edges"], want["edges"])
          and np.array_equal(got["pos"].view(np.int64), want["pos"].view(np.int64)))
    print(f"{name}: {st.iterations} batches, V={st.units}, E={st.connections}, "
          f"matches oracle: {ok}", flush=True)
    assert ok

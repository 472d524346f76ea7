"""Golden run of the reference's SINGLE-signal engine (engine.py:368-462).

Run here (the container with /root/reference, oracle/_ref built):
    python tests/golden/make_single_golden.py
Writes tests/golden/run_single.npz: final network + RunState of
growsurf.run(SphereSource(1.0), EngineParams(theta0=0.35, max_signals=20000), 3)
with the compiled backend, plus numpy's version (streams are numpy-specific).
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

from make_golden import dump_network  # noqa: E402  (also puts oracle/_ref on sys.path)

from growsurf import run  # noqa: E402
from growsurf.engine import EngineParams  # noqa: E402
from growsurf.sampling import SphereSource  # noqa: E402
import growsurf.engine as ge  # noqa: E402


def main():
    params = EngineParams(theta0=0.35, max_signals=20_000)
    captured = {}
    orig = ge.update_single

    def spy(net, params_, signal, wr, state, grid=None):  # keep the RunState for dumping
        captured["state"] = state
        return orig(net, params_, signal, wr, state, grid)

    ge.update_single = spy
    try:
        net, st = run(SphereSource(1.0), params, 3, checkpoints=(10, 40))
    finally:
        ge.update_single = orig
    blob = dump_network(net, captured["state"])
    for k in ("iterations", "signals", "discarded", "units", "connections", "converged"):
        blob[f"stat_{k}"] = np.int64(getattr(st, k))
    blob["checkpoint_units"] = np.array([c[0] for c in st.checkpoints], np.int64)
    blob["checkpoint_signals"] = np.array([c[1] for c in st.checkpoints], np.int64)
    blob["numpy_version"] = np.array(np.__version__)
    np.savez_compressed(os.path.join(HERE, "run_single.npz"), **blob)
    print("run_single:", st.signals, "signals, V =", st.units, "E =", st.connections,
          "converged =", st.converged)


if __name__ == "__main__":
    main()

"""Calibrate BASELINE config 3 (1M-point genus-2 cloud) on the B200 engine.

The engine is bit-exact with the reference, so convergence found here is
the reference's convergence on the same seeded stream."""
import os, sys, time
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import numpy as np
from paper_1503_08294_b200 import (CloudSource, DoubleTorusSource, EngineParams, extract_mesh,
                                   genus, manifold_check, run_multi)

t = time.time()
pts = DoubleTorusSource().sample(np.random.Generator(np.random.Philox(2026)), 1_000_000)
print(f"cloud {pts.shape} in {time.time()-t:.1f}s", flush=True)
src = CloudSource(pts, label="double-torus-1M")
grid = [(float(a), int(b)) for a, b in (x.split(":") for x in sys.argv[1:])] or \
    [(0.2, 1024), (0.2, 4096), (0.15, 4096), (0.1, 4096), (0.15, 16384), (0.1, 16384)]
for theta0, m in grid:
    p = EngineParams(theta0=theta0, batch_floor=m, batch_cap=m, max_signals=60_000_000)
    net, st = run_multi(src, p, 7)
    mesh = extract_mesh(net)
    cls = manifold_check(mesh)
    g = genus(mesh) if cls == "closed" else None
    print(f"theta0={theta0} m={m}: conv={st.converged} V={st.units} E={st.connections} "
          f"iters={st.iterations} signals={st.signals} disc={st.discarded} total={st.total_s:.2f}s "
          f"find={st.find_s:.2f} update={st.update_s:.2f} sample={st.sample_s:.2f} "
          f"manifold={cls} genus={g} rate={st.signals/st.total_s/1e6:.2f}M/s", flush=True)

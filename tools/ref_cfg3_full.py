"""Full reference run of config 3 (CPU, this container) for the record:
time-to-converge of the unmodified reference on the same seeded stream."""
import os, sys, time, json
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(REPO, "oracle", "_ref"))
sys.path.insert(0, REPO)
import numpy as np
from paper_1503_08294_b200.sampling import DoubleTorusSource
from growsurf import CloudSource, EngineParams, run_multi, extract_mesh, manifold_check, genus
from growsurf.parallel import ExecConfig, parallel_executor
pts = DoubleTorusSource().sample(np.random.Generator(np.random.Philox(2026)), 1_000_000)
src = CloudSource(pts, label="double-torus-1M")
p = EngineParams(theta0=0.1, batch_floor=4096, batch_cap=4096, max_signals=60_000_000)
t = time.time()
net, st = run_multi(src, p, 7, parallel_executor(ExecConfig(workers=os.cpu_count())), variant="multi-parallel")
mesh = extract_mesh(net); cls = manifold_check(mesh)
rec = dict(config="cfg3 double-torus 1M theta0=0.1 m=4096 seed 7", cores=os.cpu_count(),
           converged=st.converged, units=st.units, edges=st.connections, iterations=st.iterations,
           signals=st.signals, discarded=st.discarded, total_s=st.total_s, find_s=st.find_s,
           update_s=st.update_s, sample_s=st.sample_s, manifold=cls,
           genus=genus(mesh) if cls == "closed" else None, numpy=np.__version__)
print(json.dumps(rec), flush=True)
ids, pos, hab, theta = net.state_arrays()
np.savez_compressed(sys.argv[1] if len(sys.argv) > 1 else "/tmp/ref_cfg3_final.npz", ids=ids, pos=pos, hab=hab, theta=theta,
                    edges=np.array(net.edges(), np.int64))

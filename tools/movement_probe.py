"""Per-batch maximum unit displacement and nearest-unit gaps of a config-3
run (host batches, positions exported after every batch for the batches
probed): the movement bound a speculative find against the previous
snapshot would have to absorb.  Usage: python tools/movement_probe.py"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402,F401
import numpy as np  # noqa: E402

from paper_1503_08294_b200 import _lib, workloads  # noqa: E402
from paper_1503_08294_b200.network import Network  # noqa: E402
from paper_1503_08294_b200.params import batch_size  # noqa: E402

src, params, seed, _ = workloads.make("cfg3")
lib = _lib.load_library()
rng = np.random.Generator(np.random.Philox(seed))
net = Network(params, capacity=8192)
for s in src.sample(rng, 2):
    net.add_unit(s, params.theta0)
st = _lib.GsBatchStats()
units = 2
prev = None
probe = set(range(100, 110)) | set(range(600, 610)) | set(range(1500, 1510)) | set(range(4000, 4010))
for b in range(4010):
    m = batch_size(units, params.batch_cap, params.batch_floor)
    batch = np.ascontiguousarray(src.sample(rng, m))
    if b in probe or b - 1 in probe:
        ex = net.export()
        cur = dict(zip(ex["ids"].tolist(), ex["pos"]))
        if b - 1 in probe and prev is not None:
            common = [i for i in cur if i in prev]
            d = np.array([np.linalg.norm(cur[i] - prev[i]) for i in common])
            P = np.array([cur[i] for i in common])
            # nearest-unit distances of the batch's signals (2nd minus 1st)
            D = np.sqrt(((batch[:512, None, :] - P[None, :, :]) ** 2).sum(-1))
            D.sort(axis=1)
            gap = D[:, 1] - D[:, 0]
            print(f"batch {b-1}: V={len(cur)} max disp {d.max():.3e} p99 {np.percentile(d,99):.3e} "
                  f"median {np.median(d):.3e}; signals' d1 median {np.median(D[:,0]):.3e}, "
                  f"d2-d1 median {np.median(gap):.3e}, d3-d2 median {np.median(D[:,2]-D[:,1]):.3e}", flush=True)
        prev = cur
    _lib.check(lib.gs_engine_step(net.handle, batch, m, C.byref(st)))
    net._touch()
    units = int(st.units)
    if st.converged:
        break

"""Per-batch critical path of the find -> update chain from a timeline
profiling build (-DGS_PROF_TL=0: globaltimer stamps kept on the device, no
printing): one config-3 run through run_multi, then the stamps.
Usage: GS_LIB_PATH=<tl build> python tools/tl_gaps.py [batches] [workload]"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1503_08294_b200 import _lib, workloads  # noqa: E402
from paper_1503_08294_b200.multi import run_multi  # noqa: E402

nb = int(sys.argv[1]) if len(sys.argv) > 1 else 8000
NAME = sys.argv[2] if len(sys.argv) > 2 else "cfg3"
src, params, seed, _ = workloads.make(NAME)
params = type(params)(**{**params.__dict__, "max_signals": nb * params.batch_cap})
net, st = run_multi(src, params, seed, capacity=8192)
n = min(st.iterations + 1, 8192)
lib = _lib.load_library()
f = np.zeros((8192, 3), np.uint64)
u = np.zeros((8192, 3), np.uint64)
lib.gs_debug_tl_find(f.ctypes.data_as(C.c_void_p), 8192)
lib.gs_debug_tl_update(u.ctypes.data_as(C.c_void_p), 8192)
f = f.astype(np.float64)
u = u.astype(np.float64)
rows = []
for b in range(2, n):
    if f[b, 2] == 0 or u[b, 1] == 0 or u[b - 1, 2] == 0:
        continue  # not a screened-find batch
    rows.append((b, (f[b, 0] - u[b - 1, 2]) / 1e3, (f[b, 1] - f[b, 0]) / 1e3,
                 (u[b, 1] - f[b, 1]) / 1e3, (u[b, 2] - u[b, 1]) / 1e3,
                 (u[b, 2] - u[b - 1, 2]) / 1e3))
r = np.array(rows)
print(f"{len(r)} batches with stamps (of {st.iterations})")
print("batches            upd_end->find_rel  find_run  find_end->upd_rel  upd_run  batch_total (us, mean)")
for lo, hi in [(0, 64), (64, 130), (130, 650), (650, 2000), (2000, 8192)]:
    m = (r[:, 0] >= lo) & (r[:, 0] < hi)
    if m.any():
        mu = r[m, 1:].mean(axis=0)
        print(f"[{lo:5d},{hi:5d}) n={m.sum():5d}  " + "  ".join(f"{x:8.2f}" for x in mu))
tot = r[:, 5].sum() / 1e3
print(f"sum of batch totals {tot:.1f} ms; gaps {r[:, 1].sum() / 1e3:.1f} + {r[:, 3].sum() / 1e3:.1f} ms, "
      f"find {r[:, 2].sum() / 1e3:.1f} ms, update {r[:, 4].sum() / 1e3:.1f} ms")

"""Where the update's tail goes (a -DGS_PROF_TL=0 build): per batch, the
latest CTA past the last cluster barrier, the latest snapshot flag, CTA 0's
end, and the next find's release (CTA 0), relative to the update's start.
Usage: GS_LIB_PATH=<tl build> python tools/tl_flags.py [batches] [workload]"""
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
u2 = np.zeros((8192, 2), np.uint64)
lib.gs_debug_tl_find(f.ctypes.data_as(C.c_void_p), 8192)
lib.gs_debug_tl_update(u.ctypes.data_as(C.c_void_p), 8192)
lib.gs_debug_tl_update2(u2.ctypes.data_as(C.c_void_p), 8192)
f2 = np.zeros((8192, 3), np.uint64)
has_f2 = hasattr(lib, "gs_debug_tl_find2")
if has_f2:
    lib.gs_debug_tl_find2(f2.ctypes.data_as(C.c_void_p), 8192)
f2 = f2.astype(np.float64)
f, u, u2 = f.astype(np.float64), u.astype(np.float64), u2.astype(np.float64)
rows = []
for b in range(2, n - 1):
    if u[b, 1] == 0 or u2[b, 1] == 0 or f[b + 1, 0] == 0:
        continue
    t0 = u[b, 1]
    rows.append((b, (u2[b, 0] - t0) / 1e3, (u2[b, 1] - t0) / 1e3, (u[b, 2] - t0) / 1e3,
                 (f[b + 1, 0] - t0) / 1e3, (f2[b + 1, 0] - t0) / 1e3, (f2[b + 1, 1] - t0) / 1e3,
                 (f2[b + 1, 2] - t0) / 1e3))
r = np.array(rows)
print("batches  last_barrier  last_flag  cta0_end  next_find_release  find0_entry  find0_poll  findlast_poll  (us after the update's start)")
for lo, hi in [(0, 130), (130, 650), (650, 2000), (2000, 8192)]:
    m = (r[:, 0] >= lo) & (r[:, 0] < hi)
    if m.any():
        print(f"[{lo:5d},{hi:5d}) n={m.sum():5d} " + " ".join(f"{x:9.2f}" for x in r[m, 1:].mean(axis=0)))

"""Where the end-to-end run_multi time goes (GPU box)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1503_08294_b200 import workloads, _lib
from paper_1503_08294_b200.multi import run_multi
from paper_1503_08294_b200.network import Network
from paper_1503_08294_b200.device_sampling import DeviceCloudSampler

src, params, seed, desc = workloads.make("cfg3")
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    net = Network(params, capacity=8192)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    s = DeviceCloudSampler(src.points, np.random.Generator(np.random.Philox(seed)))
    torch.cuda.synchronize(); t2 = time.perf_counter()
    net.close(); s.close()
    t3 = time.perf_counter()
    net2, st = run_multi(src, params, seed, capacity=8192)
    torch.cuda.synchronize(); t4 = time.perf_counter()
    print(f"rep {rep}: Network() {1e3*(t1-t0):.1f} ms, sampler+H2D {1e3*(t2-t1):.1f} ms, "
          f"run_multi {1e3*(t4-t3):.1f} ms (RunStats.total_s {1e3*st.total_s:.1f} ms, "
          f"find {1e3*st.find_s:.1f}, update {1e3*st.update_s:.1f}), V={st.units}", flush=True)
    net2.close()

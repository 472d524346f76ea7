import os, sys, time
sys.path.insert(0, "/root/repo")
import torch
from paper_1503_08294_b200 import workloads
from paper_1503_08294_b200.multi import run_multi
src, params, seed, desc = workloads.make("cfg3")
for pt in (True, False, True, False):
    ts = []
    for _ in range(3):
        torch.cuda.synchronize(); t = time.perf_counter()
        net, st = run_multi(src, params, seed, phase_timing=pt)
        torch.cuda.synchronize(); ts.append(1e3 * (time.perf_counter() - t))
        net.close()
    print("phase_timing", pt, ["%.0f" % x for x in ts], flush=True)

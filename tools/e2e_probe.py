"""Where run_multi's time outside the batch loop goes (GPU box)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1503_08294_b200 import workloads, _lib
from paper_1503_08294_b200.network import Network
from paper_1503_08294_b200.device_sampling import DeviceCloudSampler

src, params, seed, desc = workloads.make("cfg3")
for i in range(6):
    T = [time.perf_counter()]
    rng = np.random.Generator(np.random.Philox(seed))
    net = Network(params, capacity=8192); T.append(time.perf_counter())
    net.watch_age_limit(params.max_age)
    seeds = src.sample(rng, 2)
    for k in range(2):
        net.add_unit(seeds[k], params.theta0)
    T.append(time.perf_counter())
    s = DeviceCloudSampler(src.points, rng); T.append(time.perf_counter())
    net.reserve(net.next_id + params.batch_cap * 10); T.append(time.perf_counter())
    net.set_async(8); T.append(time.perf_counter())
    net.set_async(0); s.close(); T.append(time.perf_counter())
    net.close(); T.append(time.perf_counter())
    names = ["Network()", "add_units", "sampler", "reserve", "set_async", "teardown", "close"]
    print(f"rep {i}: " + " ".join(f"{n}={1e3*(b-a):.1f}" for n, a, b in zip(names, T, T[1:])), flush=True)

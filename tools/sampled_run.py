"""run_multi on a workload with device sampling for a fixed number of batches
(launch-list captures of the device-resident pipeline)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1503_08294_b200 import workloads
from paper_1503_08294_b200.multi import run_multi

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
src, params, seed, desc = workloads.make(name)
params = type(params)(**{**params.__dict__, "max_signals": nb * params.batch_cap})
t0 = time.perf_counter()
net, st = run_multi(src, params, seed, capacity=8192)
print(f"{name}: {st.iterations} batches, {st.signals} signals, V={st.units}, conv={st.converged}, "
      f"{time.perf_counter() - t0:.2f}s")

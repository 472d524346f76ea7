"""Run a workload for a fixed number of batches (for ncu captures) and print
per-batch engine statistics (events, windows) of the last batches."""
import ctypes as C, os, sys, time
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import numpy as np
from paper_1503_08294_b200 import _lib, workloads
from paper_1503_08294_b200.network import Network

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 100000
mode = int(sys.argv[3]) if len(sys.argv) > 3 else _lib.FIND_AUTO
src, params, seed, desc = workloads.make(name)
lib = _lib.load_library()
rng = np.random.Generator(np.random.Philox(seed))
net = Network(params, capacity=8192, find_mode=mode)
for s in src.sample(rng, 2):
    net.add_unit(s, params.theta0)
st = _lib.GsBatchStats()
units, signals = 2, 0
ev = win = proc = 0
t0 = time.perf_counter()
for b in range(nb):
    from paper_1503_08294_b200.params import batch_size
    m = batch_size(units, params.batch_cap, params.batch_floor)
    batch = np.ascontiguousarray(src.sample(rng, m))
    _lib.check(lib.gs_engine_step(net.handle, batch, m, C.byref(st)))
    units = int(st.units); signals += m
    ev += st.events; win += st.windows; proc += st.processed
    if os.environ.get("GS_FB"):
        fb = np.zeros(2, np.int64)
        _lib.check(lib.gs_find_last_fallback_counts(_lib.default_context().handle, fb))
        fbs = globals().setdefault("fbs", [])
        fbs.append(int(fb[0]))
    if st.converged:
        break
print(f"{name}: batches={b+1} signals={signals} V={units} conv={bool(st.converged)} "
      f"events/batch={ev/(b+1):.2f} windows/batch={win/(b+1):.2f} processed/batch={proc/(b+1):.0f} "
      f"maxdeg={st.max_degree} wall={time.perf_counter()-t0:.1f}s causes: create={st.ev_create} "
      f"insert={st.ev_insert} prune={st.ev_prune} sweep={st.ev_sweep} "
      f"serial-cycles={st.cyc_serial/max(1,st.cyc_total):.3f} of {st.cyc_total/1.9e9:.3f}s", flush=True)
if os.environ.get("GS_FB"):
    print("find fallbacks per batch: mean %.1f, last-100 mean %.1f, max %d" % (
        np.mean(fbs), np.mean(fbs[-100:]), max(fbs)))
names = {0: "A+scan", 2: "B", 3: "C1", 6: "walk", 7: "reset", 4: "ev:connect+moves",
         5: "ev:insert+prune", 1: "ev:reclass", 8: "ev:adapt", 9: "ev:barrier"}
print("  update phases (s): " + " ".join(f"{n}={st.cyc_phase[i]/1.9e9:.3f}" for i, n in names.items()))

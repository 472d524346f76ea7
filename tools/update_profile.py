"""Per-batch update-kernel time over one cfg3 run (GPU box): deciles of the
run by batch index with mean update/find us, processed signals, events and
windows per batch -- where the update's time goes along a run."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1503_08294_b200 import _lib, workloads
from paper_1503_08294_b200.network import Network
from paper_1503_08294_b200.device_sampling import DeviceCloudSampler, philox_state_words

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
src, params, seed, desc = workloads.make(name)
lib = _lib.load_library()
m = params.batch_cap
rng = np.random.Generator(np.random.Philox(seed))
seeds = src.sample(rng, 2)
state0 = philox_state_words(rng)
pts = torch.from_numpy(src.points).cuda()
smp = DeviceCloudSampler(None, device_ptr=pts.data_ptr(), npts=src.points.shape[0])
net = Network(params, capacity=8192)
net.reserve(8192)
st = _lib.GsBatchStats()
ph = np.zeros(2)
rows = []
for rep in range(2):
    net.reset()
    for s in seeds:
        net.add_unit(s, params.theta0)
    _lib.check(lib.gs_sampler_set_state(smp.handle, state0))
    _lib.check(lib.gs_engine_phase_ms(net.handle, 1, ph))
    prev = ph.copy()
    rows = []
    off = 0
    while off < params.max_signals:
        _lib.check(lib.gs_engine_step_sampled(net.handle, smp.handle, m, C.byref(st)))
        _lib.check(lib.gs_engine_phase_ms(net.handle, -1, ph))
        off += m
        rows.append((ph[0] - prev[0], ph[1] - prev[1], st.processed, st.events, st.windows,
                     st.units, st.inserted, st.ev_create, st.ev_insert, st.ev_prune, st.ev_sweep,
                     st.cyc_total) + tuple(st.cyc_phase[q] for q in range(12)))
        prev = ph.copy()
        if st.converged:
            break
r = np.array(rows, dtype=np.float64)
print(f"{name}: {len(r)} batches, find {r[:,0].sum():.1f} ms, update {r[:,1].sum():.1f} ms")
print("decile  find_us  upd_us  processed  events  windows  units  inserted  ev_create ev_insert ev_prune ev_sweep")
for d, part in enumerate(np.array_split(r, 10)):
    mu = part.mean(axis=0)
    print(f"{d:6d} {1e3*mu[0]:8.1f} {1e3*mu[1]:7.1f} {mu[2]:10.0f} {mu[3]:7.1f} {mu[4]:8.1f} {mu[5]:6.0f} {mu[6]:9.2f} "
          f"{mu[7]:9.2f} {mu[8]:9.2f} {mu[9]:8.2f} {mu[10]:8.2f}")
# 3 / 10 / 11: profiling builds only (GS_PROF_B: slowest B / walk chain;
# GS_PROF_TAIL: tail barrier / row snapshot / compaction check)
PH = {0: "A+scan", 2: "B", 3: "x3", 10: "x10", 11: "x11", 6: "walk", 7: "reset", 4: "ev:conn+mv", 5: "ev:ins+prune",
      1: "ev:reclass", 8: "ev:adapt", 9: "ev:barrier"}
cyc = np.diff(np.concatenate([np.zeros((1, 13)), r[:, 11:24]]), axis=0) / 1.9e3  # us at 1.9 GHz
nb = len(r)
cuts = [0] + [nb * k // 100 for k in range(1, 11)] + [nb]
print("first tenth in 1% slices (us per batch); columns: upd_us events windows total " + " ".join(PH.values()))
for lo, hi in zip(cuts, cuts[1:]):
    c = cyc[lo:hi].mean(axis=0)
    print(f"[{lo:5d},{hi:5d}) {1e3*r[lo:hi,1].mean():7.1f} {r[lo:hi,3].mean():6.1f} {r[lo:hi,4].mean():6.1f} "
          f"{c[0]:7.1f} " + " ".join(f"{c[1+q]:7.1f}" for q in PH))
# serial-path causes per batch by slice (increments of the cumulative counters)
evc = np.diff(np.concatenate([np.zeros((1, 4)), r[:, 7:11]]), axis=0)
print("event causes per batch: events create insert prune sweep (an event may have several)")
for lo, hi in zip(cuts, cuts[1:]):
    c = evc[lo:hi].mean(axis=0)
    print(f"[{lo:5d},{hi:5d}) {r[lo:hi, 3].mean():7.2f} " + " ".join(f"{x:7.2f}" for x in c))
# update time vs events: least squares us = a + b*windows + c*events
A = np.stack([np.ones(len(r)), r[:, 4], r[:, 3], r[:, 2]], 1)
coef = np.linalg.lstsq(A, 1e3 * r[:, 1], rcond=None)[0]
print("fit upd_us = %.1f + %.2f*windows + %.2f*events + %.4f*processed" % tuple(coef))

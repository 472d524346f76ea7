#!/usr/bin/env python
"""Benchmark: signals/s and time-to-converge of the multi-signal SOAM run.

Contract (driver): ``python bench.py --gpus N --steps K --warmup W`` (torchrun
for N > 1) prints ONE JSON line on rank 0.

* workload (default ``cfg3``): BASELINE config 3 -- SOAM on a 1M-point
  synthetic genus-2 cloud, m = 4096, theta0 = 0.1, seed 7.  One STEP is one
  complete seeded run from the two seed units to convergence (26.5 M
  signals, V = 1958, closed genus-2 mesh); ms_per_step is the
  time-to-converge.  The run is bit-identical to the reference's.  At N > 1
  every batch's find is sharded over the ranks (the engine's own NCCL
  communicator, one ncclAllGather of winner records per batch, replicated
  update: distributed.py), so the per-N lines are the same run.
* value: whole-job signals/s with the cloud resident in HBM; every batch's
  signals are drawn ON THE DEVICE inside the timed region from the same
  Philox stream as the reference (csrc/sample.cu, bit-identical to numpy);
  CUDA events on the engine stream, 256 MiB L2 flush before each step; max
  over ranks.
* e2e: the same metric through the public API (``run_multi``, or
  ``distributed.run_multi_sharded`` at N > 1) from host memory: the cloud's
  H2D copy, the sampler state and every batch's stats (written by the
  update kernel into pinned host memory) are inside the timed region.
* cpu_baseline / --impl reference: the unmodified reference (growsurf built
  from /root/reference into oracle/_ref, Cython kernel, parallel_executor on
  every host core) resumed from its OWN pickled state at the start of each
  of 8 equal slices of the run (tests/golden/make_ref_checkpoints.py) for a
  bounded time each: the whole run's time-to-converge is estimated as the
  sum over slices of (batches in the slice x measured seconds per batch), a
  stratified sample of the full run.  ``--ref-full-cfg3`` runs the stock
  ``growsurf.run_multi`` to convergence instead (minutes); configs 1 and 2
  are run to convergence by the stock reference in ``other_configs``.
* cfg4 (BASELINE config 4): 10M-point torus cloud, paper batch rule up to
  m = 65536, a fixed 30 M-signal budget through the public API, sharded over
  the N ranks: signals/s and all-gather time per batch.
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "signals/sec & time-to-converge (SOAM, 1M-pt cloud) at 1/2/4/8 B200 vs CPU ref"
MEASURED_PEAKS = os.path.join(REPO, "MEASURED_PEAKS.json")
NCU_SUMMARY = os.path.join(REPO, "profiles", "ncu_summary.json")
REF_CKPT = os.path.join(REPO, "tests", "golden", "ref_cfg3_checkpoints.pkl.gz")


def parse_args():
    p = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=3)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=("b200", "reference"), default="b200")
    p.add_argument("--workload", default="cfg3")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-budget-s", type=float, default=20.0)
    p.add_argument("--no-find-microbench", action="store_true")
    p.add_argument("--no-m-sweep", action="store_true")
    p.add_argument("--no-ref-full", action="store_true",
                   help="skip the stock reference's full runs of configs 1 and 2")
    p.add_argument("--ref-full-cfg3", action="store_true",
                   help="also run the stock reference's config-3 run to convergence (minutes)")
    p.add_argument("--no-cfg4", action="store_true")
    p.add_argument("--no-sharded-anchor", action="store_true")
    return p.parse_args()


# ---------------------------------------------------------------------------
# process group


def dist_setup(args, backend):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    return world, rank, local


# ---------------------------------------------------------------------------
# clocks (nvidia-smi sampled during the timed region)

_REASONS = {
    0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
    0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
    0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
}


class ClockSampler:
    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu),
                 "--query-gpu=clocks.sm,clocks.max.sm,utilization.gpu,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        return False

    def summary(self):
        rows = []
        try:
            for line in open(self.path):
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 4:
                    try:
                        rows.append((float(parts[0]), float(parts[1]), float(parts[2]),
                                     int(parts[3], 16) if parts[3].startswith("0x") else int(parts[3])))
                    except ValueError:
                        pass
        finally:
            if self.path and os.path.exists(self.path):
                os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        busy = [r for r in rows if r[2] > 0] or rows
        reasons = set()
        for r in busy:
            for bit, name in _REASONS.items():
                if r[3] & bit:
                    reasons.add(name)
        reasons.discard("gpu_idle")
        return {"sm_mhz": statistics.median(r[0] for r in busy), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": sorted(reasons), "samples": len(rows), "samples_busy": len(busy)}


# ---------------------------------------------------------------------------
# CPU reference (oracle/_ref growsurf) on a bounded prefix of the same run


def reference_available():
    ref = os.path.join(REPO, "oracle", "_ref")
    if os.path.isdir(os.path.join(ref, "growsurf")):
        if ref not in sys.path:
            sys.path.insert(0, ref)
        try:
            from growsurf import kernels

            return kernels.HAVE_COMPILED
        except Exception:
            return False
    return False


def reference_prefix(points, label, wparams, seed, budget_s):
    """Run the reference driver (multi.py:134-185) with growsurf's own
    functions until the time budget is spent; returns (signals, seconds,
    batches, kind, cores)."""
    if reference_available():
        from growsurf import CloudSource, EngineParams
        from growsurf.engine import RunState, is_converged
        from growsurf.multi import batch_size, resolve_and_update
        from growsurf.network import Network
        from growsurf.parallel import ExecConfig, parallel_executor
        import numpy as np

        params = EngineParams(**wparams)
        src = CloudSource(points, label=label)
        executor = parallel_executor(ExecConfig(workers=os.cpu_count() or 1))
        t0 = time.perf_counter()
        rng = np.random.Generator(np.random.Philox(seed))
        net = Network()
        net.watch_age_limit(params.max_age)
        for s in src.sample(rng, 2):
            net.add_unit(s, params.theta0)
        state = RunState()
        signals = batches = 0
        while signals < params.max_signals:
            m = batch_size(net.unit_count, params.batch_cap, params.batch_floor)
            batch = src.sample(rng, m)
            winners = executor(net.snapshot(), batch)
            resolve_and_update(net, params, batch, winners, state)
            signals += m
            batches += 1
            if is_converged(net, params) or time.perf_counter() - t0 > budget_s:
                break
        return signals, time.perf_counter() - t0, batches, "reference", os.cpu_count() or 1
    # C oracle port (single thread)
    from oracle import oracle as O
    from paper_1503_08294_b200 import CloudSource, EngineParams
    import numpy as np

    params = EngineParams(**wparams)
    src = CloudSource(points, label=label)
    t0 = time.perf_counter()
    rng = np.random.Generator(np.random.Philox(seed))
    net = O.OracleNet(params)
    for s in src.sample(rng, 2):
        net.add_unit(s, params.theta0)
    signals = batches = 0
    units = 2
    while signals < params.max_signals:
        m = O.batch_size(units, params.batch_cap, params.batch_floor)
        net.step(src.sample(rng, m))
        signals += m
        batches += 1
        units = net.counts()["units"]
        if net.converged() or time.perf_counter() - t0 > budget_s:
            break
    return signals, time.perf_counter() - t0, batches, "port", 1


def load_ref_checkpoints(workload):
    """The reference's own pickled states at the start of each slice of its
    config-3 run (tests/golden/make_ref_checkpoints.py), or None."""
    if workload != "cfg3" or not os.path.exists(REF_CKPT) or not reference_available():
        return None
    import gzip
    import pickle

    import numpy as np

    with gzip.open(REF_CKPT, "rb") as fh:
        blob = pickle.load(fh)
    if blob.get("numpy_version") != np.__version__:
        return None  # Generator streams are numpy-version specific
    return blob


def reference_stratified(points, label, wparams, budget_s, blob, acc=None):
    """Resume the stock reference (multi.py:165-185 loop with growsurf's own
    sample / parallel executor / resolve_and_update / is_converged) from each
    checkpoint for budget_s / slices seconds; accumulates [batches, seconds]
    per slice into ``acc``."""
    import pickle

    import numpy as np
    from growsurf import CloudSource, EngineParams
    from growsurf.engine import is_converged
    from growsurf.multi import batch_size, resolve_and_update
    from growsurf.parallel import ExecConfig, parallel_executor

    params = EngineParams(**wparams)
    src = CloudSource(points, label=label)
    executor = parallel_executor(ExecConfig(workers=os.cpu_count() or 1))
    starts = list(blob["starts"]) + [blob["total_batches"]]
    k = len(blob["checkpoints"])
    if acc is None:
        acc = [[0, 0.0] for _ in range(k)]
    per = budget_s / k
    for c, raw in enumerate(blob["checkpoints"]):
        cp = pickle.loads(raw)
        net, state = cp["net"], cp["state"]
        rng = np.random.Generator(np.random.Philox(0))
        rng.bit_generator.state = cp["rng"]
        limit = starts[c + 1] - starts[c]
        n = 0
        t0 = time.perf_counter()
        while n < limit:
            m = batch_size(net.unit_count, params.batch_cap, params.batch_floor)
            batch = src.sample(rng, m)
            winners = executor(net.snapshot(), batch)
            resolve_and_update(net, params, batch, winners, state)
            n += 1
            if is_converged(net, params) or time.perf_counter() - t0 >= per:
                break
        acc[c][0] += n
        acc[c][1] += time.perf_counter() - t0
    return acc


def stratified_estimate(acc, blob):
    """Estimated time-to-converge: sum over slices of batches x s/batch."""
    starts = list(blob["starts"]) + [blob["total_batches"]]
    per_slice = [(starts[c + 1] - starts[c]) * sec / max(1, n) for c, (n, sec) in enumerate(acc)]
    return sum(per_slice), per_slice


def reference_cpu_rate(points, label, wparams, seed, budget_s, workload, steps=1, warmup=0):
    """(signals/s, ms per run, kind, cores, sample text) of the reference on
    this host: stratified over the run when its checkpoints exist, else the
    run's prefix."""
    blob = load_ref_checkpoints(workload)
    cores = os.cpu_count() or 1
    if blob is not None:
        for _ in range(warmup):
            reference_stratified(points, label, wparams, budget_s, blob)
        acc = None
        for _ in range(steps):
            acc = reference_stratified(points, label, wparams, budget_s, blob, acc)
        est, per_slice = stratified_estimate(acc, blob)
        sampled = sum(n for n, _ in acc)
        value = blob["total_signals"] / est
        sample = (f"stratified: the stock reference resumed from its own checkpoints at the start "
                  f"of each of {len(acc)} equal slices of the {blob['total_batches']}-batch "
                  f"{workload} run, {sampled} batches sampled ({sum(t for _, t in acc):.1f} s); "
                  f"estimated time-to-converge {est:.1f} s = sum of slice batches x s/batch "
                  f"(slices: " + ", ".join(f"{t:.1f}" for t in per_slice) + " s)")
        return value, 1e3 * est, "reference", cores, sample
    tot_sig = tot_s = 0.0
    kind = batches = None
    for _ in range(warmup):
        reference_prefix(points, label, wparams, seed, budget_s)
    for _ in range(steps):
        sig, sec, batches, kind, cores = reference_prefix(points, label, wparams, seed, budget_s)
        tot_sig += sig
        tot_s += sec
    sample = (f"prefix: first {int(tot_sig / steps):,} signals ({batches} batches, "
              f"~{budget_s:.0f} s budget) of the seeded {workload} run (early-run rate)")
    return tot_sig / tot_s, 1e3 * tot_s / steps, kind, cores, sample


def reference_full_run(name, workload_params=None):
    """The stock ``growsurf.run_multi`` to convergence on this host."""
    from growsurf import CloudSource, EngineParams, run_multi
    from growsurf.multi import sequential_executor
    from growsurf.parallel import ExecConfig, parallel_executor

    from paper_1503_08294_b200 import workloads

    w = workloads.WORKLOADS[name]
    pts, label = w["cloud"]()
    params = EngineParams(**(workload_params or w["params"]))
    if params.batch_cap <= 64:
        ex, how = sequential_executor(), "sequential_executor (1 core)"
    else:
        ex = parallel_executor(ExecConfig(workers=os.cpu_count() or 1))
        how = f"parallel_executor ({os.cpu_count()} cores)"
    t0 = time.perf_counter()
    net, st = run_multi(CloudSource(pts, label=label), params, w["seed"], ex)
    sec = time.perf_counter() - t0
    return {"time_to_converge_s": sec, "converged": bool(st.converged), "signals": st.signals,
            "iterations": st.iterations, "units": st.units, "edges": st.connections,
            "signals_per_s": st.signals / sec, "find_s": st.find_s, "update_s": st.update_s,
            "sample_s": st.sample_s, "executor": how, "cores": os.cpu_count(),
            "how": "stock growsurf.run_multi (oracle/_ref) on this host"}


def run_reference_arm(args):
    world, rank, _ = dist_setup(args, "gloo")
    if rank != 0:
        return
    from paper_1503_08294_b200 import workloads

    src, params, seed, desc = workloads.make(args.workload)
    wparams = dict(workloads.WORKLOADS[args.workload]["params"])
    budget = max(2.0, min(20.0, 150.0 / max(1, args.steps + args.warmup)))
    value, ms, kind, cores, sample = reference_cpu_rate(
        src.points, src.label, wparams, seed, budget, args.workload, args.steps, args.warmup)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "signals/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.workload, "desc": desc, "m": params.batch_cap,
                   "theta0": params.theta0, "seed": seed,
                   "step": "one seeded run to convergence (estimated from the stratified sample)"},
        "cpu_baseline": {"value": value, "unit": "signals/s", "cores": cores, "kind": kind,
                         "sample": sample},
        "e2e": {"value": value, "unit": "signals/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# B200 arm


def load_peaks():
    try:
        with open(MEASURED_PEAKS) as fh:
            return json.load(fh)
    except OSError:
        return {"hbm_gbs": 6650.0, "fallback": True}


def ncu_traffic(kernel: str):
    try:
        with open(NCU_SUMMARY) as fh:
            return json.load(fh).get(kernel, {}).get("dram_bytes_per_launch")
    except (OSError, ValueError):
        return None


def find_microbench(lib, ctx, fp32_peak, peak_source, sizes=(10_000, 100_000, 1_000_000),
                    m=1_000_000, reps=3, cpu_budget_s=8.0, dists=("uniform", "torus")):
    """BASELINE config 5: m = 1e6 signals vs n units, uniform in [0,1)^3
    (cli.py:252-261) and on a torus inside the unit cube, from Philox(7).
    Resident inputs, CUDA events on the launching stream, L2 flushed between
    repetitions.  Two exact modes with the same output: the FP32 filter +
    certified FP64 re-check (FP32-bound: `lines`) and the exact uniform grid
    (`grid_lines`); every line checks grid == filter bit for bit on all m
    signals (the tests check both against the oracle and the FP64 scan)."""
    import numpy as np
    import torch

    from paper_1503_08294_b200.sampling import TorusSource

    out = {"m": m, "mode": "filter (FP32 FFMA2 + certified FP64)", "lines": [],
           "grid_mode": "exact uniform grid rebuilt per call (GS_FIND_GRID; L2-latency bound)",
           "grid_lines": [], "peak_tflops": fp32_peak, "peak_source": peak_source}
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    st = torch.cuda.Stream()  # a real stream: handle 0 would mean the context's own stream

    def draw(dist, rng, k):
        if dist == "uniform":
            return rng.random((k, 3))
        return TorusSource(0.3, 0.1).sample(rng, k) + 0.5  # inside [0.1, 0.9]^3

    for dist in dists:
        for n in sizes:
            rng = np.random.Generator(np.random.Philox(7))
            pos = torch.from_numpy(draw(dist, rng, n)).cuda()
            sig = torch.from_numpy(draw(dist, rng, m)).cuda()
            idx = torch.empty((m, 2), dtype=torch.int64, device="cuda")
            d2 = torch.empty((m, 2), dtype=torch.float64, device="cuda")
            torch.cuda.synchronize()

            def timed(mode):
                def run():
                    _lib_check(lib.gs_find_device(ctx.handle, pos.data_ptr(), n, sig.data_ptr(),
                                                  m, idx.data_ptr(), d2.data_ptr(), mode,
                                                  st.cuda_stream))

                run()
                times = []
                for _ in range(reps):
                    with torch.cuda.stream(st):
                        flush.zero_()
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record(st)
                    run()
                    e1.record(st)
                    torch.cuda.synchronize()
                    times.append(e0.elapsed_time(e1))
                fb = np.zeros(2, np.int64)
                _lib_check(lib.gs_find_last_fallback_counts(ctx.handle, fb))
                return statistics.median(times), fb

            gms, gfb = timed(4)
            g_idx, g_d2 = idx.clone(), d2.clone()
            gbytes = 24 * n + 32 * n + 56 * m  # rows read, rows in cell order, signals + results
            ms, fb2 = timed(1)
            same = bool(torch.equal(g_idx, idx) and torch.equal(g_d2.view(torch.int64),
                                                                d2.view(torch.int64)))
            out["grid_lines"].append({"dist": dist, "n": n, "ms": gms,
                                      "signals_per_s": m / (gms * 1e-3),
                                      "equivalent_pairs_per_s": float(n) * m / (gms * 1e-3),
                                      "algorithmic_bytes": gbytes,
                                      "achieved_gbs": gbytes / (gms * 1e-3) / 1e9,
                                      "exhaustive_fallback_signals": int(gfb[0]),
                                      "speedup_vs_filter": ms / gms,
                                      "identical_to_filter": same})
            pairs = float(n) * m
            achieved = 8.0 * pairs / (ms * 1e-3) / 1e12
            key = {1_000_000: "filter", 100_000: "filter_n1e5"}.get(n, "") if dist == "uniform" else ""
            out["lines"].append({"dist": dist, "n": n, "ms": ms, "pairs_per_s": pairs / (ms * 1e-3),
                                 "algorithmic_bytes": 24 * n + 56 * m,
                                 "traffic": ncu_traffic(key),
                                 "achieved_tflops": achieved, "peak_tflops": fp32_peak,
                                 "frac": achieved / fp32_peak, "fallback_signals": int(fb2[0]),
                                 "fp64_rescans": int(fb2[1]), "identical_to_grid": same})
            if not same:
                raise SystemExit(f"config 5: grid and filter disagree ({dist}, n={n})")
            del pos, sig, idx, d2, g_idx, g_d2
    # the reference's raw scan (_parallel_scan, all host cores) on a bounded sample
    if reference_available():
        from growsurf import kernels as rk
        from growsurf.network import Snapshot
        from growsurf.parallel import ExecConfig, _parallel_scan
        import numpy as np

        n = sizes[0]
        rng = np.random.Generator(np.random.Philox(7))
        pos = rng.random((n, 3))
        sig = rng.random((m, 3))
        snap = Snapshot(np.arange(n, dtype=np.int64), pos)
        cfg = ExecConfig(workers=os.cpu_count() or 1, tile=1024)
        ms_sig = 4096
        t0 = time.perf_counter()
        done = 0
        while time.perf_counter() - t0 < cpu_budget_s and done + ms_sig <= m:
            _parallel_scan(snap, sig[done:done + ms_sig], cfg, backend=rk.get_backend("compiled"))
            done += ms_sig
        sec = time.perf_counter() - t0
        out["cpu_reference"] = {"pairs_per_s": float(n) * done / sec, "n": n, "signals": done,
                                "cores": os.cpu_count(), "seconds": sec,
                                "how": "growsurf.parallel._parallel_scan, compiled backend, tile 1024"}
    return out


def mesh_timing(net):
    """SURVEY 8(f) row 3 at scale: mesh extraction + manifold check on the
    device for a grown network (and the topology of a 1M-vertex torus grid),
    beside the reference's host loops (metrics.py:148-240) on the same
    network."""
    import numpy as np

    from paper_1503_08294_b200 import TriMesh, extract_mesh, manifold_check

    extract_mesh(net)  # warm-up (allocator, module load)
    t0 = time.perf_counter()
    mesh = extract_mesh(net)
    cls = manifold_check(mesh)
    dev_s = time.perf_counter() - t0
    n = 1000
    i, j = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    a, b = i * n + j, i * n + (j + 1) % n
    c, d = ((i + 1) % n) * n + j, ((i + 1) % n) * n + (j + 1) % n
    grid = np.stack([np.stack([a, b, d], -1), np.stack([a, d, c], -1)], 2).reshape(-1, 3)
    gmesh = TriMesh(np.zeros((n * n, 3)), grid.astype(np.int64))
    manifold_check(gmesh)
    t0 = time.perf_counter()
    gcls = manifold_check(gmesh)
    grid_s = time.perf_counter() - t0
    out = {"units": int(net.unit_count), "faces": int(len(mesh.faces)), "manifold": cls,
           "device_extract_and_check_s": dev_s,
           "torus_grid_1M_vertices": {"faces": int(len(grid)), "manifold": gcls,
                                      "device_check_s": grid_s}}
    if reference_available():
        import growsurf.metrics as rm

        t0 = time.perf_counter()
        rmesh = rm.extract_mesh(net)
        rcls = rm.manifold_check(rmesh)
        out["reference_host_s"] = time.perf_counter() - t0
        out["same_faces"] = bool(np.array_equal(rmesh.faces, mesh.faces)) and rcls == cls
    return out


def fp32_peak(lib, ctx, sm_mhz, peaks):
    """(TFLOP/s, source): the FFMA2 probe measured on this GPU, else nominal."""
    t, ms = C.c_double(), C.c_double()
    try:
        _lib_check(lib.gs_fp32_peak(ctx.handle, C.byref(t), C.byref(ms)))
        return t.value, (f"measured: packed FFMA2 chains on all {ctx.sm_count} SMs "
                         f"(gs_fp32_peak, best of 5, {ms.value:.2f} ms)")
    except Exception:  # noqa: BLE001 - report the nominal figure instead
        return (2 * 128 * ctx.sm_count * sm_mhz * 1e6 / 1e12,
                f"nominal FP32 2x128 lanes x {ctx.sm_count} SMs at {sm_mhz:.0f} MHz")


def m_sweep(lib, src, wparams, seed, ms=(256, 1024, 4096, 16384, 65536), budget_s=20.0):
    """BASELINE config 3's m sweep: the same seeded run at each fixed batch
    size, device sampling + asynchronous loop, timed with CUDA events on the
    engine stream; a run that has not converged after budget_s seconds of
    device time (or the signal cap) is reported as such."""
    import numpy as np
    import torch

    from paper_1503_08294_b200 import EngineParams, _lib
    from paper_1503_08294_b200.device_sampling import DeviceCloudSampler
    from paper_1503_08294_b200.network import Network

    out = []
    pts_dev = torch.from_numpy(src.points).cuda()
    for m in ms:
        p = dict(wparams)
        p.update(batch_floor=m, batch_cap=m)
        params = EngineParams(**p)
        rng = np.random.Generator(np.random.Philox(seed))
        seeds = src.sample(rng, 2)
        net = Network(params, capacity=8192)
        net.reserve(8192)
        net.set_async(8)
        sampler = DeviceCloudSampler(None, rng, device_ptr=pts_dev.data_ptr(),
                                     npts=src.points.shape[0])
        for s_ in seeds:
            net.add_unit(s_, params.theta0)
        stream = torch.cuda.ExternalStream(net.stream_handle())
        st = _lib.GsBatchStats()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0.record(stream)
        enq = 0
        seq = C.c_int64()
        while enq * m < params.max_signals:
            _lib_check(lib.gs_engine_step_sampled(net.handle, sampler.handle, m, None))
            enq += 1
            _lib_check(lib.gs_engine_stats_lagged(net.handle, 7, C.byref(st), C.byref(seq)))
            if seq.value >= 0 and (st.converged or time.perf_counter() - t0 > budget_s):
                break
        e1.record(stream)
        _lib_check(lib.gs_engine_stats(net.handle, C.byref(st)))
        sec = e0.elapsed_time(e1) * 1e-3
        sig = int(st.batches) * m
        out.append({"m": m, "converged": bool(st.converged), "signals": sig,
                    "batches": int(st.batches), "device_s": sec, "signals_per_s": sig / sec,
                    "units": int(st.units), "edges": int(st.edges)})
        sampler.close()
        net.close()
    return out


def other_configs(lib, names=("cfg1", "cfg2"), budget_s=20.0, ref_full=True):
    """BASELINE configs 1 and 2 (the SOAM runs the reference converges on):
    time to converge from the two seed units with device sampling and the
    asynchronous loop, CUDA events on the engine stream (same run as the
    reference's, bit for bit: tests/test_gpu_engine.py golden runs)."""
    import numpy as np
    import torch

    from paper_1503_08294_b200 import _lib, workloads
    from paper_1503_08294_b200.device_sampling import DeviceCloudSampler
    from paper_1503_08294_b200.network import Network

    ref_note = {"cfg1": "reference: converges V=218 after 299,392 signals in 6.6 s on 1 core (SURVEY 8(d))",
                "cfg2": "reference: converges V=681 after 4.28 M signals in 78.8 s on 8 cores (SURVEY 8(d))"}
    out = {}
    for name in names:
        src, params, seed, desc = workloads.make(name)
        m = params.batch_cap
        pts_dev = torch.from_numpy(src.points).cuda()
        rng = np.random.Generator(np.random.Philox(seed))
        seeds = src.sample(rng, 2)
        net = Network(params, capacity=8192)
        net.reserve(8192)
        net.set_async(8)
        sampler = DeviceCloudSampler(None, rng, device_ptr=pts_dev.data_ptr(),
                                     npts=src.points.shape[0])
        for s_ in seeds:
            net.add_unit(s_, params.theta0)
        stream = torch.cuda.ExternalStream(net.stream_handle())
        st = _lib.GsBatchStats()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0.record(stream)
        enq = 0
        seq = C.c_int64()
        while enq * m < params.max_signals:
            _lib_check(lib.gs_engine_step_sampled(net.handle, sampler.handle, m, None))
            enq += 1
            if enq % 4 == 0:
                _lib_check(lib.gs_engine_stats_lagged(net.handle, 7, C.byref(st), C.byref(seq)))
                if seq.value >= 0 and (st.converged or time.perf_counter() - t0 > budget_s):
                    break
        e1.record(stream)
        _lib_check(lib.gs_engine_stats(net.handle, C.byref(st)))
        sec = e0.elapsed_time(e1) * 1e-3
        sig = int(st.batches) * m
        out[name] = {"desc": desc, "m": m, "converged": bool(st.converged), "signals": sig,
                     "batches": int(st.batches), "time_to_converge_s": sec,
                     "signals_per_s": sig / sec, "units": int(st.units), "edges": int(st.edges),
                     "reference": ref_note.get(name)}
        sampler.close()
        net.close()
        del pts_dev
        if ref_full and reference_available():
            ref = reference_full_run(name)
            ref["same_run"] = (ref["signals"], ref["units"], ref["edges"]) == (sig, int(st.units),
                                                                               int(st.edges))
            out[name]["reference_same_box"] = ref
            out[name]["speedup_time_to_converge"] = ref["time_to_converge_s"] / sec
    return out


def _lib_check(rc):
    from paper_1503_08294_b200 import _lib

    _lib.check(rc)


def run_b200_arm(args):
    import numpy as np
    import torch

    world, rank, local = dist_setup(args, "nccl")
    torch.cuda.set_device(local)
    os.environ["GS_DEVICE"] = str(local)
    from paper_1503_08294_b200 import _lib, workloads
    from paper_1503_08294_b200.distributed import attach, run_multi_sharded, shard_unique_id
    from paper_1503_08294_b200.multi import run_multi
    from paper_1503_08294_b200.network import Network

    lib = _lib.load_library()
    ctx = _lib.default_context()
    src, params, seed, desc = workloads.make(args.workload)
    if params.batch_floor != params.batch_cap:
        raise SystemExit("bench workloads use a fixed batch size")
    m = params.batch_cap
    # inputs resident in HBM: the cloud; signals are drawn on the device from
    # the same Philox stream as the reference (device_sampling.py)
    from paper_1503_08294_b200.device_sampling import DeviceCloudSampler, philox_state_words

    rng = np.random.Generator(np.random.Philox(seed))
    seeds = src.sample(rng, 2)
    state0 = philox_state_words(rng)
    pts_dev = torch.from_numpy(src.points).cuda()
    cloud_bytes = pts_dev.numel() * 8
    sampler = DeviceCloudSampler(None, device_ptr=pts_dev.data_ptr(), npts=src.points.shape[0])
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    st = _lib.GsBatchStats()
    LOOKAHEAD = 8  # batches enqueued ahead of the convergence check

    def make_net(shards):
        net = Network(params, capacity=8192)
        net.reserve(8192)
        if shards == "world":
            attach(net)  # this rank's slice of every batch + ncclAllGather
        elif shards == "world1":
            net.set_shards(1, 0, shard_unique_id())
        net.set_async(LOOKAHEAD)
        return net

    def one_run(net, trace=None):
        net.reset()
        for s in seeds:
            net.add_unit(s, params.theta0)
        _lib.check(lib.gs_sampler_set_state(sampler.handle, state0))
        if trace is None:
            # device-resident loop: the host only polls the convergence flag;
            # batches after convergence are no-ops on the device (halted)
            enq = 0
            seq = C.c_int64()
            while enq * m < params.max_signals:
                _lib.check(lib.gs_engine_step_sampled(net.handle, sampler.handle, m, None))
                enq += 1
                if enq % 4 == 0:
                    _lib.check(lib.gs_engine_stats_lagged(net.handle, LOOKAHEAD - 1, C.byref(st),
                                                          C.byref(seq)))
                    if seq.value >= 0 and st.converged:
                        break
            _lib.check(lib.gs_engine_stats(net.handle, C.byref(st)))
            return int(st.batches) * m, bool(st.converged), int(st.units), int(st.edges)
        net.set_async(0)  # synchronous: per-batch stats for the trace
        off = 0
        units = 2
        while off < params.max_signals:
            trace["pairs"] += m * units
            _lib.check(lib.gs_engine_step_sampled(net.handle, sampler.handle, m, C.byref(st)))
            off += m
            units = int(st.units)
            trace["processed"] += int(st.processed)
            trace["batches"] += 1
            if st.converged:
                break
        net.set_async(LOOKAHEAD)
        return off, bool(st.converged), int(st.units), int(st.edges)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if world > 1:
            t = torch.tensor([x], device="cuda", dtype=torch.float64)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            x = float(t.item())
        return x

    def timed_runs(net, steps, warmup, clock_gpu=None):
        stream = torch.cuda.ExternalStream(net.stream_handle())
        for _ in range(warmup):
            with torch.cuda.stream(stream):
                flush.zero_()
            one_run(net)
        barrier()
        l0 = net.launch_count()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        total = 0
        res = None
        clocks = ClockSampler(clock_gpu) if clock_gpu is not None else None
        if clocks:
            clocks.__enter__()
        ev0.record(stream)
        for _ in range(steps):
            with torch.cuda.stream(stream):
                flush.zero_()
            res = one_run(net)
            total += res[0]
        ev1.record(stream)
        barrier()
        if clocks:
            clocks.__exit__(None, None, None)
        ms = max_over_ranks(ev0.elapsed_time(ev1))
        return total, ms, res, net.launch_count() - l0, (clocks.summary() if clocks else None)

    net = make_net("world" if world > 1 else None)
    signals, ms, result, launches, clk = timed_runs(net, args.steps, args.warmup, local)
    value = signals / (ms * 1e-3)

    # per-phase device time over one extra (untimed) run: the roofline's kernel
    trace = dict(pairs=0, processed=0, batches=0)
    phase = np.zeros(2, np.float64)
    _lib.check(lib.gs_engine_phase_ms(net.handle, 1, phase))
    x0 = net.exchange_ms()
    one_run(net, trace)
    _lib.check(lib.gs_engine_phase_ms(net.handle, 0, phase))
    find_ms, update_ms = float(phase[0]), float(phase[1])
    exch_ms = net.exchange_ms() - x0
    peaks = load_peaks()
    sm_mhz = clk.get("sm_mhz") or peaks.get("sm_max_mhz", 1965.0)
    fpeak, fpeak_src = fp32_peak(lib, ctx, sm_mhz, peaks)
    counts = net.counts()
    mean_deg = 2.0 * counts["edges"] / max(1, counts["units"])
    total_phase = find_ms + exch_ms + update_ms
    f_achieved = 8.0 * trace["pairs"] / world / (find_ms * 1e-3) / 1e12
    find_roof = {"kernel": "find_small_f32_kernel (screened FP32 + exact FP64 candidates)",
                 "bound": "fp32", "achieved": f_achieved, "peak": fpeak, "unit": "TFLOP/s",
                 "frac": f_achieved / fpeak, "traffic": ncu_traffic("find"),
                 "peak_source": fpeak_src,
                 "work": "8 FLOP per (signal, live unit) pair (BASELINE.md 2) of this rank's slice",
                 "share_of_step": find_ms / total_phase,
                 "us_per_batch": 1e3 * find_ms / max(1, trace["batches"])}
    per_sig = (1 + mean_deg) * 2 * (32 + 8) + mean_deg * (8 + 8) + 16 + 24
    achieved = per_sig * trace["processed"] / (update_ms * 1e-3) / 1e9
    peak = float(peaks.get("hbm_gbs", 6650.0))
    roof = {"kernel": "k_update_batch", "bound": "hbm", "achieved": achieved, "peak": peak,
            "unit": "GB/s", "frac": achieved / peak, "traffic": ncu_traffic("update"),
            "peak_source": "MEASURED_PEAKS.json hbm_gbs" + (" (fallback)" if peaks.get("fallback") else ""),
            "work": f"{per_sig:.0f} B per processed signal (winner + {mean_deg:.2f} neighbours: "
                    "pos+hab read/write, adjacency, edge ages, record, signal)",
            "share_of_step": update_ms / total_phase,
            "us_per_batch": 1e3 * update_ms / max(1, trace["batches"]),
            "note": "sequential-semantics update on one 16-CTA cluster: bound by dependent L2 "
                    "round trips and cluster barriers, not by bandwidth"}
    if find_ms > update_ms:
        roof, find_roof = find_roof, roof

    # e2e through the public API: cloud H2D + sampler state + stats inside
    e2e = None
    if not args.no_e2e:
        # one untimed pass through the public API (allocator / module warm-up)
        if world > 1:
            run_multi_sharded(src, params, seed)
        else:
            run_multi(src, params, seed, capacity=8192)
        barrier()
        t0 = time.perf_counter()
        e_sig = e_batches = 0
        results = []  # the returned networks outlive the timed region (no teardown inside)
        for _ in range(args.steps):
            if world > 1:
                res_net, rs = run_multi_sharded(src, params, seed)
            else:
                res_net, rs = run_multi(src, params, seed, capacity=8192)
            results.append(res_net)
            e_sig += rs.signals
            e_batches += rs.iterations
        barrier()
        e_s = max_over_ranks(time.perf_counter() - t0)
        del results
        e2e = {"value": e_sig / e_s, "unit": "signals/s",
               "h2d_bytes_per_step": int(cloud_bytes + 48 + 120),
               "d2h_bytes_per_step": int(C.sizeof(_lib.GsBatchStats) * (e_batches // args.steps)),
               "ms_per_step": 1e3 * e_s / args.steps}

    # N = 1: the sharded code path with a single-rank communicator (the SCALE
    # anchor: same run, find + ncclAllGather + update per batch)
    anchor = None
    if world == 1 and not args.no_sharded_anchor:
        net1 = make_net("world1")
        a_sig, a_ms, _, a_l, _ = timed_runs(net1, max(1, min(args.steps, 3)), 1)
        ph = np.zeros(2, np.float64)
        _lib.check(lib.gs_engine_phase_ms(net1.handle, 1, ph))
        x0 = net1.exchange_ms()
        tr = dict(pairs=0, processed=0, batches=0)
        one_run(net1, tr)
        _lib.check(lib.gs_engine_phase_ms(net1.handle, 0, ph))
        anchor = {"value": a_sig / (a_ms * 1e-3), "ms_per_step": a_ms / max(1, min(args.steps, 3)),
                  "allgather_us_per_batch": 1e3 * (net1.exchange_ms() - x0) / max(1, tr["batches"]),
                  "how": "same run through the sharded engine path at world = 1 (find on the "
                         "rank's slice, ncclAllGather of records on the engine stream, update)"}
        net1.close()

    # BASELINE config 4: 10M-point torus, paper batch rule up to 65536, sharded
    cfg4 = None
    if not args.no_cfg4:
        src4, params4, seed4, desc4 = workloads.make("cfg4")
        kw = dict(capacity=65536)
        run4 = (lambda: run_multi_sharded(src4, params4, seed4, **kw)) if world > 1 else (
            lambda: run_multi(src4, params4, seed4, **kw))
        run4()  # warm-up
        barrier()
        t0 = time.perf_counter()
        net4, rs4 = run4()
        barrier()
        w_s = max_over_ranks(time.perf_counter() - t0)
        loop_s = max_over_ranks(rs4.total_s)
        x4 = net4.exchange_ms() if world > 1 else 0.0
        cfg4 = {"desc": desc4, "cloud_points": int(src4.points.shape[0]), "signals": rs4.signals,
                "batches": rs4.iterations, "units": rs4.units, "edges": rs4.connections,
                "converged": rs4.converged, "wall_s": w_s, "loop_s": loop_s,
                "signals_per_s": rs4.signals / loop_s, "signals_per_s_wall": rs4.signals / w_s,
                "find_s": rs4.find_s, "update_s": rs4.update_s,
                "allgather_us_per_batch": 1e3 * x4 / max(1, rs4.iterations),
                "timing": "signals_per_s: the batch loop of the public run_multi call (per-batch "
                          "host sampling of m, stats read each batch), max over ranks; "
                          "signals_per_s_wall adds the cloud H2D and setup",
                "parallelism": f"signal-sharded find x{world}, replicated update"}
        cfg4["mesh"] = mesh_timing(net4)
        net4.close()
        del src4

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        wparams = dict(workloads.WORKLOADS[args.workload]["params"])
        v, c_ms, kind, cores, sample = reference_cpu_rate(src.points, src.label, wparams, seed,
                                                          args.cpu_budget_s, args.workload)
        cpu = {"value": v, "unit": "signals/s", "cores": cores, "kind": kind, "sample": sample,
               "time_to_converge_s": c_ms * 1e-3}
        if args.ref_full_cfg3 and reference_available():
            cpu["full_run"] = reference_full_run(args.workload)

    sweep = None
    if rank == 0 and world == 1 and not args.no_m_sweep:
        sweep = m_sweep(lib, src, dict(workloads.WORKLOADS[args.workload]["params"]), seed)
    others = None
    if rank == 0 and world == 1 and not args.no_m_sweep:
        others = other_configs(lib, ref_full=not args.no_ref_full)
    fmb = None
    if rank == 0 and not args.no_find_microbench:
        fmb = find_microbench(lib, ctx, fpeak, fpeak_src)

    if rank == 0:
        sig, conv, units, edges = result
        line = {
            "metric": METRIC, "value": value, "unit": "signals/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": args.workload, "desc": desc, "m": m, "theta0": params.theta0,
                       "seed": seed, "cloud_points": int(src.points.shape[0]),
                       "parallelism": f"signal-sharded find x{world} (ncclAllGather of winner "
                                      "records per batch), replicated update",
                       "step": "one seeded run from the two seed units to convergence",
                       "signals_per_step": sig, "converged": conv, "units": units,
                       "edges": edges, "time_to_converge_s": ms / args.steps * 1e-3,
                       "l2": "256 MiB L2 flush before each step (cloud "
                             f"{cloud_bytes / 2**20:.0f} MiB resident in HBM)",
                       "sampling": "device Philox4x64-10 + Lemire inside the timed region, "
                                   "bit-identical to numpy",
                       "find_mode": "auto"},
            "roofline": roof,
            "find_roofline": find_roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clk,
            "phase_ms_per_step": {"find": find_ms, "allgather": exch_ms, "update": update_ms},
            "sharded_world1": anchor,
            "cfg4": cfg4,
            "find_microbench": fmb,
            "m_sweep": sweep,
            "other_configs": others,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def main():
    args = parse_args()
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_b200_arm(args)


if __name__ == "__main__":
    main()

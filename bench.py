#!/usr/bin/env python
"""Benchmark: signals/s and time-to-converge of the multi-signal SOAM run.

Contract (driver): ``python bench.py --gpus N --steps K --warmup W`` (torchrun
for N > 1) prints ONE JSON line on rank 0.

* workload (default ``cfg3``): BASELINE config 3 -- SOAM on a 1M-point
  synthetic genus-2 cloud, m = 4096, theta0 = 0.1, seed 7.  One STEP is one
  complete seeded run from the two seed units to convergence (26.5 M
  signals, V = 1958, closed genus-2 mesh); ms_per_step is the
  time-to-converge.  The run is bit-identical to the reference's.
* value: whole-job signals/s with the seeded signal stream already resident
  in HBM (pre-drawn on the host from the same Philox stream, uploaded
  before timing); CUDA events on the engine stream; max over ranks.
* e2e: the same metric through the public API (``run_multi``, or
  ``distributed.run_multi_sharded`` at N > 1): host sampling, one pinned H2D
  copy of every batch and one stats D2H per batch inside the timed region.
* cpu_baseline / --impl reference: the unmodified reference (growsurf built
  from /root/reference into oracle/_ref, Cython kernel, parallel_executor on
  every host core) on a bounded prefix of the same seeded run.  If
  oracle/_ref is absent the C oracle port stands in (kind "port").
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


def run_reference_arm(args):
    world, rank, _ = dist_setup(args, "gloo")
    if rank != 0:
        return
    from paper_1503_08294_b200 import workloads

    src, params, seed, desc = workloads.make(args.workload)
    wparams = dict(workloads.WORKLOADS[args.workload]["params"])
    budget = max(2.0, min(20.0, 150.0 / max(1, args.steps + args.warmup)))
    for _ in range(args.warmup):
        reference_prefix(src.points, src.label, wparams, seed, budget)
    tot_sig = tot_s = 0.0
    kind = cores = None
    batches = 0
    for _ in range(args.steps):
        sig, sec, batches, kind, cores = reference_prefix(src.points, src.label, wparams, seed, budget)
        tot_sig += sig
        tot_s += sec
    value = tot_sig / tot_s
    sample = (f"first {int(tot_sig / args.steps):,} signals ({batches} batches, ~{budget:.0f} s budget) "
              f"of the seeded {args.workload} run, repeated per step")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "signals/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot_s / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.workload, "desc": desc, "m": params.batch_cap,
                   "theta0": params.theta0, "seed": seed},
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


def find_microbench(lib, ctx, sm_mhz, peaks, sizes=(10_000, 100_000, 1_000_000), m=1_000_000,
                    reps=3, cpu_budget_s=8.0):
    """BASELINE config 5: m = 1e6 signals vs n units, uniform [0,1)^3 from
    Philox(7) (cli.py:252-261).  Resident inputs, FP32 filter + certified
    FP64 re-check (bit-identical to the reference scan), CUDA events on the
    launching stream, L2 flushed between repetitions (the unit-pair array of
    the largest n is 16 MB; signals 24 MB)."""
    import numpy as np
    import torch

    out = {"m": m, "mode": "filter (FP32 FFMA2 + certified FP64)", "lines": [],
           "grid_mode": "exact uniform grid rebuilt per call (GS_FIND_GRID; HBM/L2-latency bound)",
           "grid_lines": []}
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    st = torch.cuda.Stream()  # a real stream: handle 0 would mean the context's own stream
    peak = 2 * 128 * ctx.sm_count * sm_mhz * 1e6 / 1e12
    for n in sizes:
        rng = np.random.Generator(np.random.Philox(7))
        pos = torch.from_numpy(rng.random((n, 3))).cuda()
        sig = torch.from_numpy(rng.random((m, 3))).cuda()
        idx = torch.empty((m, 2), dtype=torch.int64, device="cuda")
        d2 = torch.empty((m, 2), dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()

        def timed(mode):
            def run():
                _lib_check(lib.gs_find_device(ctx.handle, pos.data_ptr(), n, sig.data_ptr(), m,
                                              idx.data_ptr(), d2.data_ptr(), mode, st.cuda_stream))

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

        # exact uniform grid (GS_FIND_GRID): same output, O(m) candidates
        gms, gfb = timed(4)
        gbytes = 24 * n + 32 * n + 56 * m  # rows read, rows in cell order, signals + results
        out["grid_lines"].append({"n": n, "ms": gms, "signals_per_s": m / (gms * 1e-3),
                                  "equivalent_pairs_per_s": float(n) * m / (gms * 1e-3),
                                  "algorithmic_bytes": gbytes,
                                  "achieved_gbs": gbytes / (gms * 1e-3) / 1e9,
                                  "exhaustive_fallback_signals": int(gfb[0])})
        ms, fb2 = timed(1)
        out["grid_lines"][-1]["speedup_vs_filter"] = ms / gms
        pairs = float(n) * m
        achieved = 8.0 * pairs / (ms * 1e-3) / 1e12
        out["lines"].append({"n": n, "ms": ms, "pairs_per_s": pairs / (ms * 1e-3),
                             "algorithmic_bytes": 24 * n + 56 * m,
                             "traffic": ncu_traffic({1_000_000: "filter", 100_000: "filter_n1e5"}.get(n, "")),
                             "achieved_tflops": achieved, "peak_tflops": peak,
                             "frac": achieved / peak, "fallback_signals": int(fb2[0]),
                             "fp64_rescans": int(fb2[1])})
        del pos, sig, idx, d2
    out["peak_source"] = (f"nominal FP32 2x128 lanes x {ctx.sm_count} SMs at the sampled "
                          f"{sm_mhz:.0f} MHz; 8 FLOP per pair (BASELINE.md 2)")
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


def other_configs(lib, names=("cfg1", "cfg2"), budget_s=20.0):
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
    from paper_1503_08294_b200.distributed import ShardedStep, run_multi_sharded
    from paper_1503_08294_b200.multi import run_multi
    from paper_1503_08294_b200.network import Network

    lib = _lib.load_library()
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
    sig_buf = torch.empty((m, 3), dtype=torch.float64, device="cuda")
    net = Network(params, capacity=8192)
    net.reserve(8192)
    sharded = ShardedStep(net) if world > 1 else None
    if sharded is None:
        net.set_async(8)
    engine_stream = torch.cuda.ExternalStream(net.stream_handle())
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    st = _lib.GsBatchStats()
    torch.cuda.synchronize()

    LOOKAHEAD = 8  # batches enqueued ahead of the convergence check

    def one_run(trace=None):
        net.reset()
        for s in seeds:
            net.add_unit(s, params.theta0)
        _lib.check(lib.gs_sampler_set_state(sampler.handle, state0))
        if trace is None and sharded is None:
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
        off = 0
        units = 2
        while off < params.max_signals:
            if trace is not None:
                trace["pairs"] += m * units
            if sharded is None:
                _lib.check(lib.gs_engine_step_sampled(net.handle, sampler.handle, m, None))
            else:
                sampler.draw(m, sig_buf.data_ptr(), net.stream_handle())
                sharded.step_device(sig_buf.data_ptr(), m)
            _lib.check(lib.gs_engine_stats(net.handle, C.byref(st)))
            off += m
            units = int(st.units)
            if trace is not None:
                trace["processed"] += int(st.processed)
                trace["batches"] += 1
            if st.converged:
                break
        return off, bool(st.converged), int(st.units), int(st.edges)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        with torch.cuda.stream(engine_stream):
            flush.zero_()
        one_run()
    barrier()
    launches0 = net.launch_count()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    signals = 0
    result = None
    with ClockSampler(local) as clocks:
        ev0.record(engine_stream)
        for _ in range(args.steps):
            with torch.cuda.stream(engine_stream):
                flush.zero_()
            sig, conv, units, edges = one_run()
            signals += sig
            result = (sig, conv, units, edges)
        ev1.record(engine_stream)
        barrier()
    launches = net.launch_count() - launches0
    ms = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    value = signals / (ms * 1e-3)
    clk = clocks.summary()

    # per-phase device time over one extra (untimed) run: the roofline's kernel
    trace = dict(pairs=0, processed=0, batches=0)
    phase = np.zeros(2, np.float64)
    _lib.check(lib.gs_engine_phase_ms(net.handle, 1, phase))
    # step_device only records events when stats are harvested synchronously
    one_run(trace)
    _lib.check(lib.gs_engine_phase_ms(net.handle, 0, phase))
    find_ms, update_ms = float(phase[0]), float(phase[1])
    peaks = load_peaks()
    counts = net.counts()
    mean_deg = 2.0 * counts["edges"] / max(1, counts["units"])
    if find_ms >= update_ms:
        sm_mhz = clk.get("sm_mhz") or peaks.get("sm_max_mhz", 1965.0)
        sms = _lib.default_context().sm_count
        peak = 2 * 128 * sms * sm_mhz * 1e6 / 1e12
        achieved = 8.0 * trace["pairs"] / (find_ms * 1e-3) / 1e12
        roof = {"kernel": "find_exact_kernel", "bound": "fp32", "achieved": achieved,
                "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                "traffic": ncu_traffic("find"),
                "peak_source": f"nominal FP32 2x128 lanes x {sms} SMs at the sampled {sm_mhz:.0f} MHz",
                "work": "8 FLOP per (signal, live unit) pair (BASELINE.md 2)",
                "share_of_step": find_ms / (find_ms + update_ms)}
    else:
        per_sig = (1 + mean_deg) * 2 * (32 + 8) + mean_deg * (8 + 8) + 16 + 24
        achieved = per_sig * trace["processed"] / (update_ms * 1e-3) / 1e9
        peak = float(peaks.get("hbm_gbs", 6650.0))
        roof = {"kernel": "k_update_batch", "bound": "hbm", "achieved": achieved, "peak": peak,
                "unit": "GB/s", "frac": achieved / peak, "traffic": ncu_traffic("update"),
                "peak_source": "MEASURED_PEAKS.json hbm_gbs" + (" (fallback)" if peaks.get("fallback") else ""),
                "work": f"{per_sig:.0f} B per processed signal (winner + {mean_deg:.2f} neighbours: "
                        "pos+hab read/write, adjacency, edge ages, record, signal)",
                "share_of_step": update_ms / (find_ms + update_ms),
                "note": "sequential-semantics update on one 16-CTA cluster: bound by dependent L2 round trips and cluster barriers, not by bandwidth"}

    # e2e through the public API: host sampling + H2D per batch + stats D2H
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
            t_run = time.perf_counter()
            if world > 1:
                res_net, rs = run_multi_sharded(src, params, seed)
            else:
                res_net, rs = run_multi(src, params, seed, capacity=8192)
            results.append(res_net)
            e_sig += rs.signals
            e_batches += rs.iterations
            if os.environ.get("GS_E2E_DEBUG"):
                print(f"e2e run: {1e3 * (time.perf_counter() - t_run):.0f} ms "
                      f"(loop {1e3 * rs.total_s:.0f} ms)", file=sys.stderr, flush=True)
        barrier()
        e_s = time.perf_counter() - t0
        del results
        if world > 1:
            t = torch.tensor([e_s], device="cuda", dtype=torch.float64)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            e_s = float(t.item())
        e2e = {"value": e_sig / e_s, "unit": "signals/s",
               "h2d_bytes_per_step": int(cloud_bytes + 48 + 120),
               "d2h_bytes_per_step": int(C.sizeof(_lib.GsBatchStats) * (e_batches // args.steps)),
               "ms_per_step": 1e3 * e_s / args.steps}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        wparams = dict(workloads.WORKLOADS[args.workload]["params"])
        sig, sec, batches, kind, cores = reference_prefix(src.points, src.label, wparams, seed,
                                                          args.cpu_budget_s)
        cpu = {"value": sig / sec, "unit": "signals/s", "cores": cores, "kind": kind,
               "sample": f"first {sig:,} signals ({batches} batches) of the same seeded "
                         f"{args.workload} run ({sec:.1f} s)"}

    sweep = None
    if rank == 0 and world == 1 and not args.no_m_sweep:
        sweep = m_sweep(lib, src, dict(workloads.WORKLOADS[args.workload]["params"]), seed)
    others = None
    if rank == 0 and world == 1 and not args.no_m_sweep:
        others = other_configs(lib)
    fmb = None
    if rank == 0 and not args.no_find_microbench:
        fmb = find_microbench(lib, _lib.default_context(),
                              clk.get("sm_mhz") or peaks.get("sm_max_mhz", 1965.0), peaks)

    if rank == 0:
        sig, conv, units, edges = result
        line = {
            "metric": METRIC, "value": value, "unit": "signals/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": args.workload, "desc": desc, "m": m, "theta0": params.theta0,
                       "seed": seed, "cloud_points": int(src.points.shape[0]),
                       "parallelism": f"signal-sharded find x{world}, replicated update",
                       "step": "one seeded run from the two seed units to convergence",
                       "signals_per_step": sig, "converged": conv, "units": units,
                       "edges": edges, "time_to_converge_s": ms / args.steps * 1e-3,
                       "l2": "256 MiB L2 flush before each step (cloud "
                             f"{cloud_bytes / 2**20:.0f} MiB resident in HBM)",
                       "sampling": "device Philox4x64-10 + Lemire, bit-identical to numpy",
                       "find_mode": "auto"},
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clk,
            "phase_ms_per_step": {"find": find_ms, "update": update_ms},
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

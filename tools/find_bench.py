"""Config 5 find-winners microbench (BASELINE.json configs[4]).

m signals vs n units drawn uniform in [0,1)^3 from Philox(7) as the
reference's kernel-bench does (cli.py:252-261); the device find runs in
the requested mode on resident inputs; CUDA events on the launching
stream, L2 flushed between repetitions.  Prints one JSON line per n.
Usage: python tools/find_bench.py [m] [n ...] [--mode 0|1] [--reps R]
"""
import argparse
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("m", type=int, nargs="?", default=1_000_000)
    ap.add_argument("n", type=int, nargs="*", default=[10_000, 100_000, 1_000_000])
    ap.add_argument("--mode", type=int, default=1)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    import numpy as np
    import torch

    from paper_1503_08294_b200 import _lib

    lib = _lib.load_library()
    ctx = _lib.default_context()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for n in args.n:
        rng = np.random.Generator(np.random.Philox(7))
        pos = torch.from_numpy(rng.random((n, 3))).cuda()
        sig = torch.from_numpy(rng.random((args.m, 3))).cuda()
        idx = torch.empty((args.m, 2), dtype=torch.int64, device="cuda")
        d2 = torch.empty((args.m, 2), dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()
        st = torch.cuda.Stream()  # a real stream: handle 0 would mean the context's own stream

        def run():
            _lib.check(lib.gs_find_device(ctx.handle, pos.data_ptr(), n, sig.data_ptr(), args.m,
                                          idx.data_ptr(), d2.data_ptr(), args.mode, st.cuda_stream))

        run()
        torch.cuda.synchronize()
        times = []
        for _ in range(args.reps):
            with torch.cuda.stream(st):
                flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            run()
            e1.record(st)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
        fb2 = np.zeros(2, np.int64)
        _lib.check(lib.gs_find_last_fallback_counts(ctx.handle, fb2))
        ms = sorted(times)[len(times) // 2]
        pairs = float(n) * args.m
        print(json.dumps({"n": n, "m": args.m, "mode": args.mode, "ms": ms,
                          "pairs_per_s": pairs / (ms * 1e-3), "tflops_8": 8 * pairs / (ms * 1e-3) / 1e12,
                          "fallbacks": int(fb2[0]), "fp64_rescans": int(fb2[1]), "times": times}), flush=True)


if __name__ == "__main__":
    main()

"""Time-to-converge of BASELINE configs 1 and 2 (and 3) with the current
library (GS_LIB_PATH for A/B builds): bench.py's own measurement, no
reference runs.  Usage: python tools/cfg_timing.py [cfg1 cfg2 ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402,F401  (before the library: see _lib._preload_nccl)
import bench  # noqa: E402
from paper_1503_08294_b200 import _lib  # noqa: E402

names = tuple(sys.argv[1:]) or ("cfg1", "cfg2")
res = bench.other_configs(_lib.load_library(), names=names, ref_full=False)
for k, v in res.items():
    print(k, "%.4f s" % v["time_to_converge_s"], v["batches"], "batches", "V=%d" % v["units"],
          "conv" if v["converged"] else "NOT converged")

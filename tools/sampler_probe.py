"""Sampler chain diagnostics on one GPU: wall time per call (device-synchronised) and the exact
scans' walk statistics (certified chunk runs / element-exact chunks / split chunks / stepped
sub-chunks and their cycle counts).  Run under ncu for per-kernel durations:
  ncu --metrics gpu__time_duration.sum --csv python tools/sampler_probe.py --reps 2
"""
import argparse
import ctypes as C
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_2303_11612_b200 import device  # noqa: E402
from paper_2303_11612_b200._lib import lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1_000_000)
ap.add_argument("--L", type=int, default=400)
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--regime", default="nearly_optimal")
a = ap.parse_args()
rng = np.random.default_rng(5)
w = torch.from_numpy(rng.standard_normal(a.n) ** 2 * 1e3).cuda()
device.sample_columns(w, a.regime, 0.2, a.L, 1, 2)
st = (C.c_ulonglong * 8)()
lib.lmra_debug_sampler_stats(st, 1)
ts = []
for r in range(a.reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    device.sample_columns(w, a.regime, 0.2, a.L, 1, 2 + r)
    torch.cuda.synchronize()
    ts.append((time.perf_counter() - t0) * 1e3)
lib.lmra_debug_sampler_stats(st, 1)
names = ["certified_chunks", "exact_chunks", "split_chunks", "stepped_subchunks", "run_cycles",
         "exact_cycles", "split_cycles", "exact_iters"]
print({"n": a.n, "ms_median": round(float(np.median(ts)), 4),
       "per_call": {k: round(st[i] / a.reps, 1) for i, k in enumerate(names)}})

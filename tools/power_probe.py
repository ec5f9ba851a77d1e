"""Power-scheme (gram_power_apply, Strategy A, q = 1) time and fp64 tensor-pipe rate on the BASELINE
mode-0 shapes: half = A^T G then c = A half (4 I J s useful flop).  Host-timed around the C-ABI
call (which synchronises); min of 10."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2303_11612_b200 import device  # noqa: E402

SHAPES = [("cfg1 m0", 200, 40000, 15), ("cfg2 m0", 400, 160000, 30), ("cfg3 m0", 100, 80, 20),
          ("cfg5 m0", 512, 157287, 50), ("cfg5 m1", 512, 12288, 50), ("cfg4 m0", 1000, 400, 60)]
if len(sys.argv) > 1:
    SHAPES = [s for s in SHAPES if s[0].split()[0] in sys.argv[1:]]
torch.manual_seed(0)
for name, I, J, s in SHAPES:
    a = torch.randn(I * J, dtype=torch.float64, device="cuda")
    g = torch.randn(I * s, dtype=torch.float64, device="cuda")
    for _ in range(2):
        device.gram_power_apply(a, I, J, g, s, 1)
    ts = []
    for _ in range(10):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        device.gram_power_apply(a, I, J, g, s, 1)
        ts.append(time.perf_counter() - t0)
    t = min(ts)
    fl = 4.0 * I * J * s
    print(f"{name}: {I} x {J}, s {s}: {t * 1e3:.3f} ms, {fl / t / 1e12:.2f} TF/s useful "
          f"({fl / t / 1e12 / 37.0:.2f} of 37 TF)", flush=True)

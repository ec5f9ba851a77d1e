"""Split-K Strategy-A power scheme on the BASELINE's latency-bound shapes under different split
sizes (LMRA_TTM_MINK rows of K per TTM split / LMRA_GRAM_MINJ columns per Gram split), timed through lmra_gram_power_apply (wall clock around the synchronous
call, median of 20; includes the two device copies of the API)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2303_11612_b200 import device  # noqa: E402

res = {}
for (I, J, s, q) in [(1000, 400, 60, 2), (200, 40000, 15, 1), (100, 80, 20, 1), (400, 8000, 30, 1)]:
    a = torch.randn(I * J, dtype=torch.float64, device="cuda")
    g = torch.randn(I * s, dtype=torch.float64, device="cuda")
    for fused in ("64/32", "16/16", "32/16"):
        mk, mj = fused.split("/")
        os.environ["LMRA_TTM_MINK"], os.environ["LMRA_GRAM_MINJ"] = mk, mj
        for _ in range(3):
            device.gram_power_apply(a, I, J, g, s, q)
        ts = []
        for _ in range(20):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            device.gram_power_apply(a, I, J, g, s, q)
            ts.append((time.perf_counter() - t0) * 1e3)
        res[f"{I}x{J} s{s} q{q} splits={fused}"] = round(float(np.median(ts)), 4)
print(res)

"""Probe: int8 mode-0 contraction time vs SMs withheld from its grid (LMRA_I8_RESERVE)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_11612_b200 as P  # noqa: E402
from paper_2303_11612_b200 import device  # noqa: E402

K, J, mu = 1000, 1_000_000, 50
x = torch.randn(K * J, dtype=torch.float64, device="cuda")
q = torch.linalg.qr(torch.randn(K, mu, dtype=torch.float64, device="cuda"))[0].T.contiguous().view(-1)
w = (x.view(J, K) ** 2).sum(1)
ctx = P.default_context(0)
for r in [0, 1, 2, 4, 8, 16, 40, 74]:
    os.environ["LMRA_I8_RESERVE"] = str(r)
    device.mode0_product_i8(x, K, J, q, mu, w, ctx=ctx)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        device.mode0_product_i8(x, K, J, q, mu, w, ctx=ctx)
        ts.append((time.perf_counter() - t0) * 1e3)
    print(f"reserve {r:3d}: {min(ts):.3f} ms (host-timed incl. launch + sync)", flush=True)

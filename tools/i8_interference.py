"""Does a few SMs of fp64 work slow the int8 core contraction?  Times lmra_mode0_product_i8 on
cfg4's shape (1000 x 10^6, mu 50) alone and beside 6 single-CTA spinners (fp64 FMA or sleeping)
on another stream.  Build tools/microbench/libspinner.so first (see spinner.cu)."""
import ctypes as C
import os
import sys
import time

import torch

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)
from paper_2303_11612_b200 import device  # noqa: E402

sp = C.CDLL(os.path.join(ROOT, "tools", "microbench", "libspinner.so"))
K, J, mu = 1000, 1_000_000, 50
x = torch.randn(K * J, dtype=torch.float64, device="cuda")
q = torch.linalg.qr(torch.randn(K, mu, dtype=torch.float64, device="cuda"))[0].t().contiguous().t()
q = q.t().contiguous().reshape(-1)  # column-major K x mu
w = (x.view(J, K) ** 2).sum(1)
out = torch.zeros(1, dtype=torch.float64, device="cuda")
side = torch.cuda.Stream()


def timed(kind, nctas, cycles=3.0e6):
    torch.cuda.synchronize()
    if kind is not None:
        sp.spin_launch(kind, nctas, C.c_longlong(int(cycles)), C.c_void_p(side.cuda_stream),
                       C.c_void_p(out.data_ptr()))
    t0 = time.perf_counter()
    device.mode0_product_i8(x, K, J, q, mu, w)
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) * 1e3


for _ in range(3):
    timed(None, 0)
res = {}
for label, kind, n in [("alone", None, 0), ("6 fp64 spinners", 0, 6), ("6 sleeping spinners", 1, 6),
                       ("24 fp64 spinners", 0, 24), ("alone again", None, 0)]:
    ts = sorted(timed(kind, n) for _ in range(5))
    res[label] = round(ts[2], 3)
print(res)
# the same with the contraction's grid reduced to the SMs the spinners leave free
os.environ["LMRA_I8_RESERVE"] = "6"
res2 = {}
for label, kind, n in [("alone, 142 CTAs", None, 0), ("6 fp64 spinners, 142 CTAs", 0, 6),
                       ("6 sleeping spinners, 142 CTAs", 1, 6)]:
    ts = sorted(timed(kind, n) for _ in range(5))
    res2[label] = round(ts[2], 3)
print(res2)

# short co-runners (~0.3 ms): a device-wide sync inside the call would show as spinner time + call
os.environ["LMRA_I8_RESERVE"] = "0"
res3 = {}
for label, kind, n in [("alone", None, 0), ("6 sleeping spinners 0.3 ms", 1, 6), ("6 fp64 spinners 0.3 ms", 0, 6),
                       ("148 sleeping spinners 0.3 ms", 1, 148)]:
    ts = sorted(timed(kind, n, 6.0e5) for _ in range(5))
    res3[label] = round(ts[2], 3)
print(res3)

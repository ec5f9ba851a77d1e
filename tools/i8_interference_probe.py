"""Probe: int8 mode-0 contraction time while orthonormalisations (Jacobi) run on other SMs."""
import os
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_11612_b200 as P  # noqa: E402
from paper_2303_11612_b200 import device  # noqa: E402

K, J, mu = 1000, 1_000_000, 50
os.environ["LMRA_I8_RESERVE"] = "8"
x = torch.randn(K * J, dtype=torch.float64, device="cuda")
q = torch.linalg.qr(torch.randn(K, mu, dtype=torch.float64, device="cuda"))[0].T.contiguous().view(-1)
w = (x.view(J, K) ** 2).sum(1)
ctx = P.default_context(0)
c = torch.randn(1000 * 60, dtype=torch.float64, device="cuda")
s2 = torch.cuda.Stream()
ctx2 = P.Context(0, s2.cuda_stream)


def t_i8(n=5):
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        device.mode0_product_i8(x, K, J, q, mu, w, ctx=ctx)
        ts.append((time.perf_counter() - t0) * 1e3)
    return min(ts), max(ts)


print("alone", t_i8(), flush=True)
t0 = time.perf_counter()
for _ in range(10):
    device.leading_left_singular_vectors(c, 1000, 60, 50, ctx=ctx2)
print("orth alone %.3f ms" % ((time.perf_counter() - t0) * 100), flush=True)
for nthr in (1, 3):
    stop = threading.Event()
    cnt = [0]

    def loop(cx):
        with torch.cuda.stream(torch.cuda.Stream()):
            while not stop.is_set():
                device.leading_left_singular_vectors(c, 1000, 60, 50, ctx=cx)
                cnt[0] += 1
    ctxs = [P.Context(0, torch.cuda.Stream().cuda_stream) for _ in range(nthr)]
    th = [threading.Thread(target=loop, args=(cx,)) for cx in ctxs]
    for t in th:
        t.start()
    time.sleep(0.2)
    c0 = cnt[0]
    t1 = time.perf_counter()
    r = t_i8(10)
    el = time.perf_counter() - t1
    stop.set()
    for t in th:
        t.join()
    print(f"with {nthr} orth loops: i8 {r}, orth calls during: {cnt[0] - c0} in {el*1e3:.1f} ms", flush=True)

"""Time the int8 tensor-core mode-0 contraction vs the DMMA one on cfg4's shape."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2303_11612_b200 as P
from paper_2303_11612_b200 import device
K = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
J = int(sys.argv[2]) if len(sys.argv) > 2 else 1000000
mu = int(sys.argv[3]) if len(sys.argv) > 3 else 50
ctx = P.Context(0, torch.cuda.current_stream().cuda_stream)
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn(K * J, dtype=torch.float64, device="cuda", generator=g)
q = torch.linalg.qr(torch.randn(K, mu, dtype=torch.float64, device="cuda", generator=g))[0].T.contiguous().T.contiguous()
qcol = q.T.contiguous().reshape(-1)  # K x mu column-major
w = device.column_sqnorms(x, [K, J], 0, ctx=ctx)
res = {}
for name, fn in [("i8", lambda: device.mode0_product_i8(x, K, J, qcol, mu, w, ctx=ctx)),
                 ("dmma", lambda: device.mode_n_product(x, [K, J], 0, q.T.contiguous(), ctx=ctx)[0])]:
    for _ in range(2):
        y = fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        y = fn()
    e1.record()
    torch.cuda.synchronize()
    res[name] = e0.elapsed_time(e1) / 5
    res[name + "_y"] = y
yi = res.pop("i8_y").reshape(J, mu)
yd = res.pop("dmma_y").reshape(J, mu)
res["rel_diff"] = float((yi - yd).norm() / yd.norm())
res["i8_GBps"] = K * J * 8 / (res["i8"] / 1e3) / 1e9
print(json.dumps(res))

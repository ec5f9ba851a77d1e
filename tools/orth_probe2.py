"""Diagnostics: Jacobi sweeps + time of the orth primitive on random and structured sketches."""
import os
import sys
import ctypes

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2303_11612_b200 as P  # noqa: E402
from paper_2303_11612_b200 import _lib, device  # noqa: E402

_lib.lib.lmra_debug_jacobi_sweeps.restype = ctypes.c_int
ctx = P.Context(0, torch.cuda.current_stream().cuda_stream)
for I, s, mu in [(200, 15, 10), (400, 30, 20), (100, 20, 15), (1000, 60, 50), (512, 50, 40)]:
    for kind in ["gauss", "graded"]:
        if kind == "gauss":
            c = torch.randn(I * s, dtype=torch.float64, device="cuda")
        else:
            u, _ = torch.linalg.qr(torch.randn(I, s, dtype=torch.float64, device="cuda"))
            v, _ = torch.linalg.qr(torch.randn(s, s, dtype=torch.float64, device="cuda"))
            sig = torch.logspace(0, -10, s, dtype=torch.float64, device="cuda")
            c = ((u * sig) @ v.T).t().contiguous().view(-1)  # column-major I x s
        device.leading_left_singular_vectors(c, I, s, mu, ctx=ctx)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        device.leading_left_singular_vectors(c, I, s, mu, ctx=ctx)
        b.record()
        b.synchronize()
        print(I, s, mu, kind, "sweeps", _lib.lib.lmra_debug_jacobi_sweeps(), "ms %.3f" % a.elapsed_time(b))

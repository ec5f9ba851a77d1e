"""Micro-timings of the device primitives (CUDA events, warm, best of N)."""
import json
import sys
import os

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_11612_b200 as P  # noqa: E402
from paper_2303_11612_b200 import device  # noqa: E402


def timeit(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


def main():
    ctx = P.Context(0, torch.cuda.current_stream().cuda_stream)
    out = {}
    for I, s, mu in [(1000, 60, 50), (512, 50, 40), (400, 30, 20), (200, 15, 10), (100, 20, 15), (3, 3, 3)]:
        c = torch.randn(I * s, dtype=torch.float64, device="cuda")
        out[f"orth_{I}x{s}_mu{mu}_ms"] = timeit(lambda: device.leading_left_singular_vectors(c, I, s, mu, ctx=ctx))
    dims = [1000, 1000, 1000]
    x = torch.randn(int(np.prod(dims)), dtype=torch.float64, device="cuda")
    for mode in range(3):
        out[f"norms_1000^3_m{mode}_ms"] = timeit(lambda: device.column_sqnorms(x, dims, mode, ctx=ctx), 5)
    for m in [10, 15, 20, 30, 40, 50, 60]:
        b = torch.randn(m, 1000, dtype=torch.float64, device="cuda")
        for mode in [0, 2]:
            ms = timeit(lambda: device.mode_n_product(x, dims, mode, b, ctx=ctx), 3)
            out[f"ttm_1000^3_m{mode}_w{m}_ms"] = ms
            out[f"ttm_1000^3_m{mode}_w{m}_tflops"] = 2 * m * 1e9 / ms / 1e9
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()

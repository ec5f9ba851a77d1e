"""Time the device sampling chain on 1e6 squared-Gaussian norms (CUDA events), for ncu launch lists."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2303_11612_b200 as P  # noqa: E402
from paper_2303_11612_b200 import _lib, device  # noqa: E402

ctx = P.Context(0, torch.cuda.current_stream().cuda_stream)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
g = torch.Generator(device="cuda").manual_seed(0)
w = torch.randn(n, dtype=torch.float64, device="cuda", generator=g) ** 2
st = (ctypes.c_ulonglong * 8)()
for regime in ["nearly_optimal", "uniform"]:
    device.sample_columns(w, regime, 0.5, 400, 1, 4, ctx=ctx)
    torch.cuda.synchronize()
    _lib.lib.lmra_debug_sampler_stats(st, 1)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    device.sample_columns(w, regime, 0.5, 400, 1, 4, ctx=ctx)
    b.record()
    b.synchronize()
    _lib.lib.lmra_debug_sampler_stats(st, 1)
    print(regime, n, "ms %.3f" % a.elapsed_time(b),
          "| walk: certified %d exact %d split %d (stepped subs %d), run cycles %d, exact cycles %d, split cycles %d, block iters %d"
          % tuple(st[:8]))

"""Time the latency-bound chain pieces at cfg4 sizes (CUDA events, warm): the device sampling
chain on chi^2_1000-like column norms (J = 1e6, L = 400, nearly-optimal) and the
orthonormalisation of a 1000 x 60 sketch (mu = 50).  Walk statistics from the sampler's
diagnostics.  Used for launch lists under ncu as well (then the times are not bench values)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2303_11612_b200 as P  # noqa: E402
from paper_2303_11612_b200 import _lib, device  # noqa: E402

ctx = P.Context(0, torch.cuda.current_stream().cuda_stream)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
g = torch.Generator(device="cuda").manual_seed(0)
w = 2.0 * torch._standard_gamma(torch.full((n,), 500.0, dtype=torch.float64, device="cuda"), generator=g)
st = (ctypes.c_ulonglong * 8)()


def timed(fn):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps


for regime in ["nearly_optimal", "uniform"]:
    _lib.lib.lmra_debug_sampler_stats(st, 1)
    ms = timed(lambda: device.sample_columns(w, regime, 0.5, 400, 1, 4, ctx=ctx))
    _lib.lib.lmra_debug_sampler_stats(st, 1)
    print(regime, n, "ms %.4f" % ms,
          "| walk/rep: certified %d exact %d split %d (stepped subs %d), run cyc %d, exact cyc %d, split cyc %d, block iters %d"
          % tuple(v // (reps + 1) for v in st[:8]))
for I, s, mu in [(1000, 60, 50), (512, 50, 40), (400, 30, 20), (200, 15, 10)]:
    c = torch.randn(I * s, dtype=torch.float64, device="cuda", generator=g)
    c = c * torch.logspace(0, -8, s, dtype=torch.float64, device="cuda").repeat_interleave(I)
    ms = timed(lambda: device.leading_left_singular_vectors(c, I, s, mu, ctx=ctx))
    print("orth %dx%d mu %d: ms %.4f sweeps %d" % (I, s, mu, ms, _lib.lib.lmra_debug_jacobi_sweeps()))

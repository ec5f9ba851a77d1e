"""Per-mode exact-sampler time and walk statistics on cfg4's own canonical norms: the run's trace
gives each mode's norm vector, then lmra_sample_columns_device runs each mode's chain alone
(host-timed, min of 10) and lmra_debug_sampler_stats reports that mode's walk counts / cycles."""
import ctypes
import os
import sys
import time

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2303_11612_b200 as P  # noqa: E402
from baseline_configs import CONFIGS  # noqa: E402
from paper_2303_11612_b200 import _lib, device  # noqa: E402
from paper_2303_11612_b200.configs import algo_config, generate_device  # noqa: E402

bc = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg4"]
ctx = P.default_context(0)
x = generate_device(bc, ctx=ctx)
cfg = algo_config(bc)
dec = P.run_algorithm(bc.alg, P.DenseTensor.device(x, list(bc.dims)), cfg, ctx=ctx, trace=True)
buf = (ctypes.c_ulonglong * 8)()
for n, w in enumerate(dec.norms):
    if w is None:
        continue
    wd = torch.from_numpy(w).cuda()
    L = len(dec.samples[n][0])
    device.sample_columns(wd, cfg.regime, cfg.regime_beta, L, cfg.seed, len(bc.dims) + n + 1, ctx=ctx)
    _lib.lib.lmra_debug_sampler_stats(buf, 1)
    ts = []
    for _ in range(10):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        device.sample_columns(wd, cfg.regime, cfg.regime_beta, L, cfg.seed, len(bc.dims) + n + 1, ctx=ctx)
        ts.append((time.perf_counter() - t0) * 1e3)
    _lib.lib.lmra_debug_sampler_stats(buf, 1)
    v = [x_ // 10 for x_ in buf]
    print(f"mode {n}: J {w.size}, L {L}: {min(ts):.3f} ms (host-timed); per run: certified chunks {v[0]}, "
          f"crossing {v[1]}, split {v[2]}; thread-0 cycles runs {v[4]}, crossing {v[5]}, split {v[6]}", flush=True)

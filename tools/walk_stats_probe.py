"""Exact-sampler walk statistics (lmra_debug_sampler_stats) for one decomposition of a config:
certified chunks taken in runs, crossing chunks walked in O(1), split chunks walked by
sub-chunks, and thread-0 cycles spent in each (diagnostics of sampler.cu chunk_walk_kernel)."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2303_11612_b200 as P  # noqa: E402
from baseline_configs import CONFIGS  # noqa: E402
from paper_2303_11612_b200 import _lib  # noqa: E402
from paper_2303_11612_b200.configs import algo_config, generate_device  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
bc = CONFIGS[name]
ctx = P.default_context(0)
x = generate_device(bc, ctx=ctx)
t = P.DenseTensor.device(x, list(bc.dims))
cfg = algo_config(bc)
r = P.run_raw(bc.alg, t, cfg, ctx=ctx)
r.free()
buf = (ctypes.c_ulonglong * 8)()
_lib.lib.lmra_debug_sampler_stats(buf, 1)
r = P.run_raw(bc.alg, t, cfg, ctx=ctx)
r.free()
torch.cuda.synchronize()
_lib.lib.lmra_debug_sampler_stats(buf, 1)
v = list(buf)
print(f"{name}: certified chunks in runs {v[0]}, crossing chunks (O(1)) {v[1]}, split chunks {v[2]}; "
      f"thread-0 cycles: runs {v[4]}, crossing/exact {v[5]}, split {v[6]}")

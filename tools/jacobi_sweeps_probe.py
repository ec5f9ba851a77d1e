"""Jacobi sweeps and orthonormalisation time on the BASELINE sketches (oracle sketches of
scaled-down configs), per mode: lmra_leading_left_singular_vectors, then
lmra_debug_jacobi_sweeps and the orth core's phase clocks (lmra_debug_orth_clocks)."""
import ctypes
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from baseline_configs import CONFIGS, generate_host, scaled  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from paper_2303_11612_b200 import _lib, device  # noqa: E402

lib = _lib.lib
lib.lmra_debug_jacobi_sweeps.restype = ctypes.c_int
lib.lmra_debug_orth_clocks.argtypes = [ctypes.POINTER(ctypes.c_longlong)]
clk = (ctypes.c_longlong * 7)()
for name, dims in [("cfg1", None), ("cfg2", None), ("cfg3", None), ("cfg4", [1000, 200, 200]),
                   ("cfg5", [512, 128, 3, 128])]:
    bc = CONFIGS[name] if dims is None else scaled(name, dims)
    x = generate_host(bc)
    c = bc.cfg
    oc = orc.AlgoConfig(rank=list(c.rank), oversampling=c.oversampling, power=c.power, alpha=c.alpha,
                        regime=c.regime, regime_beta=c.regime_beta, t_samples=c.t_samples, order=c.order,
                        seed=c.seed, strategy=c.strategy)
    ref = orc.run(bc.alg, x, bc.dims, oc)
    for n, sk in enumerate(ref.sketches):
        I, s = sk.shape
        mu = ref.factors[n].shape[1]
        cd = torch.from_numpy(np.asfortranarray(sk).ravel(order="F")).cuda()
        device.leading_left_singular_vectors(cd, I, s, mu)
        sw = lib.lmra_debug_jacobi_sweeps()
        ts = []
        for _ in range(5):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            device.leading_left_singular_vectors(cd, I, s, mu)
            ts.append((time.perf_counter() - t0) * 1e3)
        lib.lmra_debug_orth_clocks(clk)
        c7 = list(clk)
        ph = ["load", "qr", "scale", "jacobi", "order", "apply+store"]
        parts = ", ".join(f"{ph[i]} {(c7[i + 1] - c7[i]) / 1e3:.1f}k" for i in range(6))
        sv = np.linalg.svd(sk, compute_uv=False)
        print(f"{name} mode {n}: {I}x{s} mu {mu}: sweeps {sw}, {min(ts):.3f} ms (host-timed), "
              f"kappa {sv[0] / max(sv[-1], 1e-300):.2e}; core cycles: {parts}", flush=True)

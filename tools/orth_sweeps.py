"""Orth timing + Jacobi sweep count on real sketches (oracle's, scaled cfg4/cfg5/cfg2)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2303_11612_b200 as P
from paper_2303_11612_b200 import device, _lib
from paper_2303_11612_b200.configs import scaled
from oracle import oracle as O

ctx = P.Context(0, torch.cuda.current_stream().cuda_stream)
out = {}
for name, dims in [("cfg4", [1000, 1000, 60]), ("cfg2", [500, 500, 500]), ("cfg5", [120, 120, 120, 40])]:
    bc = scaled(name, dims)
    x = bc.generate_host() if hasattr(bc, "generate_host") else None
    if x is None:
        from paper_2303_11612_b200.configs import generate_device
        x = generate_device(bc, ctx=ctx).cpu().numpy()
    oc = O.AlgoConfig(rank=list(bc.cfg.rank), oversampling=bc.cfg.oversampling, power=bc.cfg.power,
                      alpha=bc.cfg.alpha, regime=bc.cfg.regime,
                      t_samples=bc.cfg.t_samples, seed=bc.cfg.seed)
    ref = O.run(bc.alg, x, bc.dims, oc)
    for n, C in enumerate(ref.sketches):
        I, s = C.shape
        mu = ref.factors[n].shape[1]
        c = torch.from_numpy(np.asfortranarray(C).ravel(order="F")).cuda()
        for _ in range(2):
            device.leading_left_singular_vectors(c, I, s, mu, ctx=ctx)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            device.leading_left_singular_vectors(c, I, s, mu, ctx=ctx)
        e1.record()
        torch.cuda.synchronize()
        sw = _lib.lib.lmra_debug_jacobi_sweeps()
        sig = np.linalg.svd(C, compute_uv=False)
        out[f"{name}_m{n}"] = {"I": I, "s": s, "mu": mu, "ms": e0.elapsed_time(e1) / 5, "sweeps": sw,
                               "kappa": float(sig[0] / max(sig[-1], 1e-300))}
        print(f"{name} mode {n}: {I}x{s} mu={mu} orth {e0.elapsed_time(e1)/5:.3f} ms sweeps {sw} kappa {sig[0]/max(sig[-1],1e-300):.3g}", flush=True)
json.dump(out, open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/orth_sweeps.json", "w"), indent=1)

"""Diagnostics for the sharded path: per-rank core vs numpy contraction with the returned factors."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np
from oracle import oracle as orc
from test_gpu_sharded import run_sharded, _tensor
from conftest import subspace_sine
from paper_2303_11612_b200 import AlgoConfig, run_algorithm

def contract(a, factors):
    t = a
    for n, f in enumerate(factors):
        t = np.moveaxis(np.tensordot(f.T, t, axes=([1], [n])), 0, n)
    return t

for alg, dims, rank, P, regime, ov in [("alg5", (40, 36, 47), (4, 5, 6), 4, "optimal", True),
                                       ("alg5", (40, 36, 47), (4, 5, 6), 4, "optimal", False),
                                       ("alg5", (40, 36, 48), (4, 5, 6), 4, "optimal", True),
                                       ("alg5", (40, 36, 47), (4, 5, 6), 2, "optimal", True),
                                       ("alg5", (40, 36, 47), (5, 5, 5), 4, "optimal", True),
                                       ("alg2", (40, 36, 47), (4, 5, 6), 4, "optimal", False),
                                       ("alg4", (40, 36, 47), (4, 5, 6), 4, "optimal", True)]:
    a = _tensor(orc, dims)
    ocfg = orc.AlgoConfig(rank=list(rank), oversampling=6, power=1, regime=regime, seed=11)
    ref = orc.run(alg, a, dims, ocfg)
    cfg = AlgoConfig(rank=list(rank), oversampling=6, power=1, regime=regime, seed=11)
    amm = alg in ("alg4", "alg5")
    outs = run_sharded(alg, a, dims, cfg, P, samples=ref.samples if (amm and ov) else None)
    A = a.reshape(dims, order="F")
    g = outs[0]
    single = run_algorithm(alg, A, cfg, samples=ref.samples if (amm and ov) else None)
    sines = [subspace_sine(ref.factors[n], g.factors[n]) for n in range(3)]
    sines1 = [subspace_sine(ref.factors[n], single.factors[n]) for n in range(3)]
    cg = contract(A, g.factors)
    print(alg, dims, rank, P, regime, "ov" if ov else "own",
          "core_vs_ref %.3g" % (np.linalg.norm(g.core - ref.core) / np.linalg.norm(ref.core)),
          "core_vs_own_factors %.3g" % (np.linalg.norm(g.core - cg) / np.linalg.norm(cg)),
          "single_core_vs_ref %.3g" % (np.linalg.norm(single.core - ref.core) / np.linalg.norm(ref.core)),
          "sines", ["%.2g" % s for s in sines], "single sines", ["%.2g" % s for s in sines1],
          "colmax", ["%.2g" % np.abs(g.factors[n] - ref.factors[n]).max() for n in range(3)], flush=True)

"""Randomised parity sweep: random shapes / ranks / algorithms / regimes / power / oversampling at
oracle-friendly sizes, the device run (own draws) against the CPU oracle -- gap-aware sines, core
and RE differences -- beside the oracle's own floor (the oracle on the input perturbed at 1e-15
relative against the unperturbed oracle: requested ranks past the signal rank leave directions
that no fp64 evaluation order determines, and ST-HOSVD carries them into the later modes' data).
A case fails when a device metric exceeds max(1e-10, 100 x the floor's) or an index differs."""
import os
import sys
import traceback

import numpy as np

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2303_11612_b200 as lmra  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from conftest import gap_blocks, relative_error, subspace_sine  # noqa: E402

n_cases = int(sys.argv[1]) if len(sys.argv) > 1 else 100
seed0 = int(sys.argv[2]) if len(sys.argv) > 2 else 0
ALL_ALGS = len(sys.argv) > 3 and sys.argv[3] == "all"  # + the QR-proxy variants and the deterministic baselines
LARGE = len(sys.argv) > 3 and sys.argv[3] == "large"  # 3-way tensors of >= 2^27 elements (the big-input paths)
rng = np.random.default_rng(seed0)
fails = 0


def align_signs(g, o):
    """g's factor columns flipped to o's signs (the core's slices with them).  Only for the QR-proxy
    variants (alg6/alg7): the reference's factor there is Q u1 with the sign rule on u1 only, so its
    column signs follow Eigen's unblocked Householder Q, which the device's TSQR reproduces for
    sketches of <= 256 rows but not, column sign by column sign, for taller ones."""
    core = g.core.copy()
    facs = []
    for n, (qg, qo) in enumerate(zip(g.factors, o.factors)):
        sg = np.sign(np.sum(qg * qo, axis=0))
        sg[sg == 0] = 1.0
        facs.append(qg * sg)
        shape = [1] * core.ndim
        shape[n] = -1
        core = core * sg.reshape(shape)
    return type(g)(core=core, factors=facs, omega=g.omega, samples=g.samples, norms=g.norms)


def metrics(g, o, a):
    """(worst gap-aware sine, core rel diff, RE rel diff) of decomposition g against o (no asserts)."""
    worst = 0.0
    for n, (qg, qo) in enumerate(zip(g.factors, o.factors)):
        sk = o.sketches[n] if o.sketches and o.sketches[n] is not None and o.sketches[n].size else None
        if sk is None:  # deterministic baselines: the gaps of the unfolding's singular values
            sig = np.linalg.svd(np.moveaxis(a, n, 0).reshape(a.shape[n], -1), compute_uv=False)
        else:
            sig = np.linalg.svd(sk, compute_uv=False)
        ks = gap_blocks(sig, qo.shape[1])
        worst = max([worst] + [subspace_sine(qo[:, :k], qg[:, :k]) for k in ks])
    cd = np.linalg.norm(g.core - o.core) / np.linalg.norm(o.core)
    re_g, re_o = relative_error(a, g.core, g.factors), relative_error(a, o.core, o.factors)
    return worst, cd, abs(re_g - re_o) / max(re_o, 1e-3)


for case in range(n_cases):
    order = int(rng.choice([3, 3, 3, 4]))
    big = int(rng.integers(0, order))
    dims = [int(rng.integers(3, 40)) for _ in range(order)]
    dims[big] = int(rng.choice([int(rng.integers(40, 300)), int(rng.integers(770, 1100))]))
    if LARGE:  # >= 2^27 elements: the split orthonormalisation, int8 contractions, CholeskyQR basis
        order = 3
        dims = [int(rng.integers(480, 1050)) for _ in range(3)]
        while np.prod(dims) < (1 << 27):
            dims[int(rng.integers(0, 3))] += 64
    rank = [max(1, min(d, int(rng.integers(1, 12)))) for d in dims]
    algs = ["alg1", "alg2", "alg4", "alg5"] + (["alg6", "alg7", "thosvd", "sthosvd", "hooi"] if ALL_ALGS else [])
    alg = str(rng.choice(algs))
    kw = dict(rank=rank, oversampling=int(rng.integers(0, 12)), power=int(rng.integers(1, 3)),
              seed=int(rng.integers(0, 1000)))
    if alg in ("alg4", "alg5"):
        kw["regime"] = str(rng.choice(["uniform", "nearly_optimal", "optimal"]))
        kw["alpha"] = float(rng.choice([0.1, 0.3, 0.6]))
    gamma = float(rng.choice([1e-1, 1e-2, 1e-4]))
    x = orc.gen_tucker_noise(dims, [min(r, 6) for r in rank], gamma, int(rng.integers(0, 1000)))
    tag = f"case {case}: {alg} dims {dims} {kw} gamma {gamma}"
    a = x.reshape(dims, order="F")
    try:
        if alg in ("thosvd", "sthosvd", "hooi"):
            kw = dict(rank=rank)
        ref = orc.run(alg, x, dims, orc.AlgoConfig(**kw))
        gpu = lmra.run_algorithm(alg, lmra.DenseTensor.from_flat(x, dims), lmra.AlgoConfig(**kw))
        same_idx = True
        if alg in ("alg4", "alg5"):
            for n in range(order):
                same_idx &= bool(np.array_equal(gpu.samples[n][0], ref.samples[n][0]))
        # the floor: the oracle itself on the input perturbed at the rounding level (1e-15 relative)
        xp = x * (1.0 + 1e-15 * np.random.default_rng(case).standard_normal(x.size))
        refp = orc.run(alg, xp, dims, orc.AlgoConfig(**kw))
        if alg in ("alg6", "alg7"):
            gpu = align_signs(gpu, ref)
        mg, mf = metrics(gpu, ref, a), metrics(refp, ref, a)
        bad = [i for i in range(3) if mg[i] > max(1e-10, 100.0 * mf[i])]
        flag = "FAIL" if bad or not same_idx else "ok  "
        if flag == "FAIL":
            fails += 1
        print(f"{flag} {tag} | gpu sine {mg[0]:.1e} core {mg[1]:.1e} re {mg[2]:.1e} | floor sine {mf[0]:.1e} "
              f"core {mf[1]:.1e} re {mf[2]:.1e} | idx {'same' if same_idx else 'DIFF'}", flush=True)
    except Exception as e:  # noqa: BLE001
        fails += 1
        print(f"ERR  {tag}: {type(e).__name__}: {str(e)[:200]}", flush=True)
print(f"{n_cases - fails}/{n_cases} within max(1e-10, 100 x the oracle's own rounding floor)")

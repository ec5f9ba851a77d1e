"""Randomised parity (tools/parity_fuzz.py, a seeded sample of it): random shapes, ranks,
algorithms, sampling regimes, power and oversampling; the device decomposition against the CPU
oracle on the gap-aware sines, the core and the RE, each within max(1e-10, 100 x the oracle's own
floor -- the oracle on the input perturbed at 1e-15 relative against itself), and the sampled
indices bit-exact.  Requested ranks past the signal rank leave directions no fp64 evaluation order
determines; the floor measures that, the 1e-10 contract holds wherever the problem fixes the answer.
"""
import numpy as np
import pytest

from conftest import gap_blocks, relative_error, subspace_sine

pytestmark = pytest.mark.gpu


def _metrics(g, o, a):
    worst = 0.0
    for qg, qo, sk in zip(g.factors, o.factors, o.sketches):
        sig = np.linalg.svd(sk, compute_uv=False)
        worst = max([worst] + [subspace_sine(qo[:, :k], qg[:, :k]) for k in gap_blocks(sig, qo.shape[1])])
    cd = np.linalg.norm(g.core - o.core) / np.linalg.norm(o.core)
    re_g, re_o = relative_error(a, g.core, g.factors), relative_error(a, o.core, o.factors)
    return worst, cd, abs(re_g - re_o) / max(re_o, 1e-3)


@pytest.mark.parametrize("case", range(24))
def test_random_parity(gpu_ctx, lmra, orc, case):
    rng = np.random.default_rng(1000 + case)
    order = int(rng.choice([3, 3, 3, 4]))
    big = int(rng.integers(0, order))
    dims = [int(rng.integers(3, 40)) for _ in range(order)]
    dims[big] = int(rng.choice([int(rng.integers(40, 300)), int(rng.integers(770, 1100))]))
    rank = [max(1, min(d, int(rng.integers(1, 12)))) for d in dims]
    alg = str(rng.choice(["alg1", "alg2", "alg4", "alg5"]))
    kw = dict(rank=rank, oversampling=int(rng.integers(0, 12)), power=int(rng.integers(1, 3)),
              seed=int(rng.integers(0, 1000)))
    if alg in ("alg4", "alg5"):
        kw["regime"] = str(rng.choice(["uniform", "nearly_optimal", "optimal"]))
        kw["alpha"] = float(rng.choice([0.1, 0.3, 0.6]))
    gamma = float(rng.choice([1e-1, 1e-2, 1e-4]))
    x = orc.gen_tucker_noise(dims, [min(r, 6) for r in rank], gamma, int(rng.integers(0, 1000)))
    a = x.reshape(dims, order="F")
    ref = orc.run(alg, x, dims, orc.AlgoConfig(**kw))
    gpu = lmra.run_algorithm(alg, lmra.DenseTensor.from_flat(x, dims), lmra.AlgoConfig(**kw), ctx=gpu_ctx)
    if alg in ("alg4", "alg5"):
        for n in range(order):
            assert np.array_equal(gpu.samples[n][0], ref.samples[n][0]), f"mode {n}: sampled indices differ"
    xp = x * (1.0 + 1e-15 * np.random.default_rng(case).standard_normal(x.size))
    floor = _metrics(orc.run(alg, xp, dims, orc.AlgoConfig(**kw)), ref, a)
    got = _metrics(gpu, ref, a)
    for name, g, f in zip(("gap-aware sine", "core", "RE"), got, floor):
        assert g <= max(1e-10, 100.0 * f), f"{alg} {dims} {kw}: {name} {g:.3g} vs floor {f:.3g}"

"""GPU parity of the QR-proxy variants alg6 / alg7 (tucker.cpp:422-454) and their primitives
thin_qr (linalg.cpp:52-60) and qr_project_extract (linalg.cpp:89-99) against the CPU oracle.

Signs.  qr_project_extract returns Q U1 with the sign rule applied to U1 in the basis of
Householder Q (LAPACK/Eigen convention).  The device forms Q by Householder TSQR: for
I_n <= 256 (one block) that is exactly the Householder Q, so factor columns match one to one;
above, the TSQR Q spans the same space with possibly different column signs, so factor
columns match up to sign and the core up to the matching slice signs.  Subspaces, core and
RE are held to the 1e-10 contract, gap-aware on the projected spectrum and against the
measured rounding floor of the extraction itself (check_extract).
"""
import numpy as np
import pytest

from conftest import gap_blocks, relative_error, subspace_sine

pytestmark = pytest.mark.gpu

TOL = 1e-10


def _to_dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _unfold(t, n):
    return np.moveaxis(t, n, 0).reshape(t.shape[n], -1, order="F")


def _mode_product(t, b, n):
    return np.moveaxis(np.tensordot(b, t, axes=([1], [n])), 0, n)


def _align(gpu_f, ref_f, gpu_core):
    """Flip gpu factor columns onto the oracle's; flip the matching core slices."""
    core = gpu_core.copy()
    out = []
    for n, (g, r) in enumerate(zip(gpu_f, ref_f)):
        sg = np.sign(np.sum(g * r, axis=0))
        sg[sg == 0] = 1.0
        out.append(g * sg)
        shape = [1] * core.ndim
        shape[n] = -1
        core = core * sg.reshape(shape)
    return out, core


def _alt_extract(c, a_n, mu):
    """An equally valid fp64 evaluation of qr_project_extract (numpy Householder QR of the
    row-reversed sketch): its distance to the oracle is the rounding floor of the problem."""
    q, _ = np.linalg.qr(c[::-1])
    q = q[::-1]
    u = np.linalg.svd(q.T @ a_n, full_matrices=False)[0][:, :mu]
    return q @ u


def check_extract(got, want, c, a_n, mu, *, exact_signs, where=""):
    """Gap-aware sines (spectrum of the projected unfolding Q^T A_(n)) against
    max(1e-10, 100 x the measured oracle-vs-oracle floor): the extraction's noise-bulk
    directions inherit kappa(C) through Q (C = (A A^T)^q G squares the spectrum), so the
    reference's own output is determined only to that floor there.  Returns the
    worst floor and the alternative factor."""
    assert np.abs(got.T @ got - np.eye(mu)).max() <= 1e-12
    q, _ = np.linalg.qr(c)
    sig = np.linalg.svd(q.T @ a_n, compute_uv=False)
    ks = gap_blocks(sig, mu)
    alt = _alt_extract(c, a_n, mu)
    worst_floor = 0.0
    for k in ks:
        floor = subspace_sine(want[:, :k], alt[:, :k])
        worst_floor = max(worst_floor, floor)
        sine = subspace_sine(want[:, :k], got[:, :k])
        assert sine <= max(TOL, 100 * floor), f"{where} k={k}: sine {sine:.3g} (floor {floor:.3g})"
        if exact_signs and floor <= 1e-12 and (k - 1 in ks or k == 1):
            d = np.abs(got[:, k - 1] - want[:, k - 1]).max()
            assert d <= 1e3 * TOL, f"{where} column {k - 1}: sign/vector mismatch {d:.3g}"
    return worst_floor, alt


def compare_qr(gpu, ref, a, order, sequential, *, exact_signs):
    """Per mode check_extract on the oracle's sketch and working tensor; then the core
    (sign-aligned) against the oracle's when every mode is well determined (floor <= 1e-12),
    else against the GPU factors' own projection; RE within 1e-10 relative (or 100 x the RE
    floor of the alternative evaluation)."""
    work = a
    floors, alts = [], [None] * len(order)
    for n in order:
        qg, qo = gpu.factors[n], ref.factors[n]
        assert qg.shape == qo.shape, (n, qg.shape, qo.shape)
        fl, alts[n] = check_extract(qg, qo, ref.sketches[n], _unfold(work, n), qo.shape[1],
                                    exact_signs=exact_signs[n], where=f"mode {n}")
        floors.append(fl)
        if sequential:
            work = _mode_product(work, qo.T, n)
    if max(floors) <= 1e-12:
        _, core = _align(gpu.factors, ref.factors, gpu.core)
        cd = np.linalg.norm(core - ref.core) / np.linalg.norm(ref.core)
    else:
        proj = a
        for n, f in enumerate(gpu.factors):
            proj = _mode_product(proj, f.T, n)
        cd = np.linalg.norm(gpu.core - proj) / np.linalg.norm(proj)
    assert cd <= TOL, f"core rel diff {cd:.3g}"
    re_g = relative_error(a, gpu.core, gpu.factors)
    re_o = relative_error(a, ref.core, ref.factors)
    alt_core = a
    for n, f in enumerate(alts):
        alt_core = _mode_product(alt_core, f.T, n)
    re_floor = abs(relative_error(a, alt_core, alts) - re_o)
    assert abs(re_g - re_o) <= max(TOL * max(re_o, 1e-300), 100 * re_floor), \
        f"RE {re_g!r} vs {re_o!r} (floor {re_floor:.3g})"
    return floors, cd


# ---------------------------------------------------------------- primitives
@pytest.mark.parametrize("I,s", [(5, 3), (40, 20), (256, 64), (200, 15), (257, 9), (1000, 60),
                                 (3000, 64), (64, 1), (12000, 33)])
def test_thin_qr_q(gpu_ctx, orc, I, s):
    from paper_2303_11612_b200 import device
    c = np.asfortranarray(np.random.default_rng(I * 7 + s).standard_normal((I, s)))
    want = orc.thin_qr_q(c)
    got = device.thin_qr_q(_to_dev(c.ravel(order="F")), I, s, ctx=gpu_ctx).cpu().numpy().reshape((I, s), order="F")
    assert np.abs(got.T @ got - np.eye(s)).max() <= 1e-13
    if I <= 256:  # one Householder block: LAPACK's Q, signs included
        assert np.abs(got - want).max() <= 1e-12, np.abs(got - want).max()
    else:  # same columns up to sign (thin QR is unique up to the signs of diag R)
        sg = np.sign(np.sum(got * want, axis=0))
        assert np.abs(got * sg - want).max() <= 1e-11, np.abs(got * sg - want).max()


@pytest.mark.parametrize("I,s,J,mu", [(30, 8, 500, 5), (200, 15, 4000, 10), (256, 64, 300, 64),
                                      (300, 20, 70000, 12), (1000, 60, 5000, 50), (50, 20, 7, 7),
                                      (100, 30, 30, 30)])
def test_qr_project_extract(gpu_ctx, orc, I, s, J, mu):
    from paper_2303_11612_b200 import device
    rng = np.random.default_rng(I + s + J)
    # a with a decaying spectrum, c a sketch of it
    u, _ = np.linalg.qr(rng.standard_normal((I, min(I, J))))
    v, _ = np.linalg.qr(rng.standard_normal((J, min(I, J))))
    sv = np.logspace(0, -3, min(I, J))  # C = a a^T G squares it: keep kappa(C) <= 1e6
    a = np.asfortranarray((u * sv) @ v.T)
    c = np.asfortranarray(a @ (a.T @ rng.standard_normal((I, s))))
    want = orc.qr_project_extract(c, a, mu)
    got = device.qr_project_extract(_to_dev(c.ravel(order="F")), I, s, _to_dev(a.ravel(order="F")), J, mu,
                                    ctx=gpu_ctx).cpu().numpy().reshape((I, mu), order="F")
    check_extract(got, want, c, a, mu, exact_signs=I <= 256)


# ---------------------------------------------------------------- algorithms
CASES = [
    # dims, rank, oversampling, power (modes above 256 exercise the TSQR tree; [6, ...] has
    # an unfolding narrower than the sketch in alg7's last mode)
    ([24, 20, 16], [4, 5, 3], 5, 1),
    ([40, 30, 300], [6, 5, 8], 10, 2),
    ([12, 10, 8, 6], [3, 3, 2, 2], 4, 1),
    ([300, 8, 6], [10, 6, 5], 10, 1),
]


@pytest.mark.parametrize("alg", ["alg6", "alg7"])
@pytest.mark.parametrize("case", range(len(CASES)))
def test_qr_proxy_matches_oracle(gpu_ctx, lmra, orc, alg, case):
    dims, rank, p, q = CASES[case]
    x = orc.gen_tucker_noise(dims, [max(1, k - 1) for k in rank], 1e-2, 11 + case)
    kw = dict(rank=rank, oversampling=p, power=q, seed=3 + case)
    ref = orc.run(alg, x, dims, orc.AlgoConfig(**kw))
    t = lmra.DenseTensor.from_flat(x, dims)
    own = lmra.run_algorithm(alg, t, lmra.AlgoConfig(**kw))
    for n in range(len(dims)):
        assert np.array_equal(own.omega[n], ref.omega[n]), f"Omega mode {n}"
    a = x.reshape(dims, order="F")
    order = list(range(len(dims)))
    exact = [d <= 256 for d in dims]
    compare_qr(own, ref, a, order, alg == "alg7", exact_signs=exact)
    gpu = lmra.run_algorithm(alg, t, lmra.AlgoConfig(**kw), omega=ref.omega)
    compare_qr(gpu, ref, a, order, alg == "alg7", exact_signs=exact)


@pytest.mark.parametrize("alg", ["alg6", "alg7"])
def test_qr_proxy_exact_rank_recovered(gpu_ctx, lmra, orc, alg):
    # test_tucker.cpp:247-255: exact multilinear rank -> RE <= 1e-8
    dims = [24, 24, 24]
    x = orc.gen_tucker_noise(dims, [4, 4, 4], 0.0, 27)
    for seed in (1, 2, 3):
        d = lmra.run_algorithm(alg, lmra.DenseTensor.from_flat(x, dims), lmra.AlgoConfig(rank=[4, 4, 4], seed=seed))
        re = relative_error(x.reshape(dims, order="F"), d.core, d.factors)
        assert re <= 1e-8, (seed, re)


def test_qr_proxy_tracks_power_variants(gpu_ctx, lmra, orc):
    # test_tucker.cpp:267-299: on the desk tensor alg6 / alg7 stay within 5 % of alg1 / alg2
    dims = [60, 60, 60]
    x = orc.gen_tucker_noise(dims, [10, 10, 10], 0.001, 31)
    a = x.reshape(dims, order="F")
    t = lmra.DenseTensor.from_flat(x, dims)
    ok6 = ok7 = 0
    for s in range(1, 21):
        cfg = lmra.AlgoConfig(rank=[10, 10, 10], seed=s)
        re = {alg: relative_error(a, d.core, d.factors)
              for alg in ("alg1", "alg2", "alg6", "alg7")
              for d in [lmra.run_algorithm(alg, t, cfg, trace=False)]}
        ok6 += re["alg6"] <= 1.05 * re["alg1"]
        ok7 += re["alg7"] <= 1.05 * re["alg2"]
    assert ok6 >= 16 and ok7 >= 16, (ok6, ok7)


@pytest.mark.parametrize("alg", ["alg6", "alg7"])
def test_qr_proxy_deterministic(gpu_ctx, lmra, alg):
    # test_tucker.cpp:398-408
    dims = [14, 12, 10]
    x = np.random.default_rng(41).standard_normal(int(np.prod(dims)))
    t = lmra.DenseTensor.from_flat(x, dims)
    cfg = lmra.AlgoConfig(rank=[3, 3, 3], seed=99)
    a, b = lmra.run_algorithm(alg, t, cfg), lmra.run_algorithm(alg, t, cfg)
    assert np.array_equal(a.core, b.core)
    for fa, fb in zip(a.factors, b.factors):
        assert np.array_equal(fa, fb)


def test_qr_proxy_order4_exact(gpu_ctx, lmra, orc):
    # test_tucker.cpp:411-428 (alg7 at the core rank of an order-4 tensor)
    dims = [12, 12, 12, 12]
    x = orc.gen_tucker_noise(dims, [3, 3, 3, 3], 0.0, 47)
    d = lmra.run_algorithm("alg7", lmra.DenseTensor.from_flat(x, dims), lmra.AlgoConfig(rank=[3, 3, 3, 3], seed=2))
    assert list(d.core.shape) == [3, 3, 3, 3]
    assert relative_error(x.reshape(dims, order="F"), d.core, d.factors) <= 1e-8


def test_qr_proxy_rank_clamped(gpu_ctx, lmra, orc):
    # rank_cap (tucker.cpp:65-71): mu above min(sketch width, unfolding columns) is clamped
    dims = [40, 2, 2]
    x = orc.rng_normal(51, 0, 160)
    for alg in ("alg6", "alg7"):
        kw = dict(rank=[10, 2, 2], seed=3, oversampling=2)
        ref = orc.run(alg, x, dims, orc.AlgoConfig(**kw))
        d = lmra.run_algorithm(alg, lmra.DenseTensor.from_flat(x, dims), lmra.AlgoConfig(**kw))
        assert [f.shape for f in d.factors] == [f.shape for f in ref.factors]
        for f in d.factors:
            assert np.abs(f.T @ f - np.eye(f.shape[1])).max() <= 1e-10

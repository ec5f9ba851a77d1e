"""GPU parity: the sm_100a path (through the C ABI) against the CPU oracle.

Tolerances (BASELINE north_star): factor principal-angle sines <= 1e-10, core and
relative reconstruction error within 1e-10 relative, integer sample indices bit-exact.
Factor sines are checked on every leading block k <= mu whose sketch gap
(s_k - s_{k+1}) / s_1 >= 1e-5 (directions inside rounding-level gaps are
not determined by any fp64 evaluation order; the full-subspace sine is reported).
"""
import numpy as np
import pytest

from conftest import gap_blocks, relative_error, subspace_sine

pytestmark = pytest.mark.gpu

TOL = 1e-10


def _torch():
    import torch
    return torch


def _to_dev(a_flat):
    torch = _torch()
    return torch.from_numpy(np.ascontiguousarray(a_flat)).cuda()


def compare(gpu, ref, a, *, tol=TOL, check_core=True, check_columns=True, check_re=True, re_fn=None):
    """Returns a dict of metrics; asserts the parity contract.  re_fn(core, factors) -> RE
    replaces the numpy reconstruction (full-size tensors: device RE, lmra_relative_error)."""
    out = {"sines": [], "full_sines": []}
    for n, (qg, qo) in enumerate(zip(gpu.factors, ref.factors)):
        assert qg.shape == qo.shape, (n, qg.shape, qo.shape)
        orth = np.abs(qg.T @ qg - np.eye(qg.shape[1])).max()
        assert orth <= 1e-12, f"mode {n}: factor not orthonormal ({orth:.3g})"
        sig = np.linalg.svd(ref.sketches[n], compute_uv=False)
        ks = gap_blocks(sig, qo.shape[1])
        worst = max([subspace_sine(qo[:, :k], qg[:, :k]) for k in ks], default=0.0)
        out["sines"].append(worst)
        out["full_sines"].append(subspace_sine(qo, qg))
        assert worst <= tol, f"mode {n}: gap-aware subspace sine {worst:.3g}"
        if check_columns:
            # columns separated by gaps on both sides must match one to one (sign rule)
            single = [k for k in ks if (k - 1 in ks or k == 1)]
            for k in single:
                d = np.abs(qg[:, k - 1] - qo[:, k - 1]).max()
                assert d <= 1e3 * tol, f"mode {n} column {k - 1}: sign/vector mismatch {d:.3g}"
    if check_core:
        cd = np.linalg.norm(gpu.core - ref.core) / np.linalg.norm(ref.core)
        out["core"] = cd
        assert cd <= tol, f"core rel diff {cd:.3g}"
    if re_fn is None:
        re_g = relative_error(a, gpu.core, gpu.factors)
        re_o = relative_error(a, ref.core, ref.factors)
    else:
        re_g = re_fn(gpu.core, gpu.factors)
        re_o = re_fn(ref.core, ref.factors)
    out["re"] = (re_g, re_o)
    if check_re:
        # relative (tol) for every RE >= 1e-3 -- all BASELINE configs except the documented cfg2;
        # an absolute 1e-13 floor for decompositions exact to rounding (RE ~ 1e-15)
        assert abs(re_g - re_o) <= tol * max(re_o, 1e-3), f"RE {re_g!r} vs {re_o!r}"
    return out


# ---------------------------------------------------------------- primitives
@pytest.mark.parametrize("dims,core", [((20, 18, 16), (4, 5, 3)), ((9, 7, 5, 3), (3, 3, 2, 2)), ((64, 33), (7, 5))])
def test_device_relative_error_matches_oracle(gpu_ctx, orc, lmra, dims, core):
    # reconstruct + relative_error (tucker.cpp:222-240) on the device vs the oracle's loop
    from paper_2303_11612_b200 import device
    x = orc.gen_tucker_noise(list(dims), list(core), 3e-2, 5)
    cfg = dict(rank=list(core), seed=2)
    ref = orc.run("alg1", x, list(dims), orc.AlgoConfig(**cfg))
    want = orc.relative_error(x, list(dims), ref)
    got = device.relative_error(_to_dev(x), list(dims), ref.core, ref.factors, ctx=gpu_ctx)
    assert abs(got - want) <= 1e-13 * want, (got, want)
    # the result-handle form (reconstructs the run's own device core / factors)
    r = lmra.run_raw("alg1", lmra.DenseTensor.from_flat(x, list(dims)), lmra.AlgoConfig(**cfg), ctx=gpu_ctx)
    dec = r.to_host()
    got2 = device.result_relative_error(r, _to_dev(x), list(dims), ctx=gpu_ctx)
    r.free()
    assert abs(got2 - relative_error(x.reshape(dims, order="F"), dec.core, dec.factors)) <= 1e-13 * want
    # the reference's error surface
    with pytest.raises(lmra.LmraInvalidArgument, match="zero reference tensor"):
        device.relative_error(_to_dev(np.zeros_like(x)), list(dims), ref.core, ref.factors, ctx=gpu_ctx)



@pytest.mark.parametrize("dims,mode,m", [
    ((7, 5, 3), 0, 4), ((7, 5, 3), 1, 4), ((7, 5, 3), 2, 2),
    ((33, 40, 17), 0, 13), ((33, 40, 17), 1, 64), ((33, 40, 17), 2, 70),
    ((64, 30, 20), 1, 8), ((6, 200, 9), 1, 50), ((200, 10, 30), 0, 1), ((10, 20, 200), 2, 57),
    ((3, 4, 5, 6), 3, 5), ((2, 129, 3), 1, 33),
    # the streaming kernel for short modes (I <= 8): contiguous and strided fibres, m up to 64
    ((40, 40, 3, 64), 2, 3), ((8, 900, 5), 0, 64), ((300, 7, 20), 1, 7), ((50, 20, 1), 2, 1),
    # small contractions split along K over both resident CTAs of an SM
    ((10, 200, 200), 1, 10), ((10, 10, 200), 2, 10), ((40, 40, 3, 512), 3, 40),
    # the persistent streaming TTM (mode 0, m <= 32, >= 4 tiles per SM): even / odd K, every width
    ((100, 400, 200), 0, 15), ((99, 400, 200), 0, 20), ((64, 300, 300), 0, 32), ((30, 700, 120), 0, 7),
])
def test_ttm_matches_oracle(gpu_ctx, orc, dims, mode, m):
    from paper_2303_11612_b200 import device
    rng = np.random.default_rng(1)
    x = rng.standard_normal(int(np.prod(dims)))
    b = rng.standard_normal((m, dims[mode]))
    want = orc.mode_n_product(x, dims, mode, b)
    y, od = device.mode_n_product(_to_dev(x), dims, mode, _to_dev(b), ctx=gpu_ctx)
    got = y.cpu().numpy()
    err = np.abs(got - want).max() / max(np.abs(want).max(), 1e-300)
    assert err <= 1e-13, err


@pytest.mark.parametrize("dims", [(7, 5, 3), (33, 40, 17), (100, 3, 70), (1, 1000, 4), (65, 2, 2),
                                  (512, 40, 3), (3, 3, 3, 3),
                                  # the TMA mode-0 pass: partial 32-row chunks, partial 128-column tiles,
                                  # more tiles than SMs (a persistent CTA takes several)
                                  (18, 77, 5), (1030, 129, 2), (64, 1000, 3), (200, 300, 1), (512, 256, 3, 2)])
def test_column_sqnorms_bit_exact(gpu_ctx, orc, dims):
    from paper_2303_11612_b200 import device
    x = np.random.default_rng(2).standard_normal(int(np.prod(dims)))
    xd = _to_dev(x)
    for mode in range(len(dims)):
        want = orc.column_sqnorms(x, dims, mode)
        got = device.column_sqnorms(xd, dims, mode, ctx=gpu_ctx).cpu().numpy()
        assert np.array_equal(got, want), (mode, np.abs(got - want).max())


@pytest.mark.parametrize("I,s,mu", [(5, 3, 2), (40, 20, 10), (200, 15, 10), (400, 30, 20),
                                    (100, 20, 15), (512, 50, 40), (1000, 60, 50), (3000, 64, 64),
                                    (3, 3, 3), (64, 1, 1), (700, 33, 7), (300, 80, 70), (1000, 128, 100)])
def test_orth_matches_oracle_svd(gpu_ctx, orc, I, s, mu):
    from paper_2303_11612_b200 import device
    c = np.asfortranarray(np.random.default_rng(I + s).standard_normal((I, s)))
    want = orc.leading_left_singular_vectors(c, mu)
    got = device.leading_left_singular_vectors(_to_dev(c.ravel(order="F")), I, s, mu,
                                               ctx=gpu_ctx).cpu().numpy().reshape((I, mu), order="F")
    assert np.abs(got.T @ got - np.eye(mu)).max() <= 1e-13
    assert np.abs(got - want).max() <= 1e-11, np.abs(got - want).max()


def test_orth_rank_deficient_still_orthonormal(gpu_ctx):
    from paper_2303_11612_b200 import device
    rng = np.random.default_rng(7)
    base = rng.standard_normal((40, 4))
    c = np.asfortranarray(base @ rng.standard_normal((4, 20)))  # rank 4, 20 columns
    c[:, 7] = 0.0
    u = device.leading_left_singular_vectors(_to_dev(c.ravel(order="F")), 40, 20, 10,
                                             ctx=gpu_ctx).cpu().numpy().reshape((40, 10), order="F")
    assert np.abs(u.T @ u - np.eye(10)).max() <= 1e-12
    # the leading 4 directions span range(c)
    q, _ = np.linalg.qr(base)
    assert subspace_sine(u[:, :4], q) <= 1e-10


def _graded_sketch(I, s, decades, seed):
    rng = np.random.default_rng(seed)
    u, _ = np.linalg.qr(rng.standard_normal((I, s)))
    v, _ = np.linalg.qr(rng.standard_normal((s, s)))
    sig = 10.0 ** (-decades * np.arange(s) / max(s - 1, 1))
    return np.asfortranarray((u * sig) @ v.T), sig


@pytest.mark.parametrize("I,s,mu,decades", [(1000, 60, 50, 10), (1000, 60, 50, 15), (800, 50, 40, 14),
                                            (900, 30, 20, 8), (1280, 64, 64, 12), (1400, 64, 64, 12),
                                            (769, 16, 16, 15)])
def test_orth_cholqr_graded_sketches(gpu_ctx, orc, I, s, mu, decades, monkeypatch):
    # sketches with kappa up to 1e15 (the BASELINE sketches reach 1e16) through the
    # CholeskyQR basis (I > 768; 1400 rows exceed one cluster: Householder): leading vectors match the oracle's thin SVD where the spectrum
    # determines them (sigma_k >= 1e-4 sigma_1), the whole factor is orthonormal, and the
    # Householder-only path (LMRA_ORTH_CHOLQR=0) gives the same vectors
    from paper_2303_11612_b200 import device
    c, sig = _graded_sketch(I, s, decades, I + s + decades)
    want = orc.leading_left_singular_vectors(c, mu)
    outs = []
    for env in ("1", "0"):
        monkeypatch.setenv("LMRA_ORTH_CHOLQR", env)
        got = device.leading_left_singular_vectors(_to_dev(c.ravel(order="F")), I, s, mu,
                                                   ctx=gpu_ctx).cpu().numpy().reshape((I, mu), order="F")
        assert np.abs(got.T @ got - np.eye(mu)).max() <= 1e-13
        k = int(np.sum(sig[:mu] >= 1e-4))
        assert np.abs(got[:, :k] - want[:, :k]).max() <= 1e-10, np.abs(got[:, :k] - want[:, :k]).max()
        outs.append(got)
    k = int(np.sum(sig[:mu] >= 1e-4))
    assert np.abs(outs[0][:, :k] - outs[1][:, :k]).max() <= 1e-10


@pytest.mark.parametrize("I,s,rank,mu", [(1000, 60, 20, 30), (900, 40, 1, 10), (800, 20, 19, 20)])
def test_orth_cholqr_rank_deficient_falls_back(gpu_ctx, I, s, rank, mu):
    # an exactly rank-deficient sketch has no C R^-1 basis: the CholeskyQR flags it and the
    # gated Householder tree behind it produces the factor (orthonormal, leading block = range(C))
    from paper_2303_11612_b200 import device
    rng = np.random.default_rng(I + rank)
    base = rng.standard_normal((I, rank))
    c = np.asfortranarray(base @ rng.standard_normal((rank, s)))
    c[:, s // 2] = 0.0
    u = device.leading_left_singular_vectors(_to_dev(c.ravel(order="F")), I, s, mu,
                                             ctx=gpu_ctx).cpu().numpy().reshape((I, mu), order="F")
    assert np.all(np.isfinite(u))
    assert np.abs(u.T @ u - np.eye(mu)).max() <= 1e-12
    q, _ = np.linalg.qr(base)
    assert subspace_sine(u[:, :rank], q) <= 1e-10


@pytest.mark.parametrize("strategy", ["A", "B"])
@pytest.mark.parametrize("shape", [(37, 300, 9, 2), (1000, 400, 60, 2), (200, 5000, 15, 1), (3, 960, 3, 1),
                                   (513, 77, 33, 3), (511, 1000, 7, 1),
                                   (3, 163840, 3, 1), (200, 40000, 15, 1), (120, 90001, 30, 1)])
def test_gram_power_apply_matches_oracle(gpu_ctx, orc, strategy, shape):
    # split-K TTM / Gram launches on odd and even row counts (16-byte fibre loads need even I)
    from paper_2303_11612_b200 import device
    I, J, s, q = shape
    rng = np.random.default_rng(3 + I)
    a = np.asfortranarray(rng.standard_normal((I, J)))
    g = np.asfortranarray(rng.standard_normal((I, s)))
    want = orc.gram_power_apply(a, g, q, strategy)
    got = device.gram_power_apply(_to_dev(a.ravel(order="F")), I, J, _to_dev(g.ravel(order="F")),
                                  s, q, strategy, ctx=gpu_ctx).cpu().numpy().reshape((I, s), order="F")
    assert np.abs(got - want).max() / np.abs(want).max() <= 1e-13


# ---------------------------------------------------------------- algorithms
ALGS = ["alg1", "alg2", "alg4", "alg5"]


def _cfgs(lmra, orc, **kw):
    return lmra.AlgoConfig(**kw), orc.AlgoConfig(**kw)


@pytest.mark.parametrize("alg", ALGS)
@pytest.mark.parametrize("regime", ["uniform", "nearly_optimal", "optimal"])
def test_small_random_tensor(gpu_ctx, lmra, orc, alg, regime):
    dims = [12, 10, 8]
    x = np.random.default_rng(37).standard_normal(int(np.prod(dims)))
    kw = dict(rank=[3, 4, 2], seed=5, regime=regime)
    cg, co = _cfgs(lmra, orc, **kw)
    ref = orc.run(alg, x, dims, co)
    t = lmra.DenseTensor.from_flat(x, dims)
    own = lmra.run_algorithm(alg, t, cg)
    a = x.reshape(dims, order="F")
    check_own_draws(alg, own, ref, regime)
    # parity run: the oracle's (= reference host RNG's) draws passed to the GPU path
    gpu = lmra.run_algorithm(alg, t, cg, omega=ref.omega, samples=ref.samples)
    compare(gpu, ref, a)


@pytest.mark.parametrize("alg", ALGS)
def test_wide_sketch_matches_oracle(gpu_ctx, lmra, orc, alg):
    # sketch width mu + p above 64 (tucker.cpp:34-35 accepts any min(mu + p, I_n)): the
    # orthonormalisation goes through the wide-sketch path; everything else is unchanged
    dims = [90, 84, 12]
    x = np.random.default_rng(61).standard_normal(int(np.prod(dims)))
    kw = dict(rank=[60, 70, 6], oversampling=10, seed=9, regime="nearly_optimal",
              t_samples=[400, 400, 400] if alg == "alg4" else None)
    cg, co = _cfgs(lmra, orc, **kw)
    ref = orc.run(alg, x, dims, co)
    t = lmra.DenseTensor.from_flat(x, dims)
    own = lmra.run_algorithm(alg, t, cg)
    # (the shrunk tensor's small mode-2 fibres of this random input carry ~1e-12 relative
    # differences into their norms; the indices are still bit-exact)
    check_own_draws(alg, own, ref, "nearly_optimal", scale_tol=1e-10)
    compare(own, ref, x.reshape(dims, order="F"), check_columns=False)


def check_own_draws(alg, own, ref, regime, order=None, scale_tol=1e-12):
    """The GPU run's own Omega / sampled columns against the oracle's.

    Omega: bit-exact (same seeded host stream).  Samples: bit-exact whenever the
    probabilities are computed from the input tensor itself (T-HOSVD, the first mode of
    ST-HOSVD, or uniform sampling) -- the column norms use the canonical order shared with
    the oracle.  Later ST-HOSVD modes sample the shrunk tensor, whose last bits depend on
    the GEMM summation order (and on the factors' last bits): indices must still agree,
    scales to 1e-12 relative."""
    N = len(ref.factors)
    order = order or list(range(N))
    for n in range(N):
        assert np.array_equal(own.omega[n], ref.omega[n]), f"Omega mode {n}"
        if ref.samples[n] is None:
            continue
        assert np.array_equal(own.samples[n][0], ref.samples[n][0]), f"indices mode {n}"
        exact = alg == "alg4" or regime == "uniform" or n == order[0]
        if exact:
            assert np.array_equal(own.samples[n][1], ref.samples[n][1]), f"scales mode {n}"
        else:
            d = np.abs(own.samples[n][1] / ref.samples[n][1] - 1).max()
            assert d <= scale_tol, f"scales mode {n}: {d:.3g}"


@pytest.mark.parametrize("alg", ALGS)
def test_exact_rank_tensor_recovered(gpu_ctx, lmra, orc, alg):
    # test_tucker.cpp:247-264: exact multilinear rank -> RE <= 1e-8 (AMM 1e-6)
    dims = [24, 24, 24]
    x = orc.gen_tucker_noise(dims, [4, 4, 4], 0.0, 27)
    kw = dict(rank=[4, 4, 4], seed=1)
    if alg == "alg4":
        kw.update(regime="optimal", t_samples=[576, 576, 576])
    if alg == "alg5":
        kw.update(t_samples=[576, 96, 16])
    cg, _ = _cfgs(lmra, orc, **kw)
    gpu = lmra.run_algorithm(alg, lmra.DenseTensor.from_flat(x, dims), cg)
    re = relative_error(x.reshape(dims, order="F"), gpu.core, gpu.factors)
    assert re <= (1e-6 if alg in ("alg4", "alg5") else 1e-8), re


@pytest.mark.parametrize("alg", ALGS)
def test_deterministic_reruns(gpu_ctx, lmra, alg):
    dims = [14, 12, 10]
    x = np.random.default_rng(41).standard_normal(int(np.prod(dims)))
    cfg = lmra.AlgoConfig(rank=[3, 3, 3], seed=99, regime="nearly_optimal")
    t = lmra.DenseTensor.from_flat(x, dims)
    a = lmra.run_algorithm(alg, t, cfg)
    b = lmra.run_algorithm(alg, t, cfg)
    assert np.array_equal(a.core, b.core)
    for fa, fb in zip(a.factors, b.factors):
        assert np.array_equal(fa, fb)


def test_config_validation(gpu_ctx, lmra):
    # test_tucker.cpp:430-446 and the resolve() checks (tucker.cpp:24-52)
    x = lmra.DenseTensor.from_flat(np.random.default_rng(45).standard_normal(64), [4, 4, 4])
    bad = [
        ("alg2", dict(rank=[2, 2, 2], order=[0, 0, 2])),
        ("alg1", dict(rank=[2, 2, 2], power=0)),
        ("alg1", dict(rank=[2, 2])),
        ("alg4", dict(rank=[2, 2, 2], alpha=1.5)),
        ("alg4", dict(rank=[2, 2, 2], t_samples=[1, 2])),
        ("alg5", dict(rank=[2, 2, 2], t_samples=[3, 0, 3])),
        ("alg4", dict(rank=[2, 2, 2], regime="nearly_optimal", regime_beta=1.5)),
        ("alg1", dict(rank=[0, 2, 2])),
    ]
    for alg, kw in bad:
        with pytest.raises(lmra.LmraInvalidArgument):
            lmra.run_algorithm(alg, x, lmra.AlgoConfig(**kw))
    with pytest.raises(lmra.LmraInvalidArgument):
        lmra.run_algorithm("alg3", x, lmra.AlgoConfig(rank=[2, 2, 2]))


def test_degenerate_shapes(gpu_ctx, lmra, orc):
    # test_tucker.cpp:461-482: rank above the unfolding rank limit, tiny modes
    dims = [40, 2, 2]
    x = orc.rng_normal(51, 0, 160)
    for alg in ALGS:
        kw = dict(rank=[10, 2, 2], seed=3, t_samples=[4, 80, 80])
        cg, co = _cfgs(lmra, orc, **kw)
        gpu = lmra.run_algorithm(alg, lmra.DenseTensor.from_flat(x, dims), cg)
        for q in gpu.factors:
            assert np.abs(q.T @ q - np.eye(q.shape[1])).max() <= 1e-10
        assert gpu.factors[0].shape == (40, 10)
        re = relative_error(x.reshape(dims, order="F"), gpu.core, gpu.factors)
        assert re <= 1.0 + 1e-12


def test_oversized_rank_clamped(gpu_ctx, lmra):
    x = lmra.DenseTensor.from_flat(np.random.default_rng(43).standard_normal(120), [6, 5, 4])
    d = lmra.run_algorithm("alg1", x, lmra.AlgoConfig(rank=[10, 10, 10]))
    assert list(d.core.shape) == [6, 5, 4]


@pytest.mark.parametrize("alg", ["alg1", "alg4"])
def test_split_orthonormalisation_path(gpu_ctx, lmra, orc, alg, monkeypatch):
    # LMRA_ORTH_SPLIT=1: the core contracted with each sketch's basis Q_C, the Jacobi rotations
    # U_R' applied to the small core at the end (opt-in path, lmra_b200.cpp)
    monkeypatch.setenv("LMRA_ORTH_SPLIT", "1")
    _split_case(lmra, orc, alg, [60, 50, 40])


@pytest.mark.parametrize("alg", ["alg1", "alg4"])
@pytest.mark.parametrize("cholqr", ["1", "0"])
def test_split_orthonormalisation_cholqr_basis(gpu_ctx, lmra, orc, alg, cholqr, monkeypatch):
    # the split form with a CholeskyQR basis (first mode > 768 rows) and with the Householder one
    monkeypatch.setenv("LMRA_ORTH_SPLIT", "1")
    monkeypatch.setenv("LMRA_ORTH_CHOLQR", cholqr)
    _split_case(lmra, orc, alg, [40, 50, 800])  # mode 2 (rank 4) is contracted first


def _split_case(lmra, orc, alg, dims):
    x = orc.gen_tucker_noise(dims, [6, 5, 4], 1e-2, 13)
    kw = dict(rank=[6, 5, 4], seed=3, power=2, regime="nearly_optimal", t_samples=[300, 300, 300])
    cg, co = _cfgs(lmra, orc, **kw)
    ref = orc.run(alg, x, dims, co)
    t = lmra.DenseTensor.from_flat(x, dims)
    gpu = lmra.run_algorithm(alg, t, cg, omega=ref.omega, samples=ref.samples if alg == "alg4" else None)
    compare(gpu, ref, x.reshape(dims, order="F"))


@pytest.mark.parametrize("dims,power", [([900, 30, 20], 1), ([1000, 40, 30], 2), ([800, 50, 20], 2)])
@pytest.mark.parametrize("alg", ["alg1", "alg2"])
def test_tall_sketch_factors_householder(gpu_ctx, lmra, orc, dims, power, alg):
    # sketches above 768 rows: the factor comes from the Householder path even where CholeskyQR
    # provides the split contraction's basis (CholeskyQR factors missed the contract on these:
    # gap-aware sines 1.9e-10 / 7.8e-10)
    rank = [5, 4, 3]
    x = orc.gen_tucker_noise(dims, rank, 1e-2, 21)
    kw = dict(rank=rank, seed=5, power=power)
    ref = orc.run(alg, x, dims, orc.AlgoConfig(**kw))
    out = compare(lmra.run_algorithm(alg, lmra.DenseTensor.from_flat(x, dims), lmra.AlgoConfig(**kw)), ref,
                  x.reshape(dims, order="F"))
    assert max(out["sines"]) <= 1e-12, out["sines"]


@pytest.mark.parametrize("alg", ["alg4", "alg5"])
@pytest.mark.parametrize("regime", ["uniform", "nearly_optimal"])
def test_power_on_sampled_columns_in_place(gpu_ctx, lmra, orc, alg, regime, monkeypatch):
    # the power scheme reading the sampled columns in place (Gather: C' = A_(0)(:, idx) diag(scale)
    # never materialised; used for large C' such as cfg5's mode 0) -- forced at small size
    monkeypatch.setenv("LMRA_FUSED_GATHER_MIN", "1")
    dims = [40, 30, 20]
    x = orc.gen_tucker_noise(dims, [5, 4, 3], 1e-2, 9)
    kw = dict(rank=[5, 4, 3], seed=7, regime=regime, power=2, t_samples=[300, 200, 150])
    cg, co = _cfgs(lmra, orc, **kw)
    ref = orc.run(alg, x, dims, co)
    t = lmra.DenseTensor.from_flat(x, dims)
    own = lmra.run_algorithm(alg, t, cg)
    check_own_draws(alg, own, ref, regime)
    gpu = lmra.run_algorithm(alg, t, cg, omega=ref.omega, samples=ref.samples)
    compare(gpu, ref, x.reshape(dims, order="F"))


def _cudart():
    import ctypes
    for name in ("libcudart.so.12", "libcudart.so"):
        try:
            return ctypes.CDLL(name)
        except OSError:
            continue
    pytest.skip("libcudart not loadable through ctypes")


def test_result_free_after_device_pointer_read(gpu_ctx, lmra, orc):
    """A result whose device pointers were handed out synchronises at free, so a copy the caller
    queued on a stream of its own still reads the run's core after the blocks go back to the
    pool and the next run reuses them (ResultBlocks reuse without stream order)."""
    import ctypes
    torch = _torch()
    rt = _cudart()
    dims, core = [40, 36, 32], [5, 5, 5]
    cfg = lmra.AlgoConfig(rank=list(core), seed=4)
    xa = orc.gen_tucker_noise(dims, core, 1e-2, 8)
    xb = orc.gen_tucker_noise(dims, core, 1e-2, 9)
    ra = lmra.run_raw("alg1", lmra.DenseTensor.from_flat(xa, dims), cfg, ctx=gpu_ctx)
    want = ra.to_host(with_trace=False).core.ravel(order="F").copy()
    dst = torch.zeros(want.size, dtype=torch.float64, device="cuda")
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        torch.cuda._sleep(50_000_000)  # the copy below starts well after free() returns
    rc = rt.cudaMemcpyAsync(ctypes.c_void_p(dst.data_ptr()), ctypes.c_void_p(ra.core_device_ptr()),
                            ctypes.c_size_t(want.size * 8), ctypes.c_int(3), ctypes.c_void_p(side.cuda_stream))
    assert rc == 0
    ra.free()
    rb = lmra.run_raw("alg1", lmra.DenseTensor.from_flat(xb, dims), cfg, ctx=gpu_ctx)
    other = rb.to_host(with_trace=False).core.ravel(order="F")
    side.synchronize()
    rb.free()
    assert not np.array_equal(other, want)
    assert np.array_equal(dst.cpu().numpy(), want)

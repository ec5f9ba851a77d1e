"""The mode-0 contraction on the int8 tensor cores (ttm_i8.cu) against an fp64 reference.

Exact digit products with int32 accumulation: the error comes only from the 46-bit fixed-point
representation and the dropped low-order digit products (< 2^-44 relative per term), so the
result agrees with fp64 GEMM to ~1e-13 relative to |q| |x_j| (tolerance here 1e-12)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _run(K, J, mu, x=None, q=None, seed=0):
    import torch
    from paper_2303_11612_b200 import device
    rng = np.random.default_rng(seed)
    if x is None:
        x = rng.standard_normal((J, K))  # row j = column j of the K x J mode-0 view
    if q is None:
        q = np.linalg.qr(rng.standard_normal((K, mu)))[0] if mu <= K else rng.standard_normal((K, mu))
    xd = torch.from_numpy(np.ascontiguousarray(x).ravel()).cuda()
    qd = torch.from_numpy(np.asfortranarray(q).ravel(order="F")).cuda()
    w = device.column_sqnorms(xd, [K, J], 0)
    y = device.mode0_product_i8(xd, K, J, qd, mu, w).cpu().numpy().reshape((J, mu)).T  # mu x J
    ref = q.T @ x.T
    scale = np.linalg.norm(q, axis=0)[:, None] * np.linalg.norm(x, axis=1)[None, :]
    err = np.abs(y - ref) / np.maximum(scale, 1e-300)
    return float(err.max()), y, ref


@pytest.mark.parametrize("K,J,mu", [(1000, 4096, 50), (64, 1000, 8), (512, 300, 40), (2, 129, 1),
                                    (998, 777, 56), (4096, 256, 64), (256, 128, 17), (32, 5, 3)])
def test_ttm_i8_matches_fp64(K, J, mu):
    err, _, _ = _run(K, J, mu)
    assert err <= 1e-12, err


def test_ttm_i8_dynamic_range_and_zero_columns():
    K, J, mu = 200, 300, 24
    rng = np.random.default_rng(5)
    x = rng.standard_normal((J, K)) * (10.0 ** rng.uniform(-150, 150, size=(J, 1)))
    x[7] = 0.0
    x[11, :] = 0.0
    x[11, 3] = 2.0 ** 60  # single spike
    err, y, _ = _run(K, J, mu, x=x)
    assert err <= 1e-12, err
    assert np.all(y[:, 7] == 0.0)


def test_ttm_i8_rejects_unsupported():
    from paper_2303_11612_b200 import LmraInvalidArgument
    with pytest.raises(LmraInvalidArgument):
        _run(999, 10, 4)  # odd K (TMA row stride)
    with pytest.raises(LmraInvalidArgument):
        _run(100, 10, 70)  # mu > 64


# ---------------------------------------------------------------- mode-1 (inner) form
def _run_inner(R, K, O, mu, x=None, seed=0):
    """x: (O, K, R) array = X(r, k, o) at r + R (k + K o); returns max error relative to
    |q_m| |x_(r, o)| and the result (O, mu, R)."""
    from paper_2303_11612_b200 import device
    import torch
    rng = np.random.default_rng(seed)
    if x is None:
        x = rng.standard_normal((O, K, R))
    q = np.linalg.qr(rng.standard_normal((K, mu)))[0] if mu <= K else rng.standard_normal((K, mu))
    xd = torch.from_numpy(np.ascontiguousarray(x).ravel()).cuda()
    qd = torch.from_numpy(np.asfortranarray(q).ravel(order="F")).cuda()
    y = device.mode1_product_i8(xd, R, K, O, qd, mu).cpu().numpy().reshape((O, mu, R))
    ref = np.einsum("okr,km->omr", x, q)
    scale = np.linalg.norm(q, axis=0)[None, :, None] * np.linalg.norm(x, axis=1)[:, None, :]
    err = np.abs(y - ref) / np.maximum(scale, 1e-300)
    return float(err.max()), y, ref


@pytest.mark.parametrize("R,K,O,mu", [(50, 1000, 37, 50), (40, 512, 7, 40), (2, 64, 5, 3), (64, 4096, 3, 64),
                                      (10, 100, 33, 17), (6, 1, 9, 4), (50, 333, 1, 16)])
def test_ttm_i8_inner_matches_fp64(R, K, O, mu):
    err, _, _ = _run_inner(R, K, O, mu)
    assert err <= 1e-12, err


def test_ttm_i8_inner_dynamic_range_and_zero_columns():
    R, K, O, mu = 24, 200, 11, 20
    rng = np.random.default_rng(9)
    x = rng.standard_normal((O, K, R)) * (10.0 ** rng.uniform(-150, 150, size=(O, 1, R)))
    x[3, :, 5] = 0.0
    x[4, :, 7] = 0.0
    x[4, 17, 7] = -(2.0 ** 70)  # single spike
    err, y, _ = _run_inner(R, K, O, mu, x=x)
    assert err <= 1e-12, err
    assert np.all(y[3, :, 5] == 0.0)


def test_ttm_i8_inner_rejects_unsupported():
    from paper_2303_11612_b200 import LmraInvalidArgument
    with pytest.raises(LmraInvalidArgument):
        _run_inner(7, 10, 3, 4)  # odd R (TMA row stride)
    with pytest.raises(LmraInvalidArgument):
        _run_inner(66, 10, 3, 4)  # R > 64


def test_core_chain_uses_int8_mode1_and_matches_fp64():
    """alg4 with even ranks: the core's first two contractions run on the int8 tensor cores
    (the second taking its scales from the first's exponents); the core matches an fp64
    evaluation of the same factors far inside the parity tolerance."""
    import torch
    import paper_2303_11612_b200 as P
    rng = np.random.default_rng(2)
    dims = [64, 48, 40]
    x = rng.standard_normal(int(np.prod(dims)))  # column-major flat (i0 fastest)
    # ascending widths: core_from_factors contracts in ascending width order (stable), so mode 0
    # (int8, canonical norms) comes first and mode 1 (int8, exponents handed over) second
    cfg = P.AlgoConfig(rank=[4, 6, 8], oversampling=4, power=1, regime="nearly_optimal",
                       t_samples=[60, 60, 60], seed=4)
    ctx = P.Context(0, torch.cuda.current_stream().cuda_stream)
    ctx.set_profiling(1)
    r = P.run_raw("alg4", P.DenseTensor.device(torch.from_numpy(x).cuda(), dims), cfg, ctx=ctx)
    names = set(r.phases().keys())
    d = r.to_host(with_trace=False)
    r.free()
    assert "core_ttm0_i8" in names and "core_ttm1_i8" in names, names
    core = x.reshape(dims[::-1]).transpose(2, 1, 0)  # [i0, i1, i2]
    for n, U in enumerate(d.factors):
        core = np.moveaxis(np.tensordot(U.T, np.moveaxis(core, n, 0), axes=1), 0, n)
    got = np.asarray(d.core).reshape(core.shape)
    rel = np.linalg.norm(got - core) / np.linalg.norm(core)
    assert rel <= 1e-12, rel

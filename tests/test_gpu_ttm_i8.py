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

"""The deterministic baselines t_hosvd / st_hosvd / hooi (tucker.cpp:242-316) on the device
against the oracle's restatement, and the in-process multi-GPU entry point.

Factors come from the FULL unfoldings (QR of A_(n)^T + SVD of R on the device).  Parity
contract as for the randomized family (test_gpu_parity.compare): gap-aware factor sines and
core / RE within 1e-10 -- the "sketch" whose spectrum defines the gaps is the unfolding itself.
HOOI is compared at a fixed number of sweeps (hooi_tol = 0): its stopping sweep depends on a
1e-8-level test that two valid fp64 evaluations may cross one sweep apart.
"""
import numpy as np
import pytest

from conftest import relative_error
from test_gpu_parity import compare

pytestmark = pytest.mark.gpu

SHAPES = [([20, 18, 16], [4, 5, 3]), ([12, 10, 8, 6], [3, 3, 2, 2]), ([40, 2, 2], [10, 2, 2]),
          ([70, 65, 3], [8, 6, 3]), ([130, 40, 30], [9, 7, 5])]


@pytest.mark.parametrize("alg", ["thosvd", "sthosvd"])
@pytest.mark.parametrize("shape", range(len(SHAPES)))
def test_deterministic_matches_oracle(gpu_ctx, lmra, orc, alg, shape):
    dims, core = SHAPES[shape]
    x = orc.gen_tucker_noise(dims, [min(c, d) for c, d in zip(core, dims)], 1e-2, 3 + shape)
    kw = dict(rank=core, seed=1)
    ref = orc.run(alg, x, dims, orc.AlgoConfig(**kw))
    gpu = lmra.run_algorithm(alg, lmra.DenseTensor.from_flat(x, dims), lmra.AlgoConfig(**kw))
    m = compare(gpu, ref, x.reshape(dims, order="F"))
    print(alg, dims, m)


@pytest.mark.parametrize("order", [None, [2, 0, 1]])
def test_hooi_fixed_sweeps_matches_oracle(gpu_ctx, lmra, orc, order):
    dims = [24, 20, 16]
    x = orc.gen_tucker_noise(dims, [5, 4, 3], 5e-2, 11)
    kw = dict(rank=[4, 4, 3], seed=1, order=order, hooi_max_sweeps=3, hooi_tol=0.0)
    ref = orc.run("hooi", x, dims, orc.AlgoConfig(**kw))
    gpu = lmra.run_algorithm("hooi", lmra.DenseTensor.from_flat(x, dims), lmra.AlgoConfig(**kw))
    compare(gpu, ref, x.reshape(dims, order="F"))


def test_hooi_improves_on_sthosvd_and_converges(gpu_ctx, lmra, orc):
    # tucker.cpp:261-316: HOOI starts from st_hosvd and does not increase the error; on a
    # tensor of exact multilinear rank it converges in a sweep or two
    dims = [30, 26, 22]
    x = orc.gen_tucker_noise(dims, [4, 4, 4], 1e-1, 21)
    a = x.reshape(dims, order="F")
    cfg = lmra.AlgoConfig(rank=[4, 4, 4], seed=1)
    st = lmra.st_hosvd(lmra.DenseTensor.from_flat(x, dims), cfg)
    ho = lmra.hooi(lmra.DenseTensor.from_flat(x, dims), cfg)
    assert relative_error(a, ho.core, ho.factors) <= relative_error(a, st.core, st.factors) + 1e-12
    exact = orc.gen_tucker_noise(dims, [3, 3, 3], 0.0, 22)
    r = lmra.run_raw("hooi", lmra.DenseTensor.from_flat(exact, dims), lmra.AlgoConfig(rank=[3, 3, 3]))
    import ctypes as C
    conv, sweeps = C.c_int(), C.c_int()
    lmra._lib.lib.lmra_result_hooi_stats(r.handle, C.byref(conv), C.byref(sweeps))
    dec = r.to_host()
    r.free()
    assert conv.value == 1 and 1 <= sweeps.value <= 3, (conv.value, sweeps.value)
    assert relative_error(exact.reshape(dims, order="F"), dec.core, dec.factors) <= 1e-12


def test_deterministic_errors(gpu_ctx, lmra):
    x = lmra.DenseTensor.from_flat(np.random.default_rng(1).standard_normal(64), [4, 4, 4])
    for alg in ("thosvd", "sthosvd", "hooi"):
        with pytest.raises(lmra.LmraInvalidArgument):
            lmra.run_algorithm(alg, x, lmra.AlgoConfig(rank=[2, 2]))
        with pytest.raises(lmra.LmraInvalidArgument):
            lmra.run_algorithm(alg, x, lmra.AlgoConfig(rank=[2, 0, 2]))
    d = lmra.t_hosvd(x, lmra.AlgoConfig(rank=[9, 9, 9]))  # clamped to the dims (tucker.cpp:174-188)
    assert list(d.core.shape) == [4, 4, 4]


@pytest.mark.parametrize("alg", ["alg1", "alg4", "alg5"])
def test_multigpu_entry_point(gpu_ctx, lmra, orc, alg):
    # lmra_run_algorithm_multigpu: ranks as host threads with a context each; with the one GPU
    # the pool gives, two ranks share device 0 (the in-process communicator)
    import torch
    dims = [30, 24, 40]
    x = orc.gen_tucker_noise(dims, [4, 4, 4], 1e-2, 5)
    kw = dict(rank=[4, 4, 4], seed=2, regime="nearly_optimal", t_samples=[200, 200, 200])
    cfg = lmra.AlgoConfig(**kw)
    ref = orc.run(alg, x, dims, orc.AlgoConfig(**kw))
    r = lmra.run_raw_multigpu(alg, lmra.DenseTensor.from_flat(x, dims), cfg, [0, 0])
    host = r.to_host()
    r.free()
    compare(host, ref, x.reshape(dims, order="F"))
    # device input on devices[0]
    xd = torch.from_numpy(x).cuda()
    r = lmra.run_raw_multigpu(alg, lmra.DenseTensor.device(xd, dims), cfg, [0, 0, 0])
    dev = r.to_host()
    r.free()
    compare(dev, ref, x.reshape(dims, order="F"))

"""Sharded (multi-GPU) path: the tensor split along its last mode across P
ranks, every collective through the context's communicator.

The GPU pool gives one B200, so the P ranks run as host threads of this process, each with
its own lmra context and stream, exchanging through the in-process ThreadComm (device
copies + host barriers; no kernel waits on another rank).  The sharded orchestration --
slab views, norm all-gather, index localisation, Gram / half-product all-reduces, row
all-gather, partial-core all-reduce -- is the same code the NCCL communicator drives.

Checks: (1) all ranks return bitwise-identical factors and core; (2) against the oracle on
the whole tensor with the parity tolerances of test_gpu_parity (for AMM runs the oracle's
own draws are passed in, so the comparison isolates the sharded arithmetic); (3) without
overrides, the draws are bit-exact with the oracle's: modes < N-1 always (their norms are
computed locally in the canonical order and all-gathered), the sharded mode N-1 whenever the
slabs are segment-aligned (last extent >= 64 P: each rank's canonical-norm segments are
all-gathered and added in global order), and every mode in the uniform regime.
"""
import threading

import numpy as np
import pytest

from test_gpu_parity import compare

pytestmark = pytest.mark.gpu


def run_sharded(alg, a_flat, dims, cfg, P, samples=None, timeout=120):
    import torch
    from paper_2303_11612_b200 import Context, DenseTensor, ThreadGroup, run_algorithm, shard_range

    group = ThreadGroup(P)
    out, err = [None] * P, [None] * P
    per = int(np.prod(dims[:-1]))

    def worker(r):
        ctx = None
        try:
            ctx = Context(0)
            ctx.set_thread_comm(group, r)
            s0, c0 = shard_range(dims[-1], P, r)
            slab = torch.from_numpy(np.ascontiguousarray(a_flat[per * s0: per * (s0 + c0)])).cuda()
            torch.cuda.synchronize()
            x = DenseTensor.device(slab, list(dims[:-1]) + [c0])
            out[r] = run_algorithm(alg, x, cfg, ctx=ctx, samples=samples, global_dims=list(dims))
        except Exception as e:  # noqa: BLE001 -- re-raised on the main thread
            err[r] = e
        finally:
            if ctx is not None:
                ctx.close()

    threads = [threading.Thread(target=worker, args=(r,), daemon=True) for r in range(P)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout)
        assert not t.is_alive(), "sharded run did not finish (collective mismatch?)"
    for e in err:
        if e is not None:
            raise e
    return out


def assert_ranks_identical(outs):
    for r in range(1, len(outs)):
        assert np.array_equal(outs[r].core, outs[0].core), f"rank {r} core differs"
        for n, (a, b) in enumerate(zip(outs[r].factors, outs[0].factors)):
            assert np.array_equal(a, b), f"rank {r} factor {n} differs"


# alpha = 0.5: later ST-HOSVD modes sample a shrunk tensor with few columns (mu_0 mu_1 = 20
# for the last mode of the 3-way cases); alpha 0.2 would draw fewer columns than mu_{N-1}
# and leave the trailing factor columns undetermined by the sketch (rank-deficient C').
def _tensor(orc, dims, seed=3):
    core = tuple(max(1, min(d // 3, 6)) for d in dims)
    return orc.gen_tucker_noise(dims, core, 1e-3, seed)


CASES = [
    # (alg, dims, rank, P, regime)
    ("alg1", (30, 26, 40), (5, 5, 5), 2, "uniform"),
    ("alg1", (30, 26, 37), (5, 4, 6), 4, "uniform"),
    ("alg2", (30, 26, 40), (5, 5, 5), 3, "uniform"),
    ("alg4", (40, 36, 48), (5, 5, 5), 2, "nearly_optimal"),
    ("alg4", (40, 36, 45), (5, 6, 4), 4, "optimal"),
    ("alg4", (12, 10, 9, 14), (3, 3, 3, 3), 3, "nearly_optimal"),
    ("alg5", (40, 36, 48), (5, 5, 5), 2, "nearly_optimal"),
    ("alg5", (40, 36, 47), (4, 5, 6), 4, "optimal"),
    # segment-aligned slabs (last extent >= 64 P): the sharded mode's norms are exact too
    ("alg4", (20, 18, 130), (4, 4, 5), 2, "nearly_optimal"),
    ("alg4", (12, 10, 300), (3, 3, 5), 4, "optimal"),
    ("alg4", (8, 6, 5, 200), (3, 3, 3, 4), 3, "nearly_optimal"),
    ("alg5", (16, 14, 200), (4, 4, 4), 3, "nearly_optimal"),
]


@pytest.mark.parametrize("alg,dims,rank,P,regime", CASES)
def test_sharded_matches_oracle(orc, alg, dims, rank, P, regime):
    a = _tensor(orc, dims)
    ocfg = orc.AlgoConfig(rank=list(rank), oversampling=6, power=1, regime=regime, seed=11,
                          alpha=0.5)
    ref = orc.run(alg, a, dims, ocfg)
    from paper_2303_11612_b200 import AlgoConfig
    cfg = AlgoConfig(rank=list(rank), oversampling=6, power=1, regime=regime, seed=11,
                          alpha=0.5)
    amm = alg in ("alg4", "alg5")
    samples = ref.samples if amm else None
    outs = run_sharded(alg, a, dims, cfg, P, samples=samples)
    assert_ranks_identical(outs)
    compare(outs[0], ref, a.reshape(dims, order="F"))


@pytest.mark.parametrize("alg,dims,rank,P,regime", [c for c in CASES if c[0] in ("alg4", "alg5")])
def test_sharded_own_draws(orc, alg, dims, rank, P, regime):
    """No overrides: the sharded run's own sampling chain against the oracle's draws.

    Indices must agree on every mode.  Scales are bit-exact where the norms are exact:
    T-HOSVD modes < N-1 (local canonical norms, all-gathered), the sharded mode N-1 when the
    slabs are segment-aligned, and the first ST-HOSVD mode.  Unaligned slabs' mode N-1 norms
    are rank partials added in rank order, and later ST-HOSVD modes see a shrunk tensor with
    its own rounding: 1e-13 relative."""
    a = _tensor(orc, dims, seed=5)
    ocfg = orc.AlgoConfig(rank=list(rank), oversampling=6, power=1, regime=regime, seed=2,
                          alpha=0.5)
    ref = orc.run(alg, a, dims, ocfg)
    from paper_2303_11612_b200 import AlgoConfig
    cfg = AlgoConfig(rank=list(rank), oversampling=6, power=1, regime=regime, seed=2,
                          alpha=0.5)
    outs = run_sharded(alg, a, dims, cfg, P)
    assert_ranks_identical(outs)
    N = len(dims)
    own = outs[0]
    for n in range(N):
        assert np.array_equal(own.omega[n], ref.omega[n]), f"Omega mode {n}"
        gi, gs = own.samples[n]
        oi, os_ = ref.samples[n]
        assert np.array_equal(gi, oi), f"mode {n}: sharded draws differ from the oracle's"
        aligned = dims[-1] >= 64 * P
        exact = (n < N - 1 or aligned) if alg == "alg4" else n == 0
        if exact:
            assert np.array_equal(gs, os_), f"mode {n}: scales"
        else:
            d = np.abs(gs / os_ - 1).max()
            assert d <= 1e-13, f"mode {n}: scales {d:.3g}"
    compare(own, ref, a.reshape(dims, order="F"))


@pytest.mark.parametrize("alg", ["alg4", "alg5"])
def test_sharded_uniform_bit_exact_draws(orc, alg):
    dims, rank, P = (24, 20, 30), (4, 4, 4), 3
    a = _tensor(orc, dims, seed=9)
    ocfg = orc.AlgoConfig(rank=list(rank), oversampling=5, power=2, regime="uniform", seed=4,
                          alpha=0.5)
    ref = orc.run(alg, a, dims, ocfg)
    from paper_2303_11612_b200 import AlgoConfig
    cfg = AlgoConfig(rank=list(rank), oversampling=5, power=2, regime="uniform", seed=4,
                          alpha=0.5)
    outs = run_sharded(alg, a, dims, cfg, P)
    assert_ranks_identical(outs)
    for n in range(len(dims)):
        assert np.array_equal(outs[0].samples[n][0], ref.samples[n][0]), n
    compare(outs[0], ref, a.reshape(dims, order="F"))


def test_sharded_single_rank_group_matches_unsharded(orc, gpu_ctx):
    """P = 1 through the communicator plumbing is the plain single-GPU run."""
    from paper_2303_11612_b200 import AlgoConfig, run_algorithm
    dims = (20, 18, 16)
    a = _tensor(orc, dims)
    cfg = AlgoConfig(rank=[4, 4, 4], oversampling=5, power=1, regime="nearly_optimal", seed=1)
    (one,) = run_sharded("alg4", a, dims, cfg, 1)
    plain = run_algorithm("alg4", a.reshape(dims, order="F"), cfg, ctx=gpu_ctx)
    np.testing.assert_array_equal(one.core, plain.core)


def test_sharded_rejects_too_many_ranks(orc):
    from paper_2303_11612_b200 import AlgoConfig, LmraInvalidArgument
    dims = (6, 5, 3)
    a = _tensor(orc, dims)
    cfg = AlgoConfig(rank=[2, 2, 2], oversampling=2)
    with pytest.raises(LmraInvalidArgument):
        run_sharded("alg1", a, dims, cfg, 4)

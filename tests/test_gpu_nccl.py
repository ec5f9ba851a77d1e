"""The sharded path over the NCCL communicator (NcclComm, lmra_context_set_comm): one process per
GPU, the tensor split along its last mode, every collective through NCCL -- the code path
`bench.py --gpus N` drives.  Needs >= 2 visible GPUs (the pool's boxes give one; the in-process
ThreadComm tests in test_gpu_sharded.py cover the same orchestration rank for rank there).

Checks: both ranks return bitwise-identical factors and core; the draws equal the oracle's
(segment-aligned slabs: every mode bit-exact); factors / core / RE within the parity
tolerances of the oracle on the whole tensor.
"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, alg, dims, rank_, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)  # plumbing for the NCCL id only
    try:
        import paper_2303_11612_b200 as P
        from oracle import oracle as orc
        x = orc.gen_tucker_noise(list(dims), [3] * len(dims), 1e-2, 5)
        uid = [P.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        ctx = P.Context(rank)
        ctx.set_comm(uid[0], world, rank)
        per = int(np.prod(dims[:-1]))
        s0, c0 = P.shard_range(dims[-1], world, rank)
        slab = torch.from_numpy(np.ascontiguousarray(x[per * s0: per * (s0 + c0)])).cuda(rank)
        torch.cuda.synchronize()
        cfg = P.AlgoConfig(rank=list(rank_), oversampling=4, power=2, regime="nearly_optimal",
                           t_samples=[200] * len(dims), seed=11)
        d = P.run_algorithm(alg, P.DenseTensor.device(slab, list(dims[:-1]) + [c0]), cfg, ctx=ctx,
                            global_dims=list(dims))
        q.put((rank, d.core, d.factors, d.samples, d.omega))
        ctx.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(600)
@pytest.mark.parametrize("alg", ["alg4", "alg5"])
def test_nccl_two_ranks(orc, alg):
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("NCCL sharded test needs >= 2 GPUs (one visible)")
    import torch.multiprocessing as mp
    from test_gpu_parity import check_own_draws, compare
    dims, rank_ = (24, 20, 130), (4, 4, 5)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, alg, dims, rank_, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=500) for _ in procs], key=lambda t: t[0])
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    (_, c0, f0, s0, o0), (_, c1, f1, _, _) = res
    assert np.array_equal(c0, c1)
    assert all(np.array_equal(a, b) for a, b in zip(f0, f1))
    x = orc.gen_tucker_noise(list(dims), [3] * len(dims), 1e-2, 5)
    co = orc.AlgoConfig(rank=list(rank_), oversampling=4, power=2, regime="nearly_optimal",
                        t_samples=[200] * len(dims), seed=11)
    ref = orc.run(alg, x, list(dims), co)

    class _D:  # the rank-0 decomposition in the shape compare() reads
        core, factors, samples, omega = c0, f0, s0, o0
    check_own_draws(alg, _D, ref, "nearly_optimal")
    compare(_D, ref, x.reshape(dims, order="F"))

"""Host-side check of the sharded plan on CPU: world_size 2 over gloo.

Each rank holds the slab of the last mode that lmra_shard_range assigns it and replays the
exchange steps run_sharded_impl performs (lmra_b200.cpp) in numpy, with gloo standing in
for NCCL: column-norm all-gather (modes < N-1), index localisation with zero columns for
other ranks' fibres, Gram-partial all-reduce (power scheme), half-product all-reduce + row
all-gather (mode N-1), and the partial-core all-reduce of the sharded contraction.  Every
step must reproduce the unsharded computation.
"""
import os
import socket

import numpy as np
import pytest


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _unfold(x, n):
    # reference unfolding order (tensor.cpp:60-86): column j = (i_<n, i_>n), first fastest
    return np.moveaxis(x, n, 0).reshape(x.shape[n], -1, order="F")


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2303_11612_b200 import shard_range
        rng = np.random.default_rng(0)
        dims = (7, 6, 11)
        x = rng.standard_normal(dims)
        L = dims[-1]
        s0, c0 = shard_range(L, world, rank)
        slab = x[..., s0:s0 + c0]
        shards = [shard_range(L, world, r) for r in range(world)]
        cmax = max(c for _, c in shards)

        def allreduce(a):
            t = torch.from_numpy(np.ascontiguousarray(a))
            dist.all_reduce(t)
            return t.numpy()

        def allgather(a):
            t = torch.from_numpy(np.ascontiguousarray(a))
            out = [torch.empty_like(t) for _ in range(world)]
            dist.all_gather(out, t)
            return [o.numpy() for o in out]

        s, T, power = 4, 9, 2
        errs = {}
        # ---- mode 0: columns split (j = i_1 + I_1 * i_2; slab owns i_2 in [s0, s0 + c0))
        A = _unfold(x, 0)
        per = dims[1]
        wl = np.zeros(per * cmax)
        wl[: per * c0] = (_unfold(slab, 0) ** 2).sum(axis=0)
        parts = allgather(wl)
        w = np.concatenate([parts[r][: per * c] for r, (_, c) in enumerate(shards)])
        errs["norms_mode0"] = np.abs(w - (A ** 2).sum(axis=0)).max()
        idx = np.random.default_rng(1).integers(0, A.shape[1], T)
        sc = np.random.default_rng(2).random(T) + 0.5
        loc = idx - per * s0
        loc = np.where((loc >= 0) & (loc < per * c0), loc, -1)
        Al = _unfold(slab, 0)
        Cl = np.where(loc >= 0, Al[:, np.maximum(loc, 0)], 0.0) * sc
        c = np.random.default_rng(3).standard_normal((dims[0], s))
        cf = c.copy()
        Cf = A[:, idx] * sc
        for _ in range(power):
            c = allreduce(Cl @ (Cl.T @ c))
            cf = Cf @ (Cf.T @ cf)
        errs["power_mode0"] = np.abs(c - cf).max() / np.abs(cf).max()
        # ---- mode N-1: rows split
        A2 = _unfold(x, 2)
        w2 = allreduce((_unfold(slab, 2) ** 2).sum(axis=0))
        errs["norms_mode2"] = np.abs(w2 - (A2 ** 2).sum(axis=0)).max() / w2.max()
        idx2 = np.random.default_rng(4).integers(0, A2.shape[1], T)
        C2l = _unfold(slab, 2)[:, idx2] * sc
        c2 = np.random.default_rng(5).standard_normal((L, s))
        c2f = c2.copy()
        cr = c2[s0:s0 + c0]
        C2f = A2[:, idx2] * sc
        for _ in range(power):
            h = allreduce(C2l.T @ cr)
            cr = C2l @ h
            c2f = C2f @ (C2f.T @ c2f)
        pad = np.zeros((cmax, s))
        pad[:c0] = cr
        rows = allgather(pad)
        c2 = np.concatenate([rows[r][:cnt] for r, (_, cnt) in enumerate(shards)])
        errs["power_mode2"] = np.abs(c2 - c2f).max() / np.abs(c2f).max()
        # ---- contraction of the sharded mode: local partial + all-reduce
        Q = np.linalg.qr(c2f)[0]
        part = np.tensordot(slab, Q[s0:s0 + c0], axes=([2], [0]))
        full = np.tensordot(x, Q, axes=([2], [0]))
        errs["contract_mode2"] = np.abs(allreduce(part) - full).max() / np.abs(full).max()
        q.put((rank, errs, (s0, c0)))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_shard_plan_world2_gloo():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    ranges = sorted(r[2] for r in results)
    assert ranges == [(0, 5), (5, 6)]  # floor(L*r/P) split of L = 11
    for rank, errs, _ in results:
        for k, v in errs.items():
            assert v <= 1e-13, (rank, k, v)


def test_shard_plan_is_segment_aligned(lmra):
    # lmra_shard_range: contiguous covering slabs, balanced in units of 64 rows when L >= 64 P
    for L, P in [(1000, 8), (1000, 2), (512, 8), (130, 2), (47, 4), (63, 1), (4096, 7)]:
        spans = [lmra.shard_range(L, P, r) for r in range(P)]
        assert spans[0][0] == 0 and sum(c for _, c in spans) == L
        for (s0, c0), (s1, _) in zip(spans, spans[1:]):
            assert s0 + c0 == s1
        if L >= 64 * P:
            assert all(s0 % 64 == 0 for s0, _ in spans)
            assert max(c for _, c in spans) - min(c for _, c in spans) <= 64


def _segments_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as orc
        from paper_2303_11612_b200 import shard_range
        dims = [5, 4, 300]
        x = orc.gen_tucker_noise(dims, [3, 3, 4], 1e-2, 7)
        slab_n = dims[0] * dims[1]
        s0, c0 = shard_range(dims[2], world, rank)
        slab = x[slab_n * s0: slab_n * (s0 + c0)]
        # this rank's canonical-norm segments of every mode-2 column: 64 rows each (a 64-row
        # fibre's canonical norm is exactly its segment sum)
        segs = []
        for r0 in range(0, c0, 64):
            n = min(64, c0 - r0)
            segs.append(orc.column_sqnorms(slab[slab_n * r0: slab_n * (r0 + n)], [dims[0], dims[1], n], 2))
        mine = np.stack(segs)
        got = [None] * world
        dist.all_gather_object(got, mine)
        total = np.zeros(slab_n)
        for g in got:  # global segment order = rank order, then local order
            for row in g:
                total = total + row
        want = orc.column_sqnorms(x, dims, 2)
        q.put((rank, bool(np.array_equal(total, want)), (s0, c0)))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_sharded_canonical_norms_world2_gloo():
    """The sharded mode's norms (run_sharded_impl, segment-aligned slabs): each rank's
    segment sums all-gathered and added in global order give the unsharded canonical bits."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_segments_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    assert sorted(r[2] for r in results) == [(0, 128), (128, 172)]
    assert all(r[1] for r in results)

"""TNSR tensor files (tensor_io.hpp:9-13, tensor_io.cpp:27-69) through the C ABI.

CPU: byte layout against an independent struct-packed encoding, bit-exact round trips,
the reference's error messages (test_tensor_io.cpp's cases: bad magic, truncation, version).
GPU: straight-to-HBM loads (chunked pinned staging) and device saves, bit-exact.
"""
import os
import struct

import numpy as np
import pytest


def _encode(dims, values):
    head = b"TNSR" + struct.pack("<II", 1, len(dims)) + struct.pack(f"<{len(dims)}Q", *dims)
    return head + np.asarray(values, dtype="<f8").tobytes()


def test_save_layout_and_round_trip(lmra, tmp_path):
    dims = [3, 4, 5]
    vals = np.random.default_rng(3).standard_normal(60)
    vals[7] = -0.0
    vals[8] = np.inf
    vals[9] = 5e-324
    p = str(tmp_path / "t.tnsr")
    lmra.save_tensor(p, lmra.DenseTensor.from_flat(vals, dims))
    assert open(p, "rb").read() == _encode(dims, vals)
    t = lmra.load_tensor(p)
    assert t.dims == dims
    assert t.data.tobytes() == vals.tobytes()


def test_reads_independently_written_file(lmra, tmp_path):
    dims = [2, 1, 3, 2]
    vals = np.arange(12, dtype=np.float64) / 7.0
    p = tmp_path / "x.tnsr"
    p.write_bytes(_encode(dims, vals))
    t = lmra.load_tensor(str(p))
    assert t.dims == dims and np.array_equal(t.data, vals)


def test_order_zero_and_empty_extent(lmra, tmp_path):
    p = tmp_path / "s.tnsr"
    p.write_bytes(_encode([], [2.5]))  # order 0: one value (the empty product)
    t = lmra.load_tensor(str(p))
    assert t.dims == [] and t.data.tolist() == [2.5]
    p.write_bytes(_encode([4, 0], []))
    assert lmra.load_tensor(str(p)).dims == [4, 0]


@pytest.mark.parametrize("mutate,msg", [
    (lambda b: b"TNSX" + b[4:], "bad magic in tensor file"),
    (lambda b: b[:4] + struct.pack("<I", 2) + b[8:], "unsupported tensor file version 2"),
    (lambda b: b[:-8], "tensor file truncated while reading values"),
    (lambda b: b[:14], "tensor file truncated while reading dimensions"),
    (lambda b: b[:2], "tensor file truncated while reading magic"),
])
def test_reference_errors(lmra, tmp_path, mutate, msg):
    p = tmp_path / "bad.tnsr"
    p.write_bytes(mutate(_encode([2, 3], np.ones(6))))
    with pytest.raises(lmra.LmraError, match=msg):
        lmra.load_tensor(str(p))


def test_missing_file(lmra, tmp_path):
    with pytest.raises(lmra.LmraError, match="cannot open tensor file"):
        lmra.load_tensor(str(tmp_path / "nope.tnsr"))


@pytest.mark.gpu
def test_device_load_and_save(gpu_ctx, lmra, tmp_path):
    import torch
    dims = [70, 50, 41]
    vals = np.random.default_rng(5).standard_normal(int(np.prod(dims)))
    p = str(tmp_path / "d.tnsr")
    open(p, "wb").write(_encode(dims, vals))
    t = lmra.load_tensor(p, device=True, ctx=gpu_ctx)
    assert t.on_device and t.dims == dims
    assert t.owner.cpu().numpy().tobytes() == vals.tobytes()
    q = str(tmp_path / "e.tnsr")
    lmra.save_tensor(q, t, ctx=gpu_ctx)
    assert open(q, "rb").read() == open(p, "rb").read()
    # > 2 staging chunks (64 MB each): 160 MB
    big = torch.arange(20_000_000, dtype=torch.float64, device="cuda") * 0.5
    bt = lmra.DenseTensor.device(big, [20_000_000])
    r = str(tmp_path / "big.tnsr")
    lmra.save_tensor(r, bt, ctx=gpu_ctx)
    assert os.path.getsize(r) == 12 + 8 + 8 * 20_000_000
    back = lmra.load_tensor(r, device=True, ctx=gpu_ctx)
    assert torch.equal(back.owner, big)

"""The BASELINE input generators: device (gen.cu) == host (oracle) bit for bit.

Both evaluate the definitions of paper_2303_11612_b200/csrc/gen/portable_gen.hpp with
explicit IEEE operations in fixed orders (no libm / CUDA transcendental functions), so the
CPU arm of bench.py and the oracle side of every parity test see exactly the tensor the
GPU decomposes, and a multi-GPU rank can generate its slab of the last mode alone.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _host(orc, bc):
    from baseline_configs import generate_host
    return generate_host(bc)


def _same(xd, xh):
    import torch
    xt = torch.from_numpy(xh).to(xd.device)
    # bitwise: compare the int64 views (also distinguishes -0.0 / +0.0)
    return bool(torch.equal(xd.view(torch.int64), xt.view(torch.int64)))


CASES = [("cfg1", None), ("cfg2", None), ("cfg3", None), ("cfg4", [200, 200, 200]), ("cfg4", [64, 48, 40]),
         ("cfg5", [128, 128, 3, 128]), ("cfg5", None), ("cfg1", [7, 5, 3]), ("cfg3", [9, 8, 7, 6])]


@pytest.mark.parametrize("name,dims", CASES)
def test_device_generator_equals_host(gpu_ctx, orc, name, dims):
    from baseline_configs import CONFIGS, scaled
    from paper_2303_11612_b200.configs import generate_device
    bc = CONFIGS[name] if dims is None else scaled(name, dims)
    if bc.generator == "tucker_noise":  # small shapes keep the config's core where it fits
        bc.gen_args["core_dims"] = [min(c, d) for c, d in zip(bc.gen_args["core_dims"], bc.dims)]
    xd = generate_device(bc, ctx=gpu_ctx)
    xh = _host(orc, bc)
    assert xh.size == xd.numel()
    assert _same(xd, xh), (name, bc.dims, float(np.abs(xd.cpu().numpy() - xh).max()))


@pytest.mark.parametrize("name,dims,parts", [("cfg4", [60, 50, 41], 3), ("cfg5", [64, 40, 3, 37], 4),
                                             ("cfg2", [30, 20, 17], 5), ("cfg1", [20, 10, 8], 8)])
def test_slabs_compose_to_the_whole(gpu_ctx, lmra, name, dims, parts):
    import torch
    from paper_2303_11612_b200 import device
    from baseline_configs import scaled
    from paper_2303_11612_b200.configs import generate_device, generate_device_slab
    bc = scaled(name, dims)
    if bc.generator == "tucker_noise":
        bc.gen_args["core_dims"] = [min(c, d) for c, d in zip(bc.gen_args["core_dims"], bc.dims)]
    whole = generate_device(bc, ctx=gpu_ctx)
    L = dims[-1]
    ranges = [lmra.shard_range(L, parts, r) for r in range(parts)]
    if bc.generator == "tucker_noise":
        # two-step protocol: signal + per-slice sums on every slab, exchange, then the noise
        halves = [device.gen_tucker_signal_slab(bc.dims, bc.gen_args["core_dims"], bc.gen_args["seed"], s, c,
                                                ctx=gpu_ctx) for s, c in ranges]
        sb = np.concatenate([h[1] for h in halves])
        se = np.concatenate([h[2] for h in halves])
        coef = device.noise_coef(sb, se, bc.gen_args["gamma"])
        slabs = [device.gen_add_noise_slab(h[0], bc.dims, bc.gen_args["seed"], s, c, coef, ctx=gpu_ctx)
                 for h, (s, c) in zip(halves, ranges)]
    else:
        slabs = [generate_device_slab(bc, s, c, ctx=gpu_ctx) for s, c in ranges]
    cat = torch.cat(slabs)
    assert torch.equal(cat.view(torch.int64), whole.view(torch.int64))


def test_generator_errors(gpu_ctx, lmra):
    from paper_2303_11612_b200 import device
    with pytest.raises(lmra.LmraInvalidArgument):
        device.gen_tucker_noise([10, 10], [11, 2], 1e-2, 1, ctx=gpu_ctx)
    with pytest.raises(lmra.LmraInvalidArgument):
        device.gen_hilbert([10, 10], ctx=gpu_ctx, start=8, count=5)

"""Device-side helpers for the BASELINE configurations (baseline_configs.py at the repo
root holds them as data): the synthetic inputs generated on the device -- whole tensors or
one rank's slab of the last mode -- and the conversion of a config's algorithm fields to
AlgoConfig."""
from __future__ import annotations

import dataclasses

from .tucker import AlgoConfig


def algo_config(bc) -> AlgoConfig:
    return AlgoConfig(**dataclasses.asdict(bc.cfg))


def generate_device(bc, ctx=None):
    """Synthetic input on the device (flat float64 CUDA tensor)."""
    from . import device
    if bc.generator == "tucker_noise":
        return device.gen_tucker_noise(bc.dims, bc.gen_args["core_dims"], bc.gen_args["gamma"],
                                       bc.gen_args["seed"], ctx=ctx)
    if bc.generator == "hilbert":
        return device.gen_hilbert(bc.dims, ctx=ctx)
    if bc.generator == "video":
        return device.gen_video(bc.dims, bc.gen_args["n_terms"], bc.gen_args["noise"],
                                bc.gen_args["seed"], ctx=ctx)
    raise ValueError(bc.generator)


def generate_device_slab(bc, start: int, count: int, ctx=None):
    """Slab [start, start + count) of the last mode of the synthetic input, generated on the
    device without the rest of the tensor (Hilbert and video: elementwise; the Tucker +
    noise tensor needs the all-slice norm exchange, see bench.py / device.gen_tucker_signal_slab)."""
    from . import device
    if bc.generator == "hilbert":
        return device.gen_hilbert(bc.dims, ctx=ctx, start=start, count=count)
    if bc.generator == "video":
        return device.gen_video(bc.dims, bc.gen_args["n_terms"], bc.gen_args["noise"], bc.gen_args["seed"],
                                ctx=ctx, start=start, count=count)
    raise ValueError("tucker_noise slabs need the two-step protocol (gen_tucker_signal_slab)")

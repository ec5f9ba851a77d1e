"""The five BASELINE.json configurations as data.

Each entry: dims, the generator that makes the synthetic input, the algorithm id and
the algorithm configuration (the fields of lmra::AlgoConfig, tucker.hpp:32-45), plus the
algorithmic byte / flop counts of one decomposition used for the roofline (DESIGN.md
section 6).  Importing this module loads no GPU library: bench.py's CPU (reference) arm
uses it together with the oracle only; the GPU side converts `cfg` with
paper_2303_11612_b200.configs.algo_config().
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, List, Optional

import numpy as np



@dataclass
class AlgoSpec:
    """lmra::AlgoConfig's fields (tucker.hpp:32-45), reference defaults."""
    rank: List[int]
    oversampling: int = 10
    power: int = 1
    alpha: float = 0.2
    regime: str = "uniform"
    regime_beta: float = 0.5
    t_samples: Optional[List[int]] = None
    order: Optional[List[int]] = None
    seed: int = 0
    strategy: str = "A"


@dataclass
class BaselineConfig:
    name: str
    dims: List[int]
    alg: str
    cfg: AlgoSpec
    generator: str                 # "tucker_noise" | "hilbert" | "video"
    gen_args: dict = field(default_factory=dict)
    description: str = ""


CONFIGS = {
    "cfg1": BaselineConfig(
        "cfg1", [200, 200, 200], "alg1",
        AlgoSpec(rank=[10, 10, 10], oversampling=5, power=1, seed=1),
        "tucker_noise", dict(core_dims=[10, 10, 10], gamma=1e-2, seed=1),
        "200^3 Gaussian core 10^3 x orthonormal U_n + 1e-2 relative noise; rand T-HOSVD power"),
    "cfg2": BaselineConfig(
        "cfg2", [400, 400, 400], "alg2",
        AlgoSpec(rank=[20, 20, 20], oversampling=10, power=1, order=[0, 1, 2], seed=1),
        "hilbert", {},
        "400^3 Hilbert a_ijk = 1/(i+j+k-2); rand ST-HOSVD power"),
    "cfg3": BaselineConfig(
        "cfg3", [100, 100, 100, 100], "alg5",
        AlgoSpec(rank=[15, 15, 15, 15], oversampling=5, power=1, regime="uniform",
                   t_samples=[80, 80, 80, 80], seed=1),
        "tucker_noise", dict(core_dims=[15, 15, 15, 15], gamma=1e-3, seed=1),
        "100^4 Gaussian core 15^4 + 1e-3 noise; rand ST-HOSVD AMM uniform c=4(K+p)=80"),
    "cfg4": BaselineConfig(
        "cfg4", [1000, 1000, 1000], "alg4",
        AlgoSpec(rank=[50, 50, 50], oversampling=10, power=2, regime="nearly_optimal",
                   regime_beta=0.5, t_samples=[400, 400, 400], seed=1),
        "tucker_noise", dict(core_dims=[50, 50, 50], gamma=1e-2, seed=1),
        "1000^3 (8 GB) Gaussian core 50^3 + 1e-2 noise; rand T-HOSVD AMM nearly-optimal c=400 q=2"),
    "cfg5": BaselineConfig(
        "cfg5", [512, 512, 3, 512], "alg5",
        AlgoSpec(rank=[40, 40, 3, 40], oversampling=10, power=1, regime="nearly_optimal",
                   regime_beta=0.5, alpha=0.2, seed=1),
        "video", dict(n_terms=30, noise=0.05, seed=1),
        "512x512x3x512 video: 30 separable cosine terms + U[0,0.05] noise; rand ST-HOSVD AMM "
        "nearly-optimal alpha=0.2"),
}


def scaled(name: str, dims: List[int], rank: Optional[List[int]] = None, **cfg_over) -> BaselineConfig:
    """Same structure as a BASELINE config at another size (for oracle-sized parity runs)."""
    import copy
    b = copy.deepcopy(CONFIGS[name])
    b.dims = list(dims)
    if rank is not None:
        b.cfg.rank = list(rank)
        if "core_dims" in b.gen_args:
            b.gen_args["core_dims"] = list(rank)
    for k, v in cfg_over.items():
        setattr(b.cfg, k, v)
    b.name = f"{name}@{'x'.join(map(str, dims))}"
    return b


def generate_host(bc: BaselineConfig):
    """The synthetic input on the host with the oracle's generators (the same bits as
    paper_2303_11612_b200.configs.generate_device; no GPU library is loaded)."""
    from oracle import oracle as O
    g = bc.gen_args
    if bc.generator == "tucker_noise":
        return O.gen_tucker_noise(bc.dims, g["core_dims"], g["gamma"], g["seed"])
    if bc.generator == "hilbert":
        return O.gen_hilbert(bc.dims)
    return O.gen_video(bc.dims, g["n_terms"], g["noise"], g["seed"])


def algorithmic_cost(bc: BaselineConfig) -> dict:
    """Compulsory bytes / flops of one decomposition (SURVEY.md 8d rules R1-R6).

    R1 each step reads each operand once and writes each output once (8 B/elem);
    R2 T-HOSVD steps reading the same input in the same phase share one read;
    R3 the AMM gather is fused into the first half-product, each half-product reads
       the I_n x T sampled matrix once;  R4 small operands counted;
    R5 host RNG / sampling chains / s x s SVDs count 0;  R6 2mnk flops per contraction,
       column squared norms 2 flops / element / mode.
    """
    dims = list(bc.dims)
    N = len(dims)
    cfg = bc.cfg
    mu = [min(m, d) for m, d in zip(cfg.rank, dims)]
    s = [min(m + cfg.oversampling, d) for m, d in zip(mu, dims)]
    q = cfg.power
    B = 0.0
    F = 0.0
    size = float(np.prod(dims))
    seq = bc.alg in ("alg2", "alg5", "alg7")
    amm = bc.alg in ("alg4", "alg5")
    qr = bc.alg in ("alg6", "alg7")  # QR-proxy: + projection P = Q^T A_(n), SVD via P's R factor
    order = list(cfg.order) if cfg.order else list(range(N))

    def power_cost(I, J, s_):
        # q x [half = A^T c (read A, write J x s); c = A half (read A, read J x s)]
        b = q * (2 * I * J + 2 * J * s_ + 2 * I * s_) * 8
        f = q * 4.0 * I * J * s_
        return b, f

    if not seq:
        # phase: norms (amm, non-uniform) share one read of X across modes
        if amm and cfg.regime != "uniform":
            B += size * 8 + sum(size / d for d in dims) * 8
            F += 2 * size * N
        for n in range(N):
            I = dims[n]
            J = size / I
            if amm:
                T = (cfg.t_samples or [None] * N)[n] or int(np.ceil(cfg.alpha * J))
                b, f = power_cost(I, T, s[n])
                # fused gather: the first half-product reads the sampled fibres from X
                B += b
                F += f
            else:
                b, f = power_cost(I, J, s[n])
                F += f
                B += b
        if not amm:
            # R2: the N modes' half-products share reads of X in each of the 2q phases
            B -= (N - 1) * 2 * q * size * 8
        if qr:
            # projections P_n = Q_n^T A_(n) share one read of X (R2); each P_n is written once
            # and read once by its R factor
            B += size * 8
            for n in range(N):
                J = size / dims[n]
                B += (2 * J * s[n] + dims[n] * s[n]) * 8
                F += 2.0 * size * s[n]
        # core: ascending width
        cur = list(dims)
        idx = sorted(range(N), key=lambda n: mu[n])
        for k, n in enumerate(idx):
            if qr and k == 0:  # the first contraction reads P (s rows) instead of X
                J = size / dims[n]
                B += (J * s[n] + J * mu[n] + s[n] * mu[n]) * 8
                F += 2.0 * J * s[n] * mu[n]
                cur[n] = mu[n]
                continue
            inp = float(np.prod(cur))
            out = inp / cur[n] * mu[n]
            B += (inp + out + cur[n] * mu[n]) * 8
            F += 2.0 * inp * mu[n]
            cur[n] = mu[n]
    else:
        cur = list(dims)
        for n in order:
            sz = float(np.prod(cur))
            I = cur[n]
            J = sz / I
            if amm:
                if cfg.regime != "uniform":
                    B += (sz + J) * 8
                    F += 2 * sz
                T = (cfg.t_samples or [None] * N)[n] or int(np.ceil(cfg.alpha * J))
                b, f = power_cost(I, T, s[n])
            else:
                b, f = power_cost(I, J, s[n])
            B += b
            F += f
            out = sz / I * mu[n]
            if qr:  # projection (read A, write P), R factor (read P), shrink from P
                B += (sz + 3 * J * s[n] + I * s[n] + out + s[n] * mu[n]) * 8
                F += 2.0 * sz * s[n] + 2.0 * J * s[n] * mu[n]
            else:
                B += (sz + out + I * mu[n]) * 8
                F += 2.0 * sz * mu[n]
            cur[n] = mu[n]
    return {"bytes": B, "flops": F, "tensor_bytes": size * 8}

"""GPU vs oracle on the BASELINE configurations, every one at FULL size (cfg4's
8 GB 1000^3 tensor and cfg5's 3.2 GB video tensor included) plus oracle-sized scalings.

Each case checks, on identical input bits (device generator == host generator, asserted):
  * the product path itself -- the run with its OWN draws, i.e. what bench.py times: the fused
    norms3 pass, the device sampling chain, the int8 tensor-core contractions (core / first
    shrinks) -- against the oracle: Omega and sampled indices bit-exact, factor sines on every
    gap-aware leading block <= 1e-10, core and RE within 1e-10 relative;
  * the parity-override run (the oracle's Omega / samples passed in), same tolerances.
RE is computed on the device for both decompositions (lmra_relative_error, checked against the
oracle's loop in test_gpu_parity.py) -- a numpy reconstruction of 8 GB would need ~40 GB.

Config 2 (Hilbert, ST-HOSVD) is the documented exception: its
sketch spectrum falls below rounding after ~12 directions, so two valid fp64 evaluation
orders disagree on trailing factor directions (sines up to 1), on the core (~1e-8) and on
RE.  The test asserts the gap-aware leading block to 1e-10 and reports the full-subspace /
core / RE differences against the measured oracle-vs-oracle floor.

Set LMRA_PARITY_LOG=path to append one JSON line of metrics per case.
"""
import json
import os

import numpy as np
import pytest

from test_gpu_parity import check_own_draws, compare

pytestmark = pytest.mark.gpu


def _input(bc, ctx):
    import torch
    from baseline_configs import generate_host
    from paper_2303_11612_b200.configs import generate_device
    xd = generate_device(bc, ctx=ctx)
    xh = generate_host(bc)
    same = torch.equal(xd.view(torch.int64), torch.from_numpy(xh).to(xd.device).view(torch.int64))
    assert same, "device and host generators differ"
    return xd, xh


def _orc_cfg(orc, c, threads=4):
    return orc.AlgoConfig(rank=list(c.rank), oversampling=c.oversampling, power=c.power,
                          alpha=c.alpha, regime=c.regime, regime_beta=c.regime_beta,
                          t_samples=c.t_samples, order=c.order, seed=c.seed, strategy=c.strategy,
                          mode_threads=threads)


def _log(case, what, m):
    path = os.environ.get("LMRA_PARITY_LOG")
    if not path:
        return
    row = {"case": case, "run": what}
    for k, v in m.items():
        row[k] = [float(x) for x in v] if isinstance(v, (list, tuple)) else float(v)
    with open(path, "a") as f:
        f.write(json.dumps(row) + "\n")


CASES = {
    "cfg1": ("cfg1", None, 0),
    "cfg3": ("cfg3", None, 0),
    "cfg4_200": ("cfg4", [200, 200, 200], 0),
    "cfg4_160x180x200": ("cfg4", [160, 180, 200], 0),
    "cfg5_128": ("cfg5", [128, 128, 3, 128], 0),
    "cfg5_96x80x3x64": ("cfg5", [96, 80, 3, 64], 0),
    # full size: host RAM for the oracle (tensor + unfoldings + GPU copy back)
    "cfg5_full": ("cfg5", None, 24),
    "cfg4_full": ("cfg4", None, 48),
}


@pytest.mark.parametrize("case", list(CASES))
def test_config_parity(gpu_ctx, lmra, orc, case):
    from baseline_configs import CONFIGS, scaled
    from paper_2303_11612_b200 import device
    from paper_2303_11612_b200.configs import algo_config
    name, dims, need_gb = CASES[case]
    if need_gb:
        import psutil
        avail = psutil.virtual_memory().available / 2**30
        if avail < need_gb:
            pytest.skip(f"{case}: needs ~{need_gb} GB of host RAM for the oracle, {avail:.0f} GB available")
    bc = CONFIGS[name] if dims is None else scaled(name, dims)
    xd, x = _input(bc, gpu_ctx)
    ref = orc.run(bc.alg, x, bc.dims, _orc_cfg(orc, bc.cfg, 3 if need_gb else 4))
    t = lmra.DenseTensor.device(xd, bc.dims)
    cfg = algo_config(bc)
    re_fn = lambda core, factors: device.relative_error(xd, bc.dims, core, factors, ctx=gpu_ctx)  # noqa: E731
    # the benchmarked path: own draws (fused norms, device sampler, int8 contractions)
    own = lmra.run_algorithm(bc.alg, t, cfg, ctx=gpu_ctx)
    check_own_draws(bc.alg, own, ref, bc.cfg.regime, bc.cfg.order)
    m_own = compare(own, ref, None, re_fn=re_fn)
    _log(case, "own_draws", m_own)
    # the parity-override run (oracle Omega / samples passed in)
    gpu = lmra.run_algorithm(bc.alg, t, cfg, omega=ref.omega, samples=ref.samples, ctx=gpu_ctx)
    m_ov = compare(gpu, ref, None, re_fn=re_fn)
    _log(case, "overrides", m_ov)
    print(case, "own", m_own, "override", m_ov)


def test_cfg2_hilbert_gap_aware(gpu_ctx, lmra, orc):
    from baseline_configs import CONFIGS
    from paper_2303_11612_b200 import device
    from paper_2303_11612_b200.configs import algo_config
    bc = CONFIGS["cfg2"]
    xd, x = _input(bc, gpu_ctx)
    ref = orc.run(bc.alg, x, bc.dims, _orc_cfg(orc, bc.cfg))
    t = lmra.DenseTensor.device(xd, bc.dims)
    re_fn = lambda core, factors: device.relative_error(xd, bc.dims, core, factors, ctx=gpu_ctx)  # noqa: E731
    own = lmra.run_algorithm(bc.alg, t, algo_config(bc), ctx=gpu_ctx)
    check_own_draws(bc.alg, own, ref, bc.cfg.regime, bc.cfg.order)
    m = compare(own, ref, None, check_core=False, check_columns=False, check_re=False, tol=1e-10, re_fn=re_fn)
    # floor report: the oracle itself with another BLAS thread count (another valid order)
    orc.set_blas_threads(1)
    ref1 = orc.run(bc.alg, x, bc.dims, _orc_cfg(orc, bc.cfg))
    orc.set_blas_threads(os.cpu_count() or 1)
    from conftest import subspace_sine
    floor_full = [subspace_sine(a1, b1) for a1, b1 in zip(ref.factors, ref1.factors)]
    m["floor_full_sines"] = floor_full
    _log("cfg2", "own_draws", m)
    print("cfg2 gpu-vs-oracle full sines", m["full_sines"], "RE", m["re"],
          "| oracle-vs-oracle floor sines", floor_full)
    # RE of both is ~1.5e-8 relative; differences at the 1e-9 level are rounding
    re_g, re_o = m["re"]
    assert abs(re_g - re_o) <= 5e-9, (re_g, re_o)

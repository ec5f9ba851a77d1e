"""GPU vs oracle on the BASELINE configurations: configs 1-3 at full size,
configs 4 and 5 at oracle-sized scalings with the same structure (rank, p, q, c /
alpha, regime), all on identical input bits generated on the device.

Config 2 (Hilbert, ST-HOSVD) is the documented exception: its
sketch spectrum falls below rounding after ~12 directions, so two valid fp64
evaluation orders disagree on trailing factor directions (sines up to 1), on the core
(~1e-8) and on RE.  The test asserts the gap-aware leading block to 1e-10 and reports
the full-subspace / core / RE differences against the measured oracle-vs-oracle floor.
"""
import numpy as np
import pytest

from conftest import relative_error
from test_gpu_parity import check_own_draws, compare

pytestmark = pytest.mark.gpu


def _input(lmra, bc):
    from paper_2303_11612_b200.configs import generate_device
    x = generate_device(bc)
    return x, x.cpu().numpy()


def _orc_cfg(orc, c):
    return orc.AlgoConfig(rank=list(c.rank), oversampling=c.oversampling, power=c.power,
                          alpha=c.alpha, regime=c.regime, regime_beta=c.regime_beta,
                          t_samples=c.t_samples, order=c.order, seed=c.seed, strategy=c.strategy,
                          mode_threads=4)


CASES = {
    "cfg1": ("cfg1", None, None),
    "cfg3": ("cfg3", None, None),
    "cfg4_200": ("cfg4", [200, 200, 200], None),
    "cfg4_160x180x200": ("cfg4", [160, 180, 200], None),
    "cfg5_128": ("cfg5", [128, 128, 3, 128], None),
    "cfg5_96x80x3x64": ("cfg5", [96, 80, 3, 64], None),
}


@pytest.mark.parametrize("case", list(CASES))
def test_config_parity(gpu_ctx, lmra, orc, case):
    from paper_2303_11612_b200.configs import CONFIGS, scaled
    name, dims, rank = CASES[case]
    bc = CONFIGS[name] if dims is None else scaled(name, dims, rank)
    xd, x = _input(lmra, bc)
    ref = orc.run(bc.alg, x, bc.dims, _orc_cfg(orc, bc.cfg))
    t = lmra.DenseTensor.device(xd, bc.dims)
    own = lmra.run_algorithm(bc.alg, t, bc.cfg)
    check_own_draws(bc.alg, own, ref, bc.cfg.regime, bc.cfg.order)
    gpu = lmra.run_algorithm(bc.alg, t, bc.cfg, omega=ref.omega, samples=ref.samples)
    m = compare(gpu, ref, x.reshape(bc.dims, order="F"))
    print(case, {k: v for k, v in m.items()})


def test_cfg2_hilbert_gap_aware(gpu_ctx, lmra, orc):
    from paper_2303_11612_b200.configs import CONFIGS
    bc = CONFIGS["cfg2"]
    xd, x = _input(lmra, bc)
    # the Hilbert generator is bit-identical on host and device
    assert np.array_equal(x, orc.gen_hilbert(bc.dims))
    ref = orc.run(bc.alg, x, bc.dims, _orc_cfg(orc, bc.cfg))
    t = lmra.DenseTensor.device(xd, bc.dims)
    gpu = lmra.run_algorithm(bc.alg, t, bc.cfg, omega=ref.omega)
    a = x.reshape(bc.dims, order="F")
    m = compare(gpu, ref, a, check_core=False, check_columns=False, check_re=False, tol=1e-10)
    # floor report: the oracle itself with another BLAS thread count (another valid order)
    orc.set_blas_threads(1)
    ref1 = orc.run(bc.alg, x, bc.dims, _orc_cfg(orc, bc.cfg))
    import os
    orc.set_blas_threads(os.cpu_count() or 1)
    from conftest import subspace_sine
    floor_full = [subspace_sine(a1, b1) for a1, b1 in zip(ref.factors, ref1.factors)]
    print("cfg2 gpu-vs-oracle full sines", m["full_sines"], "RE", m["re"],
          "| oracle-vs-oracle floor sines", floor_full)
    # RE of both is ~1.5e-8 relative; differences at the 1e-9 level are rounding
    re_g, re_o = m["re"]
    assert abs(re_g - re_o) <= 5e-9, (re_g, re_o)

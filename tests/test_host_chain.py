"""The product's host-side restatements (csrc/host/host_chain.cpp), reached through the C ABI
without a GPU, against the oracle: the sampling chain and the config rules must be bit-exact.
(On the device path the same chain runs in sampler.cu -- tests/test_gpu_sampler.py.)"""
import os

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("regime", ["optimal", "nearly_optimal", "uniform"])
def test_probabilities_bit_exact(lmra, orc, regime):
    rng = np.random.default_rng(3)
    for w in [rng.standard_normal(50_000) ** 2, np.ones(777), rng.random(1000) * 1e-200,
              np.concatenate([np.zeros(10), rng.random(90)])]:
        assert np.array_equal(lmra.probabilities(w, regime), orc.probabilities(w, regime))


def test_randsample_bit_exact(lmra, orc):
    rng = np.random.default_rng(4)
    p = orc.probabilities(rng.random(20_000), "nearly_optimal")
    for L, seed, stream in [(1, 0, 0), (400, 1, 4), (5000, 7, 9)]:
        i1, s1 = lmra.randsample(L, p, seed, stream)
        i2, s2 = orc.randsample(L, p, seed, stream)
        assert np.array_equal(i1, i2) and np.array_equal(s1, s2)


def test_amm_sample_counts_match(lmra, orc):
    for dims, kw in [([60, 60, 60], dict(rank=[10, 10, 10])),
                     ([512, 512, 3, 512], dict(rank=[40, 40, 3, 40])),
                     ([100, 100, 100, 100], dict(rank=[15] * 4, t_samples=[80] * 4)),
                     ([7, 5, 3], dict(rank=[2, 9, 1], alpha=0.37, order=[2, 0, 1]))]:
        for seq in (False, True):
            assert lmra.amm_sample_counts(dims, lmra.AlgoConfig(**kw), seq) == \
                orc.amm_sample_counts(dims, orc.AlgoConfig(**kw), seq)


def test_error_surface(lmra):
    with pytest.raises(lmra.LmraInvalidArgument):  # total > 0, a negative weight survives
        lmra.probabilities(np.array([3.0, -1.0]), "optimal")
    # total <= 0 falls back to uniform before any sign check (tucker.cpp:119-121)
    assert np.all(lmra.probabilities(np.array([1.0, -2.0]), "optimal") == 0.5)
    with pytest.raises(lmra.LmraInvalidArgument):
        lmra.probabilities(np.array([1.0, 2.0]), "nearly_optimal", 1.5)
    with pytest.raises(lmra.LmraInvalidArgument):
        lmra.amm_sample_counts([4, 4], lmra.AlgoConfig(rank=[2, 2], alpha=1.0), False)
    with pytest.raises(lmra.LmraInvalidArgument):
        lmra.randsample(0, np.array([1.0]), 1, 1)
    with pytest.raises(lmra.LmraInvalidArgument):
        lmra.run_algorithm("alg3", np.zeros((2, 2)), lmra.AlgoConfig(rank=[1, 1]))


def test_algorithm_ids_and_knobs(lmra, monkeypatch):
    # tucker.cpp:164-220: ids in the reference's order, parse / id round trips, thread_cap
    ids = lmra.all_algorithm_ids()
    assert ids == ["thosvd", "sthosvd", "hooi", "alg1", "alg2", "alg4", "alg5", "alg6", "alg7"]
    for a in ids:
        assert lmra.parse_algorithm(a) == a
        assert lmra.algorithm_id(a) == a
    assert lmra.parse_algorithm("alg3") is None and lmra.parse_algorithm("") is None
    assert lmra.algorithm_id(99) == "?"
    assert lmra.thread_cap() >= 1
    assert lmra.device_cap() == 1  # no device visible here (or LMRA_NUM_GPUS unset)


def test_knob_semantics_in_fresh_process():
    # the caps are read once per process (static, as tucker.cpp:164-172): check the env idiom
    import subprocess
    import sys
    code = ("import sys; sys.path.insert(0, %r); import paper_2303_11612_b200 as P; "
            "print(P.thread_cap())" % ROOT)
    for env, want in (({"LMRA_NUM_THREADS": "7"}, "7"), ({"LMRA_NUM_THREADS": "500"}, "64"),
                      ({"LMRA_NUM_THREADS": "0"}, "1"), ({}, "1")):
        e = {k: v for k, v in os.environ.items() if k != "LMRA_NUM_THREADS"}
        e.update(env)
        out = subprocess.run([sys.executable, "-c", code], env=e, capture_output=True, text=True, check=True)
        assert out.stdout.strip() == want, (env, out.stdout, out.stderr)

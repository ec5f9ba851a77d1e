"""Pin the oracle (and the product's host RNG, through the C ABI -- no GPU needed) to the
reference itself: golden vectors produced by the reference's own rng.hpp
(tests/golden/rng_reference.json, see make_golden.py) and the known-answer values in the
reference test suite."""
import json
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "rng_reference.json")


@pytest.fixture(scope="module")
def golden():
    with open(GOLDEN) as f:
        return json.load(f)["streams"]


def test_pcg32_known_answer(orc):
    # test_sketching.cpp:16-23: (seed, stream) = (42, 54)
    want = [0xa15c02b7, 0x7b47f409, 0xba1d3330, 0x83d2f293, 0xbfa4784b, 0xcbed606e]
    assert [int(v) for v in orc.rng_u32(42, 54, 6)] == want


def test_oracle_rng_matches_reference_rng_hpp(orc, golden):
    for s in golden:
        assert [int(v) for v in orc.rng_u32(s["seed"], s["stream"], len(s["u32"]))] == s["u32"]
        d = orc.rng_double(s["seed"], s["stream"], len(s["double_hex"]))
        assert [float.hex(float(v)) for v in d] == [float.hex(float.fromhex(h)) for h in s["double_hex"]]
        nrm = orc.rng_normal(s["seed"], s["stream"], len(s["normal_hex"]))
        assert np.array_equal(nrm, np.array([float.fromhex(h) for h in s["normal_hex"]]))


def test_oracle_jump_ahead_is_sequential(orc):
    seq = orc.rng_u32(9, 1, 300)
    assert np.array_equal(orc.rng_u32(9, 1, 100, skip=200), seq[200:])


def test_gaussian_matrix_is_the_normal_stream_in_storage_order(orc, golden):
    # sketching.cpp:164-173: column-major fill; large sizes use threaded jump-ahead
    for s in golden:
        n = len(s["normal_hex"])
        g = orc.gaussian_matrix(n, 1, s["seed"], s["stream"])
        assert np.array_equal(g.ravel(order="F"), [float.fromhex(h) for h in s["normal_hex"]])
    big = orc.gaussian_matrix(1500, 800, 3, 2)  # 1.2e6 normals: the threaded path
    assert np.array_equal(big.ravel(order="F"), orc.rng_normal(3, 2, 1200000))


def test_product_host_rng_matches_reference(lmra, orc, golden):
    # the product's own restatement (csrc/host/host_chain.cpp), bit-exact, via the C ABI
    for s in golden:
        n = len(s["normal_hex"])
        g = lmra.gaussian_matrix(n, 1, s["seed"], s["stream"])
        assert np.array_equal(g.ravel(order="F"), [float.fromhex(h) for h in s["normal_hex"]])
    assert np.array_equal(lmra.gaussian_matrix(1000, 60, 1, 1), orc.gaussian_matrix(1000, 60, 1, 1))

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a kernels)")
    config.addinivalue_line("markers", "slow: full-size BASELINE configurations")


@pytest.fixture(scope="session")
def orc():
    from oracle import oracle
    oracle.lib()
    return oracle


@pytest.fixture(scope="session")
def lmra():
    import paper_2303_11612_b200 as P
    return P


@pytest.fixture(scope="session")
def gpu_ctx(lmra):
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test selected but no CUDA device is visible")
    return lmra.default_context(0)


# ---------------------------------------------------------------- parity metrics
def subspace_sine(u: np.ndarray, v: np.ndarray) -> float:
    """sin of the largest principal angle between span(u) and span(v), stable form
    sigma_max(v - u (u^T v)) (sqrt(1-cos^2) has a 1e-8 floor)."""
    if u.shape[1] == 0:
        return 0.0
    r = v - u @ (u.T @ v)
    return float(np.linalg.norm(r, 2))


def gap_blocks(sig: np.ndarray, mu: int, rel_gap: float = 1e-5):
    """Leading block sizes k <= mu whose sketch gap (s_k - s_{k+1}) / s_1 >= rel_gap."""
    s1 = sig[0] if sig.size and sig[0] > 0 else 1.0
    ks = []
    for k in range(1, mu + 1):
        nxt = sig[k] if k < sig.size else 0.0
        if (sig[k - 1] - nxt) / s1 >= rel_gap:
            ks.append(k)
    return ks


def reconstruct(core: np.ndarray, factors) -> np.ndarray:
    t = core
    for n, f in enumerate(factors):
        t = np.moveaxis(np.tensordot(f, t, axes=([1], [n])), 0, n)
    return t


def relative_error(a: np.ndarray, core, factors) -> float:
    r = reconstruct(core, factors)
    return float(np.sqrt(np.sum((a - r) ** 2) / np.sum(a * a)))

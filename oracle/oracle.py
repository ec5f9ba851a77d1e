"""ctypes front-end of the CPU oracle (oracle/lmra_oracle.cpp).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py -- never by the product package.
"""
from __future__ import annotations

import ctypes as C
import glob
import os
import subprocess
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "build", "liblmra_oracle.so")

ALG = {"alg1": 1, "alg2": 2, "alg4": 4, "alg5": 5, "alg6": 6, "alg7": 7, "thosvd": 10, "sthosvd": 11, "hooi": 12}
REGIME = {"optimal": 0, "nearly_optimal": 1, "uniform": 2}

u64p = C.POINTER(C.c_uint64)
dblp = C.POINTER(C.c_double)
i64p = C.POINTER(C.c_int64)


class OrcConfig(C.Structure):
    _fields_ = [
        ("rank", u64p), ("oversampling", C.c_uint64), ("power", C.c_int32), ("alpha", C.c_double),
        ("regime", C.c_int32), ("regime_beta", C.c_double), ("t_samples", u64p), ("order", u64p),
        ("seed", C.c_uint64), ("strategy", C.c_int32), ("mode_threads", C.c_int32),
        ("keep_trace", C.c_int32), ("hooi_max_sweeps", C.c_int32), ("hooi_tol", C.c_double),
    ]


class OracleError(RuntimeError):
    pass


class OracleInvalidArgument(OracleError, ValueError):
    pass


def build() -> str:
    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)
    return LIB_PATH


def _blas_path() -> str:
    import numpy
    libs = glob.glob(os.path.join(os.path.dirname(os.path.dirname(numpy.__file__)), "numpy.libs",
                                  "libscipy_openblas64_*.so"))
    if not libs:
        raise OracleError("numpy's bundled OpenBLAS (ILP64) not found")
    return libs[0]


_lib = None


def lib():
    global _lib
    if _lib is None:
        try:
            build()  # make: no-op when up to date
        except (OSError, subprocess.CalledProcessError):
            if not os.path.exists(LIB_PATH):
                raise
        L = C.CDLL(LIB_PATH)
        L.orc_last_error.restype = C.c_char_p
        L.orc_stable_sum.restype = C.c_double
        L.orc_result_seconds.restype = C.c_double
        L.orc_relative_error.restype = C.c_double
        L.orc_result_num_samples.restype = C.c_uint64
        L.orc_result_num_norms.restype = C.c_uint64
        L.orc_stable_sum.argtypes = [dblp, C.c_size_t]
        if L.orc_init_blas(_blas_path().encode()) != 0:
            raise OracleError(L.orc_last_error().decode())
        _lib = L
    return _lib


def _check(rc: int):
    if rc != 0:
        msg = lib().orc_last_error().decode()
        raise (OracleInvalidArgument if rc == 1 else OracleError)(msg)


def _u64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint64))


def _f64(a) -> np.ndarray:
    return np.require(np.asarray(a, dtype=np.float64), requirements=["C"])


def _p(a: np.ndarray, t):
    return a.ctypes.data_as(t)


def set_blas_threads(n: int):
    lib().orc_set_blas_threads(int(n))


# ---------------------------------------------------------------- RNG
def rng_u32(seed: int, stream: int, n: int, skip: int = 0) -> np.ndarray:
    out = np.empty(n, dtype=np.uint32)
    lib().orc_rng_u32(C.c_uint64(seed), C.c_uint64(stream), C.c_uint64(skip),
                      out.ctypes.data_as(C.POINTER(C.c_uint32)), C.c_size_t(n))
    return out


def rng_double(seed: int, stream: int, n: int) -> np.ndarray:
    out = np.empty(n)
    lib().orc_rng_double(C.c_uint64(seed), C.c_uint64(stream), _p(out, dblp), C.c_size_t(n))
    return out


def rng_normal(seed: int, stream: int, n: int) -> np.ndarray:
    out = np.empty(n)
    lib().orc_rng_normal(C.c_uint64(seed), C.c_uint64(stream), _p(out, dblp), C.c_size_t(n))
    return out


def gaussian_matrix(rows: int, cols: int, seed: int, stream: int) -> np.ndarray:
    """Column-major rows x cols, returned as a numpy array with shape (rows, cols) (Fortran order)."""
    out = np.empty(rows * cols)
    _check(lib().orc_gaussian_matrix(C.c_uint64(rows), C.c_uint64(cols), C.c_uint64(seed),
                                     C.c_uint64(stream), _p(out, dblp)))
    return out.reshape((rows, cols), order="F")


# ---------------------------------------------------------------- sampling
def stable_sum(v) -> float:
    v = _f64(v).ravel()
    return lib().orc_stable_sum(_p(v, dblp), v.size)


def column_sqnorms(x: np.ndarray, dims: Sequence[int], mode: int) -> np.ndarray:
    x = _f64(x).ravel(order="K")
    d = _u64(dims)
    J = int(np.prod(dims)) // int(dims[mode])
    w = np.empty(J)
    _check(lib().orc_column_sqnorms(_p(x, dblp), _p(d, u64p), len(dims), mode, _p(w, dblp)))
    return w


def probabilities(w, regime: str, beta: float = 0.5) -> np.ndarray:
    w = _f64(w).ravel()
    p = np.empty_like(w)
    _check(lib().orc_probabilities(_p(w, dblp), C.c_uint64(w.size), REGIME[regime], C.c_double(beta),
                                   _p(p, dblp)))
    return p


def randsample(L: int, p, seed: int, stream: int):
    p = _f64(p).ravel()
    idx = np.empty(L, dtype=np.int64)
    sc = np.empty(L)
    _check(lib().orc_randsample(C.c_uint64(L), _p(p, dblp), C.c_uint64(p.size), C.c_uint64(seed),
                                C.c_uint64(stream), _p(idx, i64p), _p(sc, dblp)))
    return idx, sc


# ---------------------------------------------------------------- config / algorithms
@dataclass
class AlgoConfig:
    """Mirror of lmra::AlgoConfig (tucker.hpp:32-45)."""
    rank: Sequence[int]
    oversampling: int = 10
    power: int = 1
    alpha: float = 0.2
    regime: str = "uniform"
    regime_beta: float = 0.5
    t_samples: Optional[Sequence[int]] = None
    order: Optional[Sequence[int]] = None
    seed: int = 0
    strategy: str = "A"
    mode_threads: int = 1
    keep_trace: bool = True
    hooi_max_sweeps: int = 50
    hooi_tol: float = 1e-8
    _keep: list = field(default_factory=list, repr=False)

    def to_c(self, n_modes: int) -> OrcConfig:
        rank = _u64(self.rank)
        if rank.size != n_modes:
            raise OracleInvalidArgument("rank vector length must equal tensor order")
        ts = _u64(self.t_samples) if self.t_samples is not None else None
        if ts is not None and ts.size != n_modes:
            raise OracleInvalidArgument("sample count override length must equal tensor order")
        od = _u64(self.order) if self.order is not None else None
        if od is not None and od.size != n_modes:
            raise OracleInvalidArgument("processing order length must equal tensor order")
        self._keep = [rank, ts, od]
        return OrcConfig(
            _p(rank, u64p), self.oversampling, self.power, self.alpha, REGIME[self.regime],
            self.regime_beta, _p(ts, u64p) if ts is not None else None,
            _p(od, u64p) if od is not None else None, self.seed, 0 if self.strategy == "A" else 1,
            self.mode_threads, 1 if self.keep_trace else 0, self.hooi_max_sweeps, self.hooi_tol)


@dataclass
class Decomposition:
    core: np.ndarray            # shape = core dims, Fortran order (first index fastest)
    factors: list               # I_n x mu_n, Fortran order
    seconds: float
    omega: list                 # per mode (I_n x s) or None
    samples: list               # per mode (idx, scales) or None
    norms: list                 # per mode w or None
    sketches: list = field(default_factory=list)  # per mode C (I_n x s)


def amm_sample_counts(dims: Sequence[int], cfg: AlgoConfig, sequential: bool) -> list:
    d = _u64(dims)
    out = np.empty(len(dims), dtype=np.uint64)
    c = cfg.to_c(len(dims))
    _check(lib().orc_amm_sample_counts(_p(d, u64p), len(dims), C.byref(c), int(sequential),
                                       _p(out, u64p)))
    return [int(v) for v in out]


def run(alg: str, x: np.ndarray, dims: Sequence[int], cfg: AlgoConfig) -> Decomposition:
    L = lib()
    xv = _f64(x).ravel(order="K") if x.flags.c_contiguous or x.ndim == 1 else np.asfortranarray(x).ravel(order="F")
    d = _u64(dims)
    N = len(dims)
    c = cfg.to_c(N)
    h = C.c_void_p()
    _check(L.orc_run(ALG[alg], _p(xv, dblp), _p(d, u64p), N, C.byref(c), C.byref(h)))
    try:
        cd = np.empty(N, dtype=np.uint64)
        L.orc_result_core_dims(h, _p(cd, u64p))
        core = np.empty(int(np.prod(cd)))
        L.orc_result_core(h, _p(core, dblp))
        factors, omegas, samples, norms, sketches = [], [], [], [], []
        for n in range(N):
            r, k = C.c_uint64(), C.c_uint64()
            L.orc_result_factor_dims(h, n, C.byref(r), C.byref(k))
            f = np.empty(r.value * k.value)
            L.orc_result_factor(h, n, _p(f, dblp))
            factors.append(f.reshape((r.value, k.value), order="F"))
            if cfg.keep_trace:
                L.orc_result_omega_dims(h, n, C.byref(r), C.byref(k))
                g = np.empty(r.value * k.value)
                if g.size:
                    L.orc_result_omega(h, n, _p(g, dblp))
                omegas.append(g.reshape((r.value, k.value), order="F"))
                L.orc_result_sketch_dims(h, n, C.byref(r), C.byref(k))
                c = np.empty(r.value * k.value)
                if c.size:
                    L.orc_result_sketch(h, n, _p(c, dblp))
                sketches.append(c.reshape((r.value, k.value), order="F"))
                T = L.orc_result_num_samples(h, n)
                if T:
                    idx = np.empty(T, dtype=np.int64)
                    sc = np.empty(T)
                    L.orc_result_samples(h, n, _p(idx, i64p), _p(sc, dblp))
                    samples.append((idx, sc))
                else:
                    samples.append(None)
                W = L.orc_result_num_norms(h, n)
                if W:
                    w = np.empty(W)
                    L.orc_result_norms(h, n, _p(w, dblp))
                    norms.append(w)
                else:
                    norms.append(None)
        seconds = L.orc_result_seconds(h)
        re_core = core.reshape(tuple(int(v) for v in cd), order="F")
        return Decomposition(re_core, factors, seconds, omegas, samples, norms, sketches)
    finally:
        L.orc_result_free(h)


def mode_n_product(x: np.ndarray, dims: Sequence[int], mode: int, b: np.ndarray) -> np.ndarray:
    xv = _f64(x).ravel(order="K")
    d = _u64(dims)
    bm = np.asfortranarray(b, dtype=np.float64)
    out_dims = list(dims)
    out_dims[mode] = bm.shape[0]
    y = np.empty(int(np.prod(out_dims)))
    _check(lib().orc_mode_n_product(_p(xv, dblp), _p(d, u64p), len(dims), mode,
                                    bm.ctypes.data_as(dblp), C.c_uint64(bm.shape[0]), _p(y, dblp)))
    return y


def gram_power_apply(a: np.ndarray, g: np.ndarray, q: int, strategy: str = "A") -> np.ndarray:
    a = np.asfortranarray(a, dtype=np.float64)
    g = np.asfortranarray(g, dtype=np.float64)
    if g.shape[0] != a.shape[0]:  # linalg.cpp:64-65 (the C entry takes G's rows from A)
        raise OracleInvalidArgument("gram_power_apply: G must have as many rows as A")
    c = np.empty((a.shape[0], g.shape[1]), order="F")
    _check(lib().orc_gram_power_apply(a.ctypes.data_as(dblp), C.c_uint64(a.shape[0]), C.c_uint64(a.shape[1]),
                                      g.ctypes.data_as(dblp), C.c_uint64(g.shape[1]), q,
                                      0 if strategy == "A" else 1, c.ctypes.data_as(dblp)))
    return c


def leading_left_singular_vectors(c: np.ndarray, mu: int) -> np.ndarray:
    c = np.asfortranarray(c, dtype=np.float64)
    u = np.empty((c.shape[0], mu), order="F")
    _check(lib().orc_leading_left_singular_vectors(c.ctypes.data_as(dblp), C.c_uint64(c.shape[0]),
                                                   C.c_uint64(c.shape[1]), C.c_uint64(mu),
                                                   u.ctypes.data_as(dblp)))
    return u


def thin_qr_q(m: np.ndarray) -> np.ndarray:
    m = np.asfortranarray(m, dtype=np.float64)
    q = np.empty(m.shape, order="F")
    _check(lib().orc_thin_qr_q(m.ctypes.data_as(dblp), C.c_uint64(m.shape[0]), C.c_uint64(m.shape[1]),
                               q.ctypes.data_as(dblp)))
    return q


def qr_project_extract(c: np.ndarray, a: np.ndarray, mu: int) -> np.ndarray:
    """linalg.cpp:89-99."""
    c = np.asfortranarray(c, dtype=np.float64)
    a = np.asfortranarray(a, dtype=np.float64)
    out = np.empty((c.shape[0], mu), order="F")
    _check(lib().orc_qr_project_extract(c.ctypes.data_as(dblp), C.c_uint64(c.shape[0]), C.c_uint64(c.shape[1]),
                                        a.ctypes.data_as(dblp), C.c_uint64(a.shape[1]), C.c_uint64(mu),
                                        out.ctypes.data_as(dblp)))
    return out


def relative_error(x: np.ndarray, dims: Sequence[int], dec: Decomposition) -> float:
    """||a - reconstruct(d)|| / ||a|| with the reference's loop (tucker.cpp:222-240)."""
    xv = _f64(x).ravel(order="K")
    recon = dec.core.ravel(order="F")
    cur_dims = list(dec.core.shape)
    for n, f in enumerate(dec.factors):
        recon = mode_n_product(recon, cur_dims, n, f)
        cur_dims[n] = f.shape[0]
    num = float(np.sum((xv - recon) ** 2))
    den = float(np.sum(xv * xv))
    return float(np.sqrt(num / den))


# ---------------------------------------------------------------- generators
def gen_tucker_noise(dims, core_dims, gamma: float, seed: int) -> np.ndarray:
    d, cd = _u64(dims), _u64(core_dims)
    out = np.empty(int(np.prod(dims)))
    _check(lib().orc_gen_tucker_noise(_p(d, u64p), _p(cd, u64p), len(dims), C.c_double(gamma),
                                      C.c_uint64(seed), _p(out, dblp)))
    return out


def gen_hilbert(dims) -> np.ndarray:
    d = _u64(dims)
    out = np.empty(int(np.prod(dims)))
    _check(lib().orc_gen_hilbert(_p(d, u64p), len(dims), _p(out, dblp)))
    return out


def gen_video(dims, n_terms: int = 30, noise: float = 0.05, seed: int = 1) -> np.ndarray:
    d = _u64(dims)
    out = np.empty(int(np.prod(dims)))
    _check(lib().orc_gen_video(_p(d, u64p), len(dims), C.c_uint64(n_terms), C.c_double(noise),
                               C.c_uint64(seed), _p(out, dblp)))
    return out

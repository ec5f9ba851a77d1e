"""Device-side helpers over the C ABI, with torch as the allocator (plumbing only).

Primitives on device buffers (mode_n_product, gram_power_apply,
leading_left_singular_vectors, column_sqnorms) and the BASELINE input generators.
All tensors here are flat float64 CUDA tensors in the reference's layout (first
index fastest) together with explicit dims.
"""
from __future__ import annotations

import ctypes as C
from typing import Sequence

import numpy as np

from . import _lib
from ._lib import check, lib
from .tucker import Context, default_context


def _torch():
    import torch
    return torch


def _u64(v):
    return np.ascontiguousarray(np.asarray(v, dtype=np.uint64))


def _ptr(t) -> C.c_void_p:
    return C.c_void_p(t.data_ptr())


def empty(n: int, device: int = 0):
    torch = _torch()
    return torch.empty(int(n), dtype=torch.float64, device=f"cuda:{device}")


def mode_n_product(x, dims: Sequence[int], mode: int, b, ctx: Context = None):
    """y = x x_mode b  (tensor.cpp:118-139); b: torch (rows x I_mode) row-major -> passed
    column-major as the reference's Eigen matrix."""
    ctx = ctx or default_context()
    torch = _torch()
    bc = b.t().contiguous().view(-1) if b.dim() == 2 else b  # column-major flat
    rows = b.shape[0]
    out_dims = list(dims)
    out_dims[mode] = rows
    y = empty(int(np.prod(out_dims)), ctx.device)
    d = _u64(dims)
    torch.cuda.current_stream().synchronize()
    check(lib.lmra_mode_n_product(ctx.handle, _ptr(x), d.ctypes.data_as(_lib.u64p), len(dims), mode,
                                  _ptr(bc), rows, _ptr(y)))
    return y, out_dims


def mode0_product_i8(x, K: int, J: int, q, mu: int, w, ctx: Context = None):
    """y (mu x J, column-major) = q^T x on the int8 tensor cores (lmra_mode0_product_i8);
    x: K x J (columns contiguous), q: K x mu column-major, w: squared column norms of x."""
    ctx = ctx or default_context()
    _torch().cuda.current_stream().synchronize()
    y = empty(mu * J, ctx.device)
    check(lib.lmra_mode0_product_i8(ctx.handle, _ptr(x), K, J, _ptr(q), mu, _ptr(w), _ptr(y)))
    return y


def mode1_product_i8(x, R: int, K: int, O: int, q, mu: int, ctx: Context = None):
    """y (R x mu x O, R fastest) = x x_1 q^T on the int8 tensor cores (lmra_mode1_product_i8);
    x: R x K x O (R fastest), q: K x mu column-major."""
    ctx = ctx or default_context()
    _torch().cuda.current_stream().synchronize()
    y = empty(R * mu * O, ctx.device)
    check(lib.lmra_mode1_product_i8(ctx.handle, _ptr(x), R, K, O, _ptr(q), mu, _ptr(y)))
    return y


def gram_power_apply(a_colmajor, rows: int, cols: int, g_colmajor, s: int, q: int,
                     strategy: str = "A", ctx: Context = None):
    ctx = ctx or default_context()
    _torch().cuda.current_stream().synchronize()
    c = empty(rows * s, ctx.device)
    check(lib.lmra_gram_power_apply(ctx.handle, _ptr(a_colmajor), rows, cols, _ptr(g_colmajor), s, q,
                                    0 if strategy == "A" else 1, _ptr(c)))
    return c


def leading_left_singular_vectors(c_colmajor, rows: int, cols: int, mu: int, ctx: Context = None):
    ctx = ctx or default_context()
    _torch().cuda.current_stream().synchronize()
    u = empty(rows * mu, ctx.device)
    check(lib.lmra_leading_left_singular_vectors(ctx.handle, _ptr(c_colmajor), rows, cols, mu, _ptr(u)))
    return u


def thin_qr_q(c_colmajor, rows: int, cols: int, ctx: Context = None):
    """linalg.cpp:52-60 thin_qr(c).Q on the device (Householder TSQR)."""
    ctx = ctx or default_context()
    _torch().cuda.current_stream().synchronize()
    q = empty(rows * cols, ctx.device)
    check(lib.lmra_thin_qr_q(ctx.handle, _ptr(c_colmajor), rows, cols, _ptr(q)))
    return q


def qr_project_extract(c_colmajor, rows: int, cols: int, a_colmajor, a_cols: int, mu: int,
                       ctx: Context = None):
    """linalg.cpp:89-99: Q U1 with Q = thin_qr(c).Q and U1 the top-mu left singular vectors
    of Q^T a (c: rows x cols, a: rows x a_cols, column-major device buffers)."""
    ctx = ctx or default_context()
    _torch().cuda.current_stream().synchronize()
    out = empty(rows * mu, ctx.device)
    check(lib.lmra_qr_project_extract(ctx.handle, _ptr(c_colmajor), rows, cols, _ptr(a_colmajor), a_cols,
                                      mu, _ptr(out)))
    return out


def column_sqnorms(x, dims: Sequence[int], mode: int, ctx: Context = None):
    ctx = ctx or default_context()
    _torch().cuda.current_stream().synchronize()
    J = int(np.prod(dims)) // int(dims[mode])
    w = empty(J, ctx.device)
    d = _u64(dims)
    check(lib.lmra_column_sqnorms(ctx.handle, _ptr(x), d.ctypes.data_as(_lib.u64p), len(dims), mode,
                                  _ptr(w)))
    return w


def sample_columns(w, regime: str, beta: float, L: int, seed: int, stream: int, ctx: Context = None):
    """Device sampling chain (tucker.cpp:110-130 + sketching.cpp:96-131) on norms w.
    Returns (idx int64, scales, p) as CUDA tensors."""
    ctx = ctx or default_context()
    torch = _torch()
    torch.cuda.current_stream().synchronize()
    n = int(w.numel())
    idx = torch.empty(L, dtype=torch.int64, device=w.device)
    sc = empty(L, ctx.device)
    p = empty(n, ctx.device)
    regime_code = {"optimal": 0, "nearly_optimal": 1, "uniform": 2}[regime]
    check(lib.lmra_sample_columns_device(ctx.handle, _ptr(w), n, regime_code, C.c_double(beta), L,
                                         C.c_uint64(seed), C.c_uint64(stream), _ptr(idx), _ptr(sc),
                                         _ptr(p)))
    return idx, sc, p


# ---------------------------------------------------------------- BASELINE generators
# (definitions: csrc/gen/portable_gen.hpp; the oracle's host generators give the same bits)
def _slab(dims, start, count):
    L = int(dims[-1])
    if count is None:
        start, count = 0, L
    n = int(np.prod(dims[:-1])) * int(count)
    return int(start), int(count), n


def gen_tucker_noise(dims, core_dims, gamma: float, seed: int, ctx: Context = None):
    ctx = ctx or default_context()
    x = empty(int(np.prod(dims)), ctx.device)
    _torch().cuda.current_stream().synchronize()
    check(lib.lmra_gen_tucker_noise(ctx.handle, _u64(dims).ctypes.data_as(_lib.u64p),
                                    _u64(core_dims).ctypes.data_as(_lib.u64p), len(dims),
                                    C.c_double(gamma), C.c_uint64(seed), _ptr(x)))
    return x


def gen_tucker_signal_slab(dims, core_dims, seed: int, start: int, count: int, ctx: Context = None):
    """First half of a slab of the Tucker + noise tensor: (x = signal slab, slice sums of
    squares of the signal and of the noise, host arrays of `count` entries)."""
    ctx = ctx or default_context()
    start, count, n = _slab(dims, start, count)
    x = empty(n, ctx.device)
    nsl = count if len(dims) > 1 else 1
    sb, se = np.empty(nsl), np.empty(nsl)
    _torch().cuda.current_stream().synchronize()
    check(lib.lmra_gen_tucker_signal_slab(ctx.handle, _u64(dims).ctypes.data_as(_lib.u64p),
                                          _u64(core_dims).ctypes.data_as(_lib.u64p), len(dims), C.c_uint64(seed),
                                          start, count, _ptr(x), sb.ctypes.data_as(_lib.dblp),
                                          se.ctypes.data_as(_lib.dblp)))
    return x, sb, se


def noise_coef(slice_b, slice_e, gamma: float) -> float:
    sb, se = np.ascontiguousarray(slice_b, dtype=np.float64), np.ascontiguousarray(slice_e, dtype=np.float64)
    out = C.c_double()
    check(lib.lmra_gen_noise_coef(sb.ctypes.data_as(_lib.dblp), se.ctypes.data_as(_lib.dblp), sb.size,
                                  C.c_double(gamma), C.byref(out)))
    return out.value


def gen_add_noise_slab(x, dims, seed: int, start: int, count: int, coef: float, ctx: Context = None):
    ctx = ctx or default_context()
    start, count, _ = _slab(dims, start, count)
    _torch().cuda.current_stream().synchronize()
    check(lib.lmra_gen_add_noise_slab(ctx.handle, _u64(dims).ctypes.data_as(_lib.u64p), len(dims),
                                      C.c_uint64(seed), start, count, C.c_double(coef), _ptr(x)))
    return x


def gen_hilbert(dims, ctx: Context = None, start: int = 0, count: int = None):
    ctx = ctx or default_context()
    start, count, n = _slab(dims, start, count)
    x = empty(n, ctx.device)
    _torch().cuda.current_stream().synchronize()
    check(lib.lmra_gen_hilbert_slab(ctx.handle, _u64(dims).ctypes.data_as(_lib.u64p), len(dims), start, count,
                                    _ptr(x)))
    return x


def gen_video(dims, n_terms: int = 30, noise: float = 0.05, seed: int = 1, ctx: Context = None,
              start: int = 0, count: int = None):
    ctx = ctx or default_context()
    start, count, n = _slab(dims, start, count)
    x = empty(n, ctx.device)
    _torch().cuda.current_stream().synchronize()
    check(lib.lmra_gen_video_slab(ctx.handle, _u64(dims).ctypes.data_as(_lib.u64p), len(dims),
                                  C.c_uint64(n_terms), C.c_double(noise), C.c_uint64(seed), start, count,
                                  _ptr(x)))
    return x


# ---------------------------------------------------------------- verification
def relative_error(x, dims, core, factors, ctx: Context = None) -> float:
    """||x - reconstruct(core, factors)|| / ||x|| on the device (tucker.cpp:222-240).  x: flat
    float64 CUDA tensor; core (numpy, reference layout) and factors (numpy I_n x mu_n) are
    uploaded.  Used for both sides of the parity checks."""
    ctx = ctx or default_context()
    torch = _torch()
    core = np.asarray(core)
    cdims = list(core.shape)
    rec = empty(int(np.prod(dims)), ctx.device)
    cd = torch.from_numpy(np.ascontiguousarray(core.ravel(order="F"))).cuda(ctx.device)
    fs = [torch.from_numpy(np.ascontiguousarray(np.asarray(f).ravel(order="F"))).cuda(ctx.device)
          for f in factors]
    ptrs = (C.c_void_p * len(fs))(*[f.data_ptr() for f in fs])
    rows = _u64([np.asarray(f).shape[0] for f in factors])
    torch.cuda.current_stream().synchronize()
    check(lib.lmra_reconstruct(ctx.handle, _ptr(cd), _u64(cdims).ctypes.data_as(_lib.u64p), len(cdims), ptrs,
                               rows.ctypes.data_as(_lib.u64p), _lib.LMRA_DEVICE, _ptr(rec), _lib.LMRA_DEVICE))
    out = C.c_double()
    check(lib.lmra_relative_error(ctx.handle, _ptr(x), _ptr(rec), _u64(dims).ctypes.data_as(_lib.u64p), len(dims),
                                  _lib.LMRA_DEVICE, C.byref(out)))
    return out.value


def result_relative_error(result, x, dims, ctx: Context = None) -> float:
    """relative_error of a raw result (run_raw) against the device tensor x it decomposed."""
    ctx = ctx or default_context()
    out = C.c_double()
    _torch().cuda.current_stream().synchronize()
    check(lib.lmra_result_relative_error(ctx.handle, result.handle, _ptr(x), _u64(dims).ctypes.data_as(_lib.u64p),
                                         len(dims), _lib.LMRA_DEVICE, C.byref(out)))
    return out.value

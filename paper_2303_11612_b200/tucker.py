"""Host-side mirror of the reference's Tucker interface (proj/include/lmra/tucker.hpp).

Same names, argument meaning and error behaviour as the reference's C++ API:

    reference (namespace lmra)                       here
    struct AlgoConfig          tucker.hpp:32-45      AlgoConfig
    struct TuckerDecomposition tucker.hpp:27-30      TuckerDecomposition
    rand_thosvd_power          tucker.hpp:91         rand_thosvd_power   (alg1)
    rand_sthosvd_power         tucker.hpp:95         rand_sthosvd_power  (alg2)
    rand_thosvd_amm            tucker.hpp:99         rand_thosvd_amm     (alg4)
    rand_sthosvd_amm           tucker.hpp:102        rand_sthosvd_amm    (alg5)
    run_algorithm              tucker.hpp:110        run_algorithm
    amm_sample_counts          tucker.hpp:116        amm_sample_counts
    parse_algorithm / algorithm_id / all_algorithm_ids (tucker.hpp:59-61)

std::invalid_argument surfaces as LmraInvalidArgument (a ValueError), runtime_error
as LmraError.  Every call goes through the C ABI (include/lmra_b200.h) into the
sm_100a kernels -- there is no CPU path.

Tensor convention: the reference's linearisation, first index fastest
(tensor.hpp:9-12).  A numpy ndarray `a` is read as a[i0, i1, ...] (Fortran-order
flattening); device data is passed as DenseTensor.on_device(ptr_or_torch, dims).
"""
from __future__ import annotations

import ctypes as C
import os
import threading
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _lib
from ._lib import LmraError, LmraInvalidArgument, check, lib

ALGORITHM_IDS = ["thosvd", "sthosvd", "hooi", "alg1", "alg2", "alg4", "alg5", "alg6", "alg7"]
_ALG_CODE = {"alg1": 1, "alg2": 2, "alg4": 4, "alg5": 5, "alg6": 6, "alg7": 7,
             "thosvd": 10, "sthosvd": 11, "hooi": 12}
_REGIME = {"optimal": 0, "nearly_optimal": 1, "uniform": 2}
_STRATEGY = {"A": 0, "B": 1}


def parse_algorithm(name: str) -> Optional[str]:
    """tucker.cpp:190-201 (lmra_parse_algorithm): the id if known, else None."""
    code = C.c_int()
    return name if lib.lmra_parse_algorithm(name.encode(), C.byref(code)) else None


def algorithm_id(a) -> str:
    """tucker.cpp:203-215 (lmra_algorithm_id): id of an algorithm (name or ABI code); "?" if unknown."""
    code = _ALG_CODE.get(a, -1) if isinstance(a, str) else int(a)
    return lib.lmra_algorithm_id(code).decode()


def all_algorithm_ids() -> List[str]:
    """tucker.cpp:217-220 (lmra_all_algorithm_ids), in the reference's order."""
    buf = (C.c_char_p * 16)()
    n = lib.lmra_all_algorithm_ids(buf, 16)
    return [buf[k].decode() for k in range(n)]


def thread_cap() -> int:
    """tucker.cpp:164-172: LMRA_NUM_THREADS, default 1, clamped to [1, 64]."""
    return int(lib.lmra_thread_cap())


def device_cap() -> int:
    """LMRA_NUM_GPUS, default 1, clamped to the visible devices (the multi-GPU knob)."""
    return int(lib.lmra_device_cap())


@dataclass
class AlgoConfig:
    """lmra::AlgoConfig (tucker.hpp:32-45) with the reference's defaults."""
    rank: Sequence[int]
    oversampling: int = 10
    power: int = 1
    alpha: float = 0.2
    regime: str = "uniform"          # "optimal" | "nearly_optimal" | "uniform"
    regime_beta: float = 0.5
    t_samples: Optional[Sequence[int]] = None
    order: Optional[Sequence[int]] = None
    seed: int = 0
    strategy: str = "A"              # GramStrategy
    hooi_max_sweeps: int = 50
    hooi_tol: float = 1e-8

    def _to_c(self):
        if self.regime not in _REGIME:
            raise LmraInvalidArgument(f"unknown probability regime {self.regime!r}")
        if self.strategy not in _STRATEGY:
            raise LmraInvalidArgument(f"unknown Gram strategy {self.strategy!r}")
        keep = []

        def arr(v):
            if v is None:
                return None, 0
            a = np.ascontiguousarray(np.asarray(v, dtype=np.uint64))
            keep.append(a)
            return a.ctypes.data_as(_lib.u64p), a.size

        for name, v in (("rank", self.rank), ("t_samples", self.t_samples), ("order", self.order)):
            if v is not None and any(int(x) < 0 for x in v):
                raise LmraInvalidArgument(f"{name} entries must be non-negative")
        c = _lib.LmraAlgoConfig()
        lib.lmra_algo_config_init(C.byref(c))
        c.rank, c.n_rank = arr(self.rank)
        c.oversampling = int(self.oversampling)
        c.power = int(self.power)
        c.alpha = float(self.alpha)
        c.regime = _REGIME[self.regime]
        c.regime_beta = float(self.regime_beta)
        c.t_samples, c.n_t_samples = arr(self.t_samples)
        c.order, c.n_order = arr(self.order)
        c.seed = int(self.seed)
        c.strategy = _STRATEGY[self.strategy]
        c.hooi_max_sweeps = int(self.hooi_max_sweeps)
        c.hooi_tol = float(self.hooi_tol)
        return c, keep


class DenseTensor:
    """Dense fp64 tensor in the reference's layout (first index fastest).

    Host: `data` is a flat numpy float64 array.  Device: `ptr` is a device address
    (int), optionally with the owning torch tensor kept alive in `owner`.
    """

    def __init__(self, dims: Sequence[int], data: Optional[np.ndarray] = None, ptr: int = 0,
                 owner=None):
        self.dims = [int(d) for d in dims]
        self.data = data
        self.ptr = int(ptr)
        self.owner = owner

    @property
    def on_device(self) -> bool:
        return self.data is None

    @staticmethod
    def from_array(a: np.ndarray) -> "DenseTensor":
        a = np.asarray(a, dtype=np.float64)
        return DenseTensor(list(a.shape), np.ascontiguousarray(a.ravel(order="F")))

    @staticmethod
    def from_flat(flat: np.ndarray, dims: Sequence[int]) -> "DenseTensor":
        flat = np.ascontiguousarray(np.asarray(flat, dtype=np.float64).ravel())
        if flat.size != int(np.prod(dims)):
            raise LmraInvalidArgument("value count does not match tensor shape")
        return DenseTensor(dims, flat)

    @staticmethod
    def device(t, dims: Sequence[int]) -> "DenseTensor":
        """t: a contiguous float64 CUDA torch tensor (any shape; read flat) or a raw pointer."""
        if isinstance(t, int):
            return DenseTensor(dims, None, t)
        if t.dtype.__repr__() != "torch.float64" or not t.is_cuda or not t.is_contiguous():
            raise LmraInvalidArgument("device tensors must be contiguous float64 CUDA tensors")
        if t.numel() != int(np.prod(dims)):
            raise LmraInvalidArgument("value count does not match tensor shape")
        return DenseTensor(dims, None, t.data_ptr(), owner=t)

    def size(self) -> int:
        return int(np.prod(self.dims))

    def to_array(self) -> np.ndarray:
        if self.on_device:
            raise LmraError("device tensor: copy it to the host first")
        return self.data.reshape(self.dims, order="F")


def _tnsr_header(path: str) -> List[int]:
    order = C.c_int()
    dims = np.zeros(64, dtype=np.uint64)
    check(lib.lmra_tnsr_read_header(os.fsencode(path), C.byref(order), dims.ctypes.data_as(_lib.u64p), 64))
    return [int(d) for d in dims[:order.value]]


def load_tensor(path: str, device: bool = False, ctx: Optional["Context"] = None) -> DenseTensor:
    """tensor_io.hpp:13 load_tensor.  device=True streams the values straight into HBM (a
    float64 CUDA torch tensor owned by the returned DenseTensor)."""
    dims = _tnsr_header(path)
    n = int(np.prod(dims)) if dims else 1
    if not device:
        out = np.empty(n, dtype=np.float64)
        check(lib.lmra_tnsr_load(None, os.fsencode(path), out.ctypes.data_as(C.c_void_p), 0))
        return DenseTensor(dims, out)
    import torch
    ctx = ctx or default_context()
    t = torch.empty(n, dtype=torch.float64, device=f"cuda:{ctx.device}")
    torch.cuda.current_stream().synchronize()
    check(lib.lmra_tnsr_load(ctx.handle, os.fsencode(path), C.c_void_p(t.data_ptr()), 1))
    return DenseTensor(dims, None, t.data_ptr(), owner=t)


def save_tensor(path: str, t: DenseTensor, ctx: Optional["Context"] = None) -> None:
    """tensor_io.hpp:12 save_tensor (host or device tensor)."""
    dims = np.asarray(t.dims, dtype=np.uint64)
    if t.on_device:
        ctx = ctx or default_context()
        _torch_sync()
        check(lib.lmra_tnsr_save(ctx.handle, os.fsencode(path), C.c_void_p(t.ptr), 1,
                                 dims.ctypes.data_as(_lib.u64p), len(t.dims)))
    else:
        flat = np.ascontiguousarray(t.data, dtype=np.float64)
        check(lib.lmra_tnsr_save(None, os.fsencode(path), flat.ctypes.data_as(C.c_void_p), 0,
                                 dims.ctypes.data_as(_lib.u64p), len(t.dims)))


def _torch_sync():
    import torch
    torch.cuda.current_stream().synchronize()


@dataclass
class TuckerDecomposition:
    """lmra::TuckerDecomposition (tucker.hpp:27-30) plus the run's trace."""
    core: np.ndarray                     # shape = core dims (a[i0, i1, ...] indexing)
    factors: List[np.ndarray]            # I_n x mu_n, orthonormal columns
    omega: List[np.ndarray] = field(default_factory=list)
    samples: List[Optional[tuple]] = field(default_factory=list)
    norms: List[Optional[np.ndarray]] = field(default_factory=list)
    timings_ms: dict = field(default_factory=dict)


class Context:
    """One lmra_context (device + stream [+ NCCL communicator])."""

    def __init__(self, device: int = 0, stream: Optional[int] = None):
        h = C.c_void_p()
        check(lib.lmra_context_create(int(device), C.c_void_p(stream or 0), C.byref(h)))
        self.handle = h
        self.device = device

    def set_stream(self, stream: int):
        check(lib.lmra_context_set_stream(self.handle, C.c_void_p(stream)))

    def synchronize(self):
        check(lib.lmra_context_synchronize(self.handle))

    def set_trace(self, on: bool):
        """Keep host copies of drawn samples / column norms in results (default on)."""
        check(lib.lmra_context_set_trace(self.handle, int(bool(on))))

    def set_profiling(self, on):
        """Per-launch CUDA events -> _Result.phases(): True / 1 every phase, 2 only the
        phases on the context's own stream (light), 3 only the mode-0 core / shrink
        contraction, False / 0 none."""
        level = on if isinstance(on, int) and not isinstance(on, bool) else int(bool(on))
        check(lib.lmra_context_set_profiling(self.handle, level))

    def set_comm(self, unique_id: bytes, nranks: int, rank: int):
        """NCCL communicator (one process per GPU): later runs on this context are sharded
        along the last mode (this rank's slab = shard_range(dims[-1], nranks, rank))."""
        buf = C.create_string_buffer(bytes(unique_id), 128)
        check(lib.lmra_context_set_comm(self.handle, buf, int(nranks), int(rank)))

    def set_thread_comm(self, group: "ThreadGroup", rank: int):
        """In-process communicator: several ranks as host threads of one process (each with
        its own Context), exchanging through device copies -- the sharded run checked
        rank-for-rank on one GPU."""
        check(lib.lmra_context_set_thread_comm(self.handle, group.handle, int(rank)))
        self._group = group

    def close(self):
        if self.handle:
            lib.lmra_context_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    check(lib.lmra_nccl_unique_id(buf))
    return buf.raw


class ThreadGroup:
    """Rendezvous for Context.set_thread_comm (lmra_thread_group_create)."""

    def __init__(self, nranks: int):
        h = C.c_void_p()
        check(lib.lmra_thread_group_create(int(nranks), C.byref(h)))
        self.handle = h
        self.nranks = int(nranks)

    def __del__(self):
        try:
            if self.handle:
                lib.lmra_thread_group_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


def shard_range(extent: int, nranks: int, rank: int):
    s, c = C.c_uint64(), C.c_uint64()
    check(lib.lmra_shard_range(C.c_uint64(extent), int(nranks), int(rank), C.byref(s), C.byref(c)))
    return s.value, c.value


_default = {}
_default_lock = threading.Lock()


def default_context(device: int = 0) -> Context:
    with _default_lock:
        if device not in _default:
            _default[device] = Context(device)
        return _default[device]


def _overrides(n_modes: int, omega=None, samples=None):
    if omega is None and samples is None:
        return None, []
    keep = []
    ov = _lib.LmraOverrides()
    if omega is not None:
        arr = (_lib.dblp * n_modes)()
        for n, g in enumerate(omega):
            if g is None:
                continue
            gf = np.asfortranarray(np.asarray(g, dtype=np.float64))
            keep.append(gf)
            arr[n] = gf.ctypes.data_as(_lib.dblp)
        keep.append(arr)
        ov.omega = C.cast(arr, C.POINTER(_lib.dblp))
    if samples is not None:
        ia = (_lib.i64p * n_modes)()
        sa = (_lib.dblp * n_modes)()
        na = np.zeros(n_modes, dtype=np.uint64)
        for n, sm in enumerate(samples):
            if sm is None:
                continue
            idx = np.ascontiguousarray(np.asarray(sm[0], dtype=np.int64))
            sc = np.ascontiguousarray(np.asarray(sm[1], dtype=np.float64))
            keep += [idx, sc]
            ia[n] = idx.ctypes.data_as(_lib.i64p)
            sa[n] = sc.ctypes.data_as(_lib.dblp)
            na[n] = idx.size
        keep += [ia, sa, na]
        ov.sample_idx = C.cast(ia, C.POINTER(_lib.i64p))
        ov.sample_scale = C.cast(sa, C.POINTER(_lib.dblp))
        ov.n_samples = na.ctypes.data_as(_lib.u64p)
    return ov, keep


class _Result:
    """Owning wrapper of an lmra_result handle (device-resident core and factors)."""

    def __init__(self, handle, order: int):
        self.handle = handle
        self.order = order

    def core_dims(self):
        d = np.zeros(self.order, dtype=np.uint64)
        lib.lmra_result_core_dims(self.handle, d.ctypes.data_as(_lib.u64p))
        return [int(v) for v in d]

    def factor_dims(self, n):
        r, c = C.c_uint64(), C.c_uint64()
        lib.lmra_result_factor_dims(self.handle, n, C.byref(r), C.byref(c))
        return r.value, c.value

    def core_device_ptr(self) -> int:
        return lib.lmra_result_core_device(self.handle) or 0

    def factor_device_ptr(self, n) -> int:
        return lib.lmra_result_factor_device(self.handle, n) or 0

    def to_host(self, with_trace: bool = True) -> TuckerDecomposition:
        cd = self.core_dims()
        core = np.empty(int(np.prod(cd)))
        check(lib.lmra_result_copy_core(self.handle, C.c_void_p(core.ctypes.data), _lib.LMRA_HOST))
        factors, omega, samples, norms = [], [], [], []
        for n in range(self.order):
            r, c = self.factor_dims(n)
            f = np.empty(r * c)
            check(lib.lmra_result_copy_factor(self.handle, n, C.c_void_p(f.ctypes.data), _lib.LMRA_HOST))
            factors.append(f.reshape((r, c), order="F"))
            if with_trace:
                orow, ocol = C.c_uint64(), C.c_uint64()
                lib.lmra_result_omega_dims(self.handle, n, C.byref(orow), C.byref(ocol))
                g = np.empty(orow.value * ocol.value)
                if g.size:
                    lib.lmra_result_copy_omega(self.handle, n, g.ctypes.data_as(_lib.dblp))
                omega.append(g.reshape((orow.value, ocol.value), order="F"))
                T = lib.lmra_result_num_samples(self.handle, n)
                if T:
                    idx = np.empty(T, dtype=np.int64)
                    sc = np.empty(T)
                    lib.lmra_result_copy_samples(self.handle, n, idx.ctypes.data_as(_lib.i64p),
                                                 sc.ctypes.data_as(_lib.dblp))
                    samples.append((idx, sc))
                else:
                    samples.append(None)
                W = lib.lmra_result_num_norms(self.handle, n)
                if W:
                    w = np.empty(W)
                    lib.lmra_result_copy_norms(self.handle, n, w.ctypes.data_as(_lib.dblp))
                    norms.append(w)
                else:
                    norms.append(None)
        return TuckerDecomposition(core.reshape(cd, order="F"), factors, omega, samples, norms,
                                   self.timings())

    def phases(self) -> dict:
        """{phase: (device ms, launches)} for profiling contexts."""
        out = {}
        buf = C.create_string_buffer(64)
        for i in range(lib.lmra_result_num_phases(self.handle)):
            ms, cnt = C.c_double(), C.c_int()
            check(lib.lmra_result_phase(self.handle, i, buf, 64, C.byref(ms), C.byref(cnt)))
            out[buf.value.decode()] = (ms.value, cnt.value)
        return out

    def timings(self) -> dict:
        t = np.zeros(5)
        lib.lmra_result_timings(self.handle, t.ctypes.data_as(_lib.dblp))
        return {"total_ms": t[0], "host_rng_ms": t[1], "host_sampling_ms": t[2],
                "device_ms": t[3], "launches": int(t[4])}

    def free(self):
        if self.handle:
            lib.lmra_result_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def _as_tensor(a) -> DenseTensor:
    if isinstance(a, DenseTensor):
        return a
    return DenseTensor.from_array(np.asarray(a))


def run_raw(alg: str, a, cfg: AlgoConfig, *, ctx: Optional[Context] = None, omega=None,
            samples=None, trace: bool = False,
            global_dims: Optional[Sequence[int]] = None) -> _Result:
    """run_algorithm returning the device-resident result handle (no copy-out).
    trace=True also keeps host copies of the drawn samples and column norms.
    global_dims: on a sharded context `a` is this rank's slab of the last mode and
    global_dims the whole tensor's dims (default: a's own dims, i.e. unsharded)."""
    if alg not in _ALG_CODE:
        raise LmraInvalidArgument("unknown algorithm")
    t = _as_tensor(a)
    ctx = ctx or default_context()
    ctx.set_trace(trace)
    dims = np.asarray(t.dims if global_dims is None else list(global_dims), dtype=np.uint64)
    if global_dims is not None:
        if len(global_dims) != len(t.dims) or list(global_dims[:-1]) != list(t.dims[:-1]):
            raise LmraInvalidArgument("slab dims must equal the global dims except the last")
    c, keep = cfg._to_c()
    ov, keep2 = _overrides(len(t.dims), omega, samples)
    h = C.c_void_p()
    if t.on_device:
        xp, loc = C.c_void_p(t.ptr), _lib.LMRA_DEVICE
    else:
        xp, loc = C.c_void_p(t.data.ctypes.data), _lib.LMRA_HOST
    rc = lib.lmra_run_algorithm(ctx.handle, _ALG_CODE[alg], xp, dims.ctypes.data_as(_lib.u64p),
                                len(t.dims), loc, C.byref(c), C.byref(ov) if ov is not None else None,
                                C.byref(h))
    del keep, keep2
    check(rc)
    return _Result(h, len(t.dims))


def run_algorithm(alg: str, a, cfg: AlgoConfig, *, ctx: Optional[Context] = None, omega=None,
                  samples=None, trace: bool = True,
                  global_dims: Optional[Sequence[int]] = None) -> TuckerDecomposition:
    """tucker.cpp:456-470.  omega / samples: per-mode parity overrides (None = seeded RNG).
    trace: also return the drawn samples / column norms (host copies).
    global_dims: sharded contexts only (see run_raw)."""
    r = run_raw(alg, a, cfg, ctx=ctx, omega=omega, samples=samples, trace=trace,
                global_dims=global_dims)
    try:
        return r.to_host()
    finally:
        r.free()


def rand_thosvd_power(a, cfg: AlgoConfig, **kw) -> TuckerDecomposition:
    return run_algorithm("alg1", a, cfg, **kw)


def rand_sthosvd_power(a, cfg: AlgoConfig, **kw) -> TuckerDecomposition:
    return run_algorithm("alg2", a, cfg, **kw)


def rand_thosvd_amm(a, cfg: AlgoConfig, **kw) -> TuckerDecomposition:
    return run_algorithm("alg4", a, cfg, **kw)


def rand_sthosvd_amm(a, cfg: AlgoConfig, **kw) -> TuckerDecomposition:
    return run_algorithm("alg5", a, cfg, **kw)


def rand_thosvd_power_qr(a, cfg: AlgoConfig, **kw) -> TuckerDecomposition:
    """tucker.cpp:422-436 (alg6): power-scheme sketch, QR-proxy extraction."""
    return run_algorithm("alg6", a, cfg, **kw)


def rand_sthosvd_power_qr(a, cfg: AlgoConfig, **kw) -> TuckerDecomposition:
    """tucker.cpp:438-454 (alg7): sequential modes, QR-proxy extraction."""
    return run_algorithm("alg7", a, cfg, **kw)


def t_hosvd(a, cfg: AlgoConfig, **kw) -> TuckerDecomposition:
    """tucker.cpp:242-248: factors from the full unfoldings (deterministic baseline)."""
    return run_algorithm("thosvd", a, cfg, **kw)


def st_hosvd(a, cfg: AlgoConfig, **kw) -> TuckerDecomposition:
    """tucker.cpp:250-259: sequentially truncated HOSVD (deterministic baseline)."""
    return run_algorithm("sthosvd", a, cfg, **kw)


def hooi(a, cfg: AlgoConfig, **kw) -> TuckerDecomposition:
    """tucker.cpp:261-316: higher-order orthogonal iteration from the st_hosvd start; stops when
    |delta ||core||| / ||a|| < cfg.hooi_tol or after cfg.hooi_max_sweeps sweeps."""
    return run_algorithm("hooi", a, cfg, **kw)


def run_raw_multigpu(alg: str, a, cfg: AlgoConfig, devices: Sequence[int]) -> "_Result":
    """run_algorithm on several devices from this process (lmra_run_algorithm_multigpu): one
    host thread and context per device, the tensor split along its last mode.  `a`: host
    DenseTensor / ndarray, or a device tensor on devices[0]."""
    if alg not in _ALG_CODE:
        raise LmraInvalidArgument("unknown algorithm")
    t = _as_tensor(a)
    dims = np.asarray(t.dims, dtype=np.uint64)
    devs = (C.c_int * len(devices))(*[int(d) for d in devices])
    c, keep = cfg._to_c()
    h = C.c_void_p()
    if t.on_device:
        xp, loc = C.c_void_p(t.ptr), _lib.LMRA_DEVICE
    else:
        xp, loc = C.c_void_p(t.data.ctypes.data), _lib.LMRA_HOST
    _torch_sync()
    rc = lib.lmra_run_algorithm_multigpu(len(devices), devs, _ALG_CODE[alg], xp, dims.ctypes.data_as(_lib.u64p),
                                         len(t.dims), loc, C.byref(c), None, C.byref(h))
    del keep
    check(rc)
    return _Result(h, len(t.dims))


def amm_sample_counts(dims: Sequence[int], cfg: AlgoConfig, sequential: bool) -> List[int]:
    d = np.asarray(dims, dtype=np.uint64)
    out = np.zeros(len(dims), dtype=np.uint64)
    c, keep = cfg._to_c()
    check(lib.lmra_amm_sample_counts(d.ctypes.data_as(_lib.u64p), len(dims), C.byref(c),
                                     int(bool(sequential)), out.ctypes.data_as(_lib.u64p)))
    return [int(v) for v in out]


# ---------------------------------------------------------------- host restatements on the path
def gaussian_matrix(rows: int, cols: int, seed: int, stream: int) -> np.ndarray:
    out = np.empty(rows * cols)
    check(lib.lmra_gaussian_matrix(rows, cols, seed, stream, out.ctypes.data_as(_lib.dblp)))
    return out.reshape((rows, cols), order="F")


def probabilities(w, regime: str, beta: float = 0.5) -> np.ndarray:
    w = np.ascontiguousarray(np.asarray(w, dtype=np.float64))
    p = np.empty_like(w)
    check(lib.lmra_probabilities(w.ctypes.data_as(_lib.dblp), w.size, _REGIME[regime], beta,
                                 p.ctypes.data_as(_lib.dblp)))
    return p


def randsample(L: int, p, seed: int, stream: int):
    p = np.ascontiguousarray(np.asarray(p, dtype=np.float64))
    idx = np.empty(L, dtype=np.int64)
    sc = np.empty(L)
    check(lib.lmra_randsample(L, p.ctypes.data_as(_lib.dblp), p.size, seed, stream,
                              idx.ctypes.data_as(_lib.i64p), sc.ctypes.data_as(_lib.dblp)))
    return idx, sc

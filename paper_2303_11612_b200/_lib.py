"""ctypes binding of the C ABI (include/lmra_b200.h) -> paper_2303_11612_b200/lib/liblmra_b200.so.

The product path has no CPU fallback: if the shared library is missing or cannot
be loaded this module raises, loudly, at import.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "liblmra_b200.so")

u64p = C.POINTER(C.c_uint64)
i64p = C.POINTER(C.c_int64)
dblp = C.POINTER(C.c_double)
vp = C.c_void_p

LMRA_OK, LMRA_EINVAL, LMRA_ERUNTIME, LMRA_ECUDA = 0, 1, 2, 3
LMRA_HOST, LMRA_DEVICE = 0, 1


class LmraAlgoConfig(C.Structure):
    _fields_ = [
        ("rank", u64p), ("n_rank", C.c_uint64), ("oversampling", C.c_uint64), ("power", C.c_int32),
        ("alpha", C.c_double), ("regime", C.c_int32), ("regime_beta", C.c_double),
        ("t_samples", u64p), ("n_t_samples", C.c_uint64), ("order", u64p), ("n_order", C.c_uint64),
        ("seed", C.c_uint64), ("strategy", C.c_int32), ("hooi_max_sweeps", C.c_int32), ("hooi_tol", C.c_double),
    ]


class LmraOverrides(C.Structure):
    _fields_ = [
        ("omega", C.POINTER(dblp)), ("sample_idx", C.POINTER(i64p)),
        ("sample_scale", C.POINTER(dblp)), ("n_samples", u64p),
    ]


class LmraError(RuntimeError):
    """runtime_error / CUDA failure surfaced through the C ABI."""


class LmraInvalidArgument(LmraError, ValueError):
    """std::invalid_argument of the reference (tucker.cpp / linalg.cpp checks)."""


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(make -C paper_2303_11612_b200/csrc). There is no CPU fallback.")
    L = C.CDLL(LIB_PATH)
    sig = {
        "lmra_last_error": (C.c_char_p, []),
        "lmra_version": (C.c_char_p, []),
        "lmra_algo_config_init": (None, [C.POINTER(LmraAlgoConfig)]),
        "lmra_context_create": (C.c_int, [C.c_int, vp, C.POINTER(vp)]),
        "lmra_context_destroy": (None, [vp]),
        "lmra_context_set_stream": (C.c_int, [vp, vp]),
        "lmra_context_synchronize": (C.c_int, [vp]),
        "lmra_nccl_unique_id": (C.c_int, [vp]),
        "lmra_context_set_comm": (C.c_int, [vp, vp, C.c_int, C.c_int]),
        "lmra_shard_range": (C.c_int, [C.c_uint64, C.c_int, C.c_int, u64p, u64p]),
        "lmra_thread_group_create": (C.c_int, [C.c_int, C.POINTER(vp)]),
        "lmra_thread_group_destroy": (None, [vp]),
        "lmra_context_set_thread_comm": (C.c_int, [vp, vp, C.c_int]),
        "lmra_run_algorithm": (C.c_int, [vp, C.c_int, vp, u64p, C.c_int, C.c_int,
                                         C.POINTER(LmraAlgoConfig), C.POINTER(LmraOverrides),
                                         C.POINTER(vp)]),
        "lmra_result_order": (C.c_int, [vp]),
        "lmra_result_hooi_stats": (None, [vp, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
        "lmra_result_core_dims": (None, [vp, u64p]),
        "lmra_result_copy_core": (C.c_int, [vp, vp, C.c_int]),
        "lmra_result_factor_dims": (None, [vp, C.c_int, u64p, u64p]),
        "lmra_result_copy_factor": (C.c_int, [vp, C.c_int, vp, C.c_int]),
        "lmra_result_core_device": (vp, [vp]),
        "lmra_result_factor_device": (vp, [vp, C.c_int]),
        "lmra_result_omega_dims": (None, [vp, C.c_int, u64p, u64p]),
        "lmra_result_copy_omega": (C.c_int, [vp, C.c_int, dblp]),
        "lmra_result_num_samples": (C.c_uint64, [vp, C.c_int]),
        "lmra_result_copy_samples": (C.c_int, [vp, C.c_int, i64p, dblp]),
        "lmra_result_num_norms": (C.c_uint64, [vp, C.c_int]),
        "lmra_result_copy_norms": (C.c_int, [vp, C.c_int, dblp]),
        "lmra_result_timings": (C.c_int, [vp, dblp]),
        "lmra_result_free": (None, [vp]),
        "lmra_context_set_profiling": (C.c_int, [vp, C.c_int]),
        "lmra_context_set_trace": (C.c_int, [vp, C.c_int]),
        "lmra_sample_columns_device": (C.c_int, [vp, vp, C.c_uint64, C.c_int, C.c_double, C.c_uint64,
                                                 C.c_uint64, C.c_uint64, vp, vp, vp]),
        "lmra_result_num_phases": (C.c_int, [vp]),
        "lmra_result_phase": (C.c_int, [vp, C.c_int, C.c_char_p, C.c_size_t, dblp,
                                        C.POINTER(C.c_int)]),
        "lmra_mode_n_product": (C.c_int, [vp, vp, u64p, C.c_int, C.c_int, vp, C.c_uint64, vp]),
        "lmra_mode0_product_i8": (C.c_int, [vp, vp, C.c_uint64, C.c_uint64, vp, C.c_int, vp, vp]),
        "lmra_mode1_product_i8": (C.c_int, [vp, vp, C.c_uint64, C.c_uint64, C.c_uint64, vp, C.c_int, vp]),
        "lmra_gram_power_apply": (C.c_int, [vp, vp, C.c_uint64, C.c_uint64, vp, C.c_uint64,
                                            C.c_int, C.c_int, vp]),
        "lmra_leading_left_singular_vectors": (C.c_int, [vp, vp, C.c_uint64, C.c_uint64,
                                                         C.c_uint64, vp]),
        "lmra_thin_qr_q": (C.c_int, [vp, vp, C.c_uint64, C.c_uint64, vp]),
        "lmra_tnsr_read_header": (C.c_int, [C.c_char_p, C.POINTER(C.c_int), u64p, C.c_int]),
        "lmra_tnsr_load": (C.c_int, [vp, C.c_char_p, vp, C.c_int]),
        "lmra_tnsr_save": (C.c_int, [vp, C.c_char_p, vp, C.c_int, u64p, C.c_int]),
        "lmra_qr_project_extract": (C.c_int, [vp, vp, C.c_uint64, C.c_uint64, vp, C.c_uint64,
                                              C.c_uint64, vp]),
        "lmra_column_sqnorms": (C.c_int, [vp, vp, u64p, C.c_int, C.c_int, vp]),
        "lmra_gaussian_matrix": (C.c_int, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, dblp]),
        "lmra_probabilities": (C.c_int, [dblp, C.c_uint64, C.c_int, C.c_double, dblp]),
        "lmra_randsample": (C.c_int, [C.c_uint64, dblp, C.c_uint64, C.c_uint64, C.c_uint64, i64p,
                                      dblp]),
        "lmra_amm_sample_counts": (C.c_int, [u64p, C.c_int, C.POINTER(LmraAlgoConfig), C.c_int,
                                             u64p]),
        "lmra_gen_tucker_noise": (C.c_int, [vp, u64p, u64p, C.c_int, C.c_double, C.c_uint64, vp]),
        "lmra_gen_hilbert": (C.c_int, [vp, u64p, C.c_int, vp]),
        "lmra_gen_video": (C.c_int, [vp, u64p, C.c_int, C.c_uint64, C.c_double, C.c_uint64, vp]),
        "lmra_gen_tucker_signal_slab": (C.c_int, [vp, u64p, u64p, C.c_int, C.c_uint64, C.c_uint64, C.c_uint64,
                                                  vp, dblp, dblp]),
        "lmra_gen_noise_coef": (C.c_int, [dblp, dblp, C.c_uint64, C.c_double, dblp]),
        "lmra_gen_add_noise_slab": (C.c_int, [vp, u64p, C.c_int, C.c_uint64, C.c_uint64, C.c_uint64,
                                              C.c_double, vp]),
        "lmra_gen_hilbert_slab": (C.c_int, [vp, u64p, C.c_int, C.c_uint64, C.c_uint64, vp]),
        "lmra_gen_video_slab": (C.c_int, [vp, u64p, C.c_int, C.c_uint64, C.c_double, C.c_uint64, C.c_uint64,
                                          C.c_uint64, vp]),
        "lmra_reconstruct": (C.c_int, [vp, vp, u64p, C.c_int, C.POINTER(vp), u64p, C.c_int, vp, C.c_int]),
        "lmra_relative_error": (C.c_int, [vp, vp, vp, u64p, C.c_int, C.c_int, dblp]),
        "lmra_result_relative_error": (C.c_int, [vp, vp, vp, u64p, C.c_int, C.c_int, dblp]),
        "lmra_parse_algorithm": (C.c_int, [C.c_char_p, C.POINTER(C.c_int)]),
        "lmra_algorithm_id": (C.c_char_p, [C.c_int]),
        "lmra_all_algorithm_ids": (C.c_int, [C.POINTER(C.c_char_p), C.c_int]),
        "lmra_thread_cap": (C.c_int, []),
        "lmra_device_cap": (C.c_int, []),
        "lmra_run_algorithm_multigpu": (C.c_int, [C.c_int, C.POINTER(C.c_int), C.c_int, vp, u64p, C.c_int, C.c_int,
                                                  C.POINTER(LmraAlgoConfig), C.POINTER(LmraOverrides),
                                                  C.POINTER(vp)]),
        "lmra_device_alloc": (C.c_int, [vp, C.c_size_t, C.POINTER(vp)]),
        "lmra_device_free": (C.c_int, [vp, vp]),
        "lmra_memcpy": (C.c_int, [vp, vp, vp, C.c_size_t, C.c_int, C.c_int]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    return L


lib = _load()

# every symbol include/lmra_b200.h declares (checked by tests/test_abi.py)
EXPORTED = [
    "lmra_last_error", "lmra_version", "lmra_algo_config_init", "lmra_context_create",
    "lmra_context_destroy", "lmra_context_set_stream", "lmra_context_synchronize",
    "lmra_nccl_unique_id", "lmra_context_set_comm", "lmra_shard_range", "lmra_run_algorithm",
    "lmra_thread_group_create", "lmra_thread_group_destroy", "lmra_context_set_thread_comm",
    "lmra_result_order", "lmra_result_core_dims", "lmra_result_copy_core",
    "lmra_result_factor_dims", "lmra_result_copy_factor", "lmra_result_core_device",
    "lmra_result_factor_device", "lmra_result_omega_dims", "lmra_result_copy_omega",
    "lmra_result_num_samples", "lmra_result_copy_samples", "lmra_result_num_norms",
    "lmra_result_copy_norms", "lmra_result_timings", "lmra_result_free",
    "lmra_context_set_profiling", "lmra_result_num_phases", "lmra_result_phase",
    "lmra_context_set_trace", "lmra_sample_columns_device",
    "lmra_mode_n_product", "lmra_mode0_product_i8", "lmra_mode1_product_i8",
    "lmra_gram_power_apply", "lmra_leading_left_singular_vectors", "lmra_column_sqnorms",
    "lmra_thin_qr_q", "lmra_qr_project_extract", "lmra_tnsr_read_header", "lmra_tnsr_load",
    "lmra_tnsr_save",
    "lmra_gaussian_matrix", "lmra_probabilities", "lmra_randsample", "lmra_amm_sample_counts",
    "lmra_gen_tucker_noise", "lmra_gen_hilbert", "lmra_gen_video", "lmra_device_alloc",
    "lmra_gen_tucker_signal_slab", "lmra_gen_noise_coef", "lmra_gen_add_noise_slab", "lmra_gen_hilbert_slab",
    "lmra_gen_video_slab", "lmra_reconstruct", "lmra_relative_error", "lmra_result_relative_error",
    "lmra_parse_algorithm", "lmra_algorithm_id", "lmra_all_algorithm_ids", "lmra_thread_cap", "lmra_device_cap",
    "lmra_run_algorithm_multigpu", "lmra_result_hooi_stats",
    "lmra_device_free", "lmra_memcpy",
]


def check(rc: int):
    if rc != LMRA_OK:
        msg = lib.lmra_last_error().decode()
        if rc == LMRA_EINVAL:
            raise LmraInvalidArgument(msg)
        raise LmraError(msg)

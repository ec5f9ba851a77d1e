"""paper_2303_11612_b200 -- B200-native randomized Tucker (T-HOSVD / ST-HOSVD, power scheme
and AMM column sampling, QR-proxy extraction) behind the reference lmra API.  See DESIGN.md."""
from .tucker import (  # noqa: F401
    AlgoConfig, Context, DenseTensor, TuckerDecomposition, all_algorithm_ids, algorithm_id,
    amm_sample_counts, default_context, gaussian_matrix, nccl_unique_id, parse_algorithm,
    probabilities, rand_sthosvd_amm, rand_sthosvd_power, rand_sthosvd_power_qr, rand_thosvd_amm,
    rand_thosvd_power, rand_thosvd_power_qr,
    randsample, run_algorithm, run_raw, shard_range, ThreadGroup, load_tensor, save_tensor,
    t_hosvd, st_hosvd, hooi, thread_cap, device_cap, run_raw_multigpu,
)
from ._lib import LmraError, LmraInvalidArgument, LIB_PATH  # noqa: F401
from . import device  # noqa: F401

/* lmra_b200.h -- C ABI of the B200-native randomized Tucker hot path.
 *
 * Drop-in boundary for the reference's C++ entry points (namespace lmra,
 * /root/reference/proj/include/lmra/tucker.hpp).  Plain pointers and sizes only;
 * no torch, Eigen or CUDA types in the signatures (streams are `void*`).
 *
 *   reference (tucker.hpp)                              this ABI
 *   rand_thosvd_power   (tucker.hpp:91)       alg1  ->  lmra_run_algorithm(LMRA_ALG1, ...)
 *   rand_sthosvd_power  (tucker.hpp:95)       alg2  ->  lmra_run_algorithm(LMRA_ALG2, ...)
 *   rand_thosvd_amm     (tucker.hpp:99)       alg4  ->  lmra_run_algorithm(LMRA_ALG4, ...)
 *   rand_sthosvd_amm    (tucker.hpp:102)      alg5  ->  lmra_run_algorithm(LMRA_ALG5, ...)
 *   run_algorithm       (tucker.hpp:110-111)        ->  lmra_run_algorithm
 *   amm_sample_counts   (tucker.hpp:116-117)        ->  lmra_amm_sample_counts
 *   thread_cap          (tucker.hpp:121)            ->  lmra_thread_cap (+ lmra_device_cap: LMRA_NUM_GPUS)
 *   parse_algorithm / algorithm_id / all_algorithm_ids (tucker.hpp:59-61) -> lmra_parse_algorithm, ...
 *   t_hosvd / st_hosvd / hooi (tucker.hpp:70-89)    ->  lmra_run_algorithm(LMRA_THOSVD / STHOSVD / HOOI)
 *   AlgoConfig          (tucker.hpp:32-45)          ->  lmra_algo_config
 *   TuckerDecomposition (tucker.hpp:27-30)          ->  lmra_result (core + factors)
 *   mode_n_product      (tensor.hpp:56-57)          ->  lmra_mode_n_product
 *   gram_power_apply    (linalg.hpp:37-38)          ->  lmra_gram_power_apply
 *   leading_left_singular_vectors (linalg.hpp:41)   ->  lmra_leading_left_singular_vectors
 *   thin_qr             (linalg.hpp:35)             ->  lmra_thin_qr_q
 *   qr_project_extract  (linalg.hpp:43-46)          ->  lmra_qr_project_extract
 *   load_tensor / save_tensor (tensor_io.hpp:12-13) ->  lmra_tnsr_load / lmra_tnsr_save
 *   gaussian_matrix     (sketching.hpp:69)          ->  lmra_gaussian_matrix
 *   randsample          (sketching.hpp:56)          ->  lmra_randsample
 *   gram_sampling_probabilities (tucker.cpp:110-130)->  lmra_column_sqnorms + lmra_probabilities
 *   reconstruct         (tucker.hpp:63)             ->  lmra_reconstruct
 *   relative_error      (tucker.hpp:66)             ->  lmra_relative_error / lmra_result_relative_error
 *
 * Tensors are dense fp64 with the reference's linearisation: first index fastest
 * (tensor.hpp:9-12).  Matrices are column-major (Eigen default).
 *
 * Errors (tucker.cpp / linalg.cpp exception surface): every int-returning call
 * returns LMRA_OK or an error code; lmra_last_error() gives the thread's message.
 *   LMRA_EINVAL   <-> std::invalid_argument  (bad rank length, power < 1, bad order,
 *                                             alpha outside (0,1), t < 1, ...)
 *   LMRA_ERUNTIME <-> std::runtime_error     (SVD did not converge)
 *   LMRA_ECUDA    CUDA / NCCL failure
 * Rank clamping is a warning on stderr, as in the reference (tucker.cpp:65-72,185-186).
 */
#ifndef LMRA_B200_H
#define LMRA_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum lmra_status { LMRA_OK = 0, LMRA_EINVAL = 1, LMRA_ERUNTIME = 2, LMRA_ECUDA = 3 };
/* Algorithm ids (tucker.hpp:47-57). The randomized family: power scheme (alg1/alg2), AMM
 * (alg4/alg5) and the QR-proxy extraction (alg6/alg7, tucker.cpp:422-454). */
enum lmra_algorithm {
  LMRA_ALG1 = 1, LMRA_ALG2 = 2, LMRA_ALG4 = 4, LMRA_ALG5 = 5, LMRA_ALG6 = 6, LMRA_ALG7 = 7,
  /* the deterministic baselines (tucker.cpp:242-316): factors from the full unfoldings */
  LMRA_THOSVD = 10, LMRA_STHOSVD = 11, LMRA_HOOI = 12
};
/* ProbRegime (sketching.hpp:31) */
enum lmra_regime { LMRA_OPTIMAL = 0, LMRA_NEARLY_OPTIMAL = 1, LMRA_UNIFORM = 2 };
/* GramStrategy (linalg.hpp:26) */
enum lmra_strategy { LMRA_STRATEGY_A = 0, LMRA_STRATEGY_B = 1 };
/* where a buffer lives */
enum lmra_location { LMRA_HOST = 0, LMRA_DEVICE = 1 };

/* AlgoConfig (tucker.hpp:32-45); arrays may be NULL with length 0 = "empty vector". */
typedef struct {
  const uint64_t* rank;       /* MultilinearRank::mu */
  uint64_t n_rank;
  uint64_t oversampling;      /* default 10 */
  int32_t power;              /* q, default 1 */
  double alpha;               /* default 0.2 */
  int32_t regime;             /* lmra_regime, default LMRA_UNIFORM */
  double regime_beta;         /* default 0.5 */
  const uint64_t* t_samples;  /* per-mode sample counts or NULL */
  uint64_t n_t_samples;
  const uint64_t* order;      /* processing order (0-based) or NULL */
  uint64_t n_order;
  uint64_t seed;              /* default 0 */
  int32_t strategy;           /* lmra_strategy, default A */
  int32_t hooi_max_sweeps;    /* default 50 */
  double hooi_tol;            /* default 1e-8 */
} lmra_algo_config;

/* Fills the reference's defaults (tucker.hpp:32-45). */
void lmra_algo_config_init(lmra_algo_config* cfg);

/* parse_algorithm / algorithm_id / all_algorithm_ids (tucker.hpp:59-61, tucker.cpp:190-220):
 * lmra_parse_algorithm returns 1 and sets *algorithm for a known id ("thosvd", "sthosvd",
 * "hooi", "alg1" ... "alg7"), else 0; lmra_algorithm_id returns "?" for an unknown code;
 * lmra_all_algorithm_ids fills up to max_ids ids in the reference's order and returns 9. */
int lmra_parse_algorithm(const char* id, int* algorithm);
const char* lmra_algorithm_id(int algorithm);
int lmra_all_algorithm_ids(const char** ids, int max_ids);
/* thread_cap (tucker.hpp:121, tucker.cpp:164-172): LMRA_NUM_THREADS, default 1, in [1, 64].
 * lmra_device_cap: the same idiom for devices, LMRA_NUM_GPUS, default 1, clamped to the
 * visible device count -- the C++ drop-in (lmra_b200.hpp) runs on that many GPUs. */
int lmra_thread_cap(void);
int lmra_device_cap(void);

/* Parity overrides: per-mode Omega (I_n x s, column-major, host) and per-mode sampled
 * columns (indices + scales, host).  NULL arrays / NULL entries mean "draw them from
 * the seeded host RNG as the reference does".  Sample indices are columns of the mode-n
 * unfolding of the tensor as it is when that mode is processed. */
typedef struct {
  const double* const* omega;        /* [order] or NULL */
  const int64_t* const* sample_idx;  /* [order] or NULL */
  const double* const* sample_scale; /* [order] or NULL */
  const uint64_t* n_samples;         /* [order] or NULL */
} lmra_overrides;

typedef struct lmra_context lmra_context;
typedef struct lmra_result lmra_result;

const char* lmra_last_error(void);
const char* lmra_version(void);

/* One context per (process, device).  stream == NULL -> the context creates its own. */
int lmra_context_create(int device, void* stream, lmra_context** out);
void lmra_context_destroy(lmra_context* ctx);
int lmra_context_set_stream(lmra_context* ctx, void* stream);
int lmra_context_synchronize(lmra_context* ctx);

/* Multi-GPU (one process per GPU).  The tensor passed to lmra_run_algorithm is then
 * this rank's slab along the LAST mode (rows [start, start+count) of that mode, see
 * lmra_shard_range); dims[] are the GLOBAL dims.  Small sketch / Gram / norm partials
 * are combined with NCCL all-reduce / all-gather over NVLink. */
int lmra_nccl_unique_id(void* out128);
int lmra_context_set_comm(lmra_context* ctx, const void* unique_id128, int nranks, int rank);
/* In-process rank group: each rank is a host thread with its own context (any devices);
 * collectives are device copies + host barriers.  Used to check the sharded path with
 * several ranks on one GPU; NCCL (lmra_context_set_comm) is the multi-GPU product path. */
int lmra_thread_group_create(int nranks, void** group);
void lmra_thread_group_destroy(void* group);
int lmra_context_set_thread_comm(lmra_context* ctx, void* group, int rank);
/* Shard plan: contiguous balanced slabs, rank r owns [start, start + count). */
int lmra_shard_range(uint64_t extent, int nranks, int rank, uint64_t* start, uint64_t* count);

/* run_algorithm (tucker.cpp:456-470) for every algorithm id. x: dense tensor on the host
 * (x_location = LMRA_HOST, copied in) or device (LMRA_DEVICE, read in place, never
 * mutated).  The call returns once the result is complete on the device. */
int lmra_run_algorithm(lmra_context* ctx, int algorithm, const double* x, const uint64_t* dims,
                       int order, int x_location, const lmra_algo_config* cfg,
                       const lmra_overrides* overrides, lmra_result** out);

/* The same on ndev devices from ONE process (one host thread and context per device, the
 * tensor split along its last mode as with one process per GPU; NCCL between distinct
 * devices, else the in-process communicator).  x: the whole tensor on the host, or on
 * devices[0] (x_location = LMRA_DEVICE; each rank's slab is copied peer to peer).  The
 * result lives on devices[0]. */
int lmra_run_algorithm_multigpu(int ndev, const int* devices, int algorithm, const double* x, const uint64_t* dims,
                                int order, int x_location, const lmra_algo_config* cfg,
                                const lmra_overrides* overrides, lmra_result** out);

int lmra_result_order(const lmra_result* r);
/* HooiStats (tucker.hpp:73-76) of a hooi run: converged flag and sweeps taken (0, 0 otherwise) */
void lmra_result_hooi_stats(const lmra_result* r, int* converged, int* sweeps);
void lmra_result_core_dims(const lmra_result* r, uint64_t* dims);
int lmra_result_copy_core(const lmra_result* r, double* dst, int dst_location);
void lmra_result_factor_dims(const lmra_result* r, int mode, uint64_t* rows, uint64_t* cols);
int lmra_result_copy_factor(const lmra_result* r, int mode, double* dst, int dst_location);
const double* lmra_result_core_device(const lmra_result* r);
const double* lmra_result_factor_device(const lmra_result* r, int mode);
/* trace of the draws this run used (host copies) */
void lmra_result_omega_dims(const lmra_result* r, int mode, uint64_t* rows, uint64_t* cols);
int lmra_result_copy_omega(const lmra_result* r, int mode, double* dst);
uint64_t lmra_result_num_samples(const lmra_result* r, int mode);
int lmra_result_copy_samples(const lmra_result* r, int mode, int64_t* idx, double* scales);
uint64_t lmra_result_num_norms(const lmra_result* r, int mode);
int lmra_result_copy_norms(const lmra_result* r, int mode, double* w);
/* phase timings of the run (milliseconds): [0] total wall, [1] host RNG (Omega),
 * [2] host sampling chains, [3] device time of the run (events), [4] kernel launches */
int lmra_result_timings(const lmra_result* r, double* out5);
/* per-phase device time (CUDA events around each launch), only recorded when
 * lmra_context_set_profiling(ctx, 1) (every phase), (ctx, 2) (light: only the phases on the
 * context's own stream -- the norm pass and the contractions -- not the per-mode chains that
 * T-HOSVD runs on their own streams) or (ctx, 3) (only the mode-0 core / shrink contraction).  Phases: norms, gather, power_half, power_gram, orth,
 * core_ttm<k> (k-th contraction of core_from_factors), shrink_ttm_m<n>. */
int lmra_context_set_profiling(lmra_context* ctx, int on);
/* keep host copies of the drawn samples / column norms in the result (default on) */
int lmra_context_set_trace(lmra_context* ctx, int on);
int lmra_result_num_phases(const lmra_result* r);
int lmra_result_phase(const lmra_result* r, int i, char* name, size_t name_len, double* ms,
                      int* launches);
/* Releases the result.  Its device core / factor buffers go back to the context's block
 * cache and are reused by later runs.  If their device pointers were handed out
 * (lmra_result_core_device / lmra_result_factor_device), free synchronises the device first,
 * so reads the caller queued on its own streams complete before the blocks are reused (the
 * guarantee cudaFree gives); results only read through the copy calls skip that sync. */
void lmra_result_free(lmra_result* r);

/* ---- primitives (device pointers unless stated; all on the context's stream) ---- */
/* y = x x_mode b, b is b_rows x dims[mode] column-major (tensor.cpp:118-139) */
int lmra_mode_n_product(lmra_context* ctx, const double* x, const uint64_t* dims, int order,
                        int mode, const double* b, uint64_t b_rows, double* y);
/* y (mu x J) = q^T x for the mode-0 view of a tensor (x: K x J, column j contiguous; q: K x mu
 * column-major; w[j] = canonical squared norm of column j), computed on the int8 tensor cores
 * with exact digit products (~1e-13 relative).  Replaces, for the core's first contraction,
 * mode_n_product (tensor.hpp:56-57) as called by core_from_factors (tucker.cpp:81-92) and the
 * ST-HOSVD shrink (tucker.cpp:397-420).  Device pointers; K even <= 4096, mu <= 64. */
int lmra_mode0_product_i8(lmra_context* ctx, const double* x, uint64_t K, uint64_t J, const double* q,
                          int mu, const double* w, double* y);
/* y (R x mu x O) = x x_1 q^T for x (R x K x O, R fastest) on the int8 tensor cores: the mode-1
 * product (tensor.hpp:56-57) of a tensor whose first mode has R <= 64 (even) entries, as in the
 * core's second contraction (tucker.cpp:81-92).  Column scales from the columns' maximum
 * exponents (computed here; run_algorithm takes them from the preceding mode-0 contraction). */
int lmra_mode1_product_i8(lmra_context* ctx, const double* x, uint64_t R, uint64_t K, uint64_t O,
                          const double* q, int mu, double* y);

/* c = (A A^T)^q G  (linalg.cpp:62-80), A rows x cols, G rows x s */
int lmra_gram_power_apply(lmra_context* ctx, const double* a, uint64_t rows, uint64_t cols,
                          const double* g, uint64_t s, int q, int strategy, double* c);
/* u = top-mu left singular vectors of c with the reference's sign rule (linalg.cpp:82-87) */
int lmra_leading_left_singular_vectors(lmra_context* ctx, const double* c, uint64_t rows,
                                       uint64_t cols, uint64_t mu, double* u);
/* q (rows x cols) = thin Q of c (linalg.cpp:52-60), Householder TSQR; device pointers.
 * rows <= 256: LAPACK/Eigen HouseholderQR sign convention; above: same span, column signs
 * of the tree factorisation. */
int lmra_thin_qr_q(lmra_context* ctx, const double* c, uint64_t rows, uint64_t cols, double* q);
/* out (rows x mu) = Q U1 with Q = thin_qr(c).Q, U1 = top-mu left singular vectors of Q^T a
 * (linalg.cpp:89-99); c rows x cols, a rows x a_cols (column-major); device pointers. */
int lmra_qr_project_extract(lmra_context* ctx, const double* c, uint64_t rows, uint64_t cols,
                            const double* a, uint64_t a_cols, uint64_t mu, double* out);
/* the sampling chain on the device, bit-exact with the reference's host loops:
 * p = gram_sampling_probabilities from squared norms w (tucker.cpp:110-130), then
 * randsample(L, p, {seed, stream}) (sketching.cpp:96-131).  w, idx, scales, p: device. */
int lmra_sample_columns_device(lmra_context* ctx, const double* w, uint64_t n, int regime,
                               double beta, uint64_t L, uint64_t seed, uint64_t stream,
                               int64_t* idx, double* scales, double* p);
/* TNSR files (tensor_io.hpp:9-13): "TNSR", u32 version 1, u32 order, u64 dims, float64
 * values in storage order, little-endian.  Errors carry the reference's messages.
 * lmra_tnsr_read_header: order and dims (up to max_order of them).
 * lmra_tnsr_load: the values into dst (LMRA_HOST, or LMRA_DEVICE -- then streamed through
 * pinned staging, file reads overlapping the copies; ctx gives device and stream).
 * lmra_tnsr_save: src (host, or device with ctx) written with its dims. */
int lmra_tnsr_read_header(const char* path, int* order, uint64_t* dims, int max_order);
int lmra_tnsr_load(lmra_context* ctx, const char* path, double* dst, int dst_location);
int lmra_tnsr_save(lmra_context* ctx, const char* path, const double* src, int src_location,
                   const uint64_t* dims, int order);
/* canonical column squared norms of the mode-n unfolding (tucker.cpp:117-119) */
int lmra_column_sqnorms(lmra_context* ctx, const double* x, const uint64_t* dims, int order,
                        int mode, double* w);

/* ---- host-side reference restatements used on the path (host pointers) ---- */
int lmra_gaussian_matrix(uint64_t rows, uint64_t cols, uint64_t seed, uint64_t stream,
                         double* out);
int lmra_probabilities(const double* w, uint64_t n, int regime, double beta, double* p);
int lmra_randsample(uint64_t L, const double* p, uint64_t n, uint64_t seed, uint64_t stream,
                    int64_t* idx, double* scales);
int lmra_amm_sample_counts(const uint64_t* dims, int order, const lmra_algo_config* cfg,
                           int sequential, uint64_t* out);

/* ---- verification (tucker.hpp:63-66, tucker.cpp:222-240), on the device ----
 * lmra_reconstruct: out = core x_0 Q_0 x_1 Q_1 ... (reconstruct, mode order); core (core_dims),
 *   factors[n] (factor_rows[n] x core_dims[n], column-major) all on the host (location =
 *   LMRA_HOST) or all on the device; out (prod factor_rows) at out_location.
 * lmra_relative_error: ||a - approx||_F / ||a||_F over two tensors of dims (relative_error);
 *   LMRA_EINVAL "relative_error: zero reference tensor" when a is zero.
 * lmra_result_relative_error: the same for a result against the tensor a it decomposed,
 *   reconstructed into device scratch (shape mismatch -> "relative_error: shape mismatch"). */
int lmra_reconstruct(lmra_context* ctx, const double* core, const uint64_t* core_dims, int order,
                     const double* const* factors, const uint64_t* factor_rows, int location, double* out,
                     int out_location);
int lmra_relative_error(lmra_context* ctx, const double* a, const double* approx, const uint64_t* dims,
                        int order, int location, double* re);
int lmra_result_relative_error(lmra_context* ctx, const lmra_result* r, const double* a, const uint64_t* dims,
                               int order, int location, double* re);

/* ---- synthetic BASELINE inputs, generated on the device (x is a device buffer) ----
 * Definitions in paper_2303_11612_b200/csrc/gen/portable_gen.hpp: explicit IEEE operations in
 * fixed orders, so the oracle's host generators produce the same bits.  The _slab variants
 * write only the slab [start, start + count) of the last mode (a multi-GPU rank's share);
 * the Tucker-plus-noise tensor is then made in two steps around a host exchange:
 *   lmra_gen_tucker_signal_slab  x = the signal B on the slab; slice_b / slice_e (host, count
 *                                entries) = sums of squares of B and of the noise E per slice;
 *   lmra_gen_noise_coef          coef = gamma ||B|| / ||E|| from ALL slices' sums, in order;
 *   lmra_gen_add_noise_slab      x += coef * E on the slab. */
int lmra_gen_tucker_noise(lmra_context* ctx, const uint64_t* dims, const uint64_t* core_dims,
                          int order, double gamma, uint64_t seed, double* x);
int lmra_gen_tucker_signal_slab(lmra_context* ctx, const uint64_t* dims, const uint64_t* core_dims, int order,
                                uint64_t seed, uint64_t start, uint64_t count, double* x, double* slice_b,
                                double* slice_e);
int lmra_gen_noise_coef(const double* slice_b, const double* slice_e, uint64_t nslices, double gamma,
                        double* coef);
int lmra_gen_add_noise_slab(lmra_context* ctx, const uint64_t* dims, int order, uint64_t seed, uint64_t start,
                            uint64_t count, double coef, double* x);
int lmra_gen_hilbert(lmra_context* ctx, const uint64_t* dims, int order, double* x);
int lmra_gen_hilbert_slab(lmra_context* ctx, const uint64_t* dims, int order, uint64_t start, uint64_t count,
                          double* x);
int lmra_gen_video(lmra_context* ctx, const uint64_t* dims, int order, uint64_t n_terms,
                   double noise, uint64_t seed, double* x);
int lmra_gen_video_slab(lmra_context* ctx, const uint64_t* dims, int order, uint64_t n_terms, double noise,
                        uint64_t seed, uint64_t start, uint64_t count, double* x);

/* device memory helpers (so callers without a CUDA runtime can stage data) */
int lmra_device_alloc(lmra_context* ctx, size_t bytes, void** out);
int lmra_device_free(lmra_context* ctx, void* p);
int lmra_memcpy(lmra_context* ctx, void* dst, const void* src, size_t bytes, int dst_location,
                int src_location);

#ifdef __cplusplus
}
#endif
#endif

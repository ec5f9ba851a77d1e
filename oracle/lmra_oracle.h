/* lmra_oracle.h -- CPU restatement of the reference's randomized Tucker hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the parity checker and the CPU
 * baseline; it is never linked into, loaded by, or called from the product
 * path (paper_2303_11612_b200/).  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load it.
 *
 * It restates, function by function (file:line under /root/reference/proj):
 *   rng.hpp:20-66            RandomStream (PCG32 + Box-Muller)         -> orc_rng_*
 *   sketching.cpp:13-24      stable_sum (Neumaier)                     -> orc_stable_sum
 *   sketching.cpp:28-53      ProbabilityDistribution checks/normalize  -> orc_probabilities
 *   sketching.cpp:96-131     randsample                                -> orc_randsample
 *   sketching.cpp:164-173    gaussian_matrix                           -> orc_gaussian_matrix
 *   tucker.cpp:24-130        resolve, streams, clamps, T rules, probs
 *   tucker.cpp:318-420       alg1/alg2/alg4/alg5                       -> orc_run
 *   linalg.cpp:12-43,62-87   thin SVD + fix_signs, gram_power_apply
 *   tensor.cpp:60-139        unfold / fold / mode_n_product
 * The dense arithmetic the reference delegates to Eigen3 (absent here) goes to
 * OpenBLAS/LAPACK (numpy's bundled libscipy_openblas64_, loaded with dlopen):
 * dgemm for the GEMMs, dgesdd (divide and conquer, same class as Eigen BDCSVD)
 * for the thin SVD, dgeqrf/dorgqr for the generators' thin QR.
 *
 * Column squared norms (tucker.cpp:118, Eigen squaredNorm, order unpinned) use
 * the canonical order shared with the GPU: chunks of 32 consecutive fiber
 * entries accumulated with fma, chunk partials added sequentially.  Parity of
 * bits against Eigen itself is therefore unpinned; parity of the sampling
 * chain on top of the norms is bit-exact (integer indices).
 */
#ifndef LMRA_ORACLE_H
#define LMRA_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* algorithm ids follow tucker.hpp:47-57 */
enum { ORC_ALG1 = 1, ORC_ALG2 = 2, ORC_ALG4 = 4, ORC_ALG5 = 5, ORC_ALG6 = 6, ORC_ALG7 = 7,
       ORC_THOSVD = 10, ORC_STHOSVD = 11, ORC_HOOI = 12 };
/* ProbRegime, sketching.hpp:24 */
enum { ORC_OPTIMAL = 0, ORC_NEARLY_OPTIMAL = 1, ORC_UNIFORM = 2 };

typedef struct {
  const uint64_t* rank;      /* mu_n, length = order */
  uint64_t oversampling;     /* K (paper) / p (BASELINE) */
  int32_t power;             /* q */
  double alpha;
  int32_t regime;
  double regime_beta;
  const uint64_t* t_samples; /* NULL or length = order */
  const uint64_t* order;     /* NULL or permutation, 0-based */
  uint64_t seed;
  int32_t strategy;          /* 0 = A, 1 = B (GramStrategy) */
  int32_t mode_threads;      /* LMRA_NUM_THREADS analogue for alg1/alg4 */
  int32_t keep_trace;        /* store per-mode Omega / samples / norms */
  int32_t hooi_max_sweeps;   /* default 50 */
  double hooi_tol;           /* default 1e-8 */
} orc_config;

typedef struct orc_result orc_result;

const char* orc_last_error(void);
int orc_init_blas(const char* path);
void orc_set_blas_threads(int n);

/* RNG (rng.hpp) */
void orc_rng_u32(uint64_t seed, uint64_t stream, uint64_t skip, uint32_t* out, size_t n);
void orc_rng_double(uint64_t seed, uint64_t stream, double* out, size_t n);
void orc_rng_normal(uint64_t seed, uint64_t stream, double* out, size_t n);
int orc_gaussian_matrix(uint64_t rows, uint64_t cols, uint64_t seed, uint64_t stream, double* out);

/* sampling (sketching.cpp, tucker.cpp) */
double orc_stable_sum(const double* v, size_t n);
int orc_column_sqnorms(const double* x, const uint64_t* dims, int order, int mode, double* w);
int orc_probabilities(const double* w, uint64_t n, int regime, double beta, double* p);
int orc_randsample(uint64_t L, const double* p, uint64_t n, uint64_t seed, uint64_t stream,
                   int64_t* idx, double* scales);
int orc_amm_sample_counts(const uint64_t* dims, int order, const orc_config* cfg, int sequential,
                          uint64_t* out);

/* linalg / tensor */
int orc_mode_n_product(const double* x, const uint64_t* dims, int order, int mode,
                       const double* b, uint64_t b_rows, double* y);
int orc_gram_power_apply(const double* a, uint64_t rows, uint64_t cols, const double* g,
                         uint64_t s, int q, int strategy, double* c);
int orc_leading_left_singular_vectors(const double* c, uint64_t rows, uint64_t cols, uint64_t mu,
                                      double* u);
int orc_thin_qr_q(const double* m, uint64_t rows, uint64_t cols, double* q);
/* linalg.cpp:89-99 */
int orc_qr_project_extract(const double* c, uint64_t rows, uint64_t cols, const double* a,
                           uint64_t a_cols, uint64_t mu, double* out);

/* algorithms */
int orc_run(int alg, const double* x, const uint64_t* dims, int order, const orc_config* cfg,
            orc_result** out);
int orc_result_order(const orc_result* r);
void orc_result_core_dims(const orc_result* r, uint64_t* dims);
void orc_result_factor_dims(const orc_result* r, int n, uint64_t* rows, uint64_t* cols);
void orc_result_core(const orc_result* r, double* out);
void orc_result_factor(const orc_result* r, int n, double* out);
double orc_result_seconds(const orc_result* r);
/* trace (keep_trace != 0) */
void orc_result_omega_dims(const orc_result* r, int n, uint64_t* rows, uint64_t* cols);
void orc_result_omega(const orc_result* r, int n, double* out);
void orc_result_sketch_dims(const orc_result* r, int n, uint64_t* rows, uint64_t* cols);
void orc_result_sketch(const orc_result* r, int n, double* out); /* same dims as omega */
uint64_t orc_result_num_samples(const orc_result* r, int n);
void orc_result_samples(const orc_result* r, int n, int64_t* idx, double* scales);
uint64_t orc_result_num_norms(const orc_result* r, int n);
void orc_result_norms(const orc_result* r, int n, double* w);
void orc_result_free(orc_result* r);

double orc_relative_error(const double* x, const uint64_t* dims, int order, const orc_result* r);

/* synthetic inputs for the BASELINE configs (host, CPU tests / CPU baseline) */
int orc_gen_tucker_noise(const uint64_t* dims, const uint64_t* core_dims, int order, double gamma,
                         uint64_t seed, double* out);
int orc_gen_hilbert(const uint64_t* dims, int order, double* out);
int orc_gen_video(const uint64_t* dims, int order, uint64_t n_terms, double noise, uint64_t seed,
                  double* out);

#ifdef __cplusplus
}
#endif
#endif

// kernels.hpp -- host-side launchers for the sm_100a kernels (no torch types).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace lmra_dev {

// Tensor viewed around one mode: X3[i, r, o] = x[i + inner * (r + I * o)].
// Column j of the mode unfolding is (i, o) with j = i + inner * o (tensor.cpp:60-86).
struct ModeView {
  long long inner, I, outer;
};

// widest factor / sketch the DMMA tiles take (N of m16n8k4 padded to 8)
constexpr int kMaxWidth = 64;

// Kernel launches issued by this library from the calling thread (every launch site calls
// note_launch): the results' launch counts -- and so the bench's gpu_launches -- come from here.
inline thread_local long long g_kernel_launches = 0;
inline void note_launch() { ++g_kernel_launches; }

// SMs the persistent int8 contraction leaves free (set by the host around a launch that runs
// beside other kernels -- the split orthonormalisation's Jacobis -- so both make progress:
// the contraction's tiles are assigned statically to its CTAs, and one CTA that cannot start
// delays the whole kernel by the duration of whatever holds its SM)
inline thread_local int g_i8_reserved_sms = 0;

// Stream-ordered scratch for the launchers: served from the run's device arena when the host
// has one installed (lmra_b200.cpp ArenaScope), else from the stream-ordered pool.
cudaError_t scratch_alloc(void** p, size_t bytes, cudaStream_t st);
void scratch_free(void* p, cudaStream_t st);

// Gathered columns for the power scheme on sampled columns (mode-0 views only): column j of
// the view is x column idx[j] (< 0: a zero column) scaled by scale[j] -- C' of
// sample_columns (sketching.cpp:133-141) without materialising it.  The TTM then writes
// h_j = scale_j^2 (x_idx[j]^T b) and the Gram sums x_idx[j] h_j^T, i.e. C' C'^T b.
struct Gather {
  const long long* idx = nullptr;
  const double* scale = nullptr;
};

// Y = X x_mode B, with B given transposed: bt[r + I*k] = B[k, r] (I x m column-major).
cudaError_t launch_ttm(const double* x, ModeView v, const double* bt, int m, double* y,
                       cudaStream_t st, Gather ga = Gather{});

struct GramPlan {
  int nsplit = 1;
  long long jper = 0;
};
GramPlan plan_gram(ModeView v, int num_sms);
// z (I x s, column-major) = sum_j X(:, j) H(:, j)^T; zpart holds nsplit * I * s doubles.
cudaError_t launch_gram(const double* x, ModeView v, const double* h, int s, double* zpart,
                        const GramPlan& plan, double* z, cudaStream_t st, Gather ga = Gather{});

// C' = A_(n)(:, idx) * diag(scale), I x T column-major.
cudaError_t launch_gather(const double* x, ModeView v, const long long* idx, const double* scale,
                          long long T, double* out, cudaStream_t st);

// Canonical column squared norms of the mode-n unfolding (chunks of 32 along the fiber,
// fma within a chunk, chunk partials added in order) -- bit-identical to the oracle.
cudaError_t launch_column_sqnorms(const double* x, ModeView v, double* w, cudaStream_t st);
// The same canonical norms for all three modes of a 3-way tensor from one read (norms3.cu).
// p2_chunks (optional, ceil(I2/32) x I0 I1): mode 2's chunk partials go there instead of w2
// (a sharded slab's last mode, combined across devices).
size_t norms3_workspace_doubles(long long I0, long long I1, long long I2);
cudaError_t launch_norms3(const double* x, long long I0, long long I1, long long I2, double* w0,
                          double* w1, double* w2, double* work, cudaStream_t st, double* p2_chunks = nullptr);
// A fibre split across devices (sharded mode N-1, slab boundaries at multiples of 64 entries):
// chunk partials P[c][j] of the local rows, their segment (chunk pair) sums S[s][j], and the
// combine of every rank's segments in global order -- the canonical norm's exact bits.
struct SegCounts {
  int n[64];
};
cudaError_t launch_chunk_partials(const double* x, ModeView v, double* P, cudaStream_t st);
cudaError_t launch_segment_sums(const double* P, long long J, int nchunks, double* S, cudaStream_t st);
cudaError_t launch_segment_combine(const double* G, long long J, int nranks, int kmax, const SegCounts& counts,
                                   double* w, cudaStream_t st);

// The reference's sampling chain on the device, bit-exact (sampler.cu):
// probabilities from squared column norms w (regime 0 optimal, 1 nearly-optimal, 2 uniform)
// then L multinomial draws from PCG32 stream (seed, stream): idx (int64), scales, p (n).
// status bits: 1 bad weight, 2 zero normaliser, 4 sum != 1, 8 zero total, 16 fallback, 64 internal,
// 32 bad beta.
size_t sampler_workspace_doubles(long long n);
void sampler_walk_stats(unsigned long long* out2, bool reset);  // diagnostics
cudaError_t launch_sampler(const double* w, long long n, int regime, double beta, long long L,
                           uint64_t seed, uint64_t stream, long long* idx, double* scales,
                           double* p_out, double* work, int* status, cudaStream_t st);

// Shifted CholeskyQR3 basis of C (I x s, s <= 64) in one thread-block cluster (cholqr.cu):
// Q_C (I x s) orthonormal and R (s x s, upper, column-major) with C = Q_C R; *fail = 1 when a
// Cholesky pivot breaks down (numerically rank-deficient C): the caller then needs another path.
bool cholqr_supported(long long I, int s);
int cholqr_cluster_size(long long I);
cudaError_t launch_cholqr(const double* c, long long I, int s, double* qc, double* r, int* fail,
                          cudaStream_t st);

// Top-mu left singular vectors of C (I x s, column-major) with the reference's sign
// convention (linalg.cpp:13-43,82-87), written to U (I x mu).  Workspace: orth_workspace().
size_t orth_workspace_doubles(long long I, int s);
cudaError_t launch_orth(const double* c, long long I, int s, int mu, double* u, double* work,
                        int* status, cudaStream_t st);

// The same in two halves (orth.cu): launch_orth_basis writes Q_C (I x s), an orthonormal basis of
// C's columns (pivoted Householder TSQR, no Jacobi); launch_orth_finish then runs the s x s Jacobi
// and writes U = Q_C U_R(:, :mu) with the sign rule plus U_R' (s x mu) = U_R(:, :mu) with U's
// column signs, so X x_n U^T = (X x_n Q_C^T) x_n U_R'^T.  Same workspace for both calls.
size_t orth_split_workspace_doubles(long long I, int s);
// urs (s x mu, column-major) = qc^T u for qc (I x s) and u (I x mu): a factor's coefficients in
// the split form's basis (the factor itself from launch_orth)
cudaError_t launch_basis_coeffs(const double* qc, long long I, int s, const double* u, int mu, double* urs,
                                cudaStream_t st);
cudaError_t launch_orth_basis(const double* c, long long I, int s, double* qc, double* work, cudaStream_t st);
cudaError_t launch_orth_finish(const double* qc, long long I, int s, int mu, double* u, double* ur_signed,
                               double* work, int* status, cudaStream_t st);

// qr_project_extract (linalg.cpp:89-99) building blocks (orth.cu):
// R (s x s, column-major) of a tall m x s matrix (m >= s) by Householder TSQR.
size_t r_factor_workspace_doubles(long long m, int s);
cudaError_t launch_r_factor(const double* a, long long m, int s, double* r, double* work,
                            cudaStream_t st);
// thin Q (I x s) of C (thin_qr, linalg.cpp:52-60) by Householder TSQR.
size_t thin_q_workspace_doubles(long long I, int s);
cudaError_t launch_thin_q(const double* c, long long I, int s, double* q, double* work, cudaStream_t st);
// out (J x I column-major) = transposed mode unfolding of x (ModeView inner, I, outer).
cudaError_t launch_unfold_t(const double* x, long long inner, long long I, long long outer, double* out,
                            cudaStream_t st);

// Mode-0 contraction on the int8 tensor cores (ttm_i8.cu): y (mu x J) = q^T x with x K x J
// (column j contiguous), q K x mu column-major, w[j] the canonical squared norm of column j
// (sets the column's fixed-point scale).  ~1e-13 relative accuracy; supported for K even,
// K <= 4096, mu <= 64, x 16-byte aligned.
bool ttm_i8_supported(long long K, long long J, int mu, const double* x);
size_t ttm_i8_workspace_bytes(long long K, int mu);
// fexp_out (optional, mu x O ints, preset to INT_MIN): receives the max binary exponent of
// every mode-1 fibre (m, o) of Y, with column j = i1 + I1 o -- the scales of a following
// launch_ttm_i8_inner over i1.
cudaError_t launch_ttm_i8(const double* x, long long K, long long J, const double* q, int mu,
                          const double* w, double* y, void* work, cudaStream_t st,
                          int* fexp_out = nullptr, long long I1 = 0);
// The same contraction over the middle index of X(r, k, o) = x[r + R (k + K o)] (R <= 64, even):
// Y(r, m, o) = sum_k q[k, m] X(r, k, o), i.e. the mode-1 product of a tensor whose mode 0 has
// R entries.  fexp_in[r + R o] = max binary exponent of column (r, o) (INT_MIN: all zero).
bool ttm_i8_inner_supported(long long R, long long K, long long O, int mu, const double* x);
cudaError_t launch_ttm_i8_inner(const double* x, long long R, long long K, long long O, const double* q,
                                int mu, const int* fexp_in, double* y, void* work, cudaStream_t st);
// fexp[r + R o] = max binary exponent over k of X(r, k, o) (INT_MIN: all zero)
cudaError_t launch_column_exponents(const double* x, long long R, long long K, long long O, int* fexp,
                                    cudaStream_t st);

// ---- synthetic generators (gen.cu; definitions in gen/portable_gen.hpp, bit-identical to the host) ----
// y[a, i, o] = sum_k u[i + ldu k] x[a + inner (k + K o)], i < I (fma chain over k ascending)
cudaError_t launch_gen_ttm(const double* x, long long inner, long long K, long long I, long long outer,
                           const double* u, long long ldu, double* y, cudaStream_t st);
// out[f] = sum_i x[f d0 + i]^2 (fma chain), f < nfib
cudaError_t launch_gen_fiber_sumsq(const double* x, long long d0, long long nfib, double* out, cudaStream_t st);
// the same over the normal stream (seed, stream), elements e_base + f d0 + i (regenerated)
cudaError_t launch_gen_noise_fiber_sumsq(uint64_t seed, uint64_t stream, long long e_base, long long d0,
                                         long long nfib, double* out, cudaStream_t st);
// out[l] = sum_j fib[l per + j] (sequential), l < nslices
cudaError_t launch_gen_slice_sum(const double* fib, long long per, long long nslices, double* out,
                                 cudaStream_t st);
// x[e] = x[e] + coef * z_(e_base + e), z the normal stream (seed, stream)
cudaError_t launch_gen_add_noise(double* x, long long n, long long e_base, double coef, uint64_t seed,
                                 uint64_t stream, cudaStream_t st);
// slabs [start, start + count) of the last mode
cudaError_t launch_gen_hilbert(double* out, const long long* dims, int order, long long start, long long count,
                               cudaStream_t st);
cudaError_t launch_gen_video(double* out, const long long* dims, int order, long long start, long long count,
                             const double* profiles, const double* weights, int n_terms, double noise,
                             uint64_t seed, uint64_t stream, cudaStream_t st);

// ---- deterministic baselines (dense.cu) ----
// r (n x n) = upper triangle of a (ld lda), zeros below
cudaError_t launch_copy_upper(const double* a, long long lda, int n, double* r, cudaStream_t st);
// q (n x mu) = transpose of the first mu rows of vt (n x n)
cudaError_t launch_rows_to_cols(const double* vt, int n, int mu, double* q, cudaStream_t st);
// fix_signs (linalg.cpp:13-29) on the mu columns of u (m rows, ld ldu)
cudaError_t launch_signfix_columns(double* u, long long m, int ldu, int mu, cudaStream_t st);

// ---- verification (verify.cu): out2 = {sum (a - r)^2, sum a^2}, deterministic ----
size_t diff_sumsq_workspace_doubles();
cudaError_t launch_diff_sumsq(const double* a, const double* r, long long n, double* work, double* out2,
                              cudaStream_t st);

// sharded runs: l[t] = g[t] - off if in [0, cnt) else -1
cudaError_t launch_localize_idx(const long long* g, long long T, long long off, long long cnt,
                                long long* l, cudaStream_t st);
// out[i] = sum over ranks in order of in_dev[r][i] (in_dev: device array of device pointers)
// out[i] = sum_r in[r n + i], r = 0, 1, ... (fixed order)
cudaError_t launch_sum_ranks_strided(const double* in, int nranks, long long n, double* out, cudaStream_t st);
cudaError_t launch_sum_ranks(const double* const* in_dev, int nranks, long long n, double* out,
                             cudaStream_t st);
// at (cols x rows) = a^T
cudaError_t launch_transpose(const double* a, long long rows, long long cols, double* at,
                             cudaStream_t st);
}  // namespace lmra_dev

namespace lmra_dev {
int last_jacobi_sweeps();  // diagnostics: sweeps of the most recent converged Jacobi
void last_orth_clocks(long long* out7);  // diagnostics: phase clocks of the last full orth core
}

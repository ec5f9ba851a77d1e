// gen.cu -- device generators for the BASELINE synthetic inputs and
// small device utilities (transpose, rank sums, index localisation).
//
// The generators evaluate the definitions of gen/portable_gen.hpp element by element with
// explicit IEEE operations (no contraction, fixed summation orders), so they produce the
// same bits as the host generators (oracle/lmra_oracle.cpp) -- and any slab of the last mode
// on its own (multi-GPU ranks generate only their slab).
#include "common.cuh"
#include "../gen/portable_gen.hpp"

namespace lmra_dev {

using namespace lmra_gen;

// y[a, i, o] = sum_k U[r0 + i, k] x[a, k, o] (fma chain over k ascending): one output per thread
__global__ void gen_ttm_kernel(const double* __restrict__ x, long long inner, long long K, long long I,
                               long long outer, const double* __restrict__ u, long long ldu,
                               double* __restrict__ y) {
  const long long n = inner * I * outer;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x) {
    const long long a = e % inner, r = e / inner, i = r % I, o = r / I;
    y[e] = gp_ttm_element(x, inner, K, u, ldu, a, i, o);
  }
}

// out[f] = sum_i x[f d0 + i]^2 (fma chain), one fibre per thread
__global__ void gen_fiber_sumsq_kernel(const double* __restrict__ x, long long d0, long long nfib,
                                       double* __restrict__ out) {
  const long long f = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= nfib) return;
  const double* p = x + f * d0;
  double acc = 0.0;
  for (long long i = 0; i < d0; ++i) acc = gp_fma(p[i], p[i], acc);
  out[f] = acc;
}

// the same for the normal stream (seed, stream), elements e_base + f d0 + i, regenerated
__global__ void gen_noise_fiber_sumsq_kernel(unsigned long long seed, unsigned long long stream,
                                             long long e_base, long long d0, long long nfib,
                                             double* __restrict__ out) {
  const long long f = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= nfib) return;
  const unsigned long long b = (unsigned long long)(e_base + f * d0), e = b + (unsigned long long)d0;
  Pcg g(seed, stream);
  g.advance(4ull * (b / 2));
  double acc = 0.0;
  unsigned long long i = b;
  if (i & 1) {
    double z0, z1;
    g.normal_pair(&z0, &z1);
    acc = gp_fma(z1, z1, acc);
    ++i;
  }
  for (; i < e; i += 2) {
    double z0, z1;
    g.normal_pair(&z0, &z1);
    acc = gp_fma(z0, z0, acc);
    if (i + 1 < e) acc = gp_fma(z1, z1, acc);
  }
  out[f] = acc;
}

// out[l] = sum_j fib[l per + j] (sequential adds), one slice per thread
__global__ void gen_slice_sum_kernel(const double* __restrict__ fib, long long per, long long nslices,
                                     double* __restrict__ out) {
  const long long l = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= nslices) return;
  double acc = 0.0;
  for (long long j = 0; j < per; ++j) acc = gp_add(acc, fib[l * per + j]);
  out[l] = acc;
}

constexpr long long kRun = 64;  // elements per thread (one jump-ahead per run)

// x[e] += coef * z_(e_base + e), z the normal stream (seed, stream)
__global__ void gen_add_noise_kernel(double* __restrict__ x, long long n, long long e_base, double coef,
                                     unsigned long long seed, unsigned long long stream) {
  const long long e0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * kRun;
  if (e0 >= n) return;
  const long long e1 = min(n, e0 + kRun);
  double z[kRun + 1];
  gp_normals_range(seed, stream, z, (unsigned long long)(e_base + e0), (unsigned long long)(e_base + e1));
  for (long long e = e0; e < e1; ++e) x[e] = gp_add(x[e], gp_mul(coef, z[e - e0]));
}

struct Dims8 {
  long long d[8];
};

// Hilbert slab: a = 1 / (i_0 + ... + i_{N-1} + 1) (0-based), last index offset by start
__global__ void gen_hilbert_kernel(double* __restrict__ out, long long n, Dims8 dims, int order,
                                   long long start) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  long long rem = e, s = 0;
  for (int k = 0; k < order; ++k) {
    if (k == order - 1) {
      s += rem + start;
      break;
    }
    long long q = rem / dims.d[k];
    s += rem - q * dims.d[k];
    rem = q;
  }
  out[e] = gp_div(1.0, (double)(s + 1));
}

// video slab: sum of separable cosine terms + noise * U[0,1) (stream 400, element e_base + e)
__global__ void gen_video_kernel(double* __restrict__ out, long long n, Dims8 dims, int order, long long start,
                                 long long e_base, const double* __restrict__ profiles,
                                 const double* __restrict__ weights, int R, double noise,
                                 unsigned long long seed, unsigned long long stream) {
  const long long e0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * kRun;
  if (e0 >= n) return;
  const long long e1 = min(n, e0 + kRun);
  Pcg g(seed, stream);
  g.advance(2ull * (unsigned long long)(e_base + e0));
  for (long long e = e0; e < e1; ++e) {
    long long idx[8];
    long long rem = e;
    for (int k = 0; k < order; ++k) {
      if (k == order - 1) {
        idx[k] = rem + start;
        break;
      }
      long long q = rem / dims.d[k];
      idx[k] = rem - q * dims.d[k];
      rem = q;
    }
    const double v = gp_video_element(idx, dims.d, order, profiles, weights, R);
    out[e] = gp_add(v, gp_mul(noise, g.next_double()));
  }
}

static unsigned grid_for(long long n, int per_block) {
  long long g = (n + per_block - 1) / per_block;
  if (g < 1) g = 1;
  if (g > 148LL * 64) g = 148LL * 64;
  return (unsigned)g;
}

cudaError_t launch_gen_ttm(const double* x, long long inner, long long K, long long I, long long outer,
                           const double* u, long long ldu, double* y, cudaStream_t st) {
  if (inner * I * outer <= 0) return cudaSuccess;
  gen_ttm_kernel<<<grid_for(inner * I * outer, 256), 256, 0, st>>>(x, inner, K, I, outer, u, ldu, y); note_launch();
  return cudaGetLastError();
}

cudaError_t launch_gen_fiber_sumsq(const double* x, long long d0, long long nfib, double* out, cudaStream_t st) {
  if (nfib <= 0) return cudaSuccess;
  gen_fiber_sumsq_kernel<<<(unsigned)((nfib + 127) / 128), 128, 0, st>>>(x, d0, nfib, out); note_launch();
  return cudaGetLastError();
}

cudaError_t launch_gen_noise_fiber_sumsq(uint64_t seed, uint64_t stream, long long e_base, long long d0,
                                         long long nfib, double* out, cudaStream_t st) {
  if (nfib <= 0) return cudaSuccess;
  gen_noise_fiber_sumsq_kernel<<<(unsigned)((nfib + 127) / 128), 128, 0, st>>>(seed, stream, e_base, d0, nfib,
                                                                             out); note_launch();
  return cudaGetLastError();
}

cudaError_t launch_gen_slice_sum(const double* fib, long long per, long long nslices, double* out,
                                 cudaStream_t st) {
  if (nslices <= 0) return cudaSuccess;
  gen_slice_sum_kernel<<<(unsigned)((nslices + 127) / 128), 128, 0, st>>>(fib, per, nslices, out); note_launch();
  return cudaGetLastError();
}

cudaError_t launch_gen_add_noise(double* x, long long n, long long e_base, double coef, uint64_t seed,
                                 uint64_t stream, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const long long threads = (n + kRun - 1) / kRun;
  gen_add_noise_kernel<<<(unsigned)((threads + 127) / 128), 128, 0, st>>>(x, n, e_base, coef, seed, stream); note_launch();
  return cudaGetLastError();
}

cudaError_t launch_gen_hilbert(double* out, const long long* dims, int order, long long start, long long count,
                               cudaStream_t st) {
  if (order < 1 || order > 8) return cudaErrorInvalidValue;
  Dims8 d{};
  long long n = 1;
  for (int k = 0; k < order; ++k) {
    d.d[k] = dims[k];
    n *= k == order - 1 ? count : dims[k];
  }
  if (n <= 0) return cudaSuccess;
  gen_hilbert_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(out, n, d, order, start); note_launch();
  return cudaGetLastError();
}

cudaError_t launch_gen_video(double* out, const long long* dims, int order, long long start, long long count,
                             const double* profiles, const double* weights, int n_terms, double noise,
                             uint64_t seed, uint64_t stream, cudaStream_t st) {
  if (order < 1 || order > 8) return cudaErrorInvalidValue;
  Dims8 d{};
  long long n = 1, slice = 1;
  for (int k = 0; k < order; ++k) {
    d.d[k] = dims[k];
    n *= k == order - 1 ? count : dims[k];
    if (k < order - 1) slice *= dims[k];
  }
  if (n <= 0) return cudaSuccess;
  const long long threads = (n + kRun - 1) / kRun;
  gen_video_kernel<<<(unsigned)((threads + 127) / 128), 128, 0, st>>>(out, n, d, order, start, start * slice,
                                                                     profiles, weights, n_terms, noise, seed,
                                                                     stream); note_launch();
  return cudaGetLastError();
}

// at (cols x rows) = a^T, a rows x cols column-major
__global__ void transpose_kernel(const double* __restrict__ a, long long rows, long long cols,
                                 double* __restrict__ at) {
  __shared__ double tile[32][33];
  const long long r0 = (long long)blockIdx.x * 32, c0 = (long long)blockIdx.y * 32;
  for (int k = threadIdx.y; k < 32; k += 8) {
    long long r = r0 + threadIdx.x, c = c0 + k;
    tile[k][threadIdx.x] = (r < rows && c < cols) ? a[r + rows * c] : 0.0;
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += 8) {
    long long c = c0 + threadIdx.x, r = r0 + k;
    if (r < rows && c < cols) at[c + cols * r] = tile[threadIdx.x][k];
  }
}

cudaError_t launch_transpose(const double* a, long long rows, long long cols, double* at,
                             cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return cudaSuccess;
  dim3 grid((unsigned)((rows + 31) / 32), (unsigned)((cols + 31) / 32));
  transpose_kernel<<<grid, dim3(32, 8), 0, st>>>(a, rows, cols, at); note_launch();
  return cudaGetLastError();
}

// sharded runs: global sampled column -> this rank's local column, or -1 if another rank's
__global__ void localize_idx_kernel(const long long* __restrict__ g, long long T, long long off,
                                    long long cnt, long long* __restrict__ l) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  const long long j = g[t] - off;
  l[t] = (j >= 0 && j < cnt) ? j : -1;
}

cudaError_t launch_localize_idx(const long long* g, long long T, long long off, long long cnt,
                                long long* l, cudaStream_t st) {
  if (T <= 0) return cudaSuccess;
  localize_idx_kernel<<<(unsigned)((T + 255) / 256), 256, 0, st>>>(g, T, off, cnt, l); note_launch();
  return cudaGetLastError();
}

// out[i] = sum_r in[r][i], ranks in order (deterministic in-process all-reduce)
__global__ void sum_ranks_kernel(const double* const* __restrict__ in, int nranks, long long n,
                                 double* __restrict__ out) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    double s = in[0][i];
    for (int r = 1; r < nranks; ++r) s += in[r][i];
    out[i] = s;
  }
}

// out[i] = sum_r in[r n + i] in rank order (the all-gathered form of sum_ranks)
__global__ void sum_ranks_strided_kernel(const double* __restrict__ in, int nranks, long long n,
                                         double* __restrict__ out) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    double s = in[i];
    for (int r = 1; r < nranks; ++r) s += in[(long long)r * n + i];
    out[i] = s;
  }
}

cudaError_t launch_sum_ranks_strided(const double* in, int nranks, long long n, double* out, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  sum_ranks_strided_kernel<<<148 * 4, 256, 0, st>>>(in, nranks, n, out); note_launch();
  return cudaGetLastError();
}

cudaError_t launch_sum_ranks(const double* const* in_dev, int nranks, long long n, double* out,
                             cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  sum_ranks_kernel<<<148 * 4, 256, 0, st>>>(in_dev, nranks, n, out); note_launch();
  return cudaGetLastError();
}

}  // namespace lmra_dev

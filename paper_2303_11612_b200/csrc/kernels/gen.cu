// gen.cu -- device generators for the BASELINE synthetic inputs (DESIGN.md "Synthetic
// inputs").  The integer part (PCG32 with the reference's seeding, rng.hpp:20-36) is
// bit-identical to the host stream; the Box-Muller transform uses CUDA's log/sincos,
// so device normals may differ from glibc's in the last ulp -- the generated tensor
// is defined as what this code produces and is fed bit-identically to the oracle.
#include "common.cuh"

namespace lmra_dev {

struct Pcg {
  unsigned long long state, inc;
  __device__ Pcg(unsigned long long seed, unsigned long long stream) {
    inc = (stream << 1u) | 1u;
    state = 0;
    next();
    state += seed;
    next();
  }
  __device__ unsigned int next() {
    unsigned long long old = state;
    state = old * 6364136223846793005ULL + inc;
    unsigned int xs = (unsigned int)(((old >> 18u) ^ old) >> 27u);
    unsigned int rot = (unsigned int)(old >> 59u);
    return (xs >> rot) | (xs << ((32u - rot) & 31u));
  }
  __device__ void advance(unsigned long long delta) {
    unsigned long long cm = 6364136223846793005ULL, cp = inc, am = 1, ap = 0;
    while (delta) {
      if (delta & 1) {
        am *= cm;
        ap = ap * cm + cp;
      }
      cp = (cm + 1) * cp;
      cm *= cm;
      delta >>= 1;
    }
    state = am * state + ap;
  }
  __device__ double next_double() {
    unsigned long long hi = next(), lo = next();
    return (double)(((hi << 32) | lo) >> 11) * 0x1.0p-53;
  }
};

constexpr int kPairsPerThread = 64;

__global__ void gen_normals_kernel(double* __restrict__ out, long long n, unsigned long long seed,
                                   unsigned long long stream) {
  const long long npairs = (n + 1) / 2;
  const long long p0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * kPairsPerThread;
  if (p0 >= npairs) return;
  Pcg g(seed, stream);
  g.advance(4ull * (unsigned long long)p0);
  const long long p1 = min(npairs, p0 + kPairsPerThread);
  for (long long p = p0; p < p1; ++p) {
    double u1 = 1.0 - g.next_double();
    double u2 = g.next_double();
    double r = sqrt(-2.0 * log(u1));
    double s, c;
    sincos(6.283185307179586476925286766559 * u2, &s, &c);
    out[2 * p] = r * c;
    if (2 * p + 1 < n) out[2 * p + 1] = r * s;
  }
}

__global__ void gen_uniform_add_kernel(double* __restrict__ out, long long n, double scale,
                                       unsigned long long seed, unsigned long long stream) {
  const long long e0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * kPairsPerThread;
  if (e0 >= n) return;
  Pcg g(seed, stream);
  g.advance(2ull * (unsigned long long)e0);
  const long long e1 = min(n, e0 + kPairsPerThread);
  for (long long e = e0; e < e1; ++e) out[e] += scale * g.next_double();
}

struct Dims8 {
  long long d[8];
};

__global__ void gen_hilbert_kernel(double* __restrict__ out, long long n, Dims8 dims, int order) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  long long rem = e, s = 0;
  for (int k = 0; k < order; ++k) {
    long long q = rem / dims.d[k];
    s += rem - q * dims.d[k];
    rem = q;
  }
  out[e] = 1.0 / (double)(s + 1);
}

// out[e] = sum_t w_t prod_n P_n[i_n, t]; profiles packed mode after mode (I_n x R each).
__global__ void gen_cp_kernel(double* __restrict__ out, long long n, Dims8 dims, int order,
                              const double* __restrict__ profiles,
                              const double* __restrict__ weights, int R) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  long long idx[8];
  long long rem = e;
  for (int k = 0; k < order; ++k) {
    long long q = rem / dims.d[k];
    idx[k] = rem - q * dims.d[k];
    rem = q;
  }
  double acc = 0.0;
  for (int t = 0; t < R; ++t) {
    double v = weights[t];
    long long off = 0;
    for (int k = 0; k < order; ++k) {
      v *= profiles[off + idx[k] + dims.d[k] * t];
      off += dims.d[k] * R;
    }
    acc += v;
  }
  out[e] = acc;
}

__global__ void axpby_kernel(const double* __restrict__ a, const double* __restrict__ b,
                             double coef, double* __restrict__ out, long long n) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x)
    out[e] = a[e] + coef * b[e];
}

__global__ void sumsq_kernel(const double* __restrict__ a, long long n,
                             double* __restrict__ partials) {
  __shared__ double red[256];
  double s = 0.0;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x)
    s += a[e] * a[e];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w >= 1; w >>= 1) {
    if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) partials[blockIdx.x] = red[0];
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

cudaError_t launch_gen_normals(double* out, long long n, uint64_t seed, uint64_t stream,
                               cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  long long threads = ((n + 1) / 2 + kPairsPerThread - 1) / kPairsPerThread;
  gen_normals_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(out, n, seed, stream); note_launch();
  return cudaGetLastError();
}

cudaError_t launch_gen_uniform_add(double* out, long long n, double scale, uint64_t seed,
                                   uint64_t stream, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  long long threads = (n + kPairsPerThread - 1) / kPairsPerThread;
  gen_uniform_add_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(out, n, scale, seed,
                                                                            stream); note_launch();
  return cudaGetLastError();
}

cudaError_t launch_gen_hilbert(double* out, const long long* dims, int order, cudaStream_t st) {
  if (order < 1 || order > 8) return cudaErrorInvalidValue;
  Dims8 d{};
  long long n = 1;
  for (int k = 0; k < order; ++k) {
    d.d[k] = dims[k];
    n *= dims[k];
  }
  gen_hilbert_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(out, n, d, order); note_launch();
  return cudaGetLastError();
}

cudaError_t launch_gen_cp(double* out, const long long* dims, int order, const double* profiles,
                          const double* weights, int n_terms, cudaStream_t st) {
  if (order < 1 || order > 8) return cudaErrorInvalidValue;
  Dims8 d{};
  long long n = 1;
  for (int k = 0; k < order; ++k) {
    d.d[k] = dims[k];
    n *= dims[k];
  }
  gen_cp_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(out, n, d, order, profiles, weights,
                                                            n_terms); note_launch();
  return cudaGetLastError();
}

cudaError_t launch_axpby(const double* a, const double* b, double coef, double* out, long long n,
                         cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  axpby_kernel<<<148 * 8, 256, 0, st>>>(a, b, coef, out, n); note_launch();
  return cudaGetLastError();
}

cudaError_t launch_sumsq(const double* a, long long n, double* partials, int nparts,
                         cudaStream_t st) {
  sumsq_kernel<<<nparts, 256, 0, st>>>(a, n, partials); note_launch();
  return cudaGetLastError();
}

}  // namespace lmra_dev

// norms.cu -- column squared norms of the mode-n unfolding, in place.
//
// Replaces the squaredNorm loop of gram_sampling_probabilities (tucker.cpp:117-119),
// which in the reference runs over an explicit unfold() copy.  The summation order
// is the canonical one shared with the oracle (oracle/lmra_oracle.cpp
// canonical_sqnorm): chunks of 32 consecutive fiber entries accumulated with fma,
// chunk partials added in chunk order.  Results are therefore bit-identical to the
// oracle, which is what makes the sampled indices bit-exact end to end.
//
// HBM-bound: 8 B read per element, 2 flop.  Contiguous fibers (mode 0) are staged
// through shared memory so each thread walks its own fiber; strided fibers (modes
// > 0) are read coalesced across threads (consecutive i), one thread per column.
#include "common.cuh"

namespace lmra_dev {

constexpr int kNormChunk = 32;

// mode 0: fiber j = x[I*j .. I*j + I)
__global__ void __launch_bounds__(128) sqnorm_contig_kernel(const double* __restrict__ x,
                                                            long long I, long long J,
                                                            double* __restrict__ w) {
  __shared__ double tile[128][kNormChunk + 1];
  const int tid = threadIdx.x;
  const long long j0 = (long long)blockIdx.x * 128;
  double total = 0.0;
  for (long long r0 = 0; r0 < I; r0 += kNormChunk) {
    const int n = (I - r0 < kNormChunk) ? (int)(I - r0) : kNormChunk;
    // coalesced: a warp reads 32 consecutive entries of one fiber per instruction
    const int lane = tid & 31, wrp = tid >> 5;
#pragma unroll 4
    for (int c = wrp; c < 128; c += 4) {
      long long j = j0 + c;
      double val = 0.0;
      if (j < J && lane < n) val = __ldcs(x + I * j + r0 + lane);
      tile[c][lane] = val;
    }
    __syncthreads();
    double p = 0.0;
    for (int q = 0; q < n; ++q) {
      double v = tile[tid][q];
      p = fma(v, v, p);
    }
    total = total + p;
    __syncthreads();
  }
  const long long j = j0 + tid;
  if (j < J) w[j] = total;
}

// modes > 0: fiber j = (i, o) at x[i + inner*I*o + inner*r]
__global__ void __launch_bounds__(256) sqnorm_strided_kernel(const double* __restrict__ x,
                                                             ModeView v, double* __restrict__ w) {
  const long long J = v.inner * v.outer;
  const long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= J) return;
  const long long o = j / v.inner, i = j - o * v.inner;
  const double* f = x + i + v.inner * v.I * o;
  double total = 0.0;
  long long r0 = 0;
  for (; r0 + kNormChunk <= v.I; r0 += kNormChunk) {
    double vals[kNormChunk];
#pragma unroll
    for (int q = 0; q < kNormChunk; ++q) vals[q] = __ldcs(f + v.inner * (r0 + q));
    double p = 0.0;
#pragma unroll
    for (int q = 0; q < kNormChunk; ++q) p = fma(vals[q], vals[q], p);
    total = total + p;
  }
  if (r0 < v.I) {
    double p = 0.0;
    for (long long r = r0; r < v.I; ++r) {
      double val = __ldcs(f + v.inner * r);
      p = fma(val, val, p);
    }
    total = total + p;
  }
  w[j] = total;
}

cudaError_t launch_column_sqnorms(const double* x, ModeView v, double* w, cudaStream_t st) {
  const long long J = v.inner * v.outer;
  if (J == 0) return cudaSuccess;
  if (v.inner == 1) {
    sqnorm_contig_kernel<<<(unsigned)((J + 127) / 128), 128, 0, st>>>(x, v.I, J, w); note_launch();
  } else {
    sqnorm_strided_kernel<<<(unsigned)((J + 255) / 256), 256, 0, st>>>(x, v, w); note_launch();
  }
  return cudaGetLastError();
}

}  // namespace lmra_dev

// norms3.cu -- all three modes' canonical column squared norms from ONE read of a 3-way
// tensor (T-HOSVD with sampling: every mode's probabilities come from the same input,
// so the mode passes share the read -- SURVEY 8d rule R2).
//
// Canonical order (shared with the oracle, norms.cu): a column's squared norm is the
// in-order sum of chunk partials, a chunk partial being the fma-sequential sum over 32
// consecutive fiber entries.  Each element belongs to exactly one chunk per mode, so a
// 32 x 32 x 32 brick holds complete chunks of all three modes:
//   pass 1 (this kernel, one read of X): every chunk partial of every mode -> P0, P1, P2
//          (|X|/32 doubles each)
//   pass 2 (combine): per column, the chunk partials added in chunk order.
// Traffic: |X| read + 3 |X|/32 written and read back, vs 3 |X| for three mode passes.
#include "common.cuh"

namespace lmra_dev {

constexpr int kB = 32;          // brick edge = canonical chunk length
constexpr int kN3Threads = 256;

// X[i0, i1, i2], i0 fastest.  Grid: (ceil(I1/32), ceil(I2/32), ceil(I0/32)).
// P0[c0][i1 + I1*i2]  chunk c0 of mode-0 fibers (over i0)
// P1[c1][i0 + I0*i2]  chunk c1 of mode-1 fibers (over i1)
// P2[c2][i0 + I0*i1]  chunk c2 of mode-2 fibers (over i2)
__global__ void __launch_bounds__(kN3Threads) norms3_chunks_kernel(
    const double* __restrict__ x, long long I0, long long I1, long long I2,
    double* __restrict__ P0, double* __restrict__ P1, double* __restrict__ P2) {
  __shared__ double slice[kB][kB + 1];  // [i1][i0] of one i2
  const int tid = threadIdx.x;
  const long long c1 = blockIdx.x, c2 = blockIdx.y, c0 = blockIdx.z;
  const long long i0b = c0 * kB, i1b = c1 * kB, i2b = c2 * kB;
  const int n0 = (int)(I0 - i0b < kB ? I0 - i0b : kB), n1 = (int)(I1 - i1b < kB ? I1 - i1b : kB),
            n2 = (int)(I2 - i2b < kB ? I2 - i2b : kB);
  // mode-2 accumulators: thread owns (i0 = tid % 32, i1 = tid / 32 + 8k), k < 4
  const int a0 = tid & 31, a1 = tid >> 5;
  double acc2[4] = {0.0, 0.0, 0.0, 0.0};
  for (int k2 = 0; k2 < n2; ++k2) {
    const long long i2 = i2b + k2;
    // load the 32 x 32 (i0, i1) slice: rows of 32 contiguous i0 (256 B) per warp
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int r1 = a1 + 8 * k;
      double v = 0.0;
      if (r1 < n1 && a0 < n0) v = __ldcs(x + (i0b + a0) + I0 * ((i1b + r1) + I1 * i2));
      slice[r1][a0] = v;
      acc2[k] = fma(v, v, acc2[k]);  // mode 2: over i2, in order
    }
    __syncthreads();
    if (tid < 32) {  // mode 0 chunk partial of fiber (i1 = tid, i2): over i0 in order
      if (tid < n1) {
        double p = 0.0;
        for (int q = 0; q < n0; ++q) p = fma(slice[tid][q], slice[tid][q], p);
        P0[c0 * (I1 * I2) + (i1b + tid) + I1 * i2] = p;
      }
    } else if (tid < 64) {  // mode 1 chunk partial of fiber (i0 = tid-32, i2): over i1
      const int r0 = tid - 32;
      if (r0 < n0) {
        double p = 0.0;
        for (int q = 0; q < n1; ++q) p = fma(slice[q][r0], slice[q][r0], p);
        P1[c1 * (I0 * I2) + (i0b + r0) + I0 * i2] = p;
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int r1 = a1 + 8 * k;
    if (r1 < n1 && a0 < n0) P2[c2 * (I0 * I1) + (i0b + a0) + I0 * (i1b + r1)] = acc2[k];
  }
}

// w[j] = sum_c P[c][j] in chunk order (c = 0, 1, ...): the canonical combine
__global__ void chunk_combine_kernel(const double* __restrict__ P, long long J, int nchunks,
                                     double* __restrict__ w) {
  const long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= J) return;
  double total = 0.0;
  for (int c = 0; c < nchunks; ++c) total = total + P[(long long)c * J + j];
  w[j] = total;
}

size_t norms3_workspace_doubles(long long I0, long long I1, long long I2) {
  const long long c0 = (I0 + kB - 1) / kB, c1 = (I1 + kB - 1) / kB, c2 = (I2 + kB - 1) / kB;
  return (size_t)(c0 * I1 * I2 + c1 * I0 * I2 + c2 * I0 * I1);
}

cudaError_t launch_norms3(const double* x, long long I0, long long I1, long long I2, double* w0,
                          double* w1, double* w2, double* work, cudaStream_t st) {
  const long long c0 = (I0 + kB - 1) / kB, c1 = (I1 + kB - 1) / kB, c2 = (I2 + kB - 1) / kB;
  double* P0 = work;
  double* P1 = P0 + c0 * I1 * I2;
  double* P2 = P1 + c1 * I0 * I2;
  dim3 grid((unsigned)c1, (unsigned)c2, (unsigned)c0);
  norms3_chunks_kernel<<<grid, kN3Threads, 0, st>>>(x, I0, I1, I2, P0, P1, P2);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  chunk_combine_kernel<<<(unsigned)((I1 * I2 + 255) / 256), 256, 0, st>>>(P0, I1 * I2, (int)c0, w0);
  chunk_combine_kernel<<<(unsigned)((I0 * I2 + 255) / 256), 256, 0, st>>>(P1, I0 * I2, (int)c1, w1);
  chunk_combine_kernel<<<(unsigned)((I0 * I1 + 255) / 256), 256, 0, st>>>(P2, I0 * I1, (int)c2, w2);
  return cudaGetLastError();
}

}  // namespace lmra_dev

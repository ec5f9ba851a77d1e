// verify.cu -- relative_error (tucker.cpp:229-240) on the device: the two sums of the
// reference's loop, num = sum (a - r)^2 and den = sum a^2, over tensors that stay in HBM.
//
// Deterministic: a fixed grid of 148 x 8 CTAs strides over the elements, each CTA reduces
// its threads in a fixed tree, and one thread adds the CTA partials in CTA order; reruns
// give the same bits.  (The reference sums sequentially; the two orders agree to ~1e-15
// relative, far inside the 1e-10 RE contract.)  HBM-bound: 16 B read per element pair.
#include "common.cuh"

namespace lmra_dev {

constexpr int kVerifyBlocks = 148 * 8;
constexpr int kVerifyThreads = 256;

__global__ void __launch_bounds__(kVerifyThreads) diff_sumsq_kernel(const double* __restrict__ a,
                                                                    const double* __restrict__ r, long long n,
                                                                    double* __restrict__ partials) {
  double num = 0.0, den = 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  // two independent loads in flight per thread per iteration
  for (; e + stride < n; e += 2 * stride) {
    const double a0 = __ldcs(a + e), r0 = __ldcs(r + e);
    const double a1 = __ldcs(a + e + stride), r1 = __ldcs(r + e + stride);
    const double d0 = a0 - r0, d1 = a1 - r1;
    num = fma(d0, d0, num);
    den = fma(a0, a0, den);
    num = fma(d1, d1, num);
    den = fma(a1, a1, den);
  }
  if (e < n) {
    const double a0 = a[e], d0 = a0 - r[e];
    num = fma(d0, d0, num);
    den = fma(a0, a0, den);
  }
  __shared__ double sn[kVerifyThreads], sd[kVerifyThreads];
  sn[threadIdx.x] = num;
  sd[threadIdx.x] = den;
  __syncthreads();
  for (int w = kVerifyThreads / 2; w >= 1; w >>= 1) {
    if ((int)threadIdx.x < w) {
      sn[threadIdx.x] += sn[threadIdx.x + w];
      sd[threadIdx.x] += sd[threadIdx.x + w];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    partials[2 * blockIdx.x] = sn[0];
    partials[2 * blockIdx.x + 1] = sd[0];
  }
}

__global__ void sum_pairs_kernel(const double* __restrict__ partials, int nparts, double* __restrict__ out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double num = 0.0, den = 0.0;
  for (int b = 0; b < nparts; ++b) {
    num += partials[2 * b];
    den += partials[2 * b + 1];
  }
  out[0] = num;
  out[1] = den;
}

size_t diff_sumsq_workspace_doubles() { return 2 * (size_t)kVerifyBlocks; }

cudaError_t launch_diff_sumsq(const double* a, const double* r, long long n, double* work, double* out2,
                              cudaStream_t st) {
  diff_sumsq_kernel<<<kVerifyBlocks, kVerifyThreads, 0, st>>>(a, r, n, work); note_launch();
  sum_pairs_kernel<<<1, 32, 0, st>>>(work, kVerifyBlocks, out2); note_launch();
  return cudaGetLastError();
}

}  // namespace lmra_dev

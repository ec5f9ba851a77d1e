// dense.cu -- small kernels of the deterministic baselines (t_hosvd / st_hosvd / hooi,
// tucker.cpp:242-316), whose factors come from SVDs of full unfoldings.
#include "common.cuh"

namespace lmra_dev {

// r (n x n) = upper triangle of a (lda), zeros below the diagonal
__global__ void copy_upper_kernel(const double* __restrict__ a, long long lda, int n, double* __restrict__ r) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < (long long)n * n;
       e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e % n), j = (int)(e / n);
    r[e] = i <= j ? a[i + lda * j] : 0.0;
  }
}

// q (n x mu) = the first mu rows of vt (n x n), transposed: q(i, c) = vt(c, i)
__global__ void rows_to_cols_kernel(const double* __restrict__ vt, int n, int mu, double* __restrict__ q) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < (long long)n * mu;
       e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e % n), c = (int)(e / n);
    q[e] = vt[c + (long long)n * i];
  }
}

// fix_signs (linalg.cpp:13-29): per column the largest |u| (first index on ties) made >= 0
__global__ void __launch_bounds__(256) signfix_columns_kernel(double* __restrict__ u, long long m, int ldu) {
  const int c = blockIdx.x;
  double* col = u + (size_t)ldu * c;
  double best = 0.0;
  long long bi = -1;
  for (long long i = threadIdx.x; i < m; i += blockDim.x) {
    const double a = fabs(col[i]);
    if (a > best) {
      best = a;
      bi = i;
    }
  }
  __shared__ double bv[8];
  __shared__ long long bx[8];
  __shared__ int flip;
#pragma unroll
  for (int msk = 16; msk >= 1; msk >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, msk);
    const long long oi = __shfl_xor_sync(0xffffffffu, bi, msk);
    if (ob > best || (ob == best && oi >= 0 && (bi < 0 || oi < bi))) {
      best = ob;
      bi = oi;
    }
  }
  if ((threadIdx.x & 31) == 0) {
    bv[threadIdx.x >> 5] = best;
    bx[threadIdx.x >> 5] = bi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = 0.0;
    long long ix = -1;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k)
      if (bv[k] > b || (bv[k] == b && bx[k] >= 0 && (ix < 0 || bx[k] < ix))) {
        b = bv[k];
        ix = bx[k];
      }
    flip = ix >= 0 && col[ix] < 0.0;
  }
  __syncthreads();
  if (flip)
    for (long long i = threadIdx.x; i < m; i += blockDim.x) col[i] = -col[i];
}

static unsigned grid_of(long long n) {
  long long g = (n + 255) / 256;
  return (unsigned)std::max<long long>(1, std::min<long long>(g, 148LL * 16));
}

cudaError_t launch_copy_upper(const double* a, long long lda, int n, double* r, cudaStream_t st) {
  copy_upper_kernel<<<grid_of((long long)n * n), 256, 0, st>>>(a, lda, n, r); note_launch();
  return cudaGetLastError();
}

cudaError_t launch_rows_to_cols(const double* vt, int n, int mu, double* q, cudaStream_t st) {
  rows_to_cols_kernel<<<grid_of((long long)n * mu), 256, 0, st>>>(vt, n, mu, q); note_launch();
  return cudaGetLastError();
}

cudaError_t launch_signfix_columns(double* u, long long m, int ldu, int mu, cudaStream_t st) {
  if (mu <= 0) return cudaSuccess;
  signfix_columns_kernel<<<mu, 256, 0, st>>>(u, m, ldu); note_launch();
  return cudaGetLastError();
}

}  // namespace lmra_dev

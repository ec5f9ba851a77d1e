// Per-SM throughput of the pipes a register-resident Jacobi round uses: 64-bit shuffles (as two
// SHFL.32), DFMA, LDS.64/STS.64, measured with 16 warps issuing independent streams.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_rates pipe_rates.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void k(double* out, long long* cyc, int iters) {
  __shared__ double sm[16 * 32 * 8];
  double v[8];
  for (int i = 0; i < 8; ++i) v[i] = threadIdx.x * 0.001 + i;
  for (int i = threadIdx.x; i < 16 * 32 * 8; i += blockDim.x) sm[i] = i;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) v[i] = __shfl_xor_sync(0xffffffffu, v[i], 1 + (i & 3));
      if (OP == 1) v[i] = fma(v[i], 0.999, 0.001);
      if (OP == 2) v[i] += sm[((threadIdx.x >> 5) * 8 + i) * 32 + (threadIdx.x & 31)];
      if (OP == 3) sm[((threadIdx.x >> 5) * 8 + i) * 32 + (threadIdx.x & 31)] = v[i] + it;
      if (OP == 4) v[i] = __shfl_up_sync(0xffffffffu, v[i], 1);
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  double s = 0;
  for (int i = 0; i < 8; ++i) s += v[i];
  out[threadIdx.x] = s + sm[threadIdx.x];
}

int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 8 * 1024); cudaMallocManaged(&cyc, 8);
  const char* nm[] = {"shfl_xor.f64", "dfma", "lds.64", "sts.64", "shfl_up.f64"};
  for (int warps : {1, 4, 8, 16}) {
    const int iters = 1000;
#define RUN(OP) k<OP><<<1, 32 * warps>>>(out, cyc, iters); cudaDeviceSynchronize(); \
    k<OP><<<1, 32 * warps>>>(out, cyc, iters); cudaDeviceSynchronize(); \
    printf("{\"op\": \"%s\", \"warps\": %d, \"warp_instr_per_clk_sm\": %.3f}\n", nm[OP], warps, (double)iters * 8 * warps / cyc[0]);
    RUN(0) RUN(1) RUN(2) RUN(3) RUN(4)
  }
  return 0;
}

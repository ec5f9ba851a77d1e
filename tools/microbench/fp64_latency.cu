// Dependent-chain latency (cycles) of fp64 ops on sm_100a: DFMA, DADD, div, sqrt, rsqrt,
// rcp, hypot, and fp32 equivalents, plus __syncthreads with 1024 threads.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_latency fp64_latency.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void chain(double* out, long long* cyc, int iters, double seed) {
  double x = seed + threadIdx.x * 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (OP == 0) x = fma(x, 0.999999, 1e-9);
    if (OP == 1) x = 1.0 + 0.5 / x;
    if (OP == 2) x = sqrt(x) + 0.5;
    if (OP == 3) x = rsqrt(x) + 0.5;
    if (OP == 4) x = hypot(x, 0.3);
    if (OP == 5) x = __drcp_rn(x) + 0.5;
    if (OP == 6) x = (double)(1.0f + __fdividef(0.5f, (float)x));
    if (OP == 7) x = x + 1e-9;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  out[threadIdx.x] = x;
}

__global__ void bar(long long* cyc, int iters) {
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 4096 * 8);
  cudaMallocManaged(&cyc, 8);
  const char* names[] = {"dfma", "div", "sqrt", "rsqrt", "hypot", "drcp_rn", "fp32 div + cvt", "dadd"};
  const int iters = 1000;
#define RUN(OP)                                              \
  chain<OP><<<1, 32>>>(out, cyc, iters, 1.5);                \
  cudaDeviceSynchronize();                                   \
  chain<OP><<<1, 32>>>(out, cyc, iters, 1.5);                \
  cudaDeviceSynchronize();                                   \
  printf("{\"op\": \"%s\", \"cycles_per_op\": %.1f}\n", names[OP], (double)cyc[0] / iters);
  RUN(0) RUN(1) RUN(2) RUN(3) RUN(4) RUN(5) RUN(6) RUN(7)
  for (int t : {32, 256, 1024}) {
    bar<<<1, t>>>(cyc, iters);
    cudaDeviceSynchronize();
    bar<<<1, t>>>(cyc, iters);
    cudaDeviceSynchronize();
    printf("{\"op\": \"syncthreads_%d\", \"cycles_per_op\": %.1f}\n", t, (double)cyc[0] / iters);
  }
  return 0;
}

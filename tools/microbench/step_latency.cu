// Per-step latency of a barrier-separated dependent chain (the CholeskyQR / Jacobi step shape):
// each step reads a value another warp published in the previous step, runs an fp64 chain on it
// and publishes the next one.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o step_latency step_latency.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double rsq(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double h = 0.5 * x;
  y = y * fma(-h * y, y, 1.5);
  y = y * fma(-h * y, y, 1.5);
  return y;
}
__device__ __forceinline__ void nbar(int n) { asm volatile("bar.sync 1, %0;" ::"r"(n) : "memory"); }

template <int V>
__global__ void k(double* out, long long* cyc, int steps, int nthr) {
  __shared__ double pub[2][64];
  const int tid = threadIdx.x;
  if (tid < 128) pub[tid >> 6][tid & 63] = 1.0 + tid * 1e-3;
  __syncthreads();
  double v[16];
  for (int i = 0; i < 16; ++i) v[i] = tid + i;
  const long long t0 = clock64();
  if (tid < nthr) {
    for (int st = 0; st < steps; ++st) {
      const int par = st & 1;
      double acc = 0.0;
      if (V >= 1) {
        const double d = pub[par][st & 63];
        const double l = pub[par][(tid * 4) & 63];
        double r = V >= 2 ? rsq(d) : d;
        const double m = -(r * r) * l;
        if (V >= 3) {
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = fma(m, v[i & 3] * 1e-9, v[i]);
        }
        acc = m;
        if (tid < 64) pub[par ^ 1][tid] = 1.0 + fabs(acc) * 1e-30 + (V >= 3 ? v[0] * 1e-300 : 0.0);
      }
      if (V == 4) __syncthreads(); else nbar(nthr);
    }
  }
  const long long t1 = clock64();
  if (tid == 0) cyc[0] = t1 - t0;
  double s = 0;
  for (int i = 0; i < 16; ++i) s += v[i];
  out[tid] = s;
}

template <int V>
void run(const char* name, int threads, int nthr) {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1024 * 8);
  cudaMalloc(&cyc, 8);
  const int steps = 2000;
  k<V><<<1, threads>>>(out, cyc, steps, nthr);
  k<V><<<1, threads>>>(out, cyc, steps, nthr);
  long long c = 0;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("%-34s threads %4d (in loop %4d): %6.1f cycles/step  %s\n", name, threads, nthr, (double)c / steps,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  run<0>("barrier only", 320, 320);
  run<1>("lds + publish + barrier", 320, 320);
  run<2>("+ rsqrt chain", 320, 320);
  run<3>("+ 16 dfma", 320, 320);
  run<3>("+ 16 dfma (512 thr, 320 in loop)", 512, 320);
  run<4>("+ 16 dfma, syncthreads 512", 512, 512);
  run<3>("+ 16 dfma, 128 threads", 128, 128);
  run<2>("rsqrt chain, 32 threads", 32, 32);
  return 0;
}

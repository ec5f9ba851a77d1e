// Co-runner for interference tests: `nctas` single-CTA spinners (512 threads) for `cycles` SM
// cycles each, either issuing dependent fp64 FMAs on every warp (kind 0: like the Jacobi/QR
// kernels) or sleeping (kind 1: holds the SM without drawing power).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC -o libspinner.so spinner.cu
#include <cuda_runtime.h>

__global__ void spin(int kind, long long cycles, double* out) {
  const long long t0 = clock64();
  double a = threadIdx.x * 1e-3, b = 1.0 + a, c = 2.0 + a, d = 3.0 + a;
  while (clock64() - t0 < cycles) {
    if (kind == 0) {
#pragma unroll
      for (int i = 0; i < 64; ++i) {
        a = fma(a, 0.999999, 1e-9);
        b = fma(b, 0.999999, 1e-9);
        c = fma(c, 0.999999, 1e-9);
        d = fma(d, 0.999999, 1e-9);
      }
    } else {
      __nanosleep(1000);
    }
  }
  if (a + b + c + d == 0.123) out[0] = a;
}

extern "C" int spin_launch(int kind, int nctas, long long cycles, void* stream, double* out) {
  spin<<<nctas, 512, 0, (cudaStream_t)stream>>>(kind, cycles, out);
  return (int)cudaGetLastError();
}

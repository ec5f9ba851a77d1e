// Per-phase cycles of the register-resident Jacobi (orth.cu reg_jacobi) on a graded s x s R^T.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o jacobi2_bench jacobi2_bench.cu
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>
#define LMRA_JACOBI_CLOCKS 1
#include "../../paper_2303_11612_b200/csrc/kernels/orth.cu"
using namespace lmra_dev;

__global__ void __launch_bounds__(512) jb(const double* Rt, int s, long long* out) {
  extern __shared__ double sm[];
  const QSmem q = carve_q(sm);
  double* G = sm + kQScratchBytes / 8;
  double* J = G + s * s;
  for (int e = threadIdx.x; e < s * s; e += 512) G[e] = Rt[e];
  __syncthreads();
  long long t0 = clock64();
  bool ok = reg_jacobi(G, s, J, 8.0 * s * 0x1.0p-53, q);
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = ok; }
}

int main() {
  long long* out;
  cudaMallocManaged(&out, 16);
  for (int s : {16, 30, 60}) {
    std::vector<double> h(s * s, 0.0);
    srand(1);
    for (int i = 0; i < s; ++i)
      for (int j = i; j < s; ++j)  // R upper, graded rows; G = R^T
        h[j + s * i] = ((rand() / (double)RAND_MAX) - 0.5) * pow(10.0, -10.0 * i / s) * (i == j ? 4.0 : 1.0) * 0.5;
    double* d;
    cudaMalloc(&d, s * s * 8);
    cudaMemcpy(d, h.data(), s * s * 8, cudaMemcpyHostToDevice);
    size_t smem = kQScratchBytes + (s * s + 64 * 64) * 8 + 64;
    cudaFuncSetAttribute(jb, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int rep = 0; rep < 2; ++rep) {
      unsigned long long z[8] = {0};
      cudaMemcpyToSymbol(g_jclk, z, sizeof(z));
      jb<<<1, 512, smem>>>(d, s, out);
      cudaDeviceSynchronize();
    }
    unsigned long long c[8];
    cudaMemcpyFromSymbol(c, g_jclk, sizeof(c));
    double R = (double)c[4];
    printf("{\"s\": %d, \"cycles\": %lld, \"ok\": %lld, \"sweeps\": %d, \"rounds\": %.0f, \"cyc_per_round\": %.0f, "
           "\"partials_barA\": %.0f, \"angles\": %.0f, \"barB\": %.0f, \"rotate_shift\": %.0f, \"J_wait\": %.0f, \"J_rot\": %.0f}\n",
           s, out[0], out[1], last_jacobi_sweeps(), R, out[0] / R, c[0] / R, c[1] / R, c[2] / R, c[3] / R, c[5] / R, c[6] / R);
    cudaFree(d);
  }
  return 0;
}

// Where the int8 tensor-core contraction (ttm_i8.cu) waits: per-role mbarrier wait cycles of
// CTA 0 on cfg4's shape (K = 1000, J = 10^6, mu = 50), X random normal.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lcuda -o i8_clocks i8_clocks.cu
#include <cstdio>
#include <vector>
#define LMRA_I8_CLOCKS 1
#include "../../paper_2303_11612_b200/csrc/kernels/ttm_i8.cu"
using namespace lmra_dev;

__global__ void fill(double* x, size_t n, unsigned long long seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    unsigned long long z = (i + 1) * 0x9E3779B97F4A7C15ull ^ seed;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    x[i] = ((double)(z >> 11) / 9007199254740992.0) - 0.5;
  }
}
__global__ void colnorm(const double* x, int K, long long J, double* w) {
  long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (j >= J) return;
  double s = 0;
  for (int k = 0; k < K; ++k) s = fma(x[k + K * j], x[k + K * j], s);
  w[j] = s;
}

int main(int argc, char** argv) {
  const bool with_fexp = argc > 1 && argv[1][0] == 'f';  // also hand exponents to a mode-1 pass
  const int K = 1000, mu = 50;
  const long long J = 1000000;
  double *x, *q, *w, *y;
  void* work;
  cudaMalloc(&x, (size_t)K * J * 8);
  cudaMalloc(&q, (size_t)K * mu * 8);
  cudaMalloc(&w, (size_t)J * 8);
  cudaMalloc(&y, (size_t)mu * J * 8);
  cudaMalloc(&work, ttm_i8_workspace_bytes(K, mu));
  int* fexp = nullptr;
  cudaMalloc(&fexp, (size_t)mu * 1000 * sizeof(int));
  fill<<<4096, 256>>>(x, (size_t)K * J, 1);
  fill<<<64, 256>>>(q, (size_t)K * mu, 2);
  colnorm<<<(J + 255) / 256, 256>>>(x, K, J, w);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 3; ++rep) {
    unsigned long long z[20] = {0};
    cudaMemcpyToSymbol(g_i8clk, z, sizeof(z));
    if (with_fexp) cudaMemset(fexp, 0x80, (size_t)mu * 1000 * sizeof(int));
    cudaEventRecord(e0);
    cudaError_t e = launch_ttm_i8(x, K, J, q, mu, w, y, work, 0, with_fexp ? fexp : nullptr, 1000);
    cudaEventRecord(e1);
    cudaDeviceSynchronize();
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long c[20];
    cudaMemcpyFromSymbol(c, g_i8clk, sizeof(c));
    const double cyc = (double)c[15];  // CTA 0's span in SM clocks (the clock drops under load)
    const double mhz = cyc / (ms * 1e3);
    printf("{\"ms\": %.3f, \"err\": \"%s\", \"cta0_cycles\": %.0f, \"sm_mhz\": %.0f, \"frac\": {\"x_prod_wait_empty\": %.3f, "
           "\"q_prod_wait_qempty\": %.3f, \"mma_wait_accempty\": %.3f, \"mma_wait_afull\": %.3f, "
           "\"mma_wait_qfull\": %.3f, \"slicer0_wait_full\": %.3f, \"slicer0_wait_aempty\": %.3f, "
           "\"slicer1_wait_full\": %.3f, \"slicer1_wait_aempty\": %.3f, \"epi_wait_accfull\": %.3f, "
           "\"slicer_convert\": %.3f, \"slicer_tmem_st\": %.3f, \"mma_issue\": %.3f, \"epi_busy\": %.3f, \"epi_to_release\": %.3f, \"epi_stores\": %.3f, \"epi_tmem_ld\": %.3f, \"epi_compute\": %.3f}}\n",
           ms, cudaGetErrorString(e), cyc, mhz, c[0] / cyc, c[1] / cyc, c[2] / cyc, c[3] / cyc, c[4] / cyc,
           c[5] / cyc / 4, c[6] / cyc / 4, c[9] / cyc / 4, c[10] / cyc / 4, c[7] / cyc / 8,
           c[11] / cyc / 8, c[12] / cyc / 8, c[13] / cyc, c[14] / cyc / 8, c[8] / cyc / 8, c[16] / cyc / 8, c[17] / cyc / 8, c[18] / cyc / 8);
  }
  return 0;
}

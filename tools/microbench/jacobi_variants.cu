// Cycles per Jacobi round of the three forms in orth.cu on a graded s x s R^T (one CTA of 512
// threads, G in shared memory): reg_jacobi (block barriers, warp 0 forms the angles),
// narrow_jacobi (s <= 32: G and J warps, no block barrier).  -DNO_CLOCKS: without the per-phase
// clock64 bookkeeping (which costs the narrow form ~200 cycles a round).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o jacobi_variants jacobi_variants.cu
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>
#ifndef NO_CLOCKS
#define LMRA_JACOBI_CLOCKS 1
#endif
#include "../../paper_2303_11612_b200/csrc/kernels/orth.cu"
#include "../../paper_2303_11612_b200/csrc/kernels/cholqr.cu"
using namespace lmra_dev;
namespace lmra_dev {  // host launchers orth.cu references but this benchmark never calls
cudaError_t launch_transpose(const double*, long long, long long, double*, cudaStream_t) { return cudaErrorNotSupported; }
cudaError_t scratch_alloc(void**, size_t, cudaStream_t) { return cudaErrorNotSupported; }
void scratch_free(void*, cudaStream_t) {}
}

__global__ void __launch_bounds__(512) jv(const double* Rt, int s, int variant, long long* out) {
  extern __shared__ double sm[];
  const QSmem q = carve_q(sm);
  double* G = sm + kQScratchBytes / 8;
  double* J = G + s * s;
  for (int e = threadIdx.x; e < s * s; e += 512) G[e] = Rt[e];
  __syncthreads();
  long long t0 = clock64();
  bool ok = variant == 0 ? reg_jacobi(G, s, J, 8.0 * s * 0x1.0p-53, q) : narrow_jacobi(G, s, J, 8.0 * s * 0x1.0p-53, q);
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = ok; }
}

int main() {
  long long* out;
  cudaMallocManaged(&out, 16);
  for (int s : {15, 20, 24, 30, 32}) {
    std::vector<double> h(s * s, 0.0);
    srand(1);
    for (int i = 0; i < s; ++i)
      for (int j = i; j < s; ++j)
        h[j + s * i] = ((rand() / (double)RAND_MAX) - 0.5) * pow(10.0, -6.0 * i / s) * (i == j ? 4.0 : 1.0) * 0.5;
    double* d;
    cudaMalloc(&d, s * s * 8);
    cudaMemcpy(d, h.data(), s * s * 8, cudaMemcpyHostToDevice);
    size_t smem = kQScratchBytes + (s * s + 64 * 64) * 8 + 64;
    cudaFuncSetAttribute(jv, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int variant = 0; variant < 2; ++variant) {
      jv<<<1, 512, smem>>>(d, s, variant, out);
      cudaDeviceSynchronize();
#ifdef LMRA_JACOBI_CLOCKS
      unsigned long long z[8] = {0};
      cudaMemcpyToSymbol(g_jclk, z, sizeof(z));
#endif
      cudaDeviceSynchronize();
      jv<<<1, 512, smem>>>(d, s, variant, out);
      cudaDeviceSynchronize();
      const int sw = last_jacobi_sweeps();
      const int P = (s + 1) / 2;
      unsigned long long c[8] = {0};
#ifdef LMRA_JACOBI_CLOCKS
      cudaMemcpyFromSymbol(c, g_jclk, sizeof(c));
#endif
      const double R = variant ? (double)c[4] : 1.0;
      printf("s %2d %-7s: %8lld cycles, ok %lld, sweeps %d, %.0f cycles/round  %s", s, variant ? "narrow" : "block",
             out[0], out[1], sw, out[0] / (double)(sw * (2 * P - 1)), cudaGetErrorString(cudaGetLastError()));
      if (variant && c[4]) printf("  [G warp: dots+angle %.0f, barrier %.0f, rotate+move %.0f]", c[0] / R, c[1] / R, c[2] / R);
      printf("\n");
    }
    cudaFree(d);
  }
  return 0;
}

// Cycles per Householder step of the register-resident QR / apply (orth.cu reg_qr,
// reg_apply) on an m x s block, one CTA of 512 threads.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o qr_bench qr_bench.cu
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>
#define LMRA_QR_CLOCKS 1
#include "../../paper_2303_11612_b200/csrc/kernels/orth.cu"
#include "../../paper_2303_11612_b200/csrc/kernels/cholqr.cu"
using namespace lmra_dev;
namespace lmra_dev {  // host launchers orth.cu references but this benchmark never calls
cudaError_t launch_transpose(const double*, long long, long long, double*, cudaStream_t) { return cudaErrorNotSupported; }
cudaError_t scratch_alloc(void**, size_t, cudaStream_t) { return cudaErrorNotSupported; }
void scratch_free(void*, cudaStream_t) {}
}

template <int RPL>
__global__ void __launch_bounds__(512) qb(const double* A, int m, int s, int pivot, long long* out) {
  extern __shared__ __align__(16) double sm[];
  const QSmem q = carve_q(sm);
  double* tile = sm + kQScratchBytes / 8;
  const int ldt = (32 * RPL) | 1;
  load_tile(A, m, m, s, tile, ldt, 32 * RPL);
  __syncthreads();
  double a[kCW][RPL];
  cw_load(tile, ldt, m, s, a);
  __syncthreads();
  long long t0 = clock64();
  reg_qr(a, m, s, q, pivot != 0);
  __syncthreads();
  long long t1 = clock64();
  cw_store(a, m, s, tile, ldt);
  __syncthreads();
  double y[kCW][RPL];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
#pragma unroll
  for (int j = 0; j < kCW; ++j)
#pragma unroll
    for (int i = 0; i < RPL; ++i) y[j][i] = (l + 32 * i == w + 16 * j) ? 1.0 : 0.0;
  __syncthreads();
  long long t2 = clock64();
  reg_apply(y, s, tile, ldt, q.tau, min(m, s), 0);
  __syncthreads();
  long long t3 = clock64();
  double chk = 0;
#pragma unroll
  for (int j = 0; j < kCW; ++j)
#pragma unroll
    for (int i = 0; i < RPL; ++i) chk += y[j][i];
  if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = t3 - t2; out[2] = (long long)chk; }
}

template <int RPL>
void run(int m, int s, int pivot) {
  std::vector<double> h((size_t)m * s);
  srand(1);
  for (auto& v : h) v = rand() / (double)RAND_MAX - 0.5;
  double* d;
  long long* out;
  cudaMalloc(&d, h.size() * 8);
  cudaMallocManaged(&out, 32);
  cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  size_t smem = kQScratchBytes + sizeof(double) * ((32 * RPL) | 1) * s + 64;
  cudaFuncSetAttribute(qb<RPL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int rep = 0; rep < 3; ++rep) qb<RPL><<<1, 512, smem>>>(d, m, s, pivot, out);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long c[8];
  cudaMemcpyFromSymbol(c, g_qrclk, sizeof(c));
  printf("  per step (warp 0): pivot %.0f, reflector %.0f, barrier %.0f, update %.0f, norms %.0f\n", c[0] / (double)s,
         c[1] / (double)s, c[2] / (double)s, c[3] / (double)s, c[4] / (double)s);
  printf("{\"rpl\": %d, \"m\": %d, \"s\": %d, \"pivot\": %d, \"qr_cycles\": %lld, \"qr_per_step\": %.0f, "
         "\"apply_cycles\": %lld, \"apply_per_step\": %.0f, \"err\": \"%s\"}\n",
         RPL, m, s, pivot, out[0], out[0] / (double)s, out[1], out[1] / (double)s, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<8>(250, 60, 0);
  run<8>(240, 60, 1);
  run<8>(256, 50, 0);
  run<4>(100, 50, 0);
  run<4>(100, 50, 1);
  run<4>(128, 50, 1);
  run<2>(60, 30, 0);
  run<2>(60, 30, 1);
  run<4>(120, 60, 0);
  run<2>(60, 60, 0);
  return 0;
}

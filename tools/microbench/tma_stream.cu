// TMA streaming ceiling for the int8 TTM's X access pattern: boxes of 16 doubles (128 B, 128 B
// swizzle) x R columns of a K x J column-major matrix, 1 CTA per SM, S stages, consumers only
// release stages.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2303_11612_b200/csrc/kernels
#include <cstdio>
#include <cuda.h>
#include <cudaTypedefs.h>
#include "common.cuh"
using namespace lmra_dev;

template <int S, int R, int NCONS>
__global__ void __launch_bounds__(32 * (NCONS + 1), 1) stream_kernel(const __grid_constant__ CUtensorMap map, int K, long long J) {
  extern __shared__ __align__(16) unsigned char smraw[];
  unsigned char* base = smraw + ((1024 - (smem_u32(smraw) & 1023)) & 1023);
  constexpr int kBox = 16 * R * 8;  // bytes per box
  uint64_t* full = reinterpret_cast<uint64_t*>(base + S * 2 * kBox);
  uint64_t* empty = full + S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], NCONS); }
    mbar_fence_init();
  }
  __syncthreads();
  const int nks = (K + 31) / 32;
  const long long ntiles = (J + R - 1) / R;
  if (warp == NCONS) {
    if (lane == 0) {
      long long g = 0;
      for (long long t = blockIdx.x; t < ntiles; t += gridDim.x)
        for (int ks = 0; ks < nks; ++ks, ++g) {
          const int st = (int)(g % S);
          mbar_wait(&empty[st], (unsigned)((g / S) & 1) ^ 1u);
          mbar_arrive_expect_tx(&full[st], 2 * kBox);
          unsigned char* dst = base + (size_t)st * 2 * kBox;
          asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];\n"
                       :: "r"(smem_u32(dst)), "l"(&map), "r"(smem_u32(&full[st])), "r"(ks * 32), "r"((int)(t * R)) : "memory");
          asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];\n"
                       :: "r"(smem_u32(dst + kBox)), "l"(&map), "r"(smem_u32(&full[st])), "r"(ks * 32 + 16), "r"((int)(t * R)) : "memory");
        }
    }
  } else {
    long long g = 0;
    for (long long t = blockIdx.x; t < ntiles; t += gridDim.x)
      for (int ks = 0; ks < nks; ++ks, ++g) {
        const int st = (int)(g % S);
        mbar_wait(&full[st], (unsigned)((g / S) & 1));
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
      }
  }
}

template <int S, int R, int NCONS>
float run(const CUtensorMap& map, int K, long long J) {
  const size_t smem = S * 2 * (16 * R * 8) + 2 * S * 8 + 1024;
  cudaFuncSetAttribute(stream_kernel<S, R, NCONS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  stream_kernel<S, R, NCONS><<<148, 32 * (NCONS + 1), smem>>>(map, K, J);
  cudaEventRecord(a);
  for (int i = 0; i < 5; ++i) stream_kernel<S, R, NCONS><<<148, 32 * (NCONS + 1), smem>>>(map, K, J);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("{\"S\": %d, \"R\": %d, \"ms\": %.3f, \"GBps\": %.1f, \"err\": \"%s\"}\n", S, R, ms / 5,
         (double)K * J * 8 / (ms / 5 / 1e3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  return ms / 5;
}

int main() {
  const int K = 1000; const long long J = 1000000;
  double* x; cudaMalloc(&x, (size_t)K * J * 8); cudaMemset(x, 0, (size_t)K * J * 8);
  void* p; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  for (int R : {128, 64, 256}) {
    CUtensorMap map;
    const cuuint64_t gdim[2] = {(cuuint64_t)K, (cuuint64_t)J};
    const cuuint64_t gstride[1] = {(cuuint64_t)K * 8};
    const cuuint32_t box[2] = {16, (cuuint32_t)R}, es[2] = {1, 1};
    enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, x, gdim, gstride, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (R == 128) { run<5, 128, 4>(map, K, J); run<3, 128, 4>(map, K, J); run<6, 128, 4>(map, K, J); }
    if (R == 64) { run<8, 64, 4>(map, K, J); run<12, 64, 4>(map, K, J); }
    if (R == 256) { run<3, 256, 4>(map, K, J); }
  }
  return 0;
}

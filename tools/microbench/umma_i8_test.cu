// Bring-up test for tcgen05.mma.kind::i8 with hand-built descriptors (sm_100a):
//   D (128 x N, int32, TMEM) = A (128 x K, K-major int8) * B (N x K, K-major int8)^T
// A signed, B unsigned (the Ozaki TTM mixes signed top digits with unsigned low digits).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma_i8_test umma_i8_test.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// K-major, no swizzle: core matrices of 8 rows x 16 bytes; LBO = byte stride between the two
// 16-byte K chunks of one MMA, SBO = byte stride between 8-row groups.
__device__ __forceinline__ uint64_t smem_desc(const void* p, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_u32(p) >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version (sm100)
  return d;              // base offset 0, lbo mode 0, layout SWIZZLE_NONE (0)
}

__host__ __device__ constexpr uint32_t idesc_i8(int M, int N, bool a_signed, bool b_signed) {
  return (2u << 4)                        // D format S32
         | ((a_signed ? 1u : 0u) << 7)    // A format
         | ((b_signed ? 1u : 0u) << 10)   // B format
         | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

template <int N, int K>
__global__ void test_kernel(const int8_t* A, const uint8_t* B, int32_t* D) {
  constexpr int M = 128;
  __shared__ __align__(1024) uint8_t sa[M * K];
  __shared__ __align__(1024) uint8_t sb[N * K];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t mbar;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // canonical layout per 32-byte K step: [kstep][group of 8 rows][chunk 2][row 8][16 B]
  for (int e = tid; e < M * K; e += blockDim.x) {
    const int r = e / K, k = e % K;
    const int ks = k / 32, c = (k % 32) / 16, b = k % 16;
    sa[ks * (M * 32) + (r / 8) * 256 + c * 128 + (r % 8) * 16 + b] = (uint8_t)A[r * K + k];
  }
  for (int e = tid; e < N * K; e += blockDim.x) {
    const int r = e / K, k = e % K;
    const int ks = k / 32, c = (k % 32) / 16, b = k % 16;
    sb[ks * (N * 32) + (r / 8) * 256 + c * 128 + (r % 8) * 16 + b] = B[r * K + k];
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base)), "r"(N));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  // make the generic-proxy smem writes visible to the tensor core (async proxy)
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = tmem_base;
  if (tid == 0) {
    constexpr uint32_t idesc = idesc_i8(M, N, true, false);
    for (int ks = 0; ks < K / 32; ++ks) {
      const uint64_t da = smem_desc(sa + ks * (M * 32), 128, 256);
      const uint64_t db = smem_desc(sb + ks * (N * 32), 128, 256);
      const uint32_t acc = ks > 0 ? 1u : 0u;
      asm volatile(
          "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
          " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
          "l"(da), "l"(db), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&mbar))
                 : "memory");
  }
  // wait for the MMAs
  asm volatile(
      "{\n .reg .pred P1;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n @!P1 bra W_%=;\n}\n" ::"r"(
          smem_u32(&mbar))
      : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  // warp w reads lanes 32w..32w+31 (rows), 16 columns at a time
  for (int c0 = 0; c0 < N; c0 += 16) {
    uint32_t v[16];
    const uint32_t taddr = tmem + ((uint32_t)(32 * warp) << 16) + c0;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
    const int row = 32 * warp + lane;
    for (int j = 0; j < 16; ++j) D[row * N + c0 + j] = (int32_t)v[j];
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(N));
}

// A from TMEM: each thread writes its row (lane) of A, K/4 32-bit columns, 4 int8 per column
template <int N, int K>
__global__ void test_kernel_tmemA(const int8_t* A, const uint8_t* B, int32_t* D) {
  constexpr int M = 128;
  __shared__ __align__(1024) uint8_t sb[N * K];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t mbar;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int e = tid; e < N * K; e += blockDim.x) {
    const int r = e / K, k = e % K;
    const int ks = k / 32, c = (k % 32) / 16, b = k % 16;
    sb[ks * (N * 32) + (r / 8) * 256 + c * 128 + (r % 8) * 16 + b] = B[r * K + k];
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = tmem_base;
  const uint32_t a_col = 128;  // A tiles at columns [128, 128 + K/4)
  {  // row = 32*warp + lane: 8 columns per 32-byte K step
    const int row = 32 * warp + lane;
    for (int ks = 0; ks < K / 32; ++ks) {
      uint32_t w[8];
      for (int c = 0; c < 8; ++c) {
        uint32_t v = 0;
        for (int b = 0; b < 4; ++b) v |= (uint32_t)(uint8_t)A[row * K + ks * 32 + 4 * c + b] << (8 * b);
        w[c] = v;
      }
      const uint32_t taddr = tmem + ((uint32_t)(32 * warp) << 16) + a_col + ks * 8;
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(taddr),
                   "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  if (tid == 0) {
    constexpr uint32_t idesc = idesc_i8(M, N, true, false);
    for (int ks = 0; ks < K / 32; ++ks) {
      const uint64_t db = smem_desc(sb + ks * (N * 32), 128, 256);
      const uint32_t acc = ks > 0 ? 1u : 0u;
      asm volatile(
          "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
          " tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem),
          "r"(tmem + a_col + ks * 8), "l"(db), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&mbar))
                 : "memory");
  }
  asm volatile(
      "{\n .reg .pred P1;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n @!P1 bra W_%=;\n}\n" ::"r"(
          smem_u32(&mbar))
      : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  for (int c0 = 0; c0 < N; c0 += 16) {
    uint32_t v[16];
    const uint32_t taddr = tmem + ((uint32_t)(32 * warp) << 16) + c0;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
    const int row = 32 * warp + lane;
    for (int j = 0; j < 16; ++j) D[row * N + c0 + j] = (int32_t)v[j];
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(256));
}

int main() {
  constexpr int M = 128, N = 64, K = 96;
  std::vector<int8_t> A(M * K);
  std::vector<uint8_t> B(N * K);
  srand(3);
  for (auto& a : A) a = (int8_t)((rand() % 256) - 128);
  for (auto& b : B) b = (uint8_t)(rand() % 256);
  int8_t* dA;
  uint8_t* dB;
  int32_t* dD;
  cudaMalloc(&dA, M * K);
  cudaMalloc(&dB, N * K);
  cudaMalloc(&dD, M * N * 4);
  cudaMemcpy(dA, A.data(), M * K, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), N * K, cudaMemcpyHostToDevice);
  cudaMemset(dD, 0, M * N * 4);
  long long bad = 0;
  for (int variant = 0; variant < 2; ++variant) {
  cudaMemset(dD, 0, M * N * 4);
  if (variant == 0)
    test_kernel<N, K><<<1, 128>>>(dA, dB, dD);
  else
    test_kernel_tmemA<N, K><<<1, 128>>>(dA, dB, dD);
  cudaError_t e = cudaDeviceSynchronize();
  printf("variant %d kernel: %s\n", variant, cudaGetErrorString(e));
  std::vector<int32_t> D(M * N);
  cudaMemcpy(D.data(), dD, M * N * 4, cudaMemcpyDeviceToHost);
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      long long ref = 0;
      for (int k = 0; k < K; ++k) ref += (long long)A[i * K + k] * (long long)B[j * K + k];
      if (ref != D[i * N + j]) {
        if (bad < 5) printf("mismatch (%d,%d): got %d want %lld\n", i, j, D[i * N + j], ref);
        ++bad;
      }
    }
  printf("{\"umma_i8_test_variant\": %d, \"mismatches_so_far\": %lld}\n", variant, bad);
  }
  printf("{\"umma_i8_test\": \"%s\", \"mismatches\": %lld}\n", bad ? "FAIL" : "PASS", bad);
  return bad ? 1 : 0;
}

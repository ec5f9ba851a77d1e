// tcgen05.mma.kind::i8 issue rate vs N (M = 128, K = 32, A from TMEM or smem, B from smem).
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t a) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)8 << 16) | ((uint64_t)16 << 32) | ((uint64_t)1 << 46);
}
template <int N, bool ATMEM>
__global__ void rate_kernel(long long* out, int iters) {
  __shared__ __align__(1024) uint8_t sa[128 * 32];
  __shared__ __align__(1024) uint8_t sb[256 * 32];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  for (int i = threadIdx.x; i < 128 * 32; i += blockDim.x) sa[i] = (uint8_t)i;
  for (int i = threadIdx.x; i < 256 * 32; i += blockDim.x) sb[i] = (uint8_t)(3 * i);
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint64_t da = sdesc(smem_u32(sa)), db = sdesc(smem_u32(sb));
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if (ATMEM)
        asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n"
                     ::"r"(tmem), "r"(tmem + 448), "l"(db), "r"(idesc), "r"(1));
      else
        asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                     ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(1));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&bar)) : "memory");
    asm volatile("{\n .reg .pred P1;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n @!P1 bra W_%=;\n}\n" ::"r"(smem_u32(&bar)) : "memory");
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}
template <int N, bool AT>
void run() {
  long long* d; cudaMalloc(&d, 148 * 8);
  const int iters = 4096;
  rate_kernel<N, AT><<<148, 128>>>(d, iters);
  rate_kernel<N, AT><<<148, 128>>>(d, iters);
  long long h[148]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double cyc = (double)h[0] / iters;
  double macs = 128.0 * N * 32;
  printf("{\"N\": %d, \"A_tmem\": %d, \"cycles_per_mma\": %.1f, \"MAC_per_clk\": %.0f, \"TOPS_at_1.965GHz_148SM\": %.0f, \"err\": \"%s\"}\n",
         N, (int)AT, cyc, macs / cyc, 2 * macs / cyc * 1.965e9 * 148 / 1e12, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}
int main() {
  run<64, true>(); run<64, false>(); run<128, true>(); run<128, false>(); run<192, true>(); run<192, false>(); run<256, true>(); run<256, false>(); run<32, true>(); run<16, true>();
  return 0;
}

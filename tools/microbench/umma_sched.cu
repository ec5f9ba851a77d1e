// The int8 contraction's per-K-step MMA schedule (ttm_i8.cu: 9 grouped tcgen05.mma.kind::i8,
// N = 192/128/64, A from TMEM, B from a Q-digit ring in smem) issued back to back without
// any producer / consumer: the tensor pipe's own time per K-step.  Variants: +slicer-like
// tcgen05.st traffic into the other A buffer, +epilogue-like tcgen05.ld traffic.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t a) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)8 << 16) | ((uint64_t)16 << 32) | ((uint64_t)1 << 46);
}
constexpr int N = 64, kQBytes = 6 * N * 32, kQStages = 6, kAcc = 6 * N;
template <int MODE>  // 0: MMAs only, 1: + tcgen05.st traffic, 2: + tcgen05.ld traffic, 3: both
__global__ void __launch_bounds__(256, 1) sched_kernel(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t qs[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  __shared__ int stop;
  for (int i = threadIdx.x; i < kQStages * kQBytes; i += blockDim.x) qs[i] = (uint8_t)(i * 7);
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (threadIdx.x == 0) {
    stop = 0;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = tslot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    constexpr int kSched[9][3] = {{5, 0, 3}, {5, 3, 3}, {4, 1, 2}, {4, 3, 3}, {3, 2, 2},
                                  {3, 4, 2}, {2, 3, 3}, {1, 4, 2}, {0, 5, 1}};
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const uint32_t qbase = smem_u32(qs + (it % kQStages) * kQBytes);
      const uint32_t abase = tmem + kAcc + (uint32_t)(it & 1) * 48;
#pragma unroll
      for (int gi = 0; gi < 9; ++gi) {
        const int dt = kSched[gi][0], s0 = kSched[gi][1], gl = kSched[gi][2];
        const int L = dt + s0 - 5;
        const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)((gl * N) >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
        const uint64_t bdesc = sdesc(qbase + (uint32_t)(s0 * N * 32));
        asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n"
                     ::"r"(tmem + (uint32_t)L * N), "r"(abase + (uint32_t)dt * 8), "l"(bdesc), "r"(idesc), "r"(1));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&bar)) : "memory");
    asm volatile("{\n .reg .pred P1;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n @!P1 bra W_%=;\n}\n" ::"r"(smem_u32(&bar)) : "memory");
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
    *(volatile int*)&stop = 1;
  } else if ((MODE & 1) && warp >= 4) {  // tcgen05.st into A buffers (slicer-like), 4 warps
    const uint32_t lb = (uint32_t)(32 * (warp & 3)) << 16;
    uint32_t v = threadIdx.x;
    while (!*(volatile int*)&stop) {
      for (int s = 0; s < 6; ++s)
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};\n" ::"r"(tmem + lb + kAcc + 96 + 8 * (s & 1)), "r"(v));
      asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
      __nanosleep(200);
    }
  } else if ((MODE & 2) && warp >= 1 && warp < 4) {  // tcgen05.ld traffic (epilogue-like)
    const uint32_t lb = (uint32_t)(32 * (warp & 3)) << 16;
    uint32_t acc = 0;
    while (!*(volatile int*)&stop) {
      uint32_t r[8];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                   : "r"(tmem + lb + 8 * (acc & 31)));
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
      acc += r[0] + r[7];
      __nanosleep(100);
    }
    if (acc == 12345) out[0] = 0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}
template <int MODE>
void run() {
  long long* d; cudaMalloc(&d, 148 * 8);
  const int iters = 2000;
  const int smem = kQStages * kQBytes;
  cudaFuncSetAttribute(sched_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  sched_kernel<MODE><<<148, 256, smem>>>(d, iters);
  sched_kernel<MODE><<<148, 256, smem>>>(d, iters);
  long long h[148]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("{\"mode\": %d, \"cycles_per_kstep\": %.1f, \"ideal\": 686, \"err\": \"%s\"}\n", MODE, (double)h[0] / iters,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}
int main() { run<0>(); run<1>(); run<2>(); run<3>(); return 0; }

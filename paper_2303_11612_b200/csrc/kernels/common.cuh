// common.cuh -- shared device helpers for the sm_100a fp64 kernels.
//
// fp64 on Blackwell: tcgen05.mma has no f64 kind, so fp64 tensor work is the
// warp-level mma.sync ... f64 family, which lowers to DMMA.8x8x4 in SASS
// (measured peak 37.0 TFLOP/s on B200, profiles/fp64_peaks_r01.json, vs 33.9 for
// a DFMA loop).  Tiles are staged global->shared with cp.async (LDGSTS) in a
// multi-stage ring so HBM streaming overlaps the DMMA issue.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "kernels.hpp"

namespace lmra_dev {

// Programmatic dependent launch: a kernel launched with launch_pdl may be scheduled while the
// previous kernel in its stream drains (its launch latency overlaps that tail); it must call
// pdl_wait() before touching anything the previous kernel wrote (griddepcontrol.wait returns
// once the prerequisite grid has completed and its writes are visible; it is a no-op for a
// normal launch).  pdl_trigger() lets the dependent grid launch once every CTA of this one
// has started.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  note_launch();
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}


// The canonical column squared norm (shared with the oracle, canonical_sqnorm): chunks of 32
// fibre entries summed by an fma chain from +0, pairs of chunks (64-entry segments) summed,
// segment sums added in order.  canon_add folds chunk c's partial p into (seg, total); `last`
// marks the fibre's final chunk.
__device__ __forceinline__ void canon_add(double p, long long c, bool last, double& seg, double& total) {
  seg = (c & 1) ? seg + p : p;
  if ((c & 1) || last) total = total + seg;
}

__device__ __forceinline__ long long col_base(long long j, long long inner, long long I) {
  if (inner == 1) return j * I;
  long long o = j / inner;
  long long i = j - o * inner;
  return i + inner * I * o;
}

// D(16x8) += A(16x4) * B(4x8), fp64, fragments per PTX ISA m16n8k4 .f64:
//   a0 = A[g][t], a1 = A[g+8][t]; b = B[t][g]; d0,d1 = D[g][2t..2t+1], d2,d3 = D[g+8][2t..2t+1]
// with g = lane / 4, t = lane % 4.
__device__ __forceinline__ void dmma16x8x4(double (&d)[4], double a0, double a1, double b) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
      "{%0,%1,%2,%3};\n"
      : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
      : "d"(a0), "d"(a1), "d"(b));
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// 8-byte async copy; src_bytes = 0 zero-fills the destination.
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(smem)),
               "l"(gmem), "r"(valid ? 8 : 0));
}

// 16-byte async copy (L2 only, bypass L1); src_bytes = 0 zero-fills.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(smem)),
               "l"(gmem), "r"(valid ? 16 : 0));
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }

template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// ---- mbarrier / TMA (sm_90+ async proxy) ----
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
// ---- thread-block clusters / distributed shared memory ----
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
// this CTA's shared address `saddr` as seen in the shared window of cluster CTA `rank`
__device__ __forceinline__ uint32_t dsmem_addr(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void dsmem_st_f64(uint32_t raddr, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;\n" ::"r"(raddr), "d"(v) : "memory");
}
__device__ __forceinline__ void dsmem_st_s32(uint32_t raddr, int v) {
  asm volatile("st.shared::cluster.s32 [%0], %1;\n" ::"r"(raddr), "r"(v) : "memory");
}
// arrive on an mbarrier of another CTA of the cluster, releasing this thread's prior writes
__device__ __forceinline__ void mbar_arrive_remote(uint32_t raddr_bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(raddr_bar) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred P1;\n"
      "WAITC_%=:\n"
      " mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n"
      " @!P1 bra WAITC_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

#ifndef LMRA_MBAR_SUSPEND_NS
#define LMRA_MBAR_SUSPEND_NS 0x989680
#endif
constexpr unsigned kMbarSuspendNs = LMRA_MBAR_SUSPEND_NS;
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred P1;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
      " @!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(kMbarSuspendNs)  // suspend-time hint: the warp sleeps in hardware instead of spinning
      : "memory");
}
// 3-D tiled TMA load of one box into shared memory, completion counted on `bar`
__device__ __forceinline__ void tma_load_3d(void* dst, const void* tmap, uint64_t* bar, int c0,
                                            int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4, %5}], [%2];\n" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// Leading dimension (in doubles) >= n with ld % 16 == 4: a 64-bit fragment read of
// rows t = 0..3 x cols g = 0..3 per half-warp then hits 16 distinct even banks.
__host__ __device__ constexpr int conflict_free_ld(int n) { return ((n + 11) / 16) * 16 + 4; }

// Opt a kernel into > 48 KB dynamic shared memory once per device (bitmask of devices).
inline cudaError_t ensure_smem_attr(const void* fn, size_t bytes, unsigned long long& done) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  unsigned long long bit = 1ull << (dev & 63);
  if (done & bit) return cudaSuccess;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) done |= bit;
  return e;
}

}  // namespace lmra_dev

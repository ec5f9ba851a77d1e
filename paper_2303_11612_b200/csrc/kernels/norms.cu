// norms.cu -- column squared norms of the mode-n unfolding, in place.
//
// Replaces the squaredNorm loop of gram_sampling_probabilities (tucker.cpp:117-119),
// which in the reference runs over an explicit unfold() copy.  The summation order
// is the canonical one shared with the oracle (oracle/lmra_oracle.cpp
// canonical_sqnorm): chunks of 32 consecutive fiber entries accumulated with fma,
// chunk partials added in chunk order.  Results are therefore bit-identical to the
// oracle, which is what makes the sampled indices bit-exact end to end.
//
// HBM-bound: 8 B read per element, 2 flop.  Contiguous fibers (mode 0) are staged
// through shared memory so each thread walks its own fiber; strided fibers (modes
// > 0) are read coalesced across threads (consecutive i), one thread per column.
#include <cstdlib>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"

namespace lmra_dev {

constexpr int kNormChunk = 32;

// mode 0: fiber j = x[I*j .. I*j + I)
__global__ void __launch_bounds__(128) sqnorm_contig_kernel(const double* __restrict__ x,
                                                            long long I, long long J,
                                                            double* __restrict__ w) {
  __shared__ double tile[128][kNormChunk + 1];
  const int tid = threadIdx.x;
  const long long j0 = (long long)blockIdx.x * 128;
  double total = 0.0, seg = 0.0;
  for (long long r0 = 0; r0 < I; r0 += kNormChunk) {
    const int n = (I - r0 < kNormChunk) ? (int)(I - r0) : kNormChunk;
    // coalesced: a warp reads 32 consecutive entries of one fiber per instruction
    const int lane = tid & 31, wrp = tid >> 5;
#pragma unroll 4
    for (int c = wrp; c < 128; c += 4) {
      long long j = j0 + c;
      double val = 0.0;
      if (j < J && lane < n) val = __ldcs(x + I * j + r0 + lane);
      tile[c][lane] = val;
    }
    __syncthreads();
    double p = 0.0;
    for (int q = 0; q < n; ++q) {
      double v = tile[tid][q];
      p = fma(v, v, p);
    }
    canon_add(p, r0 / kNormChunk, r0 + kNormChunk >= I, seg, total);
    __syncthreads();
  }
  const long long j = j0 + tid;
  if (j < J) w[j] = total;
}

// mode 0, pipelined: the same canonical sums, with the 32-row x 128-column tiles streamed by
// cp.async through a 3-stage ring (the one-tile kernel above alternates load and compute phases
// and reached 4.9 TB/s on cfg5's 3.2 GB tensor, long-scoreboard bound).  Column c's 32 entries
// land rotated by c (element q at (q + c) mod 32), so both the 8-byte async copies (a warp
// writes 32 consecutive entries of one column) and the per-thread column reads (32 lanes, 32
// columns, same q) hit distinct bank pairs.
constexpr int kNCStages = 3;
__global__ void __launch_bounds__(128) sqnorm_contig_pipe_kernel(const double* __restrict__ x,
                                                                 long long I, long long J,
                                                                 double* __restrict__ w) {
  extern __shared__ __align__(16) double ring[];  // [stage][128 columns][32]
  const int tid = threadIdx.x, lane = tid & 31, wrp = tid >> 5;
  const long long j0 = (long long)blockIdx.x * 128;
  const long long nch = (I + kNormChunk - 1) / kNormChunk;
  auto load = [&](long long ch) {
    double* t = ring + (ch % kNCStages) * (128 * kNormChunk);
    const long long r0 = ch * kNormChunk;
    const bool rok = r0 + lane < I;
#pragma unroll 8
    for (int c = wrp; c < 128; c += 4) {
      const long long j = j0 + c;
      const bool ok = rok && j < J;
      cp_async8(t + c * kNormChunk + ((lane + c) & (kNormChunk - 1)), ok ? x + I * j + r0 + lane : x, ok);
    }
  };
#pragma unroll
  for (int st = 0; st < kNCStages - 1; ++st) {
    if (st < nch) load(st);
    cp_async_commit();
  }
  double total = 0.0, seg = 0.0;
  for (long long ch = 0; ch < nch; ++ch) {
    cp_async_wait<kNCStages - 2>();
    __syncthreads();  // stage ch landed for every thread; stage ch - 1 is free again
    if (ch + kNCStages - 1 < nch) load(ch + kNCStages - 1);
    cp_async_commit();
    const double* t = ring + (ch % kNCStages) * (128 * kNormChunk) + tid * kNormChunk;
    const int n = (I - ch * kNormChunk < kNormChunk) ? (int)(I - ch * kNormChunk) : kNormChunk;
    double p = 0.0;
    for (int q = 0; q < n; ++q) {
      const double v = t[(q + tid) & (kNormChunk - 1)];
      p = fma(v, v, p);
    }
    canon_add(p, ch, ch + 1 == nch, seg, total);
  }
  cp_async_wait<0>();
  const long long j = j0 + tid;
  if (j < J) w[j] = total;
}

// mode 0, TMA: the same canonical sums with the tile streamed by the tensor-memory accelerator.
// A persistent CTA per SM takes 128-column tiles in turn; each 32-row chunk of a tile is two
// boxes of 16 rows x 128 columns (128 B per column, 128 B swizzle) landing in a 6-stage ring
// (32 KB a stage) filled by one producer warp and released per consumer warp through mbarriers.
// Consumer thread c owns column c: its 16-byte pairs (rows 2p, 2p + 1) of a box sit at pair slot
// p ^ (c & 7) of the column's 128-byte row -- conflict-free double2 reads -- and it runs the
// chunk's fma chain in row order (rows past I are the TMA's zero fill: fma(0, 0, p) = p, so the
// bits match the chunked loops above).  The cp.async ring above reached 5.3 TB/s on cfg5's
// 3.2 GB mode-0 pass (8-byte copies: 32 LSU ops per thread per chunk); the TMA engine moves a
// chunk with two instructions.
constexpr int kNTStages = 6;
constexpr int kNTCols = 128;
constexpr int kNTBoxBytes = 16 * kNTCols * 8;        // 16 KB
constexpr int kNTStageBytes = 2 * kNTBoxBytes;       // one 32-row chunk
constexpr int kNTThreads = kNTCols + 32;             // 4 consumer warps + the producer warp
__global__ void __launch_bounds__(kNTThreads, 1) sqnorm_contig_tma_kernel(const __grid_constant__ CUtensorMap tmap,
                                                                        long long I, long long J,
                                                                        double* __restrict__ w) {
  extern __shared__ __align__(16) unsigned char nt_raw[];
  unsigned char* base = nt_raw + ((1024 - (smem_u32(nt_raw) & 1023)) & 1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(base + kNTStages * kNTStageBytes);
  uint64_t* empty = full + kNTStages;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (tid == 0) {
    for (int st = 0; st < kNTStages; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], kNTCols / 32);
    }
    mbar_fence_init();
  }
  __syncthreads();
  pdl_wait();  // the previous kernel's outputs (programmatic dependent launch)
  pdl_trigger();
  const long long ntiles = (J + kNTCols - 1) / kNTCols;
  const long long nch = (I + kNormChunk - 1) / kNormChunk;
  if (warp == kNTCols / 32) {  // producer
    if ((tid & 31) == 0) {
      long long g = 0;
      for (long long t = blockIdx.x; t < ntiles; t += gridDim.x)
        for (long long ch = 0; ch < nch; ++ch, ++g) {
          const int st = (int)(g % kNTStages);
          mbar_wait(&empty[st], (unsigned)((g / kNTStages) & 1) ^ 1u);
          mbar_arrive_expect_tx(&full[st], kNTStageBytes);
          unsigned char* dst = base + st * kNTStageBytes;
          const int c1 = (int)(t * kNTCols), r0 = (int)(ch * kNormChunk);
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];\n" ::
                  "r"(smem_u32(dst)), "l"(&tmap), "r"(smem_u32(&full[st])), "r"(r0), "r"(c1)
              : "memory");
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];\n" ::
                  "r"(smem_u32(dst + kNTBoxBytes)), "l"(&tmap), "r"(smem_u32(&full[st])), "r"(r0 + 16), "r"(c1)
              : "memory");
        }
    }
    return;
  }
  const int c = tid;  // column within the tile
  long long g = 0;
  for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
    double total = 0.0, seg = 0.0;
    for (long long ch = 0; ch < nch; ++ch, ++g) {
      const int st = (int)(g % kNTStages);
      mbar_wait(&full[st], (unsigned)((g / kNTStages) & 1));
      const unsigned char* col = base + st * kNTStageBytes + c * 128;
      double p = 0.0;
#pragma unroll
      for (int b = 0; b < 2; ++b)
#pragma unroll
        for (int pr = 0; pr < 8; ++pr) {
          const double2 v = *reinterpret_cast<const double2*>(col + b * kNTBoxBytes + ((pr ^ (c & 7)) << 4));
          p = fma(v.x, v.x, p);
          p = fma(v.y, v.y, p);
        }
      __syncwarp();
      if ((tid & 31) == 0) mbar_arrive(&empty[st]);
      canon_add(p, ch, ch + 1 == nch, seg, total);
    }
    const long long j = t * kNTCols + c;
    if (j < J) w[j] = total;
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 norms_tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// the TMA form when it applies (even I: 16-byte row pitch; aligned base; I < 2^31 rows fit the
// box coordinates); false: the caller uses the cp.async ring
static bool launch_sqnorm_contig_tma(const double* x, long long I, long long J, double* w, cudaStream_t st,
                                     cudaError_t* err) {
  static const bool on = !(getenv("LMRA_NORMS_TMA") && getenv("LMRA_NORMS_TMA")[0] == '0');
  PFN_cuTensorMapEncodeTiled_v12000 enc = norms_tensor_map_encoder();
  if (!on || !enc || I % 2 != 0 || I < 16 || J < 1 || I >= (1LL << 31) || J >= (1LL << 31) ||
      (reinterpret_cast<uintptr_t>(x) & 15) != 0)
    return false;
  CUtensorMap tmap;
  const cuuint64_t gdim[2] = {(cuuint64_t)I, (cuuint64_t)J};
  const cuuint64_t gstride[1] = {(cuuint64_t)I * 8};
  const cuuint32_t box[2] = {16, (cuuint32_t)kNTCols}, estride[2] = {1, 1};
  if (enc(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(x), gdim, gstride, box, estride,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  static unsigned long long attr_done = 0;
  const size_t smem = (size_t)kNTStages * kNTStageBytes + 2 * kNTStages * sizeof(uint64_t) + 1024;
  *err = ensure_smem_attr(reinterpret_cast<const void*>(sqnorm_contig_tma_kernel), smem, attr_done);
  if (*err != cudaSuccess) return true;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long ntiles = (J + kNTCols - 1) / kNTCols;
  const int grid = (int)(ntiles < sms ? ntiles : sms);
  *err = launch_pdl(sqnorm_contig_tma_kernel, dim3((unsigned)grid), dim3(kNTThreads), smem, st, tmap, I, J, w);
  return true;
}

// modes > 0: fiber j = (i, o) at x[i + inner*I*o + inner*r]
__global__ void __launch_bounds__(256) sqnorm_strided_kernel(const double* __restrict__ x,
                                                             ModeView v, double* __restrict__ w) {
  const long long J = v.inner * v.outer;
  const long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= J) return;
  const long long o = j / v.inner, i = j - o * v.inner;
  const double* f = x + i + v.inner * v.I * o;
  double total = 0.0, seg = 0.0;
  long long r0 = 0;
  for (; r0 + kNormChunk <= v.I; r0 += kNormChunk) {
    double vals[kNormChunk];
#pragma unroll
    for (int q = 0; q < kNormChunk; ++q) vals[q] = __ldcs(f + v.inner * (r0 + q));
    double p = 0.0;
#pragma unroll
    for (int q = 0; q < kNormChunk; ++q) p = fma(vals[q], vals[q], p);
    canon_add(p, r0 / kNormChunk, r0 + kNormChunk >= v.I, seg, total);
  }
  if (r0 < v.I) {
    double p = 0.0;
    for (long long r = r0; r < v.I; ++r) {
      double val = __ldcs(f + v.inner * r);
      p = fma(val, val, p);
    }
    canon_add(p, r0 / kNormChunk, true, seg, total);
  }
  w[j] = total;
}

// ---- the canonical norm of a fibre split across devices (sharded mode N-1) ----
// P[c * J + j] = chunk c's partial (fma chain over its 32 entries) of column j of the view
__global__ void __launch_bounds__(256) chunk_partials_kernel(const double* __restrict__ x, ModeView v,
                                                             double* __restrict__ P) {
  const long long J = v.inner * v.outer;
  const long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long c = blockIdx.y;
  if (j >= J) return;
  const long long o = j / v.inner, i = j - o * v.inner;
  const double* f = x + i + v.inner * v.I * o;
  const long long r0 = c * kNormChunk, r1 = min(v.I, r0 + kNormChunk);
  double p = 0.0;
  for (long long r = r0; r < r1; ++r) {
    const double val = __ldcs(f + v.inner * r);
    p = fma(val, val, p);
  }
  P[c * J + j] = p;
}

// S[s * J + j] = segment s of column j: chunk 2s's partial + chunk 2s + 1's (when it exists)
__global__ void segment_sums_kernel(const double* __restrict__ P, long long J, int nchunks, double* __restrict__ S) {
  const long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int sg = blockIdx.y;
  if (j >= J) return;
  double v = P[(long long)(2 * sg) * J + j];
  if (2 * sg + 1 < nchunks) v = v + P[(long long)(2 * sg + 1) * J + j];
  S[(long long)sg * J + j] = v;
}

// w[j] = the segments of column j added in global order: rank q contributed counts[q]
// segments at G[(q * kmax + s) * J + j]
__global__ void segment_combine_kernel(const double* __restrict__ G, long long J, int nranks, int kmax,
                                       SegCounts counts, double* __restrict__ w) {
  const long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= J) return;
  double total = 0.0;
  for (int q = 0; q < nranks; ++q)
    for (int sg = 0; sg < counts.n[q]; ++sg) total = total + G[((long long)q * kmax + sg) * J + j];
  w[j] = total;
}

cudaError_t launch_chunk_partials(const double* x, ModeView v, double* P, cudaStream_t st) {
  const long long J = v.inner * v.outer, nc = (v.I + kNormChunk - 1) / kNormChunk;
  if (J == 0 || nc == 0) return cudaSuccess;
  chunk_partials_kernel<<<dim3((unsigned)((J + 255) / 256), (unsigned)nc), 256, 0, st>>>(x, v, P); note_launch();
  return cudaGetLastError();
}

cudaError_t launch_segment_sums(const double* P, long long J, int nchunks, double* S, cudaStream_t st) {
  const int nseg = (nchunks + 1) / 2;
  if (J == 0 || nseg == 0) return cudaSuccess;
  segment_sums_kernel<<<dim3((unsigned)((J + 255) / 256), (unsigned)nseg), 256, 0, st>>>(P, J, nchunks, S); note_launch();
  return cudaGetLastError();
}

cudaError_t launch_segment_combine(const double* G, long long J, int nranks, int kmax, const SegCounts& counts,
                                   double* w, cudaStream_t st) {
  if (J == 0) return cudaSuccess;
  segment_combine_kernel<<<(unsigned)((J + 255) / 256), 256, 0, st>>>(G, J, nranks, kmax, counts, w); note_launch();
  return cudaGetLastError();
}

cudaError_t launch_column_sqnorms(const double* x, ModeView v, double* w, cudaStream_t st) {
  const long long J = v.inner * v.outer;
  if (J == 0) return cudaSuccess;
  if (v.inner == 1) {
    cudaError_t te = cudaSuccess;
    if (launch_sqnorm_contig_tma(x, v.I, J, w, st, &te)) return te != cudaSuccess ? te : cudaGetLastError();
    static const bool pipe = !(getenv("LMRA_NORMS_PIPE") && getenv("LMRA_NORMS_PIPE")[0] == '0');
    if (pipe) {
      static unsigned long long attr_done = 0;
      const size_t smem = sizeof(double) * kNCStages * 128 * kNormChunk;
      cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(sqnorm_contig_pipe_kernel), smem, attr_done);
      if (e != cudaSuccess) return e;
      sqnorm_contig_pipe_kernel<<<(unsigned)((J + 127) / 128), 128, smem, st>>>(x, v.I, J, w);
    } else {
      sqnorm_contig_kernel<<<(unsigned)((J + 127) / 128), 128, 0, st>>>(x, v.I, J, w);
    }
    note_launch();
  } else {
    sqnorm_strided_kernel<<<(unsigned)((J + 255) / 256), 256, 0, st>>>(x, v, w); note_launch();
  }
  return cudaGetLastError();
}

}  // namespace lmra_dev

// norms3.cu -- all three modes' canonical column squared norms from ONE read of a 3-way
// tensor (T-HOSVD with sampling: every mode's probabilities come from the same input,
// so the mode passes share the read -- SURVEY 8d rule R2).
//
// Canonical order (shared with the oracle, norms.cu, common.cuh canon_add): a column's squared
// norm is the in-order sum of chunk-pair sums, a chunk partial being the fma-sequential sum
// over 32 consecutive fiber entries.  Each element belongs to exactly one chunk per mode, so a
// 32 x 32 x 32 brick holds complete chunks of all three modes:
//   pass 1 (this kernel, one read of X): chunk partials of modes 0 and 1 -> P0, P1
//          (|X|/32 doubles each); mode 2 combined in registers (see below)
//   pass 2 (combine): per column, the chunk partials added in chunk order.
// Traffic: |X| read + 2 |X|/32 written and read back, vs 3 |X| for three mode passes.
#include <cmath>
#include <cstdlib>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"

namespace lmra_dev {

constexpr int kB = 32;          // brick edge = canonical chunk length
constexpr int kN3Threads = 256;
constexpr int kN3Stages = 3;    // cp.async ring of 32 x 32 slices

// X[i0, i1, i2], i0 fastest.  Grid: (ceil(I0/32), ceil(I1/32)); each CTA walks the whole i2
// extent of its 32 x 32 (i0, i1) column of bricks, one (i0, i1) slice at a time:
//   mode 0 chunk partial of fibre (i1, i2) over its 32 i0  -> P0[c0][i1 + I1*i2]
//   mode 1 chunk partial of fibre (i0, i2) over its 32 i1  -> P1[c1][i0 + I0*i2]
//   mode 2 fibres (i0, i1) lie entirely in the CTA: chunk partials over 32 consecutive i2
//   are combined in chunk order in registers and written as the final w2 (no P2 round
//   trip through HBM).
// Slices stream through a 3-stage cp.async ring so loads stay in flight while the
// previous slice's partials are formed (the first version loaded synchronously and sat
// at ~60% of HBM bandwidth).
// Grids with too few (i0, i1) columns to fill the GPU also split i2 into gridDim.z segments
// of whole chunks; mode 2 then writes its chunk partials to P2 (combined by pass 2) instead
// of the in-register total.
__global__ void __launch_bounds__(kN3Threads) norms3_chunks_kernel(
    const double* __restrict__ x, long long I0, long long I1, long long I2,
    double* __restrict__ P0, double* __restrict__ P1, double* __restrict__ w2,
    double* __restrict__ P2, long long seg) {
  __shared__ __align__(16) double ring[kN3Stages][kB][kB + 1];  // [stage][i1][i0]
  const int tid = threadIdx.x;
  const long long c0 = blockIdx.x, c1 = blockIdx.y;
  const long long i0b = c0 * kB, i1b = c1 * kB;
  const int n0 = (int)(I0 - i0b < kB ? I0 - i0b : kB), n1 = (int)(I1 - i1b < kB ? I1 - i1b : kB);
  // loads / mode-2 fibres: thread owns (i0 = tid % 32, i1 = tid / 32 + 8k), k < 4
  const int a0 = tid & 31, a1 = tid >> 5;
  const double* src[4];
  bool ok[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int r1 = a1 + 8 * k;
    ok[k] = r1 < n1 && a0 < n0;
    src[k] = x + (ok[k] ? (i0b + a0) + I0 * (i1b + r1) : 0);
  }
  const long long slab = I0 * I1;
  const long long z0 = blockIdx.z * seg, z1 = z0 + seg < I2 ? z0 + seg : I2;  // i2 range
  auto issue = [&](long long i2) {
    if (i2 < z1) {
      const int st = (int)(i2 % kN3Stages);
#pragma unroll
      for (int k = 0; k < 4; ++k)
        cp_async8(&ring[st][a1 + 8 * k][a0], ok[k] ? src[k] + slab * i2 : x, ok[k]);
    }
    cp_async_commit();
  };
#pragma unroll
  for (int s = 0; s < kN3Stages - 1; ++s) issue(z0 + s);
  double part2[4] = {0.0, 0.0, 0.0, 0.0}, tot2[4] = {0.0, 0.0, 0.0, 0.0}, seg2[4] = {0.0, 0.0, 0.0, 0.0};
  for (long long i2 = z0; i2 < z1; ++i2) {
    issue(i2 + kN3Stages - 1);
    cp_async_wait<kN3Stages - 1>();
    __syncthreads();
    const double (*slice)[kB + 1] = ring[i2 % kN3Stages];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const double v = slice[a1 + 8 * k][a0];
      part2[k] = fma(v, v, part2[k]);  // mode 2: over i2, in order within the chunk
    }
    if ((i2 & (kB - 1)) == kB - 1 || i2 == I2 - 1) {  // chunk of 32 i2 complete
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (P2) {
          if (ok[k]) P2[(i2 / kB) * slab + (i0b + a0) + I0 * (i1b + a1 + 8 * k)] = part2[k];
        } else {
          canon_add(part2[k], i2 / kB, i2 == I2 - 1, seg2[k], tot2[k]);
        }
        part2[k] = 0.0;
      }
    }
    // modes 0 / 1: the 32 values first (independent loads), then the in-order fma chain;
    // entries past the tensor edge were zero-filled, and fma(0, 0, p) = p exactly
    if (tid < 64) {
      const int f = tid & 31;
      double v[kB];
      if (tid < 32) {
#pragma unroll
        for (int q = 0; q < kB; ++q) v[q] = slice[f][q];  // fibre (i1 = f, i2) over i0
      } else {
#pragma unroll
        for (int q = 0; q < kB; ++q) v[q] = slice[q][f];  // fibre (i0 = f, i2) over i1
      }
      double p = 0.0;
#pragma unroll
      for (int q = 0; q < kB; ++q) p = fma(v[q], v[q], p);
      if (tid < 32) {
        if (f < n1) P0[c0 * (I1 * I2) + (i1b + f) + I1 * i2] = p;
      } else {
        if (f < n0) P1[c1 * (I0 * I2) + (i0b + f) + I0 * i2] = p;
      }
    }
    __syncthreads();  // the slot is refilled by the next iteration's issue
  }
  if (!P2) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (ok[k]) w2[(i0b + a0) + I0 * (i1b + a1 + 8 * k)] = tot2[k];
  }
}

// ---------------------------------------------------------------------------
// TMA version (I0 even: the tensor map needs 16-byte row strides).  One producer warp
// streams each (i0, i1) slice of the CTA's 32 x 32 column as two 16 x 32 boxes (128-byte
// swizzle) into a ring of shared-memory stages guarded by mbarriers; eight consumer warps
// form the chunk partials exactly as above.  One TMA instruction per box replaces 1024
// per-element cp.async (whose issue cost, ~8 cycles per warp instruction, would itself
// approach the per-SM share of HBM bandwidth).
// ---------------------------------------------------------------------------
constexpr int kTStages = 6;
constexpr int kTCons = 256;                 // consumer threads (8 warps)
constexpr int kTThreads = kTCons + 32;      // + producer warp
constexpr int kTStageBytes = 2 * 32 * 128;  // two boxes of 32 rows x 16 doubles

// element (row r = i1 - i1b, column c = i0 - i0b) of a stage, 128-byte swizzle: the 16-byte
// chunk j of a 128-byte row r sits at chunk j ^ (r & 7)
__device__ __forceinline__ int sw_idx(int r, int c) {
  return (c >> 4) * 512 + r * 16 + ((((c & 15) >> 1) ^ (r & 7)) << 1) + (c & 1);
}

__global__ void __launch_bounds__(kTThreads, 3) norms3_tma_kernel(
    const __grid_constant__ CUtensorMap tmap, long long I0, long long I1, long long I2,
    double* __restrict__ P0, double* __restrict__ P1, double* __restrict__ w2,
    double* __restrict__ P2, long long seg) {
  extern __shared__ __align__(16) unsigned char smraw[];
  // 1024-byte alignment for the 128-byte swizzle, kept as an offset into the shared array
  // so the compiler still emits shared-memory loads (not generic ones)
  unsigned char* base = smraw + ((1024 - (smem_u32(smraw) & 1023)) & 1023);
  double* ring = reinterpret_cast<double*>(base);
  uint64_t* full = reinterpret_cast<uint64_t*>(base + kTStages * kTStageBytes);
  uint64_t* empty = full + kTStages;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const long long c0 = blockIdx.x, c1 = blockIdx.y;
  const long long i0b = c0 * kB, i1b = c1 * kB;
  const int n0 = (int)(I0 - i0b < kB ? I0 - i0b : kB), n1 = (int)(I1 - i1b < kB ? I1 - i1b : kB);
  const long long z0 = blockIdx.z * seg, z1 = z0 + seg < I2 ? z0 + seg : I2;
  if (tid == 0) {
    for (int s = 0; s < kTStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kTCons / 32);
    }
    mbar_fence_init();
  }
  __syncthreads();
  if (warp == kTCons / 32) {  // producer
    if (lane == 0) {
      int stage = 0;
      unsigned phase = 0;
      for (long long i2 = z0; i2 < z1; ++i2) {
        mbar_wait(&empty[stage], phase ^ 1);
        mbar_arrive_expect_tx(&full[stage], kTStageBytes);
        double* dst = ring + stage * (kTStageBytes / 8);
        tma_load_3d(dst, &tmap, &full[stage], (int)i0b, (int)i1b, (int)i2);
        tma_load_3d(dst + 512, &tmap, &full[stage], (int)i0b + 16, (int)i1b, (int)i2);
        if (++stage == kTStages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
    return;
  }
  const int a0 = tid & 31, a1 = tid >> 5;  // mode-2 fibres (i0 = a0, i1 = a1 + 8k)
  double part2[4] = {0.0, 0.0, 0.0, 0.0}, tot2[4] = {0.0, 0.0, 0.0, 0.0}, seg2[4] = {0.0, 0.0, 0.0, 0.0};
  int stage = 0;
  unsigned phase = 0;
  for (long long i2 = z0; i2 < z1; ++i2) {
    mbar_wait(&full[stage], phase);
    const double* sl = ring + stage * (kTStageBytes / 8);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const double v = sl[sw_idx(a1 + 8 * k, a0)];
      part2[k] = fma(v, v, part2[k]);  // mode 2: over i2, in order within the chunk
    }
    if ((i2 & (kB - 1)) == kB - 1 || i2 == I2 - 1) {  // chunk of 32 i2 complete
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (P2) {
          if (a0 < n0 && a1 + 8 * k < n1)
            P2[(i2 / kB) * (I0 * I1) + (i0b + a0) + I0 * (i1b + a1 + 8 * k)] = part2[k];
        } else {
          canon_add(part2[k], i2 / kB, i2 == I2 - 1, seg2[k], tot2[k]);
        }
        part2[k] = 0.0;
      }
    }
    if (tid < 64) {  // modes 0 / 1: the in-order fma chain over 32 entries (zero past the edge)
      const int f = tid & 31;
      double p = 0.0;
      if (tid < 32) {
#pragma unroll
        for (int q = 0; q < kB; q += 8) {
          double v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) v[u] = sl[sw_idx(f, q + u)];  // fibre (i1 = f) over i0
#pragma unroll
          for (int u = 0; u < 8; ++u) p = fma(v[u], v[u], p);
        }
        if (f < n1) P0[c0 * (I1 * I2) + (i1b + f) + I1 * i2] = p;
      } else {
#pragma unroll
        for (int q = 0; q < kB; q += 8) {
          double v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) v[u] = sl[sw_idx(q + u, f)];  // fibre (i0 = f) over i1
#pragma unroll
          for (int u = 0; u < 8; ++u) p = fma(v[u], v[u], p);
        }
        if (f < n0) P1[c1 * (I0 * I2) + (i0b + f) + I0 * i2] = p;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[stage]);
    if (++stage == kTStages) {
      stage = 0;
      phase ^= 1;
    }
  }
  if (!P2) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (a0 < n0 && a1 + 8 * k < n1) w2[(i0b + a0) + I0 * (i1b + a1 + 8 * k)] = tot2[k];
  }
}

// ---------------------------------------------------------------------------
// Segment version (the default for even I0): a CTA owns a 64 x 64 (i0, i1) column, i.e. whole
// canonical-norm SEGMENTS (two 32-entry chunks, canon_add) of the mode-0 and mode-1 fibres it
// touches, so it writes one partial per segment instead of one per chunk -- half the
// round-trip traffic of the chunk partials.  Slices stream in as four 16 x 64 boxes (128-byte
// swizzle) through a ring of 32 KB stages; 16 consumer warps.  Mode 2: the CTA's 4096 fibres
// over its i2 range, 8 per thread, in registers; with an i2 split (segments of whole 64-entry
// segments) the per-segment partials go to P2 for the combine.
// ---------------------------------------------------------------------------
constexpr int kSB = 64;                        // tile edge = one canonical segment
constexpr int kSStages = 5;
constexpr int kSCons = 512;                    // consumer threads (16 warps)
constexpr int kSThreads = kSCons + 32;         // + producer warp
constexpr int kSStageBytes = kSB * kSB * 8;    // 32 KB: four 16 (i0) x 64 (i1) boxes

__device__ __forceinline__ int sw_idx64(int r, int c) {  // r = i1 - i1b, c = i0 - i0b
  return (c >> 4) * 1024 + r * 16 + ((((c & 15) >> 1) ^ (r & 7)) << 1) + (c & 1);
}

__global__ void __launch_bounds__(kSThreads, 1) norms3_seg_kernel(
    const __grid_constant__ CUtensorMap tmap, long long I0, long long I1, long long I2,
    double* __restrict__ S0, double* __restrict__ S1, double* __restrict__ w2,
    double* __restrict__ S2, long long seg) {
  extern __shared__ __align__(16) unsigned char smraw[];
  unsigned char* base = smraw + ((1024 - (smem_u32(smraw) & 1023)) & 1023);
  double* ring = reinterpret_cast<double*>(base);
  uint64_t* full = reinterpret_cast<uint64_t*>(base + kSStages * kSStageBytes);
  uint64_t* empty = full + kSStages;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const long long c0 = blockIdx.x, c1 = blockIdx.y;  // segment indices along i0 / i1
  const long long i0b = c0 * kSB, i1b = c1 * kSB;
  const int n0 = (int)(I0 - i0b < kSB ? I0 - i0b : kSB), n1 = (int)(I1 - i1b < kSB ? I1 - i1b : kSB);
  const long long z0 = blockIdx.z * seg, z1 = z0 + seg < I2 ? z0 + seg : I2;
  if (tid == 0) {
    for (int s = 0; s < kSStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kSCons / 32);
    }
    mbar_fence_init();
  }
  __syncthreads();
  if (warp == kSCons / 32) {  // producer
    if (lane == 0) {
      int stage = 0;
      unsigned phase = 0;
      for (long long i2 = z0; i2 < z1; ++i2) {
        mbar_wait(&empty[stage], phase ^ 1);
        mbar_arrive_expect_tx(&full[stage], kSStageBytes);
        double* dst = ring + stage * (kSStageBytes / 8);
#pragma unroll
        for (int b = 0; b < 4; ++b) tma_load_3d(dst + b * 1024, &tmap, &full[stage], (int)i0b + 16 * b, (int)i1b, (int)i2);
        if (++stage == kSStages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
    return;
  }
  const int a0 = tid & 63, a1 = tid >> 6;  // mode-2 fibres (i0 = a0, i1 = a1 + 8k), k < 8
  double part2[8], seg2[8], tot2[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) part2[k] = seg2[k] = tot2[k] = 0.0;
  int stage = 0;
  unsigned phase = 0;
  for (long long i2 = z0; i2 < z1; ++i2) {
    mbar_wait(&full[stage], phase);
    const double* sl = ring + stage * (kSStageBytes / 8);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const double v = sl[sw_idx64(a1 + 8 * k, a0)];
      part2[k] = fma(v, v, part2[k]);
    }
    if ((i2 & (kB - 1)) == kB - 1 || i2 == I2 - 1) {  // a 32-entry chunk of i2 is complete
      const long long ch = i2 / kB;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (S2) {  // i2 split: this segment's partial (the segment lies in this CTA's range)
          seg2[k] = (ch & 1) ? seg2[k] + part2[k] : part2[k];
          if (((ch & 1) || i2 == I2 - 1) && a0 < n0 && a1 + 8 * k < n1)
            S2[(ch >> 1) * (I0 * I1) + (i0b + a0) + I0 * (i1b + a1 + 8 * k)] = seg2[k];
        } else {
          canon_add(part2[k], ch, i2 == I2 - 1, seg2[k], tot2[k]);
        }
        part2[k] = 0.0;
      }
    }
    if (tid < 128) {  // modes 0 / 1: one fibre segment each, two in-order fma chains of 32
      const int f = tid & 63;
      double p0 = 0.0, p1 = 0.0;
      if (tid < 64) {
#pragma unroll
        for (int q = 0; q < kB; q += 8) {
          double v[8], u[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            v[e] = sl[sw_idx64(f, q + e)];        // fibre (i1 = f) over i0, chunk 0
            u[e] = sl[sw_idx64(f, kB + q + e)];   // chunk 1
          }
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            p0 = fma(v[e], v[e], p0);
            p1 = fma(u[e], u[e], p1);
          }
        }
        if (f < n1) S0[c0 * (I1 * I2) + (i1b + f) + I1 * i2] = n0 > kB ? p0 + p1 : p0;
      } else {
#pragma unroll
        for (int q = 0; q < kB; q += 8) {
          double v[8], u[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            v[e] = sl[sw_idx64(q + e, f)];        // fibre (i0 = f) over i1, chunk 0
            u[e] = sl[sw_idx64(kB + q + e, f)];   // chunk 1
          }
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            p0 = fma(v[e], v[e], p0);
            p1 = fma(u[e], u[e], p1);
          }
        }
        if (f < n0) S1[c1 * (I0 * I2) + (i0b + f) + I0 * i2] = n1 > kB ? p0 + p1 : p0;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[stage]);
    if (++stage == kSStages) {
      stage = 0;
      phase ^= 1;
    }
  }
  if (!S2) {
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (a0 < n0 && a1 + 8 * k < n1) w2[(i0b + a0) + I0 * (i1b + a1 + 8 * k)] = tot2[k];
  }
}

// w[j] = the segment partials S[s][j] added in order (the canonical total)
__global__ void segment_total_kernel(const double* __restrict__ S, long long J, int nseg, double* __restrict__ w) {
  const long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= J) return;
  double total = 0.0;
  for (int s = 0; s < nseg; ++s) total = total + S[(long long)s * J + j];
  w[j] = total;
}

static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
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

// w[j] = the canonical combine of the chunk partials P[c][j], c = 0, 1, ... (canon_add)
__global__ void chunk_combine_kernel(const double* __restrict__ P, long long J, int nchunks,
                                     double* __restrict__ w) {
  const long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= J) return;
  double total = 0.0, seg = 0.0;
  for (int c = 0; c < nchunks; ++c) canon_add(P[(long long)c * J + j], c, c == nchunks - 1, seg, total);
  w[j] = total;
}

// i2 segments (whole chunks) so that the grid has >= 4 CTAs per SM
static long long norms3_segments(long long I0, long long I1, long long I2) {
  const long long cols = ((I0 + kB - 1) / kB) * ((I1 + kB - 1) / kB);
  const long long c2 = (I2 + kB - 1) / kB;
  long long z = (4 * 148 + cols - 1) / cols;
  return z < 1 ? 1 : (z > c2 ? c2 : z);
}

static cudaError_t launch_norms3_seg(PFN_cuTensorMapEncodeTiled_v12000 enc, const double* x, long long I0,
                                     long long I1, long long I2, double* w0, double* w1, double* w2, double* work,
                                     cudaStream_t st) {
  const long long s0 = (I0 + kSB - 1) / kSB, s1 = (I1 + kSB - 1) / kSB, s2 = (I2 + kSB - 1) / kSB;
  double* S0 = work;
  double* S1 = S0 + s0 * I1 * I2;
  double* S2buf = S1 + s1 * I0 * I2;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // i2 split into whole 64-entry segments so the grid fills whole waves (one CTA per SM)
  const long long cols = s0 * s1;
  auto fill = [&](long long z) {
    const double n = (double)(cols * z);
    return n / (std::ceil(n / sms) * sms) - (z > 1 ? 0.02 : 0.0);
  };
  long long zs = 1;
  for (long long z = 2; z <= 16 && z <= s2; ++z)
    if (fill(z) > fill(zs) + 1e-9) zs = z;
  const long long seg = ((s2 + zs - 1) / zs) * kSB;
  double* S2 = zs > 1 ? S2buf : nullptr;
  CUtensorMap tmap;
  const cuuint64_t gdim[3] = {(cuuint64_t)I0, (cuuint64_t)I1, (cuuint64_t)I2};
  const cuuint64_t gstride[2] = {(cuuint64_t)I0 * 8, (cuuint64_t)(I0 * I1) * 8};
  const cuuint32_t box[3] = {16, 64, 1}, estride[3] = {1, 1, 1};
  if (enc(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(x), gdim, gstride, box, estride,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  static unsigned long long attr_done = 0;
  const size_t smem = kSStages * kSStageBytes + 2 * kSStages * sizeof(uint64_t) + 1024;
  cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(norms3_seg_kernel), smem, attr_done);
  if (e != cudaSuccess) return e;
  dim3 grid((unsigned)s0, (unsigned)s1, (unsigned)((I2 + seg - 1) / seg));
  norms3_seg_kernel<<<grid, kSThreads, smem, st>>>(tmap, I0, I1, I2, S0, S1, w2, S2, seg); note_launch();
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  segment_total_kernel<<<(unsigned)((I1 * I2 + 255) / 256), 256, 0, st>>>(S0, I1 * I2, (int)s0, w0); note_launch();
  segment_total_kernel<<<(unsigned)((I0 * I2 + 255) / 256), 256, 0, st>>>(S1, I0 * I2, (int)s1, w1); note_launch();
  if (S2) {
    segment_total_kernel<<<(unsigned)((I0 * I1 + 255) / 256), 256, 0, st>>>(S2, I0 * I1, (int)s2, w2);
    note_launch();
  }
  return cudaGetLastError();
}

size_t norms3_workspace_doubles(long long I0, long long I1, long long I2) {
  const long long c0 = (I0 + kB - 1) / kB, c1 = (I1 + kB - 1) / kB, c2 = (I2 + kB - 1) / kB;
  return (size_t)(c0 * I1 * I2 + c1 * I0 * I2 + c2 * I0 * I1);  // P2 when i2 is split
}

cudaError_t launch_norms3(const double* x, long long I0, long long I1, long long I2, double* w0,
                          double* w1, double* w2, double* work, cudaStream_t st, double* p2_chunks) {
  const long long c0 = (I0 + kB - 1) / kB, c1 = (I1 + kB - 1) / kB, c2 = (I2 + kB - 1) / kB;
  double* P0 = work;
  double* P1 = P0 + c0 * I1 * I2;
  PFN_cuTensorMapEncodeTiled_v12000 enc = tensor_map_encoder();
  const bool tma_ok = enc && I0 % 2 == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0 &&
                      I0 < (1ll << 31) && I1 < (1ll << 31) && I2 < (1ll << 31);
  if (tma_ok && !p2_chunks && !(getenv("LMRA_NORMS3_CHUNKS") && getenv("LMRA_NORMS3_CHUNKS")[0] == '1'))
    return launch_norms3_seg(enc, x, I0, I1, I2, w0, w1, w2, work, st);
  long long zs = norms3_segments(I0, I1, I2);
  if (tma_ok) {
    // wave quantisation: the memory-bound kernel runs at full bandwidth only while every
    // SM holds its full set of CTAs, so choose the number of i2 segments whose CTA count
    // best fills whole waves (a split costs the mode-2 chunk partials' round trip, ~6% of
    // the tensor read)
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const size_t smem = kTStages * kTStageBytes + 2 * kTStages * sizeof(uint64_t) + 1024;
    static unsigned long long attr_done0 = 0;  // the occupancy query needs the smem attribute
    cudaError_t ea = ensure_smem_attr(reinterpret_cast<const void*>(norms3_tma_kernel), smem, attr_done0);
    if (ea != cudaSuccess) return ea;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, norms3_tma_kernel, kTThreads, smem);
    const double slots = (double)sms * (per_sm > 0 ? per_sm : 1);
    const long long cols = c0 * c1;
    auto fill = [&](long long z) {
      const double n = (double)(cols * z);
      return n / (std::ceil(n / slots) * slots) - (z > 1 ? 0.06 : 0.0);
    };
    long long best = 1;
    for (long long z = 2; z <= 8 && z <= c2; ++z)
      if (fill(z) > fill(best) + 1e-9) best = z;
    zs = best;
  }
  double* P2 = p2_chunks ? p2_chunks : (zs > 1 ? P1 + c1 * I0 * I2 : nullptr);
  const long long seg = ((c2 + zs - 1) / zs) * kB;
  dim3 grid((unsigned)c0, (unsigned)c1, (unsigned)((I2 + seg - 1) / seg));
  CUtensorMap tmap;
  if (tma_ok) {
    const cuuint64_t gdim[3] = {(cuuint64_t)I0, (cuuint64_t)I1, (cuuint64_t)I2};
    const cuuint64_t gstride[2] = {(cuuint64_t)I0 * 8, (cuuint64_t)(I0 * I1) * 8};
    const cuuint32_t box[3] = {16, 32, 1}, estride[3] = {1, 1, 1};
    if (enc(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(x), gdim, gstride, box,
            estride, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
    static unsigned long long attr_done = 0;
    const size_t smem = kTStages * kTStageBytes + 2 * kTStages * sizeof(uint64_t) + 1024;
    cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(norms3_tma_kernel), smem, attr_done);
    if (e != cudaSuccess) return e;
    norms3_tma_kernel<<<grid, kTThreads, smem, st>>>(tmap, I0, I1, I2, P0, P1, w2, P2, seg); note_launch();
  } else {
    norms3_chunks_kernel<<<grid, kN3Threads, 0, st>>>(x, I0, I1, I2, P0, P1, w2, P2, seg); note_launch();
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  chunk_combine_kernel<<<(unsigned)((I1 * I2 + 255) / 256), 256, 0, st>>>(P0, I1 * I2, (int)c0, w0); note_launch();
  chunk_combine_kernel<<<(unsigned)((I0 * I2 + 255) / 256), 256, 0, st>>>(P1, I0 * I2, (int)c1, w1); note_launch();
  if (P2 && !p2_chunks) {
    chunk_combine_kernel<<<(unsigned)((I0 * I1 + 255) / 256), 256, 0, st>>>(P2, I0 * I1, (int)c2, w2);
    note_launch();
  }
  return cudaGetLastError();
}

}  // namespace lmra_dev

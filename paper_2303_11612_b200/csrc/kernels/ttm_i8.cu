// ttm_i8.cu -- the fp64 mode-0 contraction Y = Q^T X on the int8 tensor cores (tcgen05).
//
// fp64 has no tcgen05 kind; DMMA (mma.sync f64) peaks at 37 TF/s, which makes the core
// contraction of cfg4 (2 * 50 * 1000 * 10^6 flop) compute-bound at ~2.7 ms.  This kernel
// emulates it exactly enough (~1e-13 relative, far inside the 1e-10 parity tolerance) with
// integer tensor-core products (the Ozaki idea: split into fixed-point digits, multiply
// digits exactly, recombine):
//   x_kj = 2^(ex_j - 47) V_kj,  V = round(x 2^(47-ex_j)),  |V| < 2^46  (ex_j from the
//          canonical column norm: 2^ex_j >= 2 ||x_j|| >= 2 max_k |x_kj|)
//   q_km = 2^(eq_m - 47) U_km   (eq_m from max_k |q_km|)
//   V = sum_t d_t 2^(8t) with balanced signed digits d_t in [-128, 128): the bytes of V + C,
//   C = 128 sum_t 2^(8t), each XOR 0x80 -- one fma (V + C lands in the low bits of
//   fma(x, 2^(47-ex), 1.5 2^52 + C)) and one LOP3 per 4 digits.
//   y_mj = 2^(ex_j + eq_m - 94) sum_{t,s} 2^(8(t+s)) sum_k d_t[k,j] e_s[k,m]
// Each digit product is an exact int8 x int8 -> int32 MMA; products with t + s >= 5 are kept
// (21 of 36) and summed per level L = t + s in TMEM (int32, exact for K <= 4096).  The
// dropped products are zero-mean (balanced digits), ~2^-46 relative to |x||q| per term,
// growing like sqrt(K): ~1e-13 relative on the BASELINE shapes.
//
// Tile: 128 columns of X (the MMA's M) x all of K, N = mu rounded up to 16 (<= 64).  Warp roles
// (one CTA per SM, persistent over tiles):
//   warp 8 (2 lanes) TMA: X K-steps (32 k x 128 j, two 16 x 128 boxes, 128 B swizzle) into a
//                    5-stage ring freed by the slicers; the K-step's pre-split Q digits (bulk
//                    copy) into a 2-stage ring freed by the MMA
//   warps 0-7        digit split, two groups of 4 warps taking alternate K-steps (one A buffer
//                    each): thread j converts its column's 32 doubles to 6 x 32 digit
//                    bytes and writes them to TMEM with tcgen05.st (the A operand is read from
//                    TMEM, so shared memory only feeds the small B operand); after the last
//                    K-step group 0 drains the 7 level accumulators, recombines in fp64, stores Y
//   warp 9 (1 lane)  tcgen05.mma.kind::i8: 26 MMAs per K-step (A = TMEM digits, B = smem Q
//                    digits), commits to the ring / A-buffer / accumulator mbarriers
// TMEM: 6 levels x N columns of accumulators + 2 buffers x 48 columns of A digits (<= 480).
// MMA grouping: the Q digits are stored as consecutive N-row blocks, so digits s..s+g-1 form
// one B operand of g N rows and one MMA computes (t, s), ..., (t, s+g-1) into the adjacent
// level accumulators t+s-5, ... (levels are adjacent N-column blocks).  int8 MMAs with N <= 64
// cost ~45 cycles regardless of N (measured, tools/microbench/umma_rate.cu) while N >= 128 runs
// at the full 8192 MAC/clk, so 9 grouped MMAs (~690 cycles per K-step) replace 21 (~955).
// Accumulators are zeroed by the epilogue warps (every MMA accumulates).
#include <climits>
#include <cmath>
#include <type_traits>
#include <cstdio>
#include <cstdlib>

#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>

#include "common.cuh"

namespace lmra_dev {

namespace {

constexpr int kI8Stages = 4;   // X ring (released by the slicers); even: the two slicer groups
                               // then own disjoint stages (with an odd count a group could wait
                               // on a stage one phase ahead and pass on the stale parity)
constexpr int kI8QStages = 6;  // Q-digit ring (released by the MMA; the L2 -> smem copy needs
                               // several K-steps of lead)
constexpr int kI8Tile = 128;                 // columns of X per tile (MMA M)
constexpr int kI8Kstep = 32;                 // k per MMA (int8)
constexpr int kI8XBytes = kI8Kstep * kI8Tile * 8;  // 32 KB per X stage
constexpr int kI8Digits = 6;
constexpr int kI8Levels = 6;                 // L = t + s in 5..10
constexpr int kI8MinLevel = 5;
constexpr unsigned long long kI8Balance = 0x808080808080ull;  // 128 in each of the 6 digits
constexpr int kI8Threads = 608;  // 2 x 4 slicer warps, X TMA warp, MMA warp, Q warp, 8 epilogue warps
constexpr int kI8ProdWarp = 8, kI8MmaWarp = 9, kI8QWarp = 10, kI8EpiWarp0 = 11;
constexpr int kI8EpiWarps = 8;
constexpr int kI8MaxN = 64;  // N = mu rounded up to 16 (M = 128 needs N % 16 == 0)
constexpr int kI8ABufs = 2;
constexpr int kI8StageLd = 9;  // epilogue output staging: 32 columns x 8 outputs, row pad 1
constexpr int kI8StageBytes = kI8EpiWarps * 32 * kI8StageLd * 8;
constexpr int kTR = 4;  // tile-id ring of the dynamic scheduler
constexpr int kTRConsumers = 1 + 1 + kI8EpiWarps + 8;  // Q producer, MMA, epilogue warps, slicer warps

__device__ __forceinline__ uint64_t umma_smem_desc(uint32_t saddr) {
  // K-major, no swizzle: 8-row x 16-byte core matrices, LBO 128 B (K chunk), SBO 256 B (rows)
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) |
         ((uint64_t)(256 >> 4) << 32) | ((uint64_t)1 << 46);
}

__host__ __device__ constexpr uint32_t umma_idesc_i8(int M, int N, bool a_signed, bool b_signed) {
  return (2u << 4) | ((a_signed ? 1u : 0u) << 7) | ((b_signed ? 1u : 0u) << 10) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const void* tmap, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
      "[%2];\n" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

// Q digits: qd[ks][s][canonical N x 32 B] (K-major core matrices), eq[m]
__global__ void q_digits_kernel(const double* __restrict__ q, int K, int mu, int N,
                                uint8_t* __restrict__ qd, int* __restrict__ eq) {
  __shared__ double red[32];
  const int m = blockIdx.x;
  double mx = 0.0;
  if (m < mu)
    for (int k = threadIdx.x; k < K; k += blockDim.x) mx = fmax(mx, fabs(q[k + (size_t)K * m]));
  for (int o = 16; o >= 1; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  mx = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) mx = fmax(mx, red[w]);
  const int e = mx > 0.0 ? ilogb(mx) + 2 : 0;
  if (threadIdx.x == 0 && m < mu) eq[m] = e;
  const int nks = (K + kI8Kstep - 1) / kI8Kstep;
  const size_t blk = (size_t)kI8Digits * N * kI8Kstep;
  for (int k = threadIdx.x; k < nks * kI8Kstep; k += blockDim.x) {
    long long U = 0;
    if (m < mu && k < K) U = __double2ll_rn(ldexp(q[k + (size_t)K * m], 47 - e));
    const unsigned long long W = (unsigned long long)U + kI8Balance;  // balanced digits: bytes ^ 0x80
    const int ks = k / kI8Kstep, kk = k % kI8Kstep;
    const size_t off = (size_t)ks * blk + (m / 8) * 256 + (kk / 16) * 128 + (m % 8) * 16 + (kk % 16);
#pragma unroll
    for (int s = 0; s < kI8Digits; ++s)
      qd[off + (size_t)s * N * kI8Kstep] = (uint8_t)(((W >> (8 * s)) & 0xFF) ^ 0x80);
  }
}

#ifdef LMRA_I8_CLOCKS  // microbenchmark only (tools/microbench/i8_clocks.cu): CTA 0 wait cycles,
                       // summed in registers and flushed once at the end of the kernel
__device__ unsigned long long g_i8clk[20];
#define I8_WAIT(idx, call)                   \
  do {                                       \
    const long long _t0 = clock64();         \
    call;                                    \
    i8acc[idx] += clock64() - _t0;           \
  } while (0)
#define I8_T0(v) const long long v = clock64()
#define I8_ACC(idx, v) i8acc[idx] += clock64() - (v)
#else
#define I8_WAIT(idx, call) call
#define I8_T0(v)
#define I8_ACC(idx, v)
#endif

// exact int32 -> fp64 without the conversion unit: 2^52 + 2^31 + x has x in its low word
__device__ __forceinline__ double i32_to_f64(uint32_t x) {
  return __hiloint2double(0x43300000, (int)(x ^ 0x80000000u)) - 4503601774854144.0;  // 2^52 + 2^31
}

__device__ __forceinline__ double pow2(int e) {  // 2^e for -1022 <= e <= 1023
  return __longlong_as_double((long long)(e + 1023) << 52);
}

// X stage layout: two boxes (k 0-15, 16-31) of 128 rows (j) x 128 B, 128-byte swizzle
__device__ __forceinline__ const double* xs_elem(const double* stage, int j, int k) {
  const int h = k >> 4, kk = k & 15;
  return stage + h * (kI8Tile * 16) + j * 16 + ((((kk >> 1) ^ (j & 7)) << 1) | (kk & 1));
}


// Geometry of one contraction.  Mode-0 form (kInner = false): X is K x J with column j
// contiguous, scales from the canonical squared column norms w.  Inner form (kInner = true):
// X(r, k, o) = x[r + R (k + K o)] with R <= 64 (the mode-1 view of a tensor whose first mode
// has already been contracted to R), contracted over k; a tile is 2 o-slices x 64 rows r
// (rows r >= R are the TMA's zero fill), scales from per-column maximum exponents fexp_in.
struct I8Geom {
  long long J;          // mode-0: columns
  int K;
  int R;                // inner: rows per o-slice (<= 64)
  long long O;          // inner: o-slices
  const double* w;      // mode-0: canonical squared column norms
  const int* fexp_in;   // inner: max binary exponent of column (r, o) at r + R o
  int* fexp_out;        // mode-0, optional: max exponent of Y's mode-1 fibres (m, o), m + mu o,
  long long I1;         //   with j = i1 + I1 o (the next contraction's columns)
  unsigned long long* tile_ctr;  // dynamic tile scheduler: next tile (zeroed before the launch)
};

// binary exponent e with |v| < 2^(e+1) (an upper bound for subnormals), INT_MIN for 0
__device__ __forceinline__ int exp_bound(double v) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(v) << 1;
  if (b == 0) return -2147483647 - 1;
  const int e = (int)(b >> 53);
  return e == 0 ? -1023 : e - 1023;
}

template <int N, bool kInner>
__global__ void __launch_bounds__(kI8Threads, 1) ttm_i8_kernel(
    const __grid_constant__ CUtensorMap xmap, const uint8_t* __restrict__ qd, const int* __restrict__ eqg,
    const I8Geom geo, int mu, double* __restrict__ y) {
  const long long J = geo.J;
  const int K = geo.K;
  constexpr int kQBytes = kI8Digits * N * kI8Kstep;
  constexpr uint32_t kAccCols = kI8Levels * N;
  constexpr uint32_t kACols = kI8Digits * 8;  // 6 digits x 32 bytes per lane
  constexpr int kAB = kI8ABufs;
  static_assert(kI8Stages % 2 == 0 && kAB == 2, "stages and A buffers are partitioned by slicer group");
  static_assert(kAccCols + kAB * kACols <= 512, "TMEM budget");
  extern __shared__ __align__(16) unsigned char smraw[];
  unsigned char* base = smraw + ((1024 - (smem_u32(smraw) & 1023)) & 1023);
  double* xs = reinterpret_cast<double*>(base);                          // stages x 32 KB
  uint8_t* qs = base + kI8Stages * kI8XBytes;                            // qstages x kQBytes
  double* ostage = reinterpret_cast<double*>(qs + kI8QStages * kQBytes);  // epilogue staging
  uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(ostage) + kI8StageBytes);
  uint64_t* full = bars;                       // [stages] X landed
  uint64_t* empty = full + kI8Stages;          // [stages] X converted (4 slicer warps)
  uint64_t* qfull = empty + kI8Stages;         // [qstages] Q digits landed
  uint64_t* qempty = qfull + kI8QStages;       // [qstages] Q digits consumed (MMA commit)
  uint64_t* afull = qempty + kI8QStages;       // [kAB]
  uint64_t* aempty = afull + kAB;              // [kAB]
  uint64_t* accfull = aempty + kAB;            // [1]
  uint64_t* accempty = accfull + 1;            // [1]
  uint64_t* tfull = accempty + 1;              // [kTR] tile id published (X producer)
  uint64_t* tempty = tfull + kTR;              // [kTR] tile id read by every other role
  long long* tring = reinterpret_cast<long long*>(tempty + kTR);  // [kTR] tile ids
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tring + kTR);
  double* qsc = reinterpret_cast<double*>(tmem_slot + 4);  // [N] 2^eq_m

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nks = (K + kI8Kstep - 1) / kI8Kstep;
  const long long ntiles = kInner ? (geo.O + 1) / 2 : (J + kI8Tile - 1) / kI8Tile;
#ifdef LMRA_I8_CLOCKS
  long long i8acc[20] = {0};
  const long long i8start = clock64();
#endif
  if (tid == 0) {
    for (int s = 0; s < kI8Stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 4);
    }
    for (int s = 0; s < kI8QStages; ++s) {
      mbar_init(&qfull[s], 1);
      mbar_init(&qempty[s], 1);
    }
    for (int b = 0; b < kAB; ++b) {
      mbar_init(&afull[b], 4);
      mbar_init(&aempty[b], 1);
    }
    mbar_init(accfull, 1);
    mbar_init(accempty, kI8EpiWarps);
    for (int r = 0; r < kTR; ++r) {
      mbar_init(&tfull[r], 1);
      mbar_init(&tempty[r], kTRConsumers);
    }
    mbar_fence_init();
  }
  if (tid < N) qsc[tid] = ldexp(1.0, tid < mu ? eqg[tid] : 0);  // 2^eq_m
  if (warp == kI8MmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // Dynamic tile scheduler: the X producer takes tiles from a global counter and publishes them
  // in a small ring; every other role follows the same sequence (a CTA that starts late --
  // its SM busy with a concurrent kernel -- simply takes fewer tiles).  take_warp: whole warp;
  // take_lane: a single-lane role.
  auto take_warp = [&](long long it) -> long long {
    const int slot = (int)(it % kTR);
    mbar_wait(&tfull[slot], (unsigned)((it / kTR) & 1));
    const long long t = tring[slot];
    __syncwarp();
    if (lane == 0) mbar_arrive(&tempty[slot]);
    return t;
  };
  auto take_lane = [&](long long it) -> long long {
    const int slot = (int)(it % kTR);
    mbar_wait(&tfull[slot], (unsigned)((it / kTR) & 1));
    const long long t = tring[slot];
    mbar_arrive(&tempty[slot]);
    return t;
  };

  if (warp == kI8ProdWarp) {  // ---------------- producers: lane 0 X tiles, lane 1 Q digits
    if (lane == 0) {
      long long g = 0;
      for (long long it = 0;; ++it) {
        const int slot = (int)(it % kTR);
        mbar_wait(&tempty[slot], (unsigned)((it / kTR) & 1) ^ 1u);
        const long long t = (long long)atomicAdd(geo.tile_ctr, 1ull);
        tring[slot] = t;
        mbar_arrive(&tfull[slot]);
        if (t >= ntiles) break;
        for (int ks = 0; ks < nks; ++ks, ++g) {
          const int st = (int)(g % kI8Stages);
          I8_WAIT(0, mbar_wait(&empty[st], (unsigned)((g / kI8Stages) & 1) ^ 1u));
          mbar_arrive_expect_tx(&full[st], kI8XBytes);
          double* dst = xs + (size_t)st * (kI8XBytes / 8);
          if (kInner) {  // one box: 64 rows r x 32 k x 2 o-slices, [o][k][r] in smem
            tma_load_3d(dst, &xmap, &full[st], 0, ks * kI8Kstep, (int)(2 * t));
          } else {
            tma_load_2d(dst, &xmap, &full[st], ks * kI8Kstep, (int)(t * kI8Tile));
            tma_load_2d(dst + kI8Tile * 16, &xmap, &full[st], ks * kI8Kstep + 16, (int)(t * kI8Tile));
          }
        }
      }
    }
  } else if (warp == kI8QWarp) {  // ---------------- Q-digit producer (own warp: a blocked wait of
                                  // the X producer must not hold it up)
    if (lane == 0) {
      long long g = 0;
      for (long long it = 0;; ++it) {
        if (take_lane(it) >= ntiles) break;
        for (int ks = 0; ks < nks; ++ks, ++g) {
          const int qsi = (int)(g % kI8QStages);
          I8_WAIT(1, mbar_wait(&qempty[qsi], (unsigned)((g / kI8QStages) & 1) ^ 1u));
          mbar_arrive_expect_tx(&qfull[qsi], kQBytes);
          bulk_load(qs + (size_t)qsi * kQBytes, qd + (size_t)ks * kQBytes, kQBytes, &qfull[qsi]);
        }
      }
    }
  } else if (warp == kI8MmaWarp) {  // ---------------- MMA issuer
    if (lane == 0) {
      long long g = 0, tcount = 0;
      for (long long it = 0;; ++it, ++tcount) {
        if (take_lane(it) >= ntiles) break;
        I8_WAIT(2, mbar_wait(accempty, (unsigned)(tcount & 1) ^ 1u));  // previous tile drained
        tc_fence_after();
        for (int ks = 0; ks < nks; ++ks, ++g) {
          const int qsi = (int)(g % kI8QStages), b = (int)(g % kAB);
          I8_WAIT(3, mbar_wait(&afull[b], (unsigned)((g / kAB) & 1)));
          I8_WAIT(4, mbar_wait(&qfull[qsi], (unsigned)((g / kI8QStages) & 1)));
          tc_fence_after();
          I8_T0(tm0);
          const uint32_t qbase = smem_u32(qs + (size_t)qsi * kQBytes);
          const uint32_t abase = tmem + kAccCols + (uint32_t)b * kACols;
          // (t, first s, number of s) groups covering s in [max(0, 5 - t), 5]
          constexpr int kSched[9][3] = {{5, 0, 3}, {5, 3, 3}, {4, 1, 2}, {4, 3, 3}, {3, 2, 2},
                                        {3, 4, 2}, {2, 3, 3}, {1, 4, 2}, {0, 5, 1}};
#pragma unroll
          for (int gi = 0; gi < 9; ++gi) {
            const int dt = kSched[gi][0], s0 = kSched[gi][1], gl = kSched[gi][2];
            const int L = dt + s0 - kI8MinLevel;
            const uint32_t idesc = umma_idesc_i8(kI8Tile, gl * N, true, true);
            const uint64_t bdesc = umma_smem_desc(qbase + (uint32_t)(s0 * N * kI8Kstep));
            // the first two groups (t = 5) cover all six levels: at a tile's first K-step they
            // overwrite, everything after accumulates (no zeroing pass)
            const uint32_t acc = (ks == 0 && gi < 2) ? 0u : 1u;
            asm volatile(
                "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                " tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem + (uint32_t)L * N),
                "r"(abase + (uint32_t)dt * 8), "l"(bdesc), "r"(idesc), "r"(acc));
          }
          tc_commit(&qempty[qsi]);  // the Q digits are consumed
          tc_commit(&aempty[b]);  // the A digit buffer is consumed
          I8_ACC(13, tm0);
        }
        tc_commit(accfull);
      }
    }
  } else if (warp >= kI8EpiWarp0) {  // ---------------- epilogue warps: drain + recombine
    // a warp reaches only the TMEM sub-partition (32 lanes) of its warp index mod 4
    const int jl = 32 * (warp & 3) + lane;  // column within the tile = TMEM lane
    const uint32_t lane_base = (uint32_t)(32 * (warp & 3)) << 16;
    double* ost = ostage + (warp - kI8EpiWarp0) * 32 * kI8StageLd;
    long long tcount = 0;
    for (long long it = 0;; ++it, ++tcount) {
      const long long t = take_warp(it);
      if (t >= ntiles) break;
      const long long j = t * kI8Tile + jl;
      const long long jw0 = t * kI8Tile + 32 * (warp & 3);  // first column of this warp
      const int rrow = jl & 63;                                // inner form: row r, slice o
      const long long ocol = 2 * t + (jl >> 6);
      int ex = 0;
      bool valid;
      if (kInner) {
        valid = rrow < geo.R && ocol < geo.O;
        const int fe = valid ? geo.fexp_in[rrow + (long long)geo.R * ocol] : INT_MIN;
        ex = fe > -1100 ? fe + 2 : 0;
      } else {
        valid = j < J;
        if (valid) {
          const double nrm = sqrt(geo.w[j]);
          ex = nrm > 0.0 ? ilogb(nrm) + 2 : 0;
        }
      }
      const double sj = ldexp(1.0, ex - 94 + 8 * kI8MinLevel);  // column part of the scale
      // mode-0 with fexp_out: the warp's 32 columns lie in one o-slice of the next contraction
      // unless they straddle a multiple of I1
      long long o_lo = 0;
      bool o_uniform = true;
      if (!kInner && geo.fexp_out) {
        const long long jhi = min(jw0 + 31, J - 1);
        o_lo = jw0 / geo.I1;
        o_uniform = o_lo == jhi / geo.I1;
      }
      I8_WAIT(7, mbar_wait(accfull, (unsigned)(tcount & 1)));
      tc_fence_after();
      I8_T0(te0);
#ifdef LMRA_I8_NO_EPILOGUE  // microbenchmark only: release at once, no output (upper bound)
      __syncwarp();
      if (lane == 0) mbar_arrive(accempty);
      continue;
#endif
      // recombine the 6 level accumulators of column j, scale by 2^(ex + eq_m - 94 + 40).  All of
      // this warp's chunks are drained first -- TMEM -> registers, the 6 levels recombined into
      // one double per output -- and the accumulators released before any output is scaled and
      // stored: the MMA warp waits for that release before the next tile's first K-step (TMEM has
      // no room for a second accumulator set), and with the stores inside the drain it waited
      // ~18 % of the kernel (tools/microbench/i8_clocks.cu, mma_wait_accempty)
      const int half = (warp - kI8EpiWarp0) >> 2;  // two warps per sub-partition split the chunks
      constexpr int kCh = N / 16;                   // chunks of 8 outputs per warp
      double sums[kCh][8];
      I8_T0(tld);
#pragma unroll
      for (int c = 0; c < kCh; ++c) {
        const int m0 = 8 * half + 16 * c;
        if (m0 >= mu) continue;  // warp-uniform: no output in this chunk
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {  // 4 outputs at a time (register budget)
          uint32_t v[kI8Levels][4];
#pragma unroll
          for (int L = 0; L < kI8Levels; ++L)
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];\n"
                         : "=r"(v[L][0]), "=r"(v[L][1]), "=r"(v[L][2]), "=r"(v[L][3])
                         : "r"(tmem + lane_base + (uint32_t)(L * N + m0 + 4 * hh)));
          asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            // sum_L S_L 2^(8L): each int32 level to fp64 exactly with the magic-number trick
            // (one LOP + one DADD), then a Horner chain from the top level down
            double sacc = i32_to_f64(v[kI8Levels - 1][u]);
#pragma unroll
            for (int L = kI8Levels - 2; L >= 0; --L) sacc = fma(sacc, 256.0, i32_to_f64(v[L][u]));
            sums[c][4 * hh + u] = sacc;
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(accempty);
      I8_ACC(17, tld);
      I8_ACC(8, te0);
#pragma unroll
      for (int c = 0; c < kCh; ++c) {
        const int m0 = 8 * half + 16 * c;
        if (m0 >= mu) continue;
        I8_T0(tcp);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int m = m0 + u;
          // scale 2^(ex + eq_m - 94 + 40) as two exact power-of-two products
          const double val = (sums[c][u] * sj) * qsc[m];
          if (kInner) {  // Y(r, m, o): rows r of one slice are consecutive -- coalesced as is
            if (valid && m < mu) y[rrow + (long long)geo.R * (m + (long long)mu * ocol)] = val;
          } else {
            ost[lane * kI8StageLd + u] = val;
          }
        }
        if (!kInner) {
          __syncwarp();
          I8_ACC(18, tcp);
          I8_T0(tst);
          // coalesced-ish stores: 4 columns x 8 outputs per instruction (64-byte runs of Y)
          unsigned hmax = 0u;  // fexp_out: |v|'s high word orders like |v| (exponent on top)
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int jj = 4 * i + (lane >> 3), mm = lane & 7;
            const long long jo = jw0 + jj;
            const double v = ost[jj * kI8StageLd + mm];
            if (m0 + mm < mu && jo < J) {
              y[(m0 + mm) + (size_t)mu * jo] = v;
              const unsigned hw = (unsigned)__double2hiint(v) & 0x7fffffffu;
              if (o_uniform)
                hmax = max(hmax, hw);
              else if (geo.fexp_out && hw != 0u)  // columns straddle two o-slices: one by one
                atomicMax(&geo.fexp_out[(m0 + mm) + (long long)mu * (jo / geo.I1)],
                          (hw >> 20) == 0 ? -1023 : (int)(hw >> 20) - 1023);
            }
          }
          if (geo.fexp_out && o_uniform) {  // max exponent of Y's mode-1 fibre (m, o): each lane
                                            // holds 8 of the warp's 32 columns of output m0 + mm
            hmax = max(hmax, __shfl_xor_sync(0xffffffffu, hmax, 8));
            hmax = max(hmax, __shfl_xor_sync(0xffffffffu, hmax, 16));
            if (lane < 8 && m0 + lane < mu && hmax != 0u)
              atomicMax(&geo.fexp_out[(m0 + lane) + (long long)mu * o_lo],
                        (hmax >> 20) == 0 ? -1023 : (int)(hmax >> 20) - 1023);
          }
          __syncwarp();  // the staging rows are rewritten by the next chunk
          I8_ACC(16, tst);
        }
      }
      I8_ACC(14, te0);
    }
  } else {  // ---------------- warps 0-7: digit split (group = K-step parity)
    const int grp = warp >> 2;
    const int jl = tid & (kI8Tile - 1);  // column within the tile = TMEM lane
    const uint32_t lane_base = (uint32_t)(32 * (warp & 3)) << 16;
    long long g = 0, tcount = 0;
    for (long long it = 0;; ++it, ++tcount) {
      const long long t = take_warp(it);
      if (t >= ntiles) break;
      const long long j = t * kI8Tile + jl;
      const int rrow = jl & 63;
      const long long ocol = 2 * t + (jl >> 6);
      bool has = false;
      int ex = 0;
      if (kInner) {
        const int fe = (rrow < geo.R && ocol < geo.O) ? geo.fexp_in[rrow + (long long)geo.R * ocol] : INT_MIN;
        if (fe > -1100) {
          ex = fe + 2;
          has = true;
        }
      } else if (j < J) {
        const double nrm = sqrt(geo.w[j]);
        if (nrm > 0.0) {
          ex = ilogb(nrm) + 2;
          has = true;
        }
      }
      // 2^(47 - ex) as s1 * s2 (s2 = 1 unless the column is below ~2^-950, where one power
      // of two would overflow); x * s1 is exact, so fma(x s1, s2, M) rounds once like
      // fma(x, 2^(47-ex), M)
      double s1 = 0.0, s2 = 1.0;
      bool big = false;
      if (has) {
        const int sh = 47 - ex, a = sh > 1000 ? 1000 : sh;
        s1 = ldexp(1.0, a);
        s2 = ldexp(1.0, sh - a);
        big = sh > 1000;
      }
      const bool warp_big = __any_sync(0xffffffffu, big);  // uniform: the two-step path only
                                                           // when a column of the warp needs it
      // V = round(x 2^(47-ex)) read off the bits of fma(x, 2^(47-ex), 1.5 2^52): for |V| < 2^51
      // the sum is exact up to the final rounding (= round-to-nearest-even of x 2^(47-ex)) and
      // its low 51 bits are V's two's complement bits, i.e. bytes 0..5 are V's digits
      constexpr double kMagic = 6755399441055744.0 + (double)kI8Balance;  // 1.5 * 2^52 + C (exact)
      for (int ks = 0; ks < nks; ++ks, ++g) {
        if ((int)(g & 1) != grp) continue;  // the other group's K-step
        const int st = (int)(g % kI8Stages), b = (int)(g % kAB);
        I8_WAIT(5 + grp * 4, mbar_wait(&full[st], (unsigned)((g / kI8Stages) & 1)));
        const double* stage = xs + (size_t)st * (kI8XBytes / 8);
        I8_T0(ts0);
        uint32_t dw[kI8Digits][8];
        // the conversion, instantiated with and without the two-step scale (warp-uniform
        // choice outside the loop: a branch inside it cost the slicers ~50 %)
        auto convert = [&](auto two_step) {
#pragma unroll
          for (int c = 0; c < 8; ++c) {  // k = 4c .. 4c+3
            double xv[4];
            if (kInner) {  // stage [o][k][r]: this row's k values at stride 64 (conflict-free)
              const double* colp = stage + (size_t)(jl >> 6) * (32 * 64) + rrow + (4 * c) * 64;
#pragma unroll
              for (int u = 0; u < 4; ++u) xv[u] = colp[u * 64];
            } else {  // two 16-byte chunks of one swizzled row
              const double* rowp = stage + (c >> 2) * (kI8Tile * 16) + jl * 16;
              const int c2 = 2 * (c & 3);
              const double2 p0 = *reinterpret_cast<const double2*>(rowp + ((c2 ^ (jl & 7)) << 1));
              const double2 p1 = *reinterpret_cast<const double2*>(rowp + (((c2 + 1) ^ (jl & 7)) << 1));
              xv[0] = p0.x;
              xv[1] = p0.y;
              xv[2] = p1.x;
              xv[3] = p1.y;
            }
            uint32_t lo[4], hi[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const double d = decltype(two_step)::value ? fma(xv[u] * s1, s2, kMagic) : fma(xv[u], s1, kMagic);
              lo[u] = (uint32_t)__double2loint(d);
              hi[u] = (uint32_t)__double2hiint(d);
            }
            // digit s of the 4 values = byte s of each V, packed little-endian
            const uint32_t l01 = __byte_perm(lo[0], lo[1], 0x5140), l23 = __byte_perm(lo[2], lo[3], 0x5140);
            const uint32_t l01b = __byte_perm(lo[0], lo[1], 0x7362), l23b = __byte_perm(lo[2], lo[3], 0x7362);
            dw[0][c] = __byte_perm(l01, l23, 0x5410) ^ 0x80808080u;    // bytes 0
            dw[1][c] = __byte_perm(l01, l23, 0x7632) ^ 0x80808080u;    // bytes 1
            dw[2][c] = __byte_perm(l01b, l23b, 0x5410) ^ 0x80808080u;  // bytes 2
            dw[3][c] = __byte_perm(l01b, l23b, 0x7632) ^ 0x80808080u;  // bytes 3
            const uint32_t h01 = __byte_perm(hi[0], hi[1], 0x5140), h23 = __byte_perm(hi[2], hi[3], 0x5140);
            dw[4][c] = __byte_perm(h01, h23, 0x5410) ^ 0x80808080u;    // bytes 4
            dw[5][c] = __byte_perm(h01, h23, 0x7632) ^ 0x80808080u;    // bytes 5
          }
        };
        if (warp_big)
          convert(std::true_type{});
        else
          convert(std::false_type{});
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);  // this warp is done with the X stage
        I8_ACC(11, ts0);
        I8_WAIT(6 + grp * 4, mbar_wait(&aempty[b], (unsigned)((g / kAB) & 1) ^ 1u));
        tc_fence_after();
        const uint32_t abase = tmem + lane_base + kAccCols + (uint32_t)b * kACols;
        I8_T0(ts1);
#pragma unroll
        for (int s = 0; s < kI8Digits; ++s)
          asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(
                           abase + (uint32_t)s * 8),
                       "r"(dw[s][0]), "r"(dw[s][1]), "r"(dw[s][2]), "r"(dw[s][3]), "r"(dw[s][4]),
                       "r"(dw[s][5]), "r"(dw[s][6]), "r"(dw[s][7]));
        asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&afull[b]);
        I8_ACC(12, ts1);
      }
    }
  }
#ifdef LMRA_I8_CLOCKS
  if (warp == kI8MmaWarp) i8acc[15] = clock64() - i8start;  // CTA 0's own span (SM clocks)
  if (blockIdx.x == 0 && lane == 0)
    for (int i = 0; i < 20; ++i)
      if (i8acc[i]) atomicAdd(&g_i8clk[i], (unsigned long long)i8acc[i]);
#endif
  tc_fence_before();
  __syncthreads();
  if (warp == kI8MmaWarp) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512));
}

PFN_cuTensorMapEncodeTiled_v12000 i8_tensor_map_encoder() {
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

// fexp[r + R o] = max_k exp_bound(x[r + R (k + K o)]) (INT_MIN for an all-zero column)
__global__ void column_exponents_kernel(const double* __restrict__ x, long long R, long long K, long long O,
                                        int* __restrict__ fexp) {
  const long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x;  // c = r + R o
  if (c >= R * O) return;
  const long long r = c % R, o = c / R;
  const double* col = x + r + R * K * o;
  int e = INT_MIN;
  for (long long k = 0; k < K; ++k) e = max(e, exp_bound(col[R * k]));
  fexp[c] = e;
}

template <int N, bool kInner>
cudaError_t launch_n(const CUtensorMap& map, const uint8_t* qd, const int* eq, const I8Geom& geo, int mu,
                     double* y, cudaStream_t st) {
  static unsigned long long done = 0;
  const size_t smem = kI8Stages * (size_t)kI8XBytes + kI8QStages * (size_t)kI8Digits * N * kI8Kstep +
                      kI8StageBytes + 512 + 1024 + 8 * N;
  cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(ttm_i8_kernel<N, kInner>), smem, done);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long ntiles = kInner ? (geo.O + 1) / 2 : (geo.J + kI8Tile - 1) / kI8Tile;
  int reserve = std::max(0, g_i8_reserved_sms);
  if (const char* env = getenv("LMRA_I8_RESERVE")) reserve = atoi(env);  // diagnostics override
  const int avail = std::max(1, sms - reserve);
  const int grid = (int)(ntiles < avail ? ntiles : avail);
  if (getenv("LMRA_I8_DEBUG")) fprintf(stderr, "ttm_i8 grid %d (sms %d, reserve %d, tiles %lld)\n", grid, sms, reserve, ntiles);
  ttm_i8_kernel<N, kInner><<<grid, kI8Threads, smem, st>>>(map, qd, eq, geo, mu, y); note_launch();
  return cudaGetLastError();
}

// Q digits + eq into the workspace (one small kernel), returns the digit / eq pointers
cudaError_t prepare_q(const double* q, long long K, int mu, void* work, uint8_t** qd, int** eq,
                      cudaStream_t st) {
  const int N = ((mu + 15) / 16) * 16;
  const long long nks = (K + kI8Kstep - 1) / kI8Kstep;
  *qd = static_cast<uint8_t*>(work);
  *eq = reinterpret_cast<int*>(*qd + ((size_t)nks * kI8Digits * N * kI8Kstep + 255) / 256 * 256);
  q_digits_kernel<<<N, 256, 0, st>>>(q, (int)K, mu, N, *qd, *eq); note_launch();
  return cudaGetLastError();
}

template <bool kInner>
cudaError_t dispatch_n(const CUtensorMap& map, const uint8_t* qd, const int* eq, const I8Geom& geo, int mu,
                       double* y, cudaStream_t st) {
  switch (((mu + 15) / 16) * 16) {
    case 16: return launch_n<16, kInner>(map, qd, eq, geo, mu, y, st);
    case 32: return launch_n<32, kInner>(map, qd, eq, geo, mu, y, st);
    case 48: return launch_n<48, kInner>(map, qd, eq, geo, mu, y, st);
    default: return launch_n<64, kInner>(map, qd, eq, geo, mu, y, st);
  }
}

}  // namespace

bool ttm_i8_supported(long long K, long long J, int mu, const double* x) {
  return i8_tensor_map_encoder() != nullptr && K % 2 == 0 && K >= 2 && K <= 4096 && mu >= 1 &&
         mu <= kI8MaxN && J >= 1 && J < (1ll << 31) && (reinterpret_cast<uintptr_t>(x) & 15) == 0;
}

bool ttm_i8_inner_supported(long long R, long long K, long long O, int mu, const double* x) {
  return i8_tensor_map_encoder() != nullptr && R >= 2 && R <= 64 && R % 2 == 0 && K >= 1 &&
         K <= 4096 && O >= 1 && O < (1ll << 31) && mu >= 1 && mu <= kI8MaxN &&
         (reinterpret_cast<uintptr_t>(x) & 15) == 0;
}

size_t ttm_i8_workspace_bytes(long long K, int mu) {
  const int N = ((mu + 15) / 16) * 16;
  const long long nks = (K + kI8Kstep - 1) / kI8Kstep;
  return (size_t)nks * kI8Digits * N * kI8Kstep + 4 * 64 + 256 + 256;  // + the tile counter
}

namespace {
// the tile counter lives in the last 256 bytes of the workspace
unsigned long long* tile_counter(void* work, long long K, int mu, cudaStream_t st, cudaError_t* e) {
  auto* c = reinterpret_cast<unsigned long long*>(static_cast<uint8_t*>(work) + ttm_i8_workspace_bytes(K, mu) - 256);
  *e = cudaMemsetAsync(c, 0, sizeof(unsigned long long), st);
  return c;
}
}  // namespace

cudaError_t launch_ttm_i8(const double* x, long long K, long long J, const double* q, int mu,
                          const double* w, double* y, void* work, cudaStream_t st, int* fexp_out,
                          long long I1) {
  if (!ttm_i8_supported(K, J, mu, x) || (fexp_out && I1 < 1)) return cudaErrorInvalidValue;
  uint8_t* qd;
  int* eq;
  cudaError_t e = prepare_q(q, K, mu, work, &qd, &eq, st);
  if (e != cudaSuccess) return e;
  CUtensorMap map;
  const cuuint64_t gdim[2] = {(cuuint64_t)K, (cuuint64_t)J};
  const cuuint64_t gstride[1] = {(cuuint64_t)K * 8};
  const cuuint32_t box[2] = {16, (cuuint32_t)kI8Tile}, estride[2] = {1, 1};
  if (i8_tensor_map_encoder()(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(x), gdim, gstride,
                              box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  unsigned long long* ctr = tile_counter(work, K, mu, st, &e);
  if (e != cudaSuccess) return e;
  I8Geom geo{J, (int)K, 0, 0, w, nullptr, fexp_out, I1, ctr};
  return dispatch_n<false>(map, qd, eq, geo, mu, y, st);
}

cudaError_t launch_column_exponents(const double* x, long long R, long long K, long long O, int* fexp,
                                    cudaStream_t st) {
  if (R < 1 || K < 1 || O < 1) return cudaErrorInvalidValue;
  const long long n = R * O;
  column_exponents_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(x, R, K, O, fexp); note_launch();
  return cudaGetLastError();
}

cudaError_t launch_ttm_i8_inner(const double* x, long long R, long long K, long long O, const double* q,
                                int mu, const int* fexp_in, double* y, void* work, cudaStream_t st) {
  if (!ttm_i8_inner_supported(R, K, O, mu, x)) return cudaErrorInvalidValue;
  uint8_t* qd;
  int* eq;
  cudaError_t e = prepare_q(q, K, mu, work, &qd, &eq, st);
  if (e != cudaSuccess) return e;
  CUtensorMap map;  // (r, k, o), box 64 x 32 x 2, rows r >= R zero-filled, no swizzle
  const cuuint64_t gdim[3] = {(cuuint64_t)R, (cuuint64_t)K, (cuuint64_t)O};
  const cuuint64_t gstride[2] = {(cuuint64_t)R * 8, (cuuint64_t)(R * K) * 8};
  const cuuint32_t box[3] = {64, (cuuint32_t)kI8Kstep, 2}, estride[3] = {1, 1, 1};
  if (i8_tensor_map_encoder()(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(x), gdim, gstride,
                              box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  unsigned long long* ctr = tile_counter(work, K, mu, st, &e);
  if (e != cudaSuccess) return e;
  I8Geom geo{0, (int)K, (int)R, O, nullptr, fexp_in, nullptr, 0, ctr};
  return dispatch_n<true>(map, qd, eq, geo, mu, y, st);
}

}  // namespace lmra_dev

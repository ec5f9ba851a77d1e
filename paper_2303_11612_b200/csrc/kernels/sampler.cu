// sampler.cu -- the reference's sampling chain on the device, bit-exact.
//
// Replaces, for the AMM variants, the host loops of
//   gram_sampling_probabilities  tucker.cpp:110-130   (naive total, w/total, beta-mix)
//   ProbabilityDistribution::normalized + ctor check   sketching.cpp:28-48 (Neumaier sums)
//   randsample                   sketching.cpp:96-131  (naive cumulative sum, upper_bound)
// The reference's sums are SEQUENTIAL fp64 recurrences (s += x); their bits are
// reproduced exactly in parallel:
//
//  * Naive sum / prefix of nonnegative x ("exact scan").  While the running sum S stays
//    in one binade [2^e, 2^(e+1)) every rounded step adds an integer number r_i of ulps
//    u = 2^(e-52): r_i = round(x_i / u), ties to even on the resulting multiple -- so a
//    tie's choice depends on the parity of S/u, a 2-state map (reset-to-even / xor) that
//    composes associatively.  x/u is exact (power-of-two scaling), so r_i and the parity
//    maps are exact integer data and the binade's run is an exact integer prefix sum.
//    A step whose exact sum reaches the next binade is evaluated directly (one IEEE add).
//    Parallel structure: chunks of 4096; each chunk's aggregate (R for start parity 0/1,
//    parity map, crossing margin) is computed assuming the binade that an approximate
//    prefix predicts (pass B).  A chunk the prediction places across exactly one binade
//    boundary is "split": pass B gives it 16 sub-chunk aggregates (256 elements) under
//    both binades.  One CTA walks the chunks in order with the exact state (pass C): runs
//    of certified chunks are taken at once (a block scan of the 2-state parity transducer
//    M -> M + R_parity(M)); a split chunk is walked sub-chunk by sub-chunk, stepping only
//    the sub-chunk that holds the crossing (one warp: a warp scan of the sub-chunk
//    transducers, the crossing sub-chunk stepped by one lane from shared memory); chunk 0
//    (dense crossings from S = 0) is processed element-exactly.
//    Pass D writes every S_i of the certified (sub-)chunks.
//  * Neumaier's stable_sum (sketching.cpp:13-24) = fl(S + c): S is the naive sum (above);
//    c is the naive sum of the exact two-sum errors e_i (computable from S_{i-1}, x_i,
//    S_i).  c is accumulated exactly (double-double, fixed tree) and the final rounding
//    fl(S + c) is certified against the maximal drift of the sequential c (<= n u sum|c_k|);
//    an uncertifiable case (measure ~1e-5) falls back to the sequential loop, verbatim.
//  * Elementwise steps use explicit IEEE intrinsics (no FMA contraction), matching the
//    oracle compiled with -ffp-contract=off.
#include <cstdint>

#include "common.cuh"

namespace lmra_dev {

constexpr int kChunk = 4096;
constexpr int kThr = 256;                 // grid passes: 16 items per thread
constexpr int kItems = kChunk / kThr;
constexpr int kCThr = 1024;               // pass C (single CTA): 4 items per thread
constexpr int kCItems = kChunk / kCThr;
constexpr int kSub = 64;                  // sub-chunk of a split chunk (the stepped unit)
constexpr int kNSub = kChunk / kSub;      // 64 sub-chunks (two per lane of the walking warp)
constexpr int kSubThr = kSub / kItems;    // 4 threads per sub-chunk in passes B/D
constexpr double kTwo53 = 9007199254740992.0;

enum SamplerStatus {
  kBadWeight = 1,      // negative / NaN weight   -> "probability weights must be nonnegative"
  kZeroNormalize = 2,  // Neumaier sum <= 0       -> "cannot normalize an all-zero distribution"
  kNotOne = 4,         // ctor check |sum-1|>1e-12 -> "probability weights must sum to one"
  kZeroAcc = 8,        // cum total <= 0          -> "randsample: all-zero distribution"
  kFallback = 16,      // informational: sequential Neumaier fallback was used
  kBadBeta = 32,       // nearly-optimal beta outside (0, 1] (checked only when total > 0)
  kInternal = 64,      // uniform closed form: segment table overflow (unreachable)
};

// ---------------------------------------------------------------- parity maps
// map(p) = (reset ? 0 : p) ^ flip, packed as bit0 = flip, bit1 = reset
__device__ __forceinline__ int map_compose(int first, int second) {  // second o first
  const int reset = (first | second) & 2;
  const int flip = (second & 2) ? (second & 1) : ((first ^ second) & 1);
  return reset | flip;
}
__device__ __forceinline__ int map_apply(int m, int p) { return ((m & 2) ? 0 : p) ^ (m & 1); }

// per-element classification relative to ulp u (y = x / u exactly):
//   r = floor(y) (+1 if frac > 1/2), tie if frac == 1/2 (r decided by parity)
struct Elem {
  double y, q;
  int tie;
  int map;  // parity map contributed when the tie is resolved
};

// parity of an integer-valued double (exact below 2^62; larger values only occur past a
// binade crossing, where the parity is never used).  CUDA's fmod is an iterative software
// routine (~50 trips near 2^52) -- far too slow for a per-element test.
__device__ __forceinline__ int parity_of(double v) {
  return v < 4.0e18 ? (int)((unsigned long long)v & 1ull) : 0;
}

__device__ __forceinline__ Elem classify(double x, int ulp_exp) {
  Elem el;
  el.y = ldexp(x, -ulp_exp);
  el.q = floor(el.y);
  const double f = el.y - el.q;
  el.tie = f == 0.5;
  const double r = el.q + (f > 0.5 ? 1.0 : 0.0);
  // tie: result parity is even -> reset, flip 0; else xor (r mod 2)
  el.map = el.tie ? 2 : parity_of(r);
  if (!el.tie) el.q = r;
  return el;
}

__device__ __forceinline__ double tie_r(double q, int pprev) {
  // smallest of {q, q+1} making (pprev + r) even
  return q + (double)((parity_of(q) ^ pprev) & 1);
}

// binade of a positive sum: returns ulp exponent and the exponent of the boundary
__device__ __forceinline__ void binade_of(double S, int& ulp_exp, int& bound_exp) {
  if (S < 0x1.0p-1022) {  // subnormal range: fixed spacing 2^-1074 up to 2^-1022
    ulp_exp = -1074;
    bound_exp = -1022;
  } else {
    const int e = ilogb(S);
    ulp_exp = e - 52;
    bound_exp = e + 1;
  }
}

// ---------------------------------------------------------------- block scan helpers
template <int NT>
struct BlockScan {
  // exclusive scan of parity maps (composition in index order); returns block map
  __device__ static int excl_map(int m, int& excl, int* sm) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int inc = m;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc = map_compose(t, inc);
    }
    if (lane == 31) sm[w] = inc;
    __syncthreads();
    if (w == 0) {
      int t = lane < NT / 32 ? sm[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int u = __shfl_up_sync(0xffffffffu, t, o);
        if (lane >= o) t = map_compose(u, t);
      }
      if (lane < NT / 32) sm[lane] = t;
    }
    __syncthreads();
    const int wbase = w > 0 ? sm[w - 1] : 0;  // identity map = 0
    int prev = __shfl_up_sync(0xffffffffu, inc, 1);
    if (lane == 0) prev = 0;
    excl = map_compose(wbase, prev);
    const int total = sm[NT / 32 - 1];
    __syncthreads();
    return total;
  }
};

// inclusive block scan returning per-thread inclusive value (helper used below)
template <int NT>
__device__ double block_incl(double v, double* sm, double& total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    double t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  if (lane == 31) sm[w] = v;
  __syncthreads();
  if (w == 0) {
    double t = lane < NT / 32 ? sm[lane] : 0.0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      double u = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += u;
    }
    if (lane < NT / 32) sm[lane] = t;
  }
  __syncthreads();
  v += w > 0 ? sm[w - 1] : 0.0;
  total = sm[NT / 32 - 1];
  __syncthreads();
  return v;
}

template <int NT>
__device__ double block_max(double v, double* sm) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  if (lane == 0) sm[w] = v;
  __syncthreads();
  double r = sm[0];
  for (int k = 1; k < NT / 32; ++k) r = fmax(r, sm[k]);
  __syncthreads();
  return r;
}

template <int NT>
__device__ long long block_min_ll(long long v, long long* sm) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  if (lane == 0) sm[w] = v;
  __syncthreads();
  long long r = sm[0];
  for (int k = 1; k < NT / 32; ++k) r = min(r, sm[k]);
  __syncthreads();
  return r;
}

// ---------------------------------------------------------------- workspace layout
struct ChunkAgg {
  double R0, R1;    // total ulps added over the chunk for start parity 0 / 1 (saturated)
  double Z0, Z1;    // max_i (Rprev_i + y_i) for start parity 0 / 1 (rounded up by margin)
  int map;          // parity map of the whole chunk
  int ulp_exp;      // assumed binade (ulp exponent); kNoBinade if ambiguous
  int bad;          // negative / NaN input seen
  int split;        // chunk-level: sub-chunk aggregates exist (two binade hypotheses)
};
constexpr int kNoBinade = 1 << 30;

// A split chunk holding one binade crossing, in O(1) for the walk (pass B): the approximate
// per-element prefix places the crossing element in a short window [w0, w1]; the elements
// before it form one segment under the lower binade (pre), those after it one under the upper
// binade (post).  The walk applies pre, steps the window with IEEE adds, applies post.
constexpr int kWin = 32;  // longest stepped window
struct CrossAgg {
  ChunkAgg pre, post;
  long long w0, w1;  // absolute element indices, window inclusive
  int ok;            // 0: no usable window (the sub-chunk walk handles the chunk)
  int pad;
};

struct ChunkStart {  // exact state at a certified chunk's start (pass C -> pass D)
  double M;          // S / u (integer < 2^53)
  int parity;
  int ulp_exp;
  int fast;          // 1: pass D writes the chunk, 0: pass C already wrote it, 2: split
                     // (sub-chunk starts), 3: crossing chunk (CrossStart)
  int pad;
};
struct CrossStart {  // pass C -> pass D for a crossing chunk written by the O(1) path
  ChunkStart pre, post;
  long long w0, w1;
};

// ---------------------------------------------------------------- sub-chunk segments
// A split chunk's sub-chunk is kSubThr consecutive threads (16 items each) in passes B and D:
// scans and reductions stay inside the kSubThr-lane segment.
__device__ __forceinline__ unsigned seg_mask() {
  static_assert(kSubThr >= 2 && kSubThr <= 16 && (kSubThr & (kSubThr - 1)) == 0, "segment width");
  return ((1u << kSubThr) - 1u) << ((threadIdx.x & 31) & ~(kSubThr - 1));
}
__device__ __forceinline__ int seg_excl_map(int m, unsigned mask, int& total) {
  const int sl = threadIdx.x & (kSubThr - 1);
  int inc = m;
#pragma unroll
  for (int o = 1; o < kSubThr; o <<= 1) {
    const int t = __shfl_up_sync(mask, inc, o, kSubThr);
    if (sl >= o) inc = map_compose(t, inc);
  }
  total = __shfl_sync(mask, inc, kSubThr - 1, kSubThr);
  int prev = __shfl_up_sync(mask, inc, 1, kSubThr);
  return sl == 0 ? 0 : prev;
}
__device__ __forceinline__ double seg_incl_sum(double v, unsigned mask, double& total) {
  const int sl = threadIdx.x & (kSubThr - 1);
#pragma unroll
  for (int o = 1; o < kSubThr; o <<= 1) {
    const double t = __shfl_up_sync(mask, v, o, kSubThr);
    if (sl >= o) v += t;
  }
  total = __shfl_sync(mask, v, kSubThr - 1, kSubThr);
  return v;
}
__device__ __forceinline__ double seg_max(double v, unsigned mask) {
#pragma unroll
  for (int o = kSubThr / 2; o >= 1; o >>= 1) v = fmax(v, __shfl_xor_sync(mask, v, o, kSubThr));
  return v;
}

// r of one element given the running parity (updated), from its classification
__device__ __forceinline__ double step_r(const Elem& e, int& par) {
  const double r = e.tie ? tie_r(e.q, par) : e.q;
  par = map_apply(e.map, par);
  return r;
}

// Per-thread pass over its items for BOTH start parities at once (classifications are
// recomputed instead of kept: the earlier version held 16 Elem + 16 prefixes per thread
// in registers, 200 registers and one CTA per SM, latency-bound).  Returns the thread's
// ulp totals run_p and zl_p = max_j (ulps before j + y_j), saturated past 2^53.
__device__ __forceinline__ void two_parity_pass(const double (&xv)[kItems], int ue, int excl,
                                                double& run0, double& run1, double& zl0,
                                                double& zl1) {
  int par0 = map_apply(excl, 0), par1 = map_apply(excl, 1);
  run0 = run1 = zl0 = zl1 = 0.0;
#pragma unroll 4
  for (int j = 0; j < kItems; ++j) {
    const Elem e = classify(xv[j] >= 0.0 ? xv[j] : 0.0, ue);
    zl0 = fmax(zl0, run0 + e.y);
    zl1 = fmax(zl1, run1 + e.y);
    run0 = fmin(run0 + step_r(e, par0), 2.0 * kTwo53);  // saturate: past 2^53 is a crossing
    run1 = fmin(run1 + step_r(e, par1), 2.0 * kTwo53);
  }
}

__device__ __forceinline__ int thread_map(const double (&xv)[kItems], int ue) {
  int tmap = 0;
#pragma unroll 4
  for (int j = 0; j < kItems; ++j)
    tmap = map_compose(tmap, classify(xv[j] >= 0.0 ? xv[j] : 0.0, ue).map);
  return tmap;
}

// this thread's kItems consecutive elements (16-byte vector loads when fully in range;
// rows past n read as 0)
__device__ __forceinline__ void load_items(const double* __restrict__ x, long long n,
                                           long long base, double (&v)[kItems]) {
  if (base + kItems <= n) {
    const double2* p = reinterpret_cast<const double2*>(x + base);
#pragma unroll
    for (int j = 0; j < kItems / 2; ++j) {
      const double2 t = p[j];
      v[2 * j] = t.x;
      v[2 * j + 1] = t.y;
    }
  } else {
#pragma unroll
    for (int j = 0; j < kItems; ++j) v[j] = base + j < n ? x[base + j] : 0.0;
  }
}

// ---------------------------------------------------------------- pass A: chunk sums
__global__ void __launch_bounds__(kThr) chunk_sums_kernel(const double* __restrict__ x, long long n,
                                                          double* __restrict__ csum, const int* __restrict__ skip) {
  pdl_wait();  // the previous kernel's outputs (programmatic dependent launch)
  pdl_trigger();
  if (skip && *skip) return;
  __shared__ double sm[32];
  double xv[kItems];
  load_items(x, n, (long long)blockIdx.x * kChunk + threadIdx.x * kItems, xv);
  double v = 0.0;
#pragma unroll
  for (int k = 0; k < kItems; ++k) v += xv[k];
  double tot;
  block_incl<kThr>(v, sm, tot);
  if (threadIdx.x == 0) csum[blockIdx.x] = tot;
}

// approximate exclusive prefix over chunk sums -> chunk binade predictions (1 CTA, block
// scan over tiles of 1024 chunks; the prediction only needs |approx - exact| <= delta)
__global__ void __launch_bounds__(1024) chunk_plan_kernel(const double* __restrict__ csum,
                                                          int nchunks, long long n,
                                                          int* __restrict__ assumed,
                                                          int* __restrict__ assumed2,
                                                          double* __restrict__ approx,
                                                          const int* __restrict__ skip) {
  pdl_wait();  // the previous kernel's outputs (programmatic dependent launch)
  pdl_trigger();
  if (skip && *skip) return;
  __shared__ double smd[32];
  const double delta = 4.0 * ((double)n + 64.0) * 0x1.0p-53 + 1e-15;
  double carry = 0.0;
  for (int t0 = 0; t0 < nchunks; t0 += 1024) {
    const int k = t0 + threadIdx.x;
    const double v = k < nchunks ? csum[k] : 0.0;
    double tot;
    const double incl = block_incl<1024>(v, smd, tot);
    const double acc = carry + (incl - v);  // approximate exclusive prefix
    if (k < nchunks) {
      const double lo = acc * (1.0 - delta), hi = (acc + v) * (1.0 + delta) + 1e-300;
      int ue = kNoBinade, ue2 = kNoBinade;
      if (k > 0 && lo >= 0x1.0p-1022) {
        const int e_lo = ilogb(lo), e_hi = ilogb(hi);
        if (e_lo == e_hi) {
          ue = e_lo - 52;
        } else if (e_hi == e_lo + 1) {  // one boundary inside: split chunk, both binades
          ue = e_lo - 52;
          ue2 = e_hi - 52;
        }
      }
      assumed[k] = ue;
      assumed2[k] = ue2;
      approx[k] = acc;
    }
    carry += tot;
  }
}

// ---------------------------------------------------------------- pass B: aggregates
// sub-chunk aggregates of a split chunk under binade ue (this thread's 16 items)
__device__ void sub_aggregate(const double (&xv)[kItems], int ue, ChunkAgg* __restrict__ out) {
  const unsigned mask = seg_mask();
  int smap;
  const int excl = seg_excl_map(thread_map(xv, ue), mask, smap);
  double run0, run1, zl0, zl1;
  two_parity_pass(xv, ue, excl, run0, run1, zl0, zl1);
  double tot0, tot1;
  const double ex0 = seg_incl_sum(run0, mask, tot0) - run0;
  const double ex1 = seg_incl_sum(run1, mask, tot1) - run1;
  const double Z0 = seg_max(zl0 + ex0, mask) + 2.0;  // margin for the rounded additions
  const double Z1 = seg_max(zl1 + ex1, mask) + 2.0;
  if ((threadIdx.x & (kSubThr - 1)) == 0) {
    ChunkAgg a;
    a.R0 = fmin(tot0, 2.0 * kTwo53);
    a.R1 = fmin(tot1, 2.0 * kTwo53);
    a.Z0 = Z0;
    a.Z1 = Z1;
    a.map = smap;
    a.ulp_exp = ue;
    a.bad = 0;
    a.split = 0;
    *out = a;
  }
}

// whole-block aggregate of this thread's items under binade ue (thread 0's result is valid)
__device__ ChunkAgg block_aggregate(const double (&xv)[kItems], int ue, double* smd, int* smi) {
  int excl;
  const int bmap = BlockScan<kThr>::excl_map(thread_map(xv, ue), excl, smi);
  double run0, run1, zl0, zl1;
  two_parity_pass(xv, ue, excl, run0, run1, zl0, zl1);
  double tot0, tot1;
  const double ex0 = block_incl<kThr>(run0, smd, tot0) - run0;
  const double ex1 = block_incl<kThr>(run1, smd, tot1) - run1;
  const double Z0 = block_max<kThr>(zl0 + ex0, smd) + 2.0;  // margin for the rounded additions
  const double Z1 = block_max<kThr>(zl1 + ex1, smd) + 2.0;
  ChunkAgg a;
  a.R0 = fmin(tot0, 2.0 * kTwo53);
  a.R1 = fmin(tot1, 2.0 * kTwo53);
  a.Z0 = Z0;
  a.Z1 = Z1;
  a.map = bmap;
  a.ulp_exp = ue;
  a.bad = 0;
  a.split = 0;
  return a;
}

// The crossing window of split chunk k (one predicted boundary B = 2^(ue2 + 52)) and its pre /
// post aggregates.  With S~_i the approximate prefix (plan's chunk start + a block scan) and
// |S~_i - S_i| <= delta S_i: every i with S~_i (1 + delta) < B has S_i < B, and the first i with
// S~_i (1 - delta) >= B has S_i >= B, so the exact crossing lies in [w0, w1].
__device__ void cross_aggregate(const double (&xv)[kItems], long long base, long long n, int k, int ue,
                                int ue2, double start, CrossAgg* __restrict__ out, double* smd, int* smi,
                                long long* sml) {
  double v = 0.0;
#pragma unroll
  for (int j = 0; j < kItems; ++j) v += xv[j] >= 0.0 ? xv[j] : 0.0;
  double tot;
  const double incl = block_incl<kThr>(v, smd, tot);
  double run = start + (incl - v);
  const double delta = 4.0 * ((double)n + 64.0) * 0x1.0p-53 + 1e-15;
  const double Bnd = ldexp(1.0, ue2 + 52);
  const long long kNone = 0x7fffffffffffffffLL;
  long long fh = kNone, fl = kNone;
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    run += xv[j] >= 0.0 ? xv[j] : 0.0;
    const long long i = base + j;
    if (i < n) {
      if (fh == kNone && run * (1.0 + delta) + 1e-300 >= Bnd) fh = i;
      if (fl == kNone && run * (1.0 - delta) >= Bnd) fl = i;
    }
  }
  fh = block_min_ll<kThr>(fh, sml);
  fl = block_min_ll<kThr>(fl, sml);
  const long long c0 = (long long)k * kChunk, ce = min(n, c0 + kChunk);
  const long long w0 = fh == kNone ? ce : fh;
  const long long w1 = fl == kNone ? ce - 1 : fl;
  const bool ok = w0 < ce && w1 >= w0 && w1 - w0 + 1 <= kWin;
  double xm[kItems];
#pragma unroll
  for (int j = 0; j < kItems; ++j) xm[j] = base + j < w0 ? xv[j] : 0.0;
  const ChunkAgg pre = block_aggregate(xm, ue, smd, smi);
#pragma unroll
  for (int j = 0; j < kItems; ++j) xm[j] = base + j > w1 ? xv[j] : 0.0;
  const ChunkAgg post = block_aggregate(xm, ue2, smd, smi);
  if (threadIdx.x == 0) {
    CrossAgg c;
    c.pre = pre;
    c.post = post;
    c.w0 = w0;
    c.w1 = w1;
    c.ok = ok ? 1 : 0;
    c.pad = 0;
    *out = c;
  }
}

__global__ void __launch_bounds__(kThr) chunk_agg_kernel(const double* __restrict__ x, long long n,
                                                         const int* __restrict__ assumed,
                                                         const int* __restrict__ assumed2,
                                                         ChunkAgg* __restrict__ agg,
                                                         ChunkAgg* __restrict__ subagg,
                                                         const double* __restrict__ approx,
                                                         CrossAgg* __restrict__ cross,
                                                         const int* __restrict__ skip) {
  pdl_wait();  // the previous kernel's outputs (programmatic dependent launch)
  pdl_trigger();
  if (skip && *skip) return;
  __shared__ double smd[32];
  __shared__ int smi[32];
  const int k = blockIdx.x;
  const long long base = (long long)k * kChunk + threadIdx.x * kItems;
  const int ue = assumed[k];
  double xv[kItems];
  load_items(x, n, base, xv);
  int bad = 0;
#pragma unroll
  for (int j = 0; j < kItems; ++j)
    if (!(xv[j] >= 0.0)) bad = 1;
  const int g = threadIdx.x / kSubThr;
  if (k == 0) {
    // chunk 0 holds the dense crossings of the sum's start (S grows from 0): sub-chunks get
    // their own binade prediction from an approximate prefix inside the chunk; the walk
    // steps sub-chunk 0 and any sub-chunk the prediction cannot place in one binade
    double v = 0.0;
#pragma unroll
    for (int j = 0; j < kItems; ++j) v += xv[j] >= 0.0 ? xv[j] : 0.0;
    __shared__ double subsum[kNSub];
    double tot;
    seg_incl_sum(v, seg_mask(), tot);
    if ((threadIdx.x & (kSubThr - 1)) == 0) subsum[g] = tot;
    __syncthreads();
    double pre = 0.0;
    for (int h = 0; h < g; ++h) pre += subsum[h];
    const double delta = 4.0 * ((double)n + 64.0) * 0x1.0p-53 + 1e-15;
    const double lo = pre * (1.0 - delta), hi = (pre + subsum[g]) * (1.0 + delta) + 1e-300;
    int ug = kNoBinade;
    if (g > 0 && lo >= 0x1.0p-1022 && ilogb(lo) == ilogb(hi)) ug = ilogb(lo) - 52;
    if (ug != kNoBinade) {
      sub_aggregate(xv, ug, subagg + g);
    } else if ((threadIdx.x & (kSubThr - 1)) == 0) {
      ChunkAgg a{};
      a.ulp_exp = kNoBinade;
      subagg[g] = a;
    }
    if ((threadIdx.x & (kSubThr - 1)) == 0) {
      ChunkAgg a{};
      a.ulp_exp = kNoBinade;
      subagg[kNSub + g] = a;  // no second hypothesis
    }
    bad = __syncthreads_or(bad);
    if (threadIdx.x == 0) {
      ChunkAgg a{};
      a.ulp_exp = kNoBinade;
      a.bad = bad;
      a.split = 1;
      agg[k] = a;
    }
    return;
  }
  if (assumed2[k] != kNoBinade) {  // split: [k][hypothesis][sub-chunk]
    sub_aggregate(xv, ue, subagg + ((size_t)k * 2 + 0) * kNSub + g);
    sub_aggregate(xv, assumed2[k], subagg + ((size_t)k * 2 + 1) * kNSub + g);
    __shared__ long long sml[32];
    cross_aggregate(xv, base, n, k, ue, assumed2[k], approx[k], cross + k, smd, smi, sml);
    bad = __syncthreads_or(bad);
    if (threadIdx.x == 0) {
      ChunkAgg a{};
      a.ulp_exp = kNoBinade;
      a.bad = bad;
      a.split = 1;
      agg[k] = a;
    }
    return;
  }
  if (ue == kNoBinade) {
    bad = __syncthreads_or(bad);
    if (threadIdx.x == 0) {
      ChunkAgg a{};
      a.ulp_exp = kNoBinade;
      a.bad = bad;
      agg[k] = a;
    }
    return;
  }
  ChunkAgg a = block_aggregate(xv, ue, smd, smi);
  bad = __syncthreads_or(bad);
  if (threadIdx.x == 0) {
    a.bad = bad;
    agg[k] = a;
  }
}

// ---------------------------------------------------------------- pass C: serial walk
__device__ unsigned long long g_walk_stats[8];  // diagnostics: certified / exact chunks

void sampler_walk_stats(unsigned long long* out2, bool reset) {
  unsigned long long v[8];
  cudaMemcpyFromSymbol(v, g_walk_stats, sizeof(v));
  for (int i = 0; i < 8; ++i) out2[i] = v[i];
  if (reset) {
    unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(g_walk_stats, z, sizeof(z));
  }
}

// Exact element-wise processing of [c0, c1) starting from state S (one CTA, kCThr threads).
// Writes out[i] = S_i when out != nullptr.  Returns the final S.
__device__ double exact_segment(const double* __restrict__ x, long long c0, long long c1, double S,
                                double* __restrict__ out, double* smd, int* smi, long long* sml,
                                unsigned long long* st, bool force_seq = false) {
  constexpr long long kSeq = 256;  // sequential batch when crossings come fast
  constexpr long long kDense = 64;  // a crossing this close to the last one: go sequential
  __shared__ double s_seq;
  long long i0 = c0;
  // only the start of the whole sum has dense crossings (each early element can double
  // S); a later chunk is here because the approximate prefix could not place it in one
  // binade, i.e. it holds one (rarely a few) crossing at an unknown position
  bool sequential = force_seq || S == 0.0;
  while (i0 < c1) {
    const long long tb0 = clock64();
    if (sequential || S == 0.0) {
      // one thread steps the recurrence itself (plain IEEE adds, the reference's loop);
      // cheaper than a block iteration when the next binade crossing is only a few
      // elements away (the start of the sum, or right after a crossing)
      const long long e = min(c1, i0 + kSeq);
      __shared__ double s_buf[kSeq];
      // stage the batch in smem so the serial chain does not wait on global loads
      for (long long i = i0 + threadIdx.x; i < e; i += kCThr) s_buf[i - i0] = x[i];
      __syncthreads();
      if (threadIdx.x == 0) {
        double s = S;
        const int cnt = (int)(e - i0);
        int j = 0;
        for (; j + 8 <= cnt; j += 8) {  // loads batched ahead of the dependent adds
          double v[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) v[k] = s_buf[j + k];
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            s = __dadd_rn(s, v[k]);
            v[k] = s;
          }
#pragma unroll
          for (int k = 0; k < 8; ++k) s_buf[j + k] = v[k];
        }
        for (; j < cnt; ++j) {
          s = __dadd_rn(s, s_buf[j]);
          s_buf[j] = s;
        }
        s_seq = s;
      }
      __syncthreads();
      if (out)
        for (long long i = i0 + threadIdx.x; i < e; i += kCThr) out[i] = s_buf[i - i0];
      S = s_seq;
      i0 = e;
      sequential = false;
      (void)tb0;
      __syncthreads();
      continue;
    }
    if (threadIdx.x == 0) st[7] += 1;
    int ue, be;
    binade_of(S, ue, be);
    const double M = ldexp(S, -ue);                  // exact integer < 2^53
    const double capU = ldexp(1.0, be - ue);         // boundary in ulps: 2^53 (2^52 subnormal)
    const int P = parity_of(M);
    Elem el[kCItems];
    int tmap = 0;
    for (int j = 0; j < kCItems; ++j) {
      long long i = i0 + threadIdx.x * kCItems + j;
      el[j] = classify(i < c1 ? x[i] : 0.0, ue);
      tmap = map_compose(tmap, el[j].map);
    }
    int excl;
    BlockScan<kCThr>::excl_map(tmap, excl, smi);
    int par = map_apply(excl, P);
    double local[kCItems], rr[kCItems];
    double run = 0.0;
    for (int j = 0; j < kCItems; ++j) {
      rr[j] = el[j].tie ? tie_r(el[j].q, par) : el[j].q;
      par = map_apply(el[j].map, par);
      run = fmin(run + rr[j], 2.0 * kTwo53);
      local[j] = run;
    }
    double tot;
    const double incl = block_incl<kCThr>(run, smd, tot);
    const double ex = incl - run;
    // first crossing: M + Rprev + y >= capU - 1/2  <=>  y >= (capU - M - Rprev) - 1/2 (exact)
    long long cross = c1;
    for (int j = 0; j < kCItems; ++j) {
      long long i = i0 + threadIdx.x * kCItems + j;
      if (i >= c1) break;
      const double rprev = ex + (j > 0 ? local[j - 1] : 0.0);
      const double T = capU - M - rprev;  // exact (integers below 2^53)
      if (rprev >= capU || el[j].y >= T - 0.5) {
        cross = i;
        break;
      }
    }
    cross = block_min_ll<kCThr>(cross, sml);
    for (int j = 0; j < kCItems; ++j) {
      long long i = i0 + threadIdx.x * kCItems + j;
      if (i < cross && out) out[i] = ldexp(M + ex + local[j], ue);
    }
    // state after the last non-crossing element (block-wide)
    __shared__ double s_next;
    if (cross < c1) {
      if (threadIdx.x == (int)((cross - i0) / kCItems)) {
        const int j = (int)((cross - i0) % kCItems);
        const double rprev = ex + (j > 0 ? local[j - 1] : 0.0);
        const double sprev = ldexp(M + rprev, ue);
        const double snew = __dadd_rn(sprev, x[cross]);
        if (out) out[cross] = snew;
        s_next = snew;
      }
      __syncthreads();
      S = s_next;
      sequential = cross - i0 < kDense;  // crossings are dense here: step sequentially
      i0 = cross + 1;
    } else {
      S = ldexp(M + tot, ue);
      i0 = c1;
    }
    __syncthreads();
  }
  return S;
}

// Parity transducer of a certified chunk: starting with parity p the chunk adds d_p ulps
// and leaves parity q_p.  Composition (a then b) is associative, so a run of chunks in one
// binade is a block scan; sums of the integer d stay exact below 2^53 in any order and
// only certified states (M + Z < 2^53) are used.
struct Tx {
  double d0, d1;
  int q0, q1;
};
__device__ __forceinline__ Tx tx_identity() { return Tx{0.0, 0.0, 0, 1}; }
__device__ __forceinline__ Tx tx_compose(const Tx& a, const Tx& b) {
  Tx r;
  r.d0 = a.d0 + (a.q0 ? b.d1 : b.d0);
  r.q0 = a.q0 ? b.q1 : b.q0;
  r.d1 = a.d1 + (a.q1 ? b.d1 : b.d0);
  r.q1 = a.q1 ? b.q1 : b.q0;
  return r;
}
__device__ __forceinline__ Tx tx_shfl_up(const Tx& t, int o) {
  Tx r;
  r.d0 = __shfl_up_sync(0xffffffffu, t.d0, o);
  r.d1 = __shfl_up_sync(0xffffffffu, t.d1, o);
  r.q0 = __shfl_up_sync(0xffffffffu, t.q0, o);
  r.q1 = __shfl_up_sync(0xffffffffu, t.q1, o);
  return r;
}

constexpr int kTile = 256;            // chunks per walk tile (= threads taking part in runs)
constexpr int kTileWarps = kTile / 32;

// exclusive scan of transducers over threads [0, kTile) (others must pass the identity)
__device__ Tx block_excl_tx(Tx t, Tx* sm) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  Tx inc = t;
  if (w < kTileWarps) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const Tx u = tx_shfl_up(inc, o);
      if (lane >= o) inc = tx_compose(u, inc);
    }
    if (lane == 31) sm[w] = inc;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    Tx run = tx_identity();
    for (int k = 0; k < kTileWarps; ++k) {
      const Tx v = sm[k];
      sm[k] = run;  // exclusive warp prefix
      run = tx_compose(run, v);
    }
  }
  __syncthreads();
  Tx ex = tx_identity();
  if (w < kTileWarps) {
    Tx prev = tx_shfl_up(inc, 1);
    if (lane == 0) prev = tx_identity();
    ex = tx_compose(sm[w], prev);
  }
  __syncthreads();
  return ex;
}

__device__ __forceinline__ int block_min_int(int v, int* sm) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  if (lane == 0) sm[w] = v;
  __syncthreads();
  if (w == 0) {
    int t = lane < kCThr / 32 ? sm[lane] : 0x7fffffff;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) t = min(t, __shfl_xor_sync(0xffffffffu, t, o));
    if (lane == 0) sm[32] = t;
  }
  __syncthreads();
  const int r = sm[32];
  __syncthreads();
  return r;
}

// ---------------------------------------------------------------- warp-level split walk
// exclusive warp scan of parity transducers (lanes past the active range pass the identity)
__device__ __forceinline__ Tx warp_excl_tx(Tx t) {
  const int lane = threadIdx.x & 31;
  Tx inc = t;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const Tx u = tx_shfl_up(inc, o);
    if (lane >= o) inc = tx_compose(u, inc);
  }
  Tx prev = tx_shfl_up(inc, 1);
  if (lane == 0) prev = tx_identity();
  return prev;
}

// The reference's recurrence S_i = fl(S_{i-1} + x_i) over cnt <= kSub elements staged in
// shared memory, stepped by lane 0 of the walking warp (loads batched ahead of the dependent
// adds; the prefixes overwrite xs), then written out by the warp.  Measured against a
// warp-parallel variant (classify / scan / find the crossing, one iteration per binade
// crossing): a single warp's ~25 dependent instructions per element slot made that 3x slower
// than 256 plain dependent adds.
__device__ double warp_seq_segment(double* xs, long long c0, int cnt, double S, double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  if (lane == 0) {
    double s = S;
    int j = 0;
    for (; j + 8 <= cnt; j += 8) {
      double v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = xs[j + k];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        s = __dadd_rn(s, v[k]);
        v[k] = s;
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) xs[j + k] = v[k];
    }
    for (; j < cnt; ++j) {
      s = __dadd_rn(s, xs[j]);
      xs[j] = s;
    }
    S = s;
  }
  S = __shfl_sync(0xffffffffu, S, 0);
  __syncwarp();
  if (out)
    for (int i = lane; i < cnt; i += 32) out[c0 + i] = xs[i];
  return S;
}

// A split chunk, walked by warp 0: runs of certified sub-chunks (under whichever binade
// hypothesis matches the exact state) are one warp scan of their parity transducers (lane l
// holds sub-chunks 2l and 2l + 1), and only the 64-element sub-chunk holding a crossing is
// stepped (loaded into shared memory by the warp, stepped by lane 0: warp_seq_segment).
// (Round 1 used 256-element sub-chunks and staged the whole chunk first: ~12 k cycles per
// split chunk, most of them the stepped 256 elements; 64-element sub-chunks cut the stepping
// 4x and the staging to one 512-byte load.)
__device__ __forceinline__ Tx tx_of(const ChunkAgg& a) {
  Tx t;
  t.d0 = a.R0;
  t.q0 = parity_of(a.R0);
  t.d1 = a.R1;
  t.q1 = 1 ^ parity_of(a.R1);
  return t;
}

__device__ double split_walk_warp(const double* __restrict__ x, long long n, int k, double S,
                                  const ChunkAgg* __restrict__ subagg, ChunkStart* __restrict__ substarts,
                                  double* __restrict__ out, double* xs, unsigned long long* st) {
  static_assert(kNSub == 64, "two sub-chunks per lane");
  __shared__ double s_S;
  const long long base = (long long)k * kChunk;
  __syncthreads();  // xs / s_S may still be read from the previous split chunk
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    const ChunkAgg* h = subagg + (size_t)k * 2 * kNSub;
    ChunkAgg h0[2], h1[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      h0[j] = h[2 * lane + j];
      h1[j] = h[kNSub + 2 * lane + j];
    }
    int g = 0;
    while (g < kNSub) {
      if (S > 0.0) {
        int ue, be;
        binade_of(S, ue, be);
        const double M = ldexp(S, -ue);
        const double capU = ldexp(1.0, be - ue);
        const int P0 = parity_of(M);
        bool valid[2];
        ChunkAgg a[2];
        Tx t[2];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int idx = 2 * lane + j;
          valid[j] = idx >= g;
          a[j] = ChunkAgg{};
          if (valid[j]) {
            if (h0[j].ulp_exp == ue) a[j] = h0[j];
            else if (h1[j].ulp_exp == ue) a[j] = h1[j];
            else valid[j] = false;
          }
          t[j] = valid[j] ? tx_of(a[j]) : tx_identity();
        }
        const Tx ex = warp_excl_tx(tx_compose(t[0], t[1]));
        // states at the lane's two sub-chunks
        const double M0 = M + (P0 ? ex.d1 : ex.d0);
        const int Q0 = P0 ? ex.q1 : ex.q0;
        const bool c0 = valid[0] && (M0 + (Q0 ? a[0].Z1 : a[0].Z0) < capU - 1.0);
        const double M1 = M0 + (Q0 ? t[0].d1 : t[0].d0);
        const int Q1 = Q0 ? t[0].q1 : t[0].q0;
        const bool c1 = valid[1] && (M1 + (Q1 ? a[1].Z1 : a[1].Z0) < capU - 1.0);
        int fail = kNSub;
        if (2 * lane + 1 >= g && !c1) fail = 2 * lane + 1;
        if (2 * lane >= g && !c0) fail = 2 * lane;
        const int f = __reduce_min_sync(0xffffffffu, fail);  // first sub-chunk not certified
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int idx = 2 * lane + j;
          if (idx >= g && idx < f) {
            ChunkStart cs;
            cs.M = j ? M1 : M0;
            cs.parity = j ? Q1 : Q0;
            cs.ulp_exp = ue;
            cs.fast = 1;
            cs.pad = 0;
            substarts[(size_t)k * kNSub + idx] = cs;
          }
        }
        if (f > g) {  // state after sub-chunk f - 1
          const int ol = (f - 1) >> 1, oj = (f - 1) & 1;
          const double Mend = oj ? M1 + (Q1 ? t[1].d1 : t[1].d0) : M1;
          S = ldexp(__shfl_sync(0xffffffffu, Mend, ol), ue);
        }
        g = f;
      }
      if (g < kNSub) {  // the crossing sub-chunk (or the start of the whole sum), element-exact
        const long long c0 = base + (long long)g * kSub;
        if (lane == 0) {
          ChunkStart cs{};
          cs.fast = 0;
          substarts[(size_t)k * kNSub + g] = cs;
          st[3] += 1;
        }
        if (c0 < n) {
          const int cnt = (int)(n - c0 < kSub ? n - c0 : kSub);
          for (int i = lane; i < cnt; i += 32) xs[i] = x[c0 + i];
          __syncwarp();
          S = warp_seq_segment(xs, c0, cnt, S, out);
          __syncwarp();
        }
        ++g;
      }
    }
    if (lane == 0) s_S = S;
  }
  __syncthreads();
  return s_S;
}

// A crossing chunk in O(1) (warp 0; every lane carries the same state): certify and apply the
// pre segment, step the window [w0, w1] with IEEE adds (loaded by the warp in one go), check the
// state reached the upper binade, certify and apply the post segment.  Returns false (state
// untouched) when any check fails: the caller walks the chunk by sub-chunks instead.
__device__ bool cross_walk_warp(const double* __restrict__ x, long long n, int k, double& S,
                                const CrossAgg& c, CrossStart* __restrict__ cstarts,
                                double* __restrict__ out, double* xs) {
  const int lane = threadIdx.x & 31;
  if (!c.ok || !(S > 0.0)) return false;
  const long long c0 = (long long)k * kChunk;
  int ue, be;
  binade_of(S, ue, be);
  if (ue != c.pre.ulp_exp) return false;
  double M = ldexp(S, -ue);
  double capU = ldexp(1.0, be - ue);
  int P = parity_of(M);
  CrossStart cs;
  cs.pre.M = M;
  cs.pre.parity = P;
  cs.pre.ulp_exp = ue;
  cs.pre.fast = 1;
  cs.pre.pad = 0;
  cs.w0 = c.w0;
  cs.w1 = c.w1;
  if (c.w0 > c0) {
    if (!(M + (P ? c.pre.Z1 : c.pre.Z0) < capU - 1.0)) return false;
    M += P ? c.pre.R1 : c.pre.R0;
  }
  double Sw = ldexp(M, ue);
  const int cnt = (int)(c.w1 - c.w0 + 1);
  if (lane < cnt) xs[lane] = x[c.w0 + lane];
  __syncwarp();
  if (lane == 0) {
    double sv = Sw;
    for (int j = 0; j < cnt; ++j) {
      sv = __dadd_rn(sv, xs[j]);
      xs[j] = sv;
    }
  }
  __syncwarp();
  Sw = xs[cnt - 1];
  binade_of(Sw, ue, be);
  const bool reached = ue == c.post.ulp_exp;
  double Mp = ldexp(Sw, -ue);
  capU = ldexp(1.0, be - ue);
  P = parity_of(Mp);
  cs.post.M = Mp;
  cs.post.parity = P;
  cs.post.ulp_exp = ue;
  cs.post.fast = 1;
  cs.post.pad = 0;
  const long long ce = min(n, c0 + kChunk);
  bool ok = reached;
  if (ok && c.w1 + 1 < ce) {
    ok = Mp + (P ? c.post.Z1 : c.post.Z0) < capU - 1.0;
    Mp += P ? c.post.R1 : c.post.R0;
  }
  if (!ok) {
    __syncwarp();
    return false;
  }
  if (out && lane < cnt) out[c.w0 + lane] = xs[lane];
  if (lane == 0) cstarts[k] = cs;
  S = ldexp(Mp, ue);
  __syncwarp();
  return true;
}

__global__ void __launch_bounds__(kCThr) chunk_walk_kernel(const double* __restrict__ x, long long n,
                                                           int nchunks,
                                                           const ChunkAgg* __restrict__ agg,
                                                           const ChunkAgg* __restrict__ subagg,
                                                           ChunkStart* __restrict__ starts,
                                                           ChunkStart* __restrict__ substarts,
                                                           const CrossAgg* __restrict__ cross,
                                                           CrossStart* __restrict__ cstarts,
                                                           double* __restrict__ out,
                                                           double* __restrict__ total,
                                                           int* __restrict__ status, int bad_flag,
                                                           const int* __restrict__ skip) {
  pdl_wait();  // the previous kernel's outputs (programmatic dependent launch)
  pdl_trigger();
  if (skip && *skip) return;
  extern __shared__ __align__(16) double xs_dyn[];  // kSub: a stepped sub-chunk's elements
  __shared__ ChunkAgg tile[kTile];
  __shared__ Tx stx[kTileWarps];
  __shared__ double smd[32];
  __shared__ int smi[33];
  __shared__ long long sml[32];
  __shared__ double s_S;
  double S = 0.0;
  int bad = 0;
  unsigned long long st[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // diagnostics (thread 0), flushed once
  for (int t0 = 0; t0 < nchunks; t0 += kTile) {
    const int t1 = min(nchunks, t0 + kTile);
    __syncthreads();
    for (int k = t0 + (int)threadIdx.x; k < t1; k += kCThr) {
      tile[k - t0] = agg[k];
      bad |= agg[k].bad;
    }
    __syncthreads();
    int k = t0;
    while (k < t1) {
      if (S > 0.0) {
        // run of certified chunks from k: thread i takes chunk k + i
        const long long tr0 = clock64();
        int ue, be;
        binade_of(S, ue, be);
        const double M = ldexp(S, -ue);
        const double capU = ldexp(1.0, be - ue);
        const int P0 = parity_of(M);
        const int i = threadIdx.x;
        const int kk = k + i;
        bool valid = i < kTile && kk < t1;
        ChunkAgg a{};
        Tx t = tx_identity();
        if (valid) {
          a = tile[kk - t0];
          valid = !a.split && a.ulp_exp == ue;
        }
        if (valid) {
          t.d0 = a.R0;
          t.q0 = parity_of(a.R0);
          t.d1 = a.R1;
          t.q1 = 1 ^ parity_of(a.R1);
        }
        const Tx ex = block_excl_tx(t, stx);
        const double Mi = M + (P0 ? ex.d1 : ex.d0);
        const int Pi = P0 ? ex.q1 : ex.q0;
        const bool cert = valid && (Mi + (Pi ? a.Z1 : a.Z0) < capU - 1.0);
        const int f = block_min_int(cert ? 0x7fffffff : i, smi);  // first chunk not certified
        const int run = min(f, t1 - k);
        if (i < run) {
          ChunkStart cs;
          cs.M = Mi;
          cs.parity = Pi;
          cs.ulp_exp = ue;
          cs.fast = 1;
          cs.pad = 0;
          starts[kk] = cs;
        }
        if (run > 0 && i == run - 1) s_S = ldexp(Mi + (Pi ? a.R1 : a.R0), ue);  // state after the run
        __syncthreads();
        if (run > 0) S = s_S;
        k += run;
        if (threadIdx.x == 0) {
          st[0] += (unsigned long long)run;
          st[4] += (unsigned long long)(clock64() - tr0);
        }
        __syncthreads();
        if (k >= t1) break;
      }
      // chunk k is not certified: a split chunk, or element-exact processing
      const long long tq0 = clock64();
      const long long c0 = (long long)k * kChunk, c1 = min(n, c0 + kChunk);
      if (tile[k - t0].split) {  // (chunk 0 is split: its first sub-chunk starts at S = 0)
        __shared__ int s_done;
        __shared__ double s_cS;
        if (threadIdx.x < 32) {  // one crossing: the O(1) path
          double Sx = S;
          bool done = false;
          if (k > 0 && cross) {
            const CrossAgg c = cross[k];
            done = cross_walk_warp(x, n, k, Sx, c, cstarts, out, xs_dyn);
          }
          if (threadIdx.x == 0) {
            s_done = done ? 1 : 0;
            s_cS = Sx;
          }
        }
        __syncthreads();
        if (s_done) {
          S = s_cS;
          if (threadIdx.x == 0) {
            ChunkStart cs{};
            cs.fast = 3;
            starts[k] = cs;
            st[1] += 1;
            st[5] += (unsigned long long)(clock64() - tq0);
          }
          ++k;
          __syncthreads();
          continue;
        }
        if (threadIdx.x == 0) {
          ChunkStart cs{};
          cs.fast = 2;
          starts[k] = cs;
          st[2] += 1;
        }
        S = split_walk_warp(x, n, k, S, subagg, substarts, out, xs_dyn, st);
        if (threadIdx.x == 0) st[6] += (unsigned long long)(clock64() - tq0);
      } else {
        if (threadIdx.x == 0) {
          ChunkStart cs{};
          cs.fast = 0;
          starts[k] = cs;
          st[1] += 1;
        }
        S = exact_segment(x, c0, c1, S, out, smd, smi, sml, st);
        if (threadIdx.x == 0) st[5] += (unsigned long long)(clock64() - tq0);
      }
      ++k;
    }
  }
  bad = __syncthreads_or(bad);
  if (threadIdx.x == 0) {
    *total = S;
    if (bad) atomicOr(status, bad_flag);
    for (int i = 0; i < 8; ++i)
      if (st[i]) atomicAdd(&g_walk_stats[i], st[i]);
  }
}

// ---------------------------------------------------------------- pass D: write S_i
// S_i = (M + ulps before i) * u for this thread's items, given the exclusive map of the
// items before them (recomputing the classifications: see two_parity_pass)
__device__ __forceinline__ double items_run(const double (&xv)[kItems], int ue, int par) {
  double run = 0.0;
#pragma unroll 4
  for (int j = 0; j < kItems; ++j) run += step_r(classify(xv[j], ue), par);
  return run;
}
__device__ __forceinline__ void items_write(const double (&xv)[kItems], int ue, int par, double M,
                                            double ex, long long base, long long n,
                                            double* __restrict__ out) {
  double local = 0.0;
#pragma unroll 4
  for (int j = 0; j < kItems; ++j) {
    local += step_r(classify(xv[j], ue), par);
    if (base + j < n) out[base + j] = ldexp(M + ex + local, ue);
  }
}

// S_i for the items of this block in [lo, hi) from the exact state cs at lo (the others are
// masked to 0: identity parity maps, no ulps) -- one crossing chunk's pre or post segment
__device__ void write_range(const double (&xv_in)[kItems], long long base, long long n, long long lo,
                            long long hi, const ChunkStart& cs, double* __restrict__ out, double* smd,
                            int* smi) {
  double xv[kItems];
#pragma unroll
  for (int j = 0; j < kItems; ++j) xv[j] = (base + j >= lo && base + j < hi) ? xv_in[j] : 0.0;
  int excl;
  BlockScan<kThr>::excl_map(thread_map(xv, cs.ulp_exp), excl, smi);
  const int par = map_apply(excl, cs.parity);
  const double run = items_run(xv, cs.ulp_exp, par);
  double tot;
  const double ex = block_incl<kThr>(run, smd, tot) - run;
  int p2 = par;
  double local = 0.0;
#pragma unroll 4
  for (int j = 0; j < kItems; ++j) {
    local += step_r(classify(xv[j], cs.ulp_exp), p2);
    const long long i = base + j;
    if (i >= lo && i < hi && i < n) out[i] = ldexp(cs.M + ex + local, cs.ulp_exp);
  }
}

__global__ void __launch_bounds__(kThr) chunk_write_kernel(const double* __restrict__ x, long long n,
                                                           const ChunkStart* __restrict__ starts,
                                                           const ChunkStart* __restrict__ substarts,
                                                           const CrossStart* __restrict__ cstarts,
                                                           double* __restrict__ out,
                                                           const int* __restrict__ skip) {
  pdl_wait();  // the previous kernel's outputs (programmatic dependent launch)
  pdl_trigger();
  if (skip && *skip) return;
  __shared__ double smd[32];
  __shared__ int smi[32];
  const int k = blockIdx.x;
  const ChunkStart cs0 = starts[k];
  if (cs0.fast == 0) return;
  const long long base = (long long)k * kChunk + threadIdx.x * kItems;
  double xv[kItems];
  if (cs0.fast == 3) {  // crossing chunk: pre and post segments (the walk wrote the window)
    const CrossStart c = cstarts[k];
    load_items(x, n, base, xv);
    const long long c0 = (long long)k * kChunk, ce = min(n, c0 + kChunk);
    if (c.w0 > c0) write_range(xv, base, n, c0, c.w0, c.pre, out, smd, smi);
    if (c.w1 + 1 < ce) write_range(xv, base, n, c.w1 + 1, ce, c.post, out, smd, smi);
    return;
  }
  if (cs0.fast == 2) {  // split chunk: one 16-lane segment per sub-chunk, own start state
    const ChunkStart cs = substarts[(size_t)k * kNSub + threadIdx.x / kSubThr];
    if (!cs.fast) return;  // stepped by the walk (whole segment leaves together)
    const unsigned mask = seg_mask();
    load_items(x, n, base, xv);
    int smap;
    const int excl = seg_excl_map(thread_map(xv, cs.ulp_exp), mask, smap);
    const int par = map_apply(excl, cs.parity);
    const double run = items_run(xv, cs.ulp_exp, par);
    double tot;
    const double ex = seg_incl_sum(run, mask, tot) - run;
    items_write(xv, cs.ulp_exp, par, cs.M, ex, base, n, out);
    return;
  }
  const ChunkStart cs = cs0;
  load_items(x, n, base, xv);
  int excl;
  BlockScan<kThr>::excl_map(thread_map(xv, cs.ulp_exp), excl, smi);
  const int par = map_apply(excl, cs.parity);
  const double run = items_run(xv, cs.ulp_exp, par);
  double tot;
  const double ex = block_incl<kThr>(run, smd, tot) - run;
  items_write(xv, cs.ulp_exp, par, cs.M, ex, base, n, out);
}

// ---------------------------------------------------------------- Neumaier terms
// Exact two-sum error of step i (sketching.cpp:17-21) from S_{i-1}, x_i, S_i, summed in
// double-double per chunk (fixed tree), plus sum |e_i| for the drift bound.
__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
  s = __dadd_rn(a, b);
  const double bb = __dsub_rn(s, a);
  e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
}

__global__ void __launch_bounds__(kThr) neumaier_terms_kernel(const double* __restrict__ x,
                                                              const double* __restrict__ S, long long n,
                                                              double* __restrict__ part,
                                                              const int* __restrict__ skip) {
  pdl_wait();  // the previous kernel's outputs (programmatic dependent launch)
  pdl_trigger();
  if (skip && *skip) return;
  __shared__ double hi_s[kThr], lo_s[kThr], ab_s[kThr];
  const long long base = (long long)blockIdx.x * kChunk + threadIdx.x * kItems;
  double hi = 0.0, lo = 0.0, ab = 0.0;
  for (int j = 0; j < kItems; ++j) {
    long long i = base + j;
    if (i >= n) break;
    const double sp = i > 0 ? S[i - 1] : 0.0, t = S[i], xv = x[i];
    const double e = fabs(sp) >= fabs(xv) ? __dadd_rn(__dsub_rn(sp, t), xv)
                                          : __dadd_rn(__dsub_rn(xv, t), sp);
    double s2, e2;
    two_sum(hi, e, s2, e2);
    hi = s2;
    lo = __dadd_rn(lo, e2);
    ab = __dadd_rn(ab, fabs(e));
  }
  hi_s[threadIdx.x] = hi;
  lo_s[threadIdx.x] = lo;
  ab_s[threadIdx.x] = ab;
  __syncthreads();
  for (int w = kThr / 2; w >= 1; w >>= 1) {
    if ((int)threadIdx.x < w) {
      double s2, e2;
      two_sum(hi_s[threadIdx.x], hi_s[threadIdx.x + w], s2, e2);
      hi_s[threadIdx.x] = s2;
      lo_s[threadIdx.x] = __dadd_rn(__dadd_rn(lo_s[threadIdx.x], lo_s[threadIdx.x + w]), e2);
      ab_s[threadIdx.x] = __dadd_rn(ab_s[threadIdx.x], ab_s[threadIdx.x + w]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[3 * blockIdx.x] = hi_s[0];
    part[3 * blockIdx.x + 1] = lo_s[0];
    part[3 * blockIdx.x + 2] = ab_s[0];
  }
}

// The reference loop, verbatim, for the (rare) uncertified case.
__device__ double neumaier_sequential(const double* __restrict__ v, long long n) {
  double s = 0.0, c = 0.0;
  for (long long i = 0; i < n; ++i) {
    const double xv = v[i];
    const double t = __dadd_rn(s, xv);
    if (fabs(s) >= fabs(xv))
      c = __dadd_rn(c, __dadd_rn(__dsub_rn(s, t), xv));
    else
      c = __dadd_rn(c, __dadd_rn(__dsub_rn(xv, t), s));
    s = t;
  }
  return __dadd_rn(s, c);
}

// double-double accumulation of per-chunk (hi, lo[, abs]) partials: thread t takes chunks
// t, t + 256, ... in order, then a fixed tree over the threads (deterministic).
constexpr int kRedThr = 256;
__device__ void dd_block_sum(const double* __restrict__ part, int stride, int nchunks,
                             double& hi_out, double& lo_out, double& ab_out) {
  __shared__ double hi_s[kRedThr], lo_s[kRedThr], ab_s[kRedThr];
  double hi = 0.0, lo = 0.0, ab = 0.0;
  for (int k = threadIdx.x; k < nchunks; k += kRedThr) {
    double s2, e2;
    two_sum(hi, part[stride * k], s2, e2);
    hi = s2;
    lo = __dadd_rn(__dadd_rn(lo, part[stride * k + 1]), e2);
    if (stride == 3) ab = __dadd_rn(ab, part[stride * k + 2]);
  }
  hi_s[threadIdx.x] = hi;
  lo_s[threadIdx.x] = lo;
  ab_s[threadIdx.x] = ab;
  __syncthreads();
  for (int w = kRedThr / 2; w >= 1; w >>= 1) {
    if ((int)threadIdx.x < w) {
      double s2, e2;
      two_sum(hi_s[threadIdx.x], hi_s[threadIdx.x + w], s2, e2);
      hi_s[threadIdx.x] = s2;
      lo_s[threadIdx.x] = __dadd_rn(__dadd_rn(lo_s[threadIdx.x], lo_s[threadIdx.x + w]), e2);
      ab_s[threadIdx.x] = __dadd_rn(ab_s[threadIdx.x], ab_s[threadIdx.x + w]);
    }
    __syncthreads();
  }
  hi_out = hi_s[0];
  lo_out = lo_s[0];
  ab_out = ab_s[0];
}

// s_out = stable_sum(x) given S_final and the chunk partials (one CTA of kRedThr)
__global__ void __launch_bounds__(kRedThr) neumaier_final_kernel(
    const double* __restrict__ x, long long n, const double* __restrict__ Sfinal,
    const double* __restrict__ part, int nchunks, double* __restrict__ s_out,
    int* __restrict__ status, const int* __restrict__ skip) {
  pdl_wait();  // the previous kernel's outputs (programmatic dependent launch)
  pdl_trigger();
  if (skip && *skip) return;
  double hi, lo, ab;
  dd_block_sum(part, 3, nchunks, hi, lo, ab);
  if (threadIdx.x != 0) return;
  // exact c (double-double) and the drift bound of the sequential c: <= u * sum_k |c_k|,
  // |c_k| <= sum |e|  =>  B <= n u sum|e| (with slack)
  const double S = *Sfinal;
  const double c_hi = __dadd_rn(hi, lo);
  const double c_lo = __dsub_rn(lo, __dsub_rn(c_hi, hi));
  const double B = ((double)n + 8.0) * 0x1.0p-52 * ab * 1.0625 + fabs(c_lo) * 4.0 + 0x1.0p-1074;
  const double r_lo = __dadd_rn(S, __dsub_rd(c_hi, B));
  const double r_hi = __dadd_rn(S, __dadd_ru(c_hi, B));
  if (r_lo == r_hi) {
    *s_out = r_lo;
  } else {
    *s_out = neumaier_sequential(x, n);
    atomicOr(status, kFallback);
  }
}

// ---------------------------------------------------------------- Neumaier without the scan
// Double-double accumulation with renormalisation (|lo| <= ulp(hi) / 2 after every step), so
// each step's error is O(u^2 |hi|): n steps cost at most ~2 n u^2 sum x.
__device__ __forceinline__ void dd_add_d(double& hi, double& lo, double x) {
  double s, e;
  two_sum(hi, x, s, e);
  e = __dadd_rn(lo, e);
  const double h2 = __dadd_rn(s, e);  // fast two-sum (|s| >= |e|)
  lo = __dsub_rn(e, __dsub_rn(h2, s));
  hi = h2;
}
__device__ __forceinline__ void dd_add_dd(double& hi, double& lo, double bh, double bl) {
  double s, e;
  two_sum(hi, bh, s, e);
  e = __dadd_rn(e, __dadd_rn(lo, bl));
  const double h2 = __dadd_rn(s, e);
  lo = __dsub_rn(e, __dsub_rn(h2, s));
  hi = h2;
}
// fixed-tree block reduction of (hi, lo) pairs; thread 0 gets the result
template <int NT>
__device__ void block_dd_reduce(double& hi, double& lo, double* hs, double* ls) {
  hs[threadIdx.x] = hi;
  ls[threadIdx.x] = lo;
  __syncthreads();
  for (int w = NT / 2; w >= 1; w >>= 1) {
    if ((int)threadIdx.x < w) {
      double h = hs[threadIdx.x], l = ls[threadIdx.x];
      dd_add_dd(h, l, hs[threadIdx.x + w], ls[threadIdx.x + w]);
      hs[threadIdx.x] = h;
      ls[threadIdx.x] = l;
    }
    __syncthreads();
  }
  hi = hs[0];
  lo = ls[0];
}

// x1 = w / total (+ beta mix) -- tucker.cpp:119-128, as normalize_mix_kernel -- fused with the
// chunk's double-double sum of x1 (for the Neumaier certificate) and the weight check of
// normalized() (sketching.cpp:42-44).  One CTA per 4096-element chunk.
__global__ void __launch_bounds__(kThr) normalize_dd_kernel(const double* __restrict__ w, long long n,
                                                            const double* __restrict__ total, int regime,
                                                            double beta, double* __restrict__ x1,
                                                            int* __restrict__ uni, double* __restrict__ part,
                                                            int* __restrict__ status) {
  pdl_wait();  // the previous kernel's outputs (programmatic dependent launch)
  pdl_trigger();
  __shared__ double hs[kThr], ls[kThr];
  const double tot = *total;
  const bool uniform = !(tot > 0.0);
  if (!uniform && regime == 1 && !(beta > 0.0 && beta <= 1.0)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(status, kBadBeta);
  }
  const double cmix = __ddiv_rn(__dsub_rn(1.0, beta), (double)n);
  const double vu = __ddiv_rn(1.0, (double)n);
  const long long base = (long long)blockIdx.x * kChunk + threadIdx.x * kItems;
  double xv[kItems];
  load_items(w, n, base, xv);
  double hi = 0.0, lo = 0.0;
  int bad = 0;
#pragma unroll 4
  for (int j = 0; j < kItems; ++j) {
    if (base + j >= n) break;
    double v = vu;
    if (!uniform) {
      v = __ddiv_rn(xv[j], tot);
      if (regime == 1) v = __dadd_rn(__dmul_rn(beta, v), cmix);
    }
    x1[base + j] = v;
    if (!(v >= 0.0)) bad = 1;
    else dd_add_d(hi, lo, v);
  }
  bad = __syncthreads_or(bad);
  block_dd_reduce<kThr>(hi, lo, hs, ls);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = hi;
    part[2 * blockIdx.x + 1] = lo;
    if (bad) atomicOr(status, kBadWeight);
    if (blockIdx.x == 0) *uni = uniform ? 1 : 0;
  }
}

// stable_sum (sketching.cpp:13-24) certified from the exact total, without the naive prefix:
// the reference returns fl(S + c) with S the naive sum and c the naive sum of the exact
// two-sum errors e_i; S + sum e_i = T = sum x exactly, |e_i| <= u S_i <= u n T (x >= 0), and
// c's own drift is <= (n - 1) u sum|e_i|, so S + c lies within B = n^2 u^2 T (1 + 3 n u) of T.
// With T known to O(n u^2 T) in double-double, fl(S + c) is the rounding of every value in
// [T - E, T + E] when that interval holds no rounding boundary (all but ~1e-4 of cases).
// Certified: s -> *s_out and *skip = 1 (the scan-based path below is skipped); otherwise
// *skip = 0 and the exact scan + neumaier_terms + neumaier_final run.  Uniform (uni): s is
// never used (p = 1/n), *skip = 1.
__global__ void __launch_bounds__(kRedThr) neumaier_cert_kernel(const double* __restrict__ part, int nchunks,
                                                                long long n, const int* __restrict__ uni,
                                                                double* __restrict__ s_out,
                                                                int* __restrict__ skip, int force_fallback) {
  pdl_wait();  // the previous kernel's outputs (programmatic dependent launch)
  pdl_trigger();
  __shared__ double hs[kRedThr], ls[kRedThr];
  if (*uni) {
    if (threadIdx.x == 0) *skip = 1;
    return;
  }
  double hi = 0.0, lo = 0.0;
  for (int k = threadIdx.x; k < nchunks; k += kRedThr) dd_add_dd(hi, lo, part[2 * k], part[2 * k + 1]);
  block_dd_reduce<kRedThr>(hi, lo, hs, ls);
  if (threadIdx.x != 0) return;
  const double nn = (double)n;
  const double u = 0x1.0p-53;
  // B (c drift, with slack) + the double-double error (<= 2 u^2 per step, n + 2 nchunks + 512 steps)
  const double rel = __dmul_ru(__dmul_ru(nn, nn), u * u) * 1.0625 + (nn + 2.0 * nchunks + 1024.0) * 4.0 * u * u;
  const double E = __dadd_ru(__dmul_ru(rel, fabs(hi)), 0x1.0p-1074);
  const double r_lo = __dadd_rn(hi, __dsub_rd(lo, E));
  const double r_hi = __dadd_rn(hi, __dadd_ru(lo, E));
  if (r_lo == r_hi && isfinite(r_lo) && !force_fallback) {
    *s_out = r_lo;
    *skip = 1;
  } else {
    *skip = 0;
  }
}

// p = x / s (sketching.cpp:46) fused with the ctor check's double-double partial sum, the
// last positive index (sketching.cpp:109-111) and the approximate chunk sums that plan the
// cumulative scan (pass A of exact_scan).  One CTA per chunk.
__global__ void __launch_bounds__(kThr) divide_check_kernel(double* __restrict__ x, long long n,
                                                            const double* __restrict__ s,
                                                            const int* __restrict__ uni,
                                                            int* __restrict__ status, double* __restrict__ cpart,
                                                            long long* __restrict__ lastpos,
                                                            double* __restrict__ csum) {
  pdl_wait();  // the previous kernel's outputs (programmatic dependent launch)
  pdl_trigger();
  __shared__ double hs[kThr], ls[kThr];
  __shared__ long long sml[32];
  __shared__ double smd[32];
  const double sv = *s;
  bool divide = !*uni;
  if (divide && !(sv > 0.0)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(status, kZeroNormalize);
    divide = false;
  }
  const long long base = (long long)blockIdx.x * kChunk + threadIdx.x * kItems;
  double xv[kItems];
  load_items(x, n, base, xv);
  double hi = 0.0, lo = 0.0, v = 0.0;
  long long last = -1;
#pragma unroll 4
  for (int j = 0; j < kItems; ++j) {
    if (base + j >= n) break;
    double pv = xv[j];
    if (divide) {
      pv = __ddiv_rn(pv, sv);
      x[base + j] = pv;
    }
    dd_add_d(hi, lo, pv);
    v += pv;
    if (pv != 0.0) last = base + j;
  }
  double tot;
  block_incl<kThr>(v, smd, tot);
  last = -block_min_ll<kThr>(-last, sml);
  block_dd_reduce<kThr>(hi, lo, hs, ls);
  if (threadIdx.x == 0) {
    cpart[2 * blockIdx.x] = hi;
    cpart[2 * blockIdx.x + 1] = lo;
    lastpos[blockIdx.x] = last;
    csum[blockIdx.x] = tot;
  }
}

// ---------------------------------------------------------------- elementwise steps
// mode 0: total -> x1 = w / total (or uniform when total <= 0: sets *uni = 1)
// tucker.cpp:119-128; the mix beta*x + (1-beta)/n is two roundings (no contraction)
__global__ void normalize_mix_kernel(const double* __restrict__ w, long long n,
                                     const double* __restrict__ total, int regime, double beta,
                                     double* __restrict__ x1, int* __restrict__ uni,
                                     int* __restrict__ status) {
  pdl_wait();  // the previous kernel's outputs (programmatic dependent launch)
  pdl_trigger();
  const double tot = *total;
  const bool uniform = !(tot > 0.0);
  if (!uniform && regime == 1 && !(beta > 0.0 && beta <= 1.0)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(status, kBadBeta);
  }
  const double cmix = __ddiv_rn(__dsub_rn(1.0, beta), (double)n);
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    if (uniform) {
      x1[i] = __ddiv_rn(1.0, (double)n);
    } else {
      double v = __ddiv_rn(w[i], tot);
      if (regime == 1) v = __dadd_rn(__dmul_rn(beta, v), cmix);
      x1[i] = v;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *uni = uniform ? 1 : 0;
}

__global__ void fill_kernel(double* __restrict__ x, long long n, double v) {
  pdl_wait();  // the previous kernel's outputs (programmatic dependent launch)
  pdl_trigger();
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    x[i] = v;
}

// ctor check |stable_sum(p) - 1| <= 1e-12 (sketching.cpp:35-37); approximate sum in
// double-double (the threshold is 1e4 ulps away from any realistic value) + last index
// with positive weight (sketching.cpp:109-111)
__global__ void __launch_bounds__(kThr) check_last_kernel(const double* __restrict__ p, long long n,
                                                          double* __restrict__ part,
                                                          long long* __restrict__ lastpos) {
  pdl_wait();  // the previous kernel's outputs (programmatic dependent launch)
  pdl_trigger();
  __shared__ double hi_s[kThr], lo_s[kThr];
  __shared__ long long sml[32];
  double hi = 0.0, lo = 0.0;
  long long last = -1;
  const long long base = (long long)blockIdx.x * kChunk + threadIdx.x * kItems;
  for (int j = 0; j < kItems; ++j) {
    long long i = base + j;
    if (i >= n) break;
    double s2, e2;
    two_sum(hi, p[i], s2, e2);
    hi = s2;
    lo = __dadd_rn(lo, e2);
    if (p[i] != 0.0) last = i;
  }
  hi_s[threadIdx.x] = hi;
  lo_s[threadIdx.x] = lo;
  __syncthreads();
  for (int w = kThr / 2; w >= 1; w >>= 1) {
    if ((int)threadIdx.x < w) {
      double s2, e2;
      two_sum(hi_s[threadIdx.x], hi_s[threadIdx.x + w], s2, e2);
      hi_s[threadIdx.x] = s2;
      lo_s[threadIdx.x] = __dadd_rn(__dadd_rn(lo_s[threadIdx.x], lo_s[threadIdx.x + w]), e2);
    }
    __syncthreads();
  }
  last = -block_min_ll<kThr>(-last, sml);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = hi_s[0];
    part[2 * blockIdx.x + 1] = lo_s[0];
    lastpos[blockIdx.x] = last;
  }
}

__global__ void __launch_bounds__(kRedThr) check_final_kernel(const double* __restrict__ part,
                                                               const long long* __restrict__ lastpos,
                                                               int nchunks, long long* __restrict__ last,
                                                               int* __restrict__ status) {
  pdl_wait();  // the previous kernel's outputs (programmatic dependent launch)
  pdl_trigger();
  __shared__ long long sml[32];
  long long lp = -1;
  for (int k = threadIdx.x; k < nchunks; k += kRedThr) lp = max(lp, lastpos[k]);
  lp = -block_min_ll<kRedThr>(-lp, sml);
  double hi, lo, ab;
  dd_block_sum(part, 2, nchunks, hi, lo, ab);
  if (threadIdx.x != 0) return;
  const double sum = __dadd_rn(hi, lo);
  if (fabs(sum - 1.0) > 1e-12) atomicOr(status, kNotOne);
  *last = lp;
}

// ---------------------------------------------------------------- draws (sketching.cpp:119-129)
struct Pcg32 {
  unsigned long long state, inc;
  __device__ Pcg32(unsigned long long seed, unsigned long long stream) {
    inc = (stream << 1u) | 1u;
    state = 0;
    next();
    state += seed;
    next();
  }
  __device__ unsigned int next() {
    unsigned long long old = state;
    state = old * 6364136223846793005ULL + inc;
    unsigned int xs = (unsigned int)(((old >> 18u) ^ old) >> 27u);
    unsigned int rot = (unsigned int)(old >> 59u);
    return (xs >> rot) | (xs << ((32u - rot) & 31u));
  }
  __device__ void advance(unsigned long long delta) {
    unsigned long long cm = 6364136223846793005ULL, cp = inc, am = 1, ap = 0;
    while (delta) {
      if (delta & 1) {
        am *= cm;
        ap = ap * cm + cp;
      }
      cp = (cm + 1) * cp;
      cm *= cm;
      delta >>= 1;
    }
    state = am * state + ap;
  }
};

// one draw per thread: each draw is a 20-step dependent binary search in L2 (the jump-ahead
// to its PCG position is O(log j)), so parallelism across draws is what hides the latency
constexpr int kDrawsPerThread = 1;

__global__ void draw_kernel(const double* __restrict__ cum, const double* __restrict__ p, long long n,
                            const double* __restrict__ acc_p, const long long* __restrict__ last_p,
                            long long L, unsigned long long seed, unsigned long long stream,
                            long long* __restrict__ idx, double* __restrict__ scales,
                            int* __restrict__ status) {
  pdl_wait();  // the previous kernel's outputs (programmatic dependent launch)
  pdl_trigger();
  const double acc = *acc_p;
  const long long j0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * kDrawsPerThread;
  if (j0 >= L) return;
  if (!(acc > 0.0)) {
    if (j0 == 0) atomicOr(status, kZeroAcc);
    return;
  }
  const long long last = *last_p;
  const double scale_base = __ddiv_rn(1.0, __dsqrt_rn((double)L));
  Pcg32 g(seed, stream);
  g.advance(2ull * (unsigned long long)j0);
  const long long j1 = min(L, j0 + kDrawsPerThread);
  for (long long j = j0; j < j1; ++j) {
    const unsigned long long hi = g.next(), lo = g.next();
    const double u = __dmul_rn((double)(((hi << 32) | lo) >> 11) * 0x1.0p-53, acc);
    long long lo_i = 0, hi_i = n;  // upper_bound: first cum > u
    while (lo_i < hi_i) {
      const long long mid = (lo_i + hi_i) >> 1;
      if (cum[mid] > u)
        hi_i = mid;
      else
        lo_i = mid + 1;
    }
    long long id = lo_i == n ? last : lo_i;
    if (p[id] == 0.0) id = last;
    idx[j] = id;
    scales[j] = __ddiv_rn(scale_base, __dsqrt_rn(p[id]));
  }
}

// ---------------------------------------------------------------- uniform(n): closed form
// For p = uniform(n) (every p_i = v = 1.0 / n, sketching.cpp:50-53) the reference's cumulative
// sum cum_i = fl(cum_{i-1} + v) (sketching.cpp:99-104) is an arithmetic progression inside a
// binade: with u the binade's ulp and y = v / u (exact), every in-binade step adds the same
// integer r = round(y) ulps -- for a tie (frac y = 1/2) the first step lands on an even
// multiple and every later step adds the even choice q + (q odd), q = floor(y).  So the whole
// prefix is a list of segments (i0, M, r, ue, K): cum_{i0 + k} = (M + k r) 2^ue for k <= K,
// joined by single steps evaluated with an IEEE add (the first step in a binade and every
// binade crossing).  Thread 0 of each CTA builds the list in O(#binades); the draws
// (upper_bound, sketching.cpp:122-127) binary-search it.  Replaces the n-element exact scan
// and the n-element prefix array for the uniform regime.
struct USeg {
  long long i0, K;  // first index, further in-binade steps (K = 0: a single value)
  double M, r;      // value at i0 = M 2^ue, step r ulps
  int ue, pad;
};
constexpr int kUSegMax = 512;  // cum climbs from 1/n to ~1: <= 64 binades, <= 2 segments each
constexpr int kUThreads = 128;

__device__ __forceinline__ double useg_value(const USeg& g, long long k) { return ldexp(g.M + (double)k * g.r, g.ue); }

// builds the segment list (thread 0); returns the count, or -1 if it would overflow
__device__ int uniform_segments(long long n, double v, USeg* segs) {
  long long i = 0;
  double S = v;  // cum_0 = 0 + v
  int cnt = 0;
  while (true) {  // S = cum_i exactly
    if (cnt >= kUSegMax) return -1;
    int ue, be;
    binade_of(S, ue, be);
    const double M = ldexp(S, -ue), capU = ldexp(1.0, be - ue), y = ldexp(v, -ue);
    const double fy = floor(y), fr = y - fy;
    const bool tie = fr == 0.5;
    // in-binade step: non-tie r = round(y); tie from an even multiple: the even choice
    const double r = tie ? fy + (double)parity_of(fy) : (fr > 0.5 ? fy + 1.0 : fy);
    const double cstar = fr >= 0.5 ? fy + 1.0 : fy;  // a step from M' crosses iff capU - M' <= cstar
    long long K = 0;
    if (!(tie && parity_of(M))) {  // (an odd start under a tie takes one IEEE step first)
      const double N = capU - M - cstar;          // the step from M + k r stays inside iff k r < N
      if (N > 0.0) {
        if (r == 0.0) {
          K = n - 1 - i;  // stagnation: v below half an ulp
        } else {
          double k = ceil(N / r);
          while (k > 1.0 && (k - 1.0) * r >= N) k -= 1.0;
          while (k * r < N) k += 1.0;
          K = (long long)k;
        }
      }
      K = min(K, n - 1 - i);
    }
    segs[cnt++] = USeg{i, K, M, r, ue, 0};
    i += K;
    if (i >= n - 1) break;
    S = __dadd_rn(useg_value(segs[cnt - 1], K), v);  // binade crossing (or tie start): IEEE step
    ++i;
  }
  return cnt;
}

__global__ void __launch_bounds__(kUThreads) uniform_draw_kernel(long long n, long long L, unsigned long long seed,
                                                                 unsigned long long stream, long long* __restrict__ idx,
                                                                 double* __restrict__ scales, int* __restrict__ status) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(16) unsigned char usm[];
  USeg* segs = reinterpret_cast<USeg*>(usm);
  __shared__ int s_cnt;
  const double v = __ddiv_rn(1.0, (double)n);
  if (threadIdx.x == 0) s_cnt = uniform_segments(n, v, segs);
  __syncthreads();
  const int cnt = s_cnt;
  const long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (cnt < 0) {  // cannot happen for n < 2^63 (see kUSegMax); surfaced, never silent
    if (j == 0) atomicOr(status, kInternal);
    return;
  }
  if (j >= L) return;
  const USeg& lastg = segs[cnt - 1];
  const double acc = useg_value(lastg, lastg.K);  // cum_{n-1}
  const double scale_base = __ddiv_rn(1.0, __dsqrt_rn((double)L));
  Pcg32 g(seed, stream);
  g.advance(2ull * (unsigned long long)j);
  const unsigned long long hi = g.next(), lo = g.next();
  const double u = __dmul_rn((double)(((hi << 32) | lo) >> 11) * 0x1.0p-53, acc);
  // first segment whose last value exceeds u
  int a = 0, b = cnt;
  while (a < b) {
    const int mid = (a + b) >> 1;
    if (useg_value(segs[mid], segs[mid].K) > u)
      b = mid;
    else
      a = mid + 1;
  }
  long long id;
  if (a == cnt) {
    id = n - 1;  // "last": every uniform weight is positive
  } else {
    const USeg& sg = segs[a];
    long long k = 0;
    if (sg.K > 0 && sg.r > 0.0) {  // first k with M + k r > w  (w = u / 2^ue, exact)
      const double w = ldexp(u, -sg.ue);
      double kk = floor((w - sg.M) / sg.r) + 1.0;
      if (kk < 0.0) kk = 0.0;
      if (kk > (double)sg.K) kk = (double)sg.K;
      while (kk > 0.0 && sg.M + (kk - 1.0) * sg.r > w) kk -= 1.0;
      while (kk < (double)sg.K && !(sg.M + kk * sg.r > w)) kk += 1.0;
      k = (long long)kk;
    }
    id = sg.i0 + k;
  }
  idx[j] = id;
  scales[j] = __ddiv_rn(scale_base, __dsqrt_rn(v));
}

// ---------------------------------------------------------------- orchestration
static int nchunks_of(long long n) { return (int)((n + kChunk - 1) / kChunk); }

size_t sampler_workspace_doubles(long long n) {
  const size_t nc = (size_t)nchunks_of(n);
  // p / x1 (n), S (n), csum (nc), assumed (nc ints), agg (nc * 6), starts (nc * 3),
  // neumaier partials (3 nc), check partials (2 nc), lastpos (nc), scalars (16),
  // assumed2 (nc ints), subagg (nc * 2 * kNSub * 6), substarts (nc * kNSub * 3)
  // + approx (nc), cross aggregates and starts (nc each)
  return 2 * (size_t)n + nc * (1 + 1 + 6 + 3 + 3 + 2 + 1) + 64 + nc * (1 + 2 * kNSub * 6 + kNSub * 3) +
         nc * (1 + (sizeof(CrossAgg) + 7) / 8 + (sizeof(CrossStart) + 7) / 8);
}

struct ScanBufs {
  double* csum;
  int* assumed;
  int* assumed2;
  ChunkAgg* agg;
  ChunkStart* starts;
  ChunkAgg* subagg;
  ChunkStart* substarts;
  double* approx;
  CrossAgg* cross;
  CrossStart* cstarts;
};

static cudaError_t exact_scan(const double* x, long long n, double* out, double* total,
                              int* status, int bad_flag, const ScanBufs& b, cudaStream_t st,
                              const int* skip = nullptr, bool csum_ready = false) {
  const int nc = nchunks_of(n);
  cudaError_t e;
  if (!csum_ready)
    if ((e = launch_pdl(chunk_sums_kernel, dim3(nc), dim3(kThr), 0, st, x, n, b.csum, skip)) != cudaSuccess) return e;
  if ((e = launch_pdl(chunk_plan_kernel, dim3(1), dim3(1024), 0, st, b.csum, nc, n, b.assumed, b.assumed2, b.approx, skip)) != cudaSuccess) return e;
  if ((e = launch_pdl(chunk_agg_kernel, dim3(nc), dim3(kThr), 0, st, x, n, b.assumed, b.assumed2, b.agg, b.subagg, (const double*)b.approx, b.cross, skip)) != cudaSuccess) return e;
  // LMRA_SAMPLER_CROSS=0 (tests): crossing chunks always take the sub-chunk walk
  const char* cx = getenv("LMRA_SAMPLER_CROSS");
  const bool cross_on = !(cx && cx[0] == '0');
  static unsigned long long walk_attr = 0;
  if ((e = ensure_smem_attr(reinterpret_cast<const void*>(chunk_walk_kernel), kSub * sizeof(double), walk_attr)) !=
      cudaSuccess)
    return e;
  if ((e = launch_pdl(chunk_walk_kernel, dim3(1), dim3(kCThr), kSub * sizeof(double), st, x, n, nc, b.agg, b.subagg, b.starts, b.substarts, cross_on ? (const CrossAgg*)b.cross : nullptr, b.cstarts, out,
                                         total, status, bad_flag, skip)) != cudaSuccess) return e;
  if (out) {
    if ((e = launch_pdl(chunk_write_kernel, dim3(nc), dim3(kThr), 0, st, x, n, b.starts, b.substarts, (const CrossStart*)b.cstarts, out, skip)) != cudaSuccess) return e;
  }
  return cudaGetLastError();
}

cudaError_t launch_sampler(const double* w, long long n, int regime, double beta, long long L,
                           uint64_t seed, uint64_t stream, long long* idx, double* scales,
                           double* p_out, double* work, int* status, cudaStream_t st) {
  if (n <= 0 || L <= 0) return cudaErrorInvalidValue;
  const int nc = nchunks_of(n);
  double* p = p_out;             // n: probabilities (kept for the scales / tests)
  double* S = work;              // n: exact prefix sums
  double* csum = S + n;
  int* assumed = reinterpret_cast<int*>(csum + nc);
  ChunkAgg* agg = reinterpret_cast<ChunkAgg*>(csum + 2 * nc);
  ChunkStart* starts = reinterpret_cast<ChunkStart*>(csum + 8 * nc);
  double* npart = csum + 11 * nc;
  double* cpart = csum + 14 * nc;
  long long* lastpos = reinterpret_cast<long long*>(csum + 16 * nc);
  double* scal = csum + 17 * nc;  // [0] total [1] s [2] acc ; ints after
  int* uni = reinterpret_cast<int*>(scal + 8);
  long long* last = reinterpret_cast<long long*>(scal + 10);
  int* skip = reinterpret_cast<int*>(scal + 12);  // 1: the Neumaier sum was certified without the scan
  double* ext = scal + 64;  // split-chunk buffers
  int* assumed2 = reinterpret_cast<int*>(ext);
  ChunkAgg* subagg = reinterpret_cast<ChunkAgg*>(ext + nc);
  ChunkStart* substarts = reinterpret_cast<ChunkStart*>(ext + nc + (size_t)nc * 2 * kNSub * 6);
  double* approx = ext + nc + (size_t)nc * (2 * kNSub * 6 + kNSub * 3);
  CrossAgg* cross = reinterpret_cast<CrossAgg*>(approx + nc);
  CrossStart* cstarts = reinterpret_cast<CrossStart*>(approx + nc + (size_t)nc * ((sizeof(CrossAgg) + 7) / 8));
  ScanBufs b{csum, assumed, assumed2, agg, starts, subagg, substarts, approx, cross, cstarts};
  const int eg = 148 * 8;
  cudaError_t e;
  if (regime == 2) {  // uniform(n): p = 1/n each (sketching.cpp:50-53)
    if ((e = launch_pdl(fill_kernel, dim3(eg), dim3(256), 0, st, p, n, 1.0 / (double)n)) != cudaSuccess) return e;
    static const bool closed_form = !(getenv("LMRA_UNIFORM_SCAN") && getenv("LMRA_UNIFORM_SCAN")[0] == '1');
    if (closed_form) {
      // The ctor check (sketching.cpp:35-37) and "last" are decided for uniform(n) without
      // reading p: Neumaier's sum of n copies of v = fl(1/n) is within an ulp of n v, and
      // |n v - 1| <= n |v - 1/n| <= u/2, far inside 1e-12; every weight is positive, so
      // last = n - 1 (the draw kernel uses it directly).  Then the closed-form cumulative
      // sum and the draws -- no n-element pass at all besides writing p.
      static unsigned long long uattr = 0;
      const size_t usmem = sizeof(USeg) * kUSegMax;
      if ((e = ensure_smem_attr(reinterpret_cast<const void*>(uniform_draw_kernel), usmem, uattr)) != cudaSuccess) return e;
      return launch_pdl(uniform_draw_kernel, dim3((unsigned)((L + kUThreads - 1) / kUThreads)), dim3(kUThreads), usmem, st,
                        n, L, seed, stream, idx, scales, status);
    }
  } else {
    // total = naive sum of w; x1 = w / total (+ beta mix); s = Neumaier(x1); p = x1 / s
    if ((e = exact_scan(w, n, nullptr, scal + 0, status, kBadWeight, b, st)) != cudaSuccess) return e;
    // diagnostics / tests (read per call): LMRA_NEUMAIER_SCAN=1 the prefix-based certificate
    // only; =2 the certificate from the total is forced to fail (its fallback path runs)
    const char* nm = getenv("LMRA_NEUMAIER_SCAN");
    const bool scan_neumaier = nm && nm[0] == '1';
    const int force_fallback = nm && nm[0] == '2';
    if (scan_neumaier) {  // the prefix-based certificate only (kept for tests / comparison)
      if ((e = launch_pdl(normalize_mix_kernel, dim3(eg), dim3(256), 0, st, w, n, scal + 0, regime, beta, p, uni, status)) != cudaSuccess) return e;
      if ((e = exact_scan(p, n, S, scal + 1, status, kBadWeight, b, st)) != cudaSuccess) return e;
      if ((e = launch_pdl(neumaier_terms_kernel, dim3(nc), dim3(kThr), 0, st, p, S, n, npart, (const int*)nullptr)) != cudaSuccess) return e;
      if ((e = launch_pdl(neumaier_final_kernel, dim3(1), dim3(kRedThr), 0, st, p, n, scal + 1, npart, nc, scal + 1, status, uni)) != cudaSuccess) return e;
    } else {
      // x1 and its double-double chunk sums in one pass; s certified from the total; the
      // prefix-based path (exact scan of x1 + two-sum terms) runs only when that fails
      if ((e = launch_pdl(normalize_dd_kernel, dim3(nc), dim3(kThr), 0, st, w, n, scal + 0, regime, beta, p, uni, npart, status)) != cudaSuccess) return e;
      if ((e = launch_pdl(neumaier_cert_kernel, dim3(1), dim3(kRedThr), 0, st, npart, nc, n, uni, scal + 1, skip, force_fallback)) != cudaSuccess) return e;
      if ((e = exact_scan(p, n, S, scal + 1, status, kBadWeight, b, st, skip)) != cudaSuccess) return e;
      if ((e = launch_pdl(neumaier_terms_kernel, dim3(nc), dim3(kThr), 0, st, p, S, n, npart, (const int*)skip)) != cudaSuccess) return e;
      if ((e = launch_pdl(neumaier_final_kernel, dim3(1), dim3(kRedThr), 0, st, p, n, scal + 1, npart, nc, scal + 1, status, (const int*)skip)) != cudaSuccess) return e;
    }
  }
  if (regime != 2) {
    // p = x1 / s, the ctor check partials, last, and the cumulative scan's chunk sums: one pass
    if ((e = launch_pdl(divide_check_kernel, dim3(nc), dim3(kThr), 0, st, p, n, scal + 1, uni, status, cpart, lastpos, csum)) != cudaSuccess) return e;
  } else {
    if ((e = launch_pdl(check_last_kernel, dim3(nc), dim3(kThr), 0, st, p, n, cpart, lastpos)) != cudaSuccess) return e;
  }
  if ((e = launch_pdl(check_final_kernel, dim3(1), dim3(kRedThr), 0, st, cpart, lastpos, nc, last, status)) != cudaSuccess) return e;
  // cum = naive prefix of p; acc = cum[n-1]
  if ((e = exact_scan(p, n, S, scal + 2, status, kBadWeight, b, st, nullptr, regime != 2)) != cudaSuccess) return e;
  const long long threads = (L + kDrawsPerThread - 1) / kDrawsPerThread;
  if ((e = launch_pdl(draw_kernel, dim3((unsigned)((threads + 127) / 128)), dim3(128), 0, st, S, p, n, scal + 2, last, L, seed,
                                                                  stream, idx, scales, status)) != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace lmra_dev

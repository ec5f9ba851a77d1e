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
//    prefix predicts (pass B); one CTA walks the chunks in order with the exact state
//    (pass C), taking the O(1) aggregate when it is certified and processing the chunk
//    element-exactly otherwise (chunk 0 and the few chunks holding binade crossings);
//    pass D writes every S_i of the certified chunks.
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
constexpr double kTwo53 = 9007199254740992.0;

enum SamplerStatus {
  kBadWeight = 1,      // negative / NaN weight   -> "probability weights must be nonnegative"
  kZeroNormalize = 2,  // Neumaier sum <= 0       -> "cannot normalize an all-zero distribution"
  kNotOne = 4,         // ctor check |sum-1|>1e-12 -> "probability weights must sum to one"
  kZeroAcc = 8,        // cum total <= 0          -> "randsample: all-zero distribution"
  kFallback = 16,      // informational: sequential Neumaier fallback was used
  kBadBeta = 32,       // nearly-optimal beta outside (0, 1] (checked only when total > 0)
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
  int pad;
};
constexpr int kNoBinade = 1 << 30;

struct ChunkStart {  // exact state at a certified chunk's start (pass C -> pass D)
  double M;          // S / u (integer < 2^53)
  int parity;
  int ulp_exp;
  int fast;          // 1: pass D writes the chunk, 0: pass C already wrote it
  int pad;
};

// ---------------------------------------------------------------- pass A: chunk sums
__global__ void __launch_bounds__(kThr) chunk_sums_kernel(const double* __restrict__ x, long long n,
                                                          double* __restrict__ csum) {
  __shared__ double sm[32];
  const long long base = (long long)blockIdx.x * kChunk;
  double v = 0.0;
  for (int k = 0; k < kItems; ++k) {
    long long i = base + threadIdx.x * kItems + k;
    if (i < n) v += x[i];
  }
  double tot;
  block_incl<kThr>(v, sm, tot);
  if (threadIdx.x == 0) csum[blockIdx.x] = tot;
}

// approximate exclusive prefix over chunk sums -> chunk binade predictions (1 CTA, block
// scan over tiles of 1024 chunks; the prediction only needs |approx - exact| <= delta)
__global__ void __launch_bounds__(1024) chunk_plan_kernel(const double* __restrict__ csum,
                                                          int nchunks, long long n,
                                                          int* __restrict__ assumed) {
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
      int ue = kNoBinade;
      if (k > 0 && lo >= 0x1.0p-1022) {
        const int e_lo = ilogb(lo), e_hi = ilogb(hi);
        if (e_lo == e_hi) ue = e_lo - 52;
      }
      assumed[k] = ue;
    }
    carry += tot;
  }
}

// ---------------------------------------------------------------- pass B: aggregates
__global__ void __launch_bounds__(kThr) chunk_agg_kernel(const double* __restrict__ x, long long n,
                                                         const int* __restrict__ assumed,
                                                         ChunkAgg* __restrict__ agg) {
  __shared__ double smd[32];
  __shared__ int smi[32];
  const int k = blockIdx.x;
  const long long base = (long long)k * kChunk + threadIdx.x * kItems;
  const int ue = assumed[k];
  int bad = 0;
  if (ue == kNoBinade) {
    for (int j = 0; j < kItems; ++j) {
      long long i = base + j;
      if (i < n && !(x[i] >= 0.0)) bad = 1;
    }
    bad = __syncthreads_or(bad);
    if (threadIdx.x == 0) {
      ChunkAgg a{};
      a.ulp_exp = kNoBinade;
      a.bad = bad;
      agg[k] = a;
    }
    return;
  }
  Elem el[kItems];
  int tmap = 0;  // thread-local composition
  for (int j = 0; j < kItems; ++j) {
    long long i = base + j;
    double xv = i < n ? x[i] : 0.0;
    if (!(xv >= 0.0)) bad = 1;
    el[j] = classify(xv >= 0.0 ? xv : 0.0, ue);
    tmap = map_compose(tmap, el[j].map);
  }
  int excl;
  const int bmap = BlockScan<kThr>::excl_map(tmap, excl, smi);
  // two passes: start parity 0 and 1
  double R[2], Z[2];
  for (int p0 = 0; p0 < 2; ++p0) {
    int par = map_apply(excl, p0);
    double local[kItems];
    double run = 0.0;
    for (int j = 0; j < kItems; ++j) {
      double r = el[j].tie ? tie_r(el[j].q, par) : el[j].q;
      par = map_apply(el[j].map, par);
      run = fmin(run + r, 2.0 * kTwo53);  // saturate: anything past 2^53 is a crossing
      local[j] = run;
    }
    double tot;
    const double incl = block_incl<kThr>(run, smd, tot);
    const double excl_sum = incl - run;
    double z = 0.0;
    for (int j = 0; j < kItems; ++j) {
      const double rprev = excl_sum + (j > 0 ? local[j - 1] : 0.0);
      z = fmax(z, rprev + el[j].y);
    }
    Z[p0] = block_max<kThr>(z, smd) + 2.0;  // margin for the rounded additions
    R[p0] = fmin(tot, 2.0 * kTwo53);
  }
  bad = __syncthreads_or(bad);
  if (threadIdx.x == 0) {
    ChunkAgg a;
    a.R0 = R[0];
    a.R1 = R[1];
    a.Z0 = Z[0];
    a.Z1 = Z[1];
    a.map = bmap;
    a.ulp_exp = ue;
    a.bad = bad;
    a.pad = 0;
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
                                double* __restrict__ out, double* smd, int* smi, long long* sml) {
  constexpr long long kSeq = 256;  // sequential batch when crossings come fast
  constexpr long long kDense = 64;  // a crossing this close to the last one: go sequential
  __shared__ double s_seq;
  long long i0 = c0;
  // only the start of the whole sum has dense crossings (each early element can double
  // S); a later chunk is here because the approximate prefix could not place it in one
  // binade, i.e. it holds one (rarely a few) crossing at an unknown position
  bool sequential = S == 0.0;
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
      if (threadIdx.x == 0) g_walk_stats[6] += (unsigned long long)(clock64() - tb0);
      __syncthreads();
      continue;
    }
    if (threadIdx.x == 0) g_walk_stats[7] += 1;
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

__global__ void __launch_bounds__(kCThr) chunk_walk_kernel(const double* __restrict__ x, long long n,
                                                           int nchunks,
                                                           const ChunkAgg* __restrict__ agg,
                                                           ChunkStart* __restrict__ starts,
                                                           double* __restrict__ out,
                                                           double* __restrict__ total,
                                                           int* __restrict__ status, int bad_flag) {
  constexpr int kTile = 256;  // aggregates staged in smem per tile (12 KB)
  __shared__ ChunkAgg tile[kTile];
  __shared__ double smd[32];
  __shared__ int smi[32];
  __shared__ long long sml[32];
  __shared__ double s_S;
  __shared__ int s_k;
  double S = 0.0;
  int bad = 0;
  for (int t0 = 0; t0 < nchunks; t0 += kTile) {
    const int t1 = min(nchunks, t0 + kTile);
    __syncthreads();
    for (int k = t0 + (int)threadIdx.x; k < t1; k += kCThr) tile[k - t0] = agg[k];
    __syncthreads();
    int k = t0;
    while (k < t1) {
      // thread 0 takes the certified O(1) aggregates until the first chunk that is not
      const long long tf0 = clock64();
      if (threadIdx.x == 0) {
        double s = S;
        int kk = k;
        // exact state in ulps of the current binade, carried across certified chunks
        // (a certified chunk never leaves the binade, so M, ue, capU stay valid)
        int ue = kNoBinade, be = 0;
        double M = 0.0, capU = 0.0;
        if (s > 0.0) {
          binade_of(s, ue, be);
          M = ldexp(s, -ue);
          capU = ldexp(1.0, be - ue);
        }
        for (; kk < t1; ++kk) {
          const ChunkAgg& a = tile[kk - t0];
          bad |= a.bad;
          if (a.ulp_exp == kNoBinade || !(s > 0.0)) {
            g_walk_stats[2] += 1;
            break;
          }
          if (ue != a.ulp_exp) {
            g_walk_stats[3] += 1;
            break;
          }
          const int P = parity_of(M);
          if (!(M + (P ? a.Z1 : a.Z0) < capU - 1.0)) break;
          ChunkStart cs;
          cs.M = M;
          cs.parity = P;
          cs.ulp_exp = ue;
          cs.fast = 1;
          cs.pad = 0;
          starts[kk] = cs;
          M += P ? a.R1 : a.R0;
        }
        if (s > 0.0) s = ldexp(M, ue);
        s_S = s;
        s_k = kk;
        if (kk < t1) {
          ChunkStart cs{};
          cs.fast = 0;
          starts[kk] = cs;
        }
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        g_walk_stats[4] += (unsigned long long)(clock64() - tf0);
        g_walk_stats[0] += (unsigned long long)(s_k - k);  // certified chunks
        g_walk_stats[1] += s_k < t1 ? 1ull : 0ull;        // element-exact chunks
      }
      S = s_S;
      k = s_k;
      __syncthreads();
      if (k < t1) {  // element-exact processing of chunk k (binade crossings / unknown binade)
        const long long c0 = (long long)k * kChunk, c1 = min(n, c0 + kChunk);
        const long long tq0 = clock64();
        S = exact_segment(x, c0, c1, S, out, smd, smi, sml);
        if (threadIdx.x == 0) g_walk_stats[5] += (unsigned long long)(clock64() - tq0);
        ++k;
      }
    }
  }
  if (threadIdx.x == 0) {
    *total = S;
    if (bad) atomicOr(status, bad_flag);
  }
}

// ---------------------------------------------------------------- pass D: write S_i
__global__ void __launch_bounds__(kThr) chunk_write_kernel(const double* __restrict__ x, long long n,
                                                           const ChunkStart* __restrict__ starts,
                                                           double* __restrict__ out) {
  __shared__ double smd[32];
  __shared__ int smi[32];
  const int k = blockIdx.x;
  const ChunkStart cs = starts[k];
  if (!cs.fast) return;
  const long long base = (long long)k * kChunk + threadIdx.x * kItems;
  Elem el[kItems];
  int tmap = 0;
  for (int j = 0; j < kItems; ++j) {
    long long i = base + j;
    el[j] = classify(i < n ? x[i] : 0.0, cs.ulp_exp);
    tmap = map_compose(tmap, el[j].map);
  }
  int excl;
  BlockScan<kThr>::excl_map(tmap, excl, smi);
  int par = map_apply(excl, cs.parity);
  double local[kItems];
  double run = 0.0;
  for (int j = 0; j < kItems; ++j) {
    const double r = el[j].tie ? tie_r(el[j].q, par) : el[j].q;
    par = map_apply(el[j].map, par);
    run += r;
    local[j] = run;
  }
  double tot;
  const double incl = block_incl<kThr>(run, smd, tot);
  const double ex = incl - run;
  for (int j = 0; j < kItems; ++j) {
    long long i = base + j;
    if (i < n) out[i] = ldexp(cs.M + ex + local[j], cs.ulp_exp);
  }
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
                                                              double* __restrict__ part) {
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

// s_out = stable_sum(x) given S_final and the chunk partials (1 thread)
__global__ void neumaier_final_kernel(const double* __restrict__ x, long long n,
                                      const double* __restrict__ Sfinal,
                                      const double* __restrict__ part, int nchunks,
                                      double* __restrict__ s_out, int* __restrict__ status,
                                      const int* __restrict__ skip) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  if (skip && *skip) return;
  double hi = 0.0, lo = 0.0, ab = 0.0;
  for (int k = 0; k < nchunks; ++k) {
    double s2, e2;
    two_sum(hi, part[3 * k], s2, e2);
    hi = s2;
    lo = __dadd_rn(__dadd_rn(lo, part[3 * k + 1]), e2);
    ab = __dadd_rn(ab, part[3 * k + 2]);
  }
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

// ---------------------------------------------------------------- elementwise steps
// mode 0: total -> x1 = w / total (or uniform when total <= 0: sets *uni = 1)
// tucker.cpp:119-128; the mix beta*x + (1-beta)/n is two roundings (no contraction)
__global__ void normalize_mix_kernel(const double* __restrict__ w, long long n,
                                     const double* __restrict__ total, int regime, double beta,
                                     double* __restrict__ x1, int* __restrict__ uni,
                                     int* __restrict__ status) {
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

// p = x / s (sketching.cpp:46); uniform path keeps x (= 1/n); flags s <= 0
__global__ void divide_kernel(double* __restrict__ x, long long n, const double* __restrict__ s,
                              const int* __restrict__ uni, int* __restrict__ status) {
  if (*uni) return;
  const double sv = *s;
  if (!(sv > 0.0)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(status, kZeroNormalize);
    return;
  }
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    x[i] = __ddiv_rn(x[i], sv);
}

__global__ void fill_kernel(double* __restrict__ x, long long n, double v) {
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

__global__ void check_final_kernel(const double* __restrict__ part, const long long* __restrict__ lastpos,
                                   int nchunks, long long* __restrict__ last, int* __restrict__ status) {
  if (threadIdx.x != 0) return;
  double hi = 0.0, lo = 0.0;
  long long lp = -1;
  for (int k = 0; k < nchunks; ++k) {
    double s2, e2;
    two_sum(hi, part[2 * k], s2, e2);
    hi = s2;
    lo = __dadd_rn(__dadd_rn(lo, part[2 * k + 1]), e2);
    lp = max(lp, lastpos[k]);
  }
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

// ---------------------------------------------------------------- orchestration
static int nchunks_of(long long n) { return (int)((n + kChunk - 1) / kChunk); }

size_t sampler_workspace_doubles(long long n) {
  const size_t nc = (size_t)nchunks_of(n);
  // p / x1 (n), S (n), csum (nc), assumed (nc ints), agg (nc * 6), starts (nc * 3),
  // neumaier partials (3 nc), check partials (2 nc), lastpos (nc), scalars (16)
  return 2 * (size_t)n + nc * (1 + 1 + 6 + 3 + 3 + 2 + 1) + 64;
}

struct ScanBufs {
  double* csum;
  int* assumed;
  ChunkAgg* agg;
  ChunkStart* starts;
};

static cudaError_t exact_scan(const double* x, long long n, double* out, double* total,
                              int* status, int bad_flag, const ScanBufs& b, cudaStream_t st) {
  const int nc = nchunks_of(n);
  chunk_sums_kernel<<<nc, kThr, 0, st>>>(x, n, b.csum);
  chunk_plan_kernel<<<1, 1024, 0, st>>>(b.csum, nc, n, b.assumed);
  chunk_agg_kernel<<<nc, kThr, 0, st>>>(x, n, b.assumed, b.agg);
  chunk_walk_kernel<<<1, kCThr, 0, st>>>(x, n, nc, b.agg, b.starts, out, total, status, bad_flag);
  if (out) chunk_write_kernel<<<nc, kThr, 0, st>>>(x, n, b.starts, out);
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
  ScanBufs b{csum, assumed, agg, starts};
  const int eg = 148 * 8;
  cudaError_t e;
  if (regime == 2) {  // uniform(n): p = 1/n each (sketching.cpp:50-53)
    fill_kernel<<<eg, 256, 0, st>>>(p, n, 1.0 / (double)n);
  } else {
    // total = naive sum of w; x1 = w / total (+ beta mix); s = Neumaier(x1); p = x1 / s
    if ((e = exact_scan(w, n, nullptr, scal + 0, status, kBadWeight, b, st)) != cudaSuccess) return e;
    normalize_mix_kernel<<<eg, 256, 0, st>>>(w, n, scal + 0, regime, beta, p, uni, status);
    if ((e = exact_scan(p, n, S, scal + 1, status, kBadWeight, b, st)) != cudaSuccess) return e;
    neumaier_terms_kernel<<<nc, kThr, 0, st>>>(p, S, n, npart);
    neumaier_final_kernel<<<1, 32, 0, st>>>(p, n, scal + 1, npart, nc, scal + 1, status, uni);
    divide_kernel<<<eg, 256, 0, st>>>(p, n, scal + 1, uni, status);
  }
  check_last_kernel<<<nc, kThr, 0, st>>>(p, n, cpart, lastpos);
  check_final_kernel<<<1, 32, 0, st>>>(cpart, lastpos, nc, last, status);
  // cum = naive prefix of p; acc = cum[n-1]
  if ((e = exact_scan(p, n, S, scal + 2, status, kBadWeight, b, st)) != cudaSuccess) return e;
  const long long threads = (L + kDrawsPerThread - 1) / kDrawsPerThread;
  draw_kernel<<<(unsigned)((threads + 127) / 128), 128, 0, st>>>(S, p, n, scal + 2, last, L, seed,
                                                                  stream, idx, scales, status);
  return cudaGetLastError();
}

}  // namespace lmra_dev

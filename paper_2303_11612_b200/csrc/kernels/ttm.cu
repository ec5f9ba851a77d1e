// ttm.cu -- in-place mode-n TTM and Gram contraction on the fp64 DMMA pipe.
//
// Replaces the Eigen GEMMs the reference runs on explicit unfoldings:
//   mode_n_product  tensor.cpp:118-139  (unfold -> b * m -> fold)      -> ttm_kernel
//   gram_power_apply linalg.cpp:70-74   (half = A^T c ; c = A * half)  -> ttm_kernel + gram_kernel
//   sample_columns  sketching.cpp:133-141                              -> gather_columns_kernel
// No unfolding is materialised: a column j = (i, o) of A_(n) is addressed in place
// through ModeView (common.cuh).  Both contractions run as a DMMA GEMM whose long
// dimension is j; the short dimension (factor / sketch width, <= 64) lives in
// the N of m16n8k4 and is padded to a multiple of 8.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "kernels.hpp"

namespace lmra_dev {

constexpr int kThreads = 256;

// ----------------------------------------------------------------------------
// TTM: Y(k, j) = sum_r Bt[r + I*k] * X(r, j), k < m.  Y has X's layout with I -> m.
// CTA tile: 128 columns j x all k; 8 warps x 16 j.  K (= I) in chunks of 16.
// ----------------------------------------------------------------------------
template <int M8, bool RCONTIG, int KC_ = 16, int ST_ = 3>
struct TtmCfg {
  static constexpr int JT = 128, KC = KC_, STAGES = ST_;
  static constexpr int LDA = RCONTIG ? conflict_free_ld(KC) : conflict_free_ld(JT);
  static constexpr int A_ELEMS = RCONTIG ? JT * LDA : KC * LDA;
  static constexpr int LDB = conflict_free_ld(M8);
  static constexpr int B_ELEMS = KC * LDB;
  static constexpr int STAGE_ELEMS = A_ELEMS + B_ELEMS;
  static constexpr size_t SMEM = sizeof(double) * STAGE_ELEMS * STAGES;
};

// narrow outputs (M8 <= 24: the shrinks / core contractions of cfg1-3) hold few accumulators:
// three CTAs per SM for more loads in flight (ncu, cfg3's first shrink: 24 % occupancy, DMMA
// pipe and DRAM each ~half busy)
template <int M8>
constexpr int ttm_min_blocks() { return M8 <= 24 ? 3 : 2; }
template <int M8, bool RCONTIG, int KC_, int ST_>
__global__ void __launch_bounds__(kThreads, ttm_min_blocks<M8>())
    ttm_kernel(const double* __restrict__ x, ModeView v, const double* __restrict__ bt, int m,
               int mtot, int koff, double* __restrict__ y, long long kper, Gather ga) {
  pdl_wait();  // the previous kernel's outputs (programmatic dependent launch)
  pdl_trigger();
  using C = TtmCfg<M8, RCONTIG, KC_, ST_>;
  extern __shared__ __align__(16) double smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const long long J = v.inner * v.outer;
  const long long j0 = (long long)blockIdx.x * C::JT;
  // split-K (blockIdx.y): this CTA sums r in [kbeg, I) and writes partial blockIdx.y
  const long long kbeg = (long long)blockIdx.y * kper;
  const long long I = min(v.I, kbeg + kper);
  const int nk = (int)((I - kbeg + C::KC - 1) / C::KC);
  y += (size_t)blockIdx.y * (size_t)J * mtot;
  // 16-byte fibre loads: every column start (stride v.I, not this split's end) and the base
  // must be 16-byte aligned (a split-K CTA of an odd-I view once took the vector path)
  const bool vec16 = ((reinterpret_cast<uintptr_t>(x) & 15) == 0) && (RCONTIG ? (v.I % 2 == 0) : (v.inner % 2 == 0));

  // per-thread fixed column(s) for the JCONTIG loader
  long long jbase = 0;
  bool jvalid = false;
  int jl = 0, rsub = 0;
  if (!RCONTIG) {
    if (vec16) {
      jl = (tid % 64) * 2;
      rsub = tid / 64;  // 0..3
    } else {
      jl = tid % 128;
      rsub = tid / 128;  // 0..1
    }
    long long j = j0 + jl;
    jvalid = j < J;
    jbase = jvalid ? col_base(j, v.inner, v.I) : 0;
  }

  // gathered columns (mode-0 views only): column j of X is x column ga.idx[j] (< 0: zero,
  // another rank's column); this thread's columns are fixed over the K loop
  constexpr int NQ = RCONTIG ? (C::JT * C::KC / 2) / kThreads : 1;
  long long gcol[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const long long j = j0 + (tid + q * kThreads) / (C::KC / 2);
    gcol[q] = j < J ? (ga.idx ? __ldg(ga.idx + j) : j) : -1;
  }

  auto load = [&](int stage, int kt) {
    double* As = smem + stage * C::STAGE_ELEMS;
    double* Bs = As + C::A_ELEMS;
    const long long k0 = kbeg + (long long)kt * C::KC;
    // B chunk from the packed row-major bk[r][M8] (zero padded): rows r0..r0+15 are
    // contiguous, 16-byte copies, conflict-free row-major stores
    for (int e = tid; e < C::KC * (M8 / 2); e += kThreads) {
      int r = e / (M8 / 2), c2 = e % (M8 / 2);
      bool ok = k0 + r < I;
      cp_async16(Bs + r * C::LDB + 2 * c2, ok ? bt + (k0 + r) * M8 + 2 * c2 : bt, ok);
    }
    if (RCONTIG) {  // X(r, j) = x[I*j + r]  ->  As[j][r]
      if (vec16) {
#pragma unroll
        for (int q = 0; q < (C::JT * C::KC / 2) / kThreads; ++q) {
          int e = tid + q * kThreads;
          int rp = e % (C::KC / 2), jj = e / (C::KC / 2);
          long long r = k0 + 2 * rp;
          bool ok = (gcol[q] >= 0) && (r < I);
          cp_async16(As + jj * C::LDA + 2 * rp, ok ? x + v.I * gcol[q] + r : x, ok);
        }
      } else {
#pragma unroll
        for (int q = 0; q < (C::JT * C::KC) / kThreads; ++q) {
          int e = tid + q * kThreads;
          int rl = e % C::KC, jj = e / C::KC;
          long long j = j0 + jj, r = k0 + rl;
          const long long cj = j < J ? (ga.idx ? __ldg(ga.idx + j) : j) : -1;
          bool ok = (cj >= 0) && (r < I);
          cp_async8(As + jj * C::LDA + rl, ok ? x + v.I * cj + r : x, ok);
        }
      }
    } else {  // X(r, j) = x[base_j + inner*r]  ->  As[r][j]
      if (vec16) {
#pragma unroll
        for (int q = 0; q < C::KC / 4; ++q) {
          int rl = rsub + 4 * q;
          long long r = k0 + rl;
          bool ok = jvalid && (r < I);
          cp_async16(As + rl * C::LDA + jl, ok ? x + jbase + v.inner * r : x, ok);
        }
      } else {
#pragma unroll
        for (int q = 0; q < C::KC / 2; ++q) {
          int rl = rsub + 2 * q;
          long long r = k0 + rl;
          bool ok = jvalid && (r < I);
          cp_async8(As + rl * C::LDA + jl, ok ? x + jbase + v.inner * r : x, ok);
        }
      }
    }
  };

  constexpr int NF = M8 / 8;
  double acc[NF][4];
#pragma unroll
  for (int f = 0; f < NF; ++f)
#pragma unroll
    for (int e = 0; e < 4; ++e) acc[f][e] = 0.0;

#pragma unroll
  for (int s = 0; s < C::STAGES - 1; ++s) {
    if (s < nk) load(s, s);
    cp_async_commit();
  }
  const int jw = warp * 16;
  for (int kt = 0; kt < nk; ++kt) {
    cp_async_wait<C::STAGES - 2>();
    __syncthreads();
    const double* As = smem + (kt % C::STAGES) * C::STAGE_ELEMS;
    const double* Bs = As + C::A_ELEMS;
#pragma unroll
    for (int kk = 0; kk < C::KC / 4; ++kk) {
      const int r = kk * 4 + t;
      double a0, a1;
      if (RCONTIG) {
        a0 = As[(jw + g) * C::LDA + r];
        a1 = As[(jw + g + 8) * C::LDA + r];
      } else {
        a0 = As[r * C::LDA + jw + g];
        a1 = As[r * C::LDA + jw + g + 8];
      }
#pragma unroll
      for (int f = 0; f < NF; ++f) dmma16x8x4(acc[f], a0, a1, Bs[r * C::LDB + f * 8 + g]);
    }
    const int nt = kt + C::STAGES - 1;
    if (nt < nk) load(nt % C::STAGES, nt);
    cp_async_commit();
  }
  cp_async_wait<0>();

  // epilogue
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    const long long j = j0 + jw + g + 8 * half;
    if (j >= J) continue;
    long long ybase;
    long long ystride;
    if (RCONTIG) {
      ybase = j * mtot + koff;
      ystride = 1;
    } else {
      long long o = j / v.inner, i = j - o * v.inner;
      ybase = i + v.inner * ((long long)mtot * o + koff);
      ystride = v.inner;
    }
    // gathered: h_t = scale_t^2 (a_t^T c), so that the Gram pass sums a_t h_t^T
    // (= C' C'^T c with C'(:, t) = scale_t a_t, sketching.cpp:133-141, never materialised)
    double sc2 = 1.0;
    if (ga.scale) {
      const double sc = ga.scale[j];
      sc2 = sc * sc;
    }
#pragma unroll
    for (int f = 0; f < NF; ++f) {
      const int k = f * 8 + 2 * t;
      if (k < m) y[ybase + ystride * k] = ga.scale ? acc[f][2 * half] * sc2 : acc[f][2 * half];
      if (k + 1 < m) y[ybase + ystride * (k + 1)] = ga.scale ? acc[f][2 * half + 1] * sc2 : acc[f][2 * half + 1];
    }
  }
}

// ----------------------------------------------------------------------------
// Gram: Zpart[split](r, k) = sum_{j in split} X(r, j) * H(k, j);  H has the TTM output
// layout with width s.  CTA tile: 64 rows r (4 warps x 16) x all k, K = j in chunks of 16.
// ----------------------------------------------------------------------------
constexpr int kGramThreads = 128;
#ifndef LMRA_GRAM_STAGES
#define LMRA_GRAM_STAGES 3
#endif
// m16 tiles per warp: two independent accumulator sets per H fragment (ncu on cfg2's mode-0
// Gram at one tile: "wait" stalls on the DMMA accumulator chains dominated)
#ifndef LMRA_GRAM_MT
#define LMRA_GRAM_MT 2
#endif
constexpr int kGramMT = LMRA_GRAM_MT;
constexpr int kGramRT = 64 * kGramMT;  // rows per CTA (4 warps x 16 x MT)

template <int M8, bool RCONTIG>
struct GramCfg {
  static constexpr int RT = kGramRT, JC = 16, STAGES = LMRA_GRAM_STAGES;
  static constexpr int LDA = RCONTIG ? conflict_free_ld(RT) : conflict_free_ld(JC);
  static constexpr int A_ELEMS = RCONTIG ? JC * LDA : RT * LDA;
  static constexpr int LDH = conflict_free_ld(M8);
  static constexpr int H_ELEMS = JC * LDH;
  static constexpr int STAGE_ELEMS = A_ELEMS + H_ELEMS;
  static constexpr size_t SMEM = sizeof(double) * STAGE_ELEMS * STAGES;
};

template <int M8, bool RCONTIG>
__global__ void __launch_bounds__(kGramThreads)
    gram_kernel(const double* __restrict__ x, ModeView v, const double* __restrict__ h, int s,
                int stot, int koff, double* __restrict__ zpart, long long jper, Gather ga) {
  pdl_wait();  // the previous kernel's outputs (programmatic dependent launch)
  pdl_trigger();
  using C = GramCfg<M8, RCONTIG>;
  extern __shared__ __align__(16) double smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const long long J = v.inner * v.outer, I = v.I;
  const long long r0 = (long long)blockIdx.x * C::RT;
  const long long jbeg = (long long)blockIdx.y * jper;
  const long long jend = min(J, jbeg + jper);
  const int nk = (int)((jend - jbeg + C::JC - 1) / C::JC);
  const bool vec16 = RCONTIG && (I % 2 == 0) && ((reinterpret_cast<uintptr_t>(x) & 15) == 0);

  auto load = [&](int stage, int kt) {
    double* As = smem + stage * C::STAGE_ELEMS;
    double* Hs = As + C::A_ELEMS;
    const long long jc0 = jbeg + (long long)kt * C::JC;
    if (RCONTIG) {  // X(r, j) = x[I*j + r] -> As[j][r]
      if (vec16) {  // row pairs: 16-byte copies (half the LSU work of 8-byte ones)
#pragma unroll
        for (int q = 0; q < (C::RT / 2 * C::JC) / kGramThreads; ++q) {
          int e = tid + q * kGramThreads;
          int rp = e % (C::RT / 2), jl = e / (C::RT / 2);
          long long j = jc0 + jl, r = r0 + 2 * rp;
          const long long cj = j < jend ? (ga.idx ? __ldg(ga.idx + j) : j) : -1;
          bool ok = (cj >= 0) && (r < I);
          cp_async16(As + jl * C::LDA + 2 * rp, ok ? x + I * cj + r : x, ok);
        }
      } else {
#pragma unroll
        for (int q = 0; q < (C::RT * C::JC) / kGramThreads; ++q) {
          int e = tid + q * kGramThreads;
          int rl = e % C::RT, jl = e / C::RT;
          long long j = jc0 + jl, r = r0 + rl;
          const long long cj = j < jend ? (ga.idx ? __ldg(ga.idx + j) : j) : -1;
          bool ok = (cj >= 0) && (r < I);
          cp_async8(As + jl * C::LDA + rl, ok ? x + I * cj + r : x, ok);
        }
      }
      for (int e = tid; e < C::JC * M8; e += kGramThreads) {
        int k = e % M8, jl = e / M8;
        long long j = jc0 + jl;
        bool ok = (j < jend) && (k < s);
        cp_async8(Hs + jl * C::LDH + k, ok ? h + j * stot + koff + k : h, ok);
      }
    } else {  // X(r, j) = x[base_j + inner*r] -> As[r][j]
      const int jl = tid % C::JC, rs = tid / C::JC;  // rs 0..7
      const long long j = jc0 + jl;
      const bool jok = j < jend;
      long long base = 0, hbase = 0;
      if (jok) {
        long long o = j / v.inner, i = j - o * v.inner;
        base = i + v.inner * I * o;
        hbase = i + v.inner * ((long long)stot * o + koff);
      }
#pragma unroll
      for (int q = 0; q < C::RT / 8; ++q) {
        int rl = rs + 8 * q;
        long long r = r0 + rl;
        bool ok = jok && (r < I);
        cp_async8(As + rl * C::LDA + jl, ok ? x + base + v.inner * r : x, ok);
      }
      for (int k = rs; k < M8; k += 8) {
        bool ok = jok && (k < s);
        cp_async8(Hs + jl * C::LDH + k, ok ? h + hbase + v.inner * k : h, ok);
      }
    }
  };

  constexpr int NF = M8 / 8;
  double acc[kGramMT][NF][4];
#pragma unroll
  for (int mt = 0; mt < kGramMT; ++mt)
#pragma unroll
    for (int f = 0; f < NF; ++f)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[mt][f][e] = 0.0;

#pragma unroll
  for (int st = 0; st < C::STAGES - 1; ++st) {
    if (st < nk) load(st, st);
    cp_async_commit();
  }
  const int rw = warp * 16 * kGramMT;
  for (int kt = 0; kt < nk; ++kt) {
    cp_async_wait<C::STAGES - 2>();
    __syncthreads();
    const double* As = smem + (kt % C::STAGES) * C::STAGE_ELEMS;
    const double* Hs = As + C::A_ELEMS;
#pragma unroll
    for (int kk = 0; kk < C::JC / 4; ++kk) {
      const int jj = kk * 4 + t;
      double a0[kGramMT], a1[kGramMT];
#pragma unroll
      for (int mt = 0; mt < kGramMT; ++mt) {
        const int rr = rw + 16 * mt + g;
        if (RCONTIG) {
          a0[mt] = As[jj * C::LDA + rr];
          a1[mt] = As[jj * C::LDA + rr + 8];
        } else {
          a0[mt] = As[rr * C::LDA + jj];
          a1[mt] = As[(rr + 8) * C::LDA + jj];
        }
      }
#pragma unroll
      for (int f = 0; f < NF; ++f) {
        const double b = Hs[jj * C::LDH + f * 8 + g];
#pragma unroll
        for (int mt = 0; mt < kGramMT; ++mt) dmma16x8x4(acc[mt][f], a0[mt], a1[mt], b);
      }
    }
    const int nt = kt + C::STAGES - 1;
    if (nt < nk) load(nt % C::STAGES, nt);
    cp_async_commit();
  }
  cp_async_wait<0>();

  double* zp = zpart + (size_t)blockIdx.y * I * stot + (size_t)I * koff;
#pragma unroll
  for (int mt = 0; mt < kGramMT; ++mt)
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const long long r = r0 + rw + 16 * mt + g + 8 * half;
      if (r >= I) continue;
#pragma unroll
      for (int f = 0; f < NF; ++f) {
        const int k = f * 8 + 2 * t;
        if (k < s) zp[r + I * k] = acc[mt][f][2 * half];
        if (k + 1 < s) zp[r + I * (k + 1)] = acc[mt][f][2 * half + 1];
      }
    }
}

// Many splits (the Gram's split-J partials: ~200 on cfg1): 8 threads per output, thread g
// summing the partials p = g (mod 8) with their loads independent, then the 8 sums added in
// g order through shared memory -- fixed order (deterministic), 8x the loads in flight of the
// one-thread-per-output loop, which was a ~200-long chain of L2 round trips.
__global__ void __launch_bounds__(256) reduce_splits8_kernel(const double* __restrict__ zpart, int nsplit,
                                                             long long n, double* __restrict__ z) {
  pdl_wait();  // the previous kernel's outputs (programmatic dependent launch)
  pdl_trigger();
  __shared__ double part[8][33];
  const int lx = threadIdx.x & 31, g = threadIdx.x >> 5;
  const long long e = (long long)blockIdx.x * 32 + lx;
  double acc = 0.0;
  if (e < n) {
    double a0 = 0.0, a1 = 0.0;
    int p = g;
    for (; p + 8 < nsplit; p += 16) {
      a0 += zpart[(size_t)p * n + e];
      a1 += zpart[(size_t)(p + 8) * n + e];
    }
    if (p < nsplit) a0 += zpart[(size_t)p * n + e];
    acc = a0 + a1;
  }
  part[g][lx] = acc;
  __syncthreads();
  if (g == 0 && e < n) {
    double t = part[0][lx];
#pragma unroll
    for (int k = 1; k < 8; ++k) t += part[k][lx];
    z[e] = t;
  }
}

static cudaError_t launch_reduce_splits(const double* zpart, int nsplit, long long n, double* z, cudaStream_t st);

// z[e] = sum_{p < nsplit} zpart[p][e], fixed order (deterministic).
__global__ void reduce_splits_kernel(const double* __restrict__ zpart, int nsplit, long long n,
                                     double* __restrict__ z) {
  pdl_wait();  // the previous kernel's outputs (programmatic dependent launch)
  pdl_trigger();
  long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  double acc = zpart[e];
  for (int p = 1; p < nsplit; ++p) acc += zpart[(size_t)p * n + e];
  z[e] = acc;
}

static cudaError_t launch_reduce_splits(const double* zpart, int nsplit, long long n, double* z, cudaStream_t st) {
  if (nsplit >= 16)
    return launch_pdl(reduce_splits8_kernel, dim3((unsigned)((n + 31) / 32)), dim3(256), 0, st, zpart, nsplit, n, z);
  return launch_pdl(reduce_splits_kernel, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, st, zpart, nsplit, n, z);
}

// C'(:, t) = X(:, idx[t]) * scale[t]  (sketching.cpp:133-141), C' is I x T column-major.
// One warp per sampled column for contiguous fibers; a 32x32 staged transpose otherwise.
__global__ void gather_contig_kernel(const double* __restrict__ x, long long I,
                                     const long long* __restrict__ idx,
                                     const double* __restrict__ scale, long long T,
                                     double* __restrict__ out) {
  pdl_wait();  // the previous kernel's outputs (programmatic dependent launch)
  pdl_trigger();
  long long tcol = (long long)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  if (tcol >= T) return;
  const int lane = threadIdx.x & 31;
  double* dst = out + tcol * I;
  const long long id = idx[tcol];
  if (id < 0) {  // column owned by another rank (sharded runs): zero
    for (long long r = lane; r < I; r += 32) dst[r] = 0.0;
    return;
  }
  const double* src = x + id * I;
  const double sc = scale[tcol];
  for (long long r = lane; r < I; r += 32) dst[r] = src[r] * sc;
}

__global__ void gather_strided_kernel(const double* __restrict__ x, ModeView v,
                                      const long long* __restrict__ idx,
                                      const double* __restrict__ scale, long long T,
                                      double* __restrict__ out) {
  pdl_wait();  // the previous kernel's outputs (programmatic dependent launch)
  pdl_trigger();
  __shared__ double tile[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  const long long t0 = (long long)blockIdx.x * 32;
  const long long tcol = t0 + tx;
  long long base = 0;
  double sc = 0.0;
  const bool ok = tcol < T && idx[tcol] >= 0;  // negative index: another rank's column -> 0
  if (ok) {
    base = col_base(idx[tcol], v.inner, v.I);
    sc = scale[tcol];
  }
  for (long long r0 = 32LL * blockIdx.y; r0 < v.I; r0 += 32LL * gridDim.y) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      int rl = ty + 8 * q;
      long long r = r0 + rl;
      tile[rl][tx] = (ok && r < v.I) ? x[base + v.inner * r] * sc : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      int tl = ty + 8 * q;
      long long tc = t0 + tl, r = r0 + tx;
      if (tc < T && r < v.I) out[tc * v.I + r] = tile[tx][tl];
    }
    __syncthreads();
  }
}

// ----------------------------------------------------------------------------
// launchers
// ----------------------------------------------------------------------------
// bk[r * M8 + k] = bt[r + I * k] for k < m, 0 for m <= k < M8 (row-major, zero padded)
__global__ void pack_b_kernel(const double* __restrict__ bt, long long I, int m, int M8,
                              double* __restrict__ bk) {
  pdl_wait();  // the previous kernel's outputs (programmatic dependent launch)
  pdl_trigger();
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= I * M8) return;
  const long long r = e / M8;
  const int k = (int)(e - r * M8);
  bk[e] = k < m ? bt[r + I * k] : 0.0;
}

template <int M8, bool RC>
static cudaError_t launch_ttm_t(const double* x, ModeView v, const double* bt_colmajor, int m,
                                int mtot, int koff, double* y, int ksplit, long long kper,
                                cudaStream_t st, Gather ga) {
  double* bt = nullptr;  // packed copy, stream-ordered scratch
  cudaError_t pe = scratch_alloc(reinterpret_cast<void**>(&bt), sizeof(double) * v.I * M8, st);
  if (pe != cudaSuccess) return pe;
  {
    const cudaError_t le = launch_pdl(pack_b_kernel, dim3((unsigned)((v.I * M8 + 255) / 256)), dim3(256), 0, st, bt_colmajor, v.I, m, M8, bt);
    if (le != cudaSuccess) return le;
  }
  struct FreeGuard {
    double* p;
    cudaStream_t s;
    ~FreeGuard() { scratch_free(p, s); }
  } free_guard{bt, st};
  // K chunk 16 x 3 stages: measured best overall against (32,2), (16,4), (32,3) on the
  // BASELINE widths (tools/ttm_variants.sh, round 1)
  auto go = [&](auto kc, auto stg) -> cudaError_t {
    constexpr int KC = decltype(kc)::value, ST = decltype(stg)::value;
    using C = TtmCfg<M8, RC, KC, ST>;
    static unsigned long long attr_done = 0;
    cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(ttm_kernel<M8, RC, KC, ST>),
                                     C::SMEM, attr_done);
    if (e != cudaSuccess) return e;
    long long J = v.inner * v.outer;
    dim3 grid((unsigned)((J + C::JT - 1) / C::JT), (unsigned)ksplit);
    {
    const cudaError_t le = launch_pdl(ttm_kernel<M8, RC, KC, ST>, dim3(grid), dim3(kThreads), C::SMEM, st, x, v, bt, m, mtot, koff, y, kper, ga);
    if (le != cudaSuccess) return le;
  }
    return cudaGetLastError();
  };
  return go(std::integral_constant<int, 16>{}, std::integral_constant<int, 3>{});
}

template <bool RC>
static cudaError_t launch_ttm_rc(const double* x, ModeView v, const double* bt, int m, int mtot,
                                 int koff, double* y, int ks, long long kper, cudaStream_t st, Gather ga) {
  switch ((m + 7) / 8) {
    case 1: return launch_ttm_t<8, RC>(x, v, bt, m, mtot, koff, y, ks, kper, st, ga);
    case 2: return launch_ttm_t<16, RC>(x, v, bt, m, mtot, koff, y, ks, kper, st, ga);
    case 3: return launch_ttm_t<24, RC>(x, v, bt, m, mtot, koff, y, ks, kper, st, ga);
    case 4: return launch_ttm_t<32, RC>(x, v, bt, m, mtot, koff, y, ks, kper, st, ga);
    case 5: return launch_ttm_t<40, RC>(x, v, bt, m, mtot, koff, y, ks, kper, st, ga);
    case 6: return launch_ttm_t<48, RC>(x, v, bt, m, mtot, koff, y, ks, kper, st, ga);
    case 7: return launch_ttm_t<56, RC>(x, v, bt, m, mtot, koff, y, ks, kper, st, ga);
    case 8: return launch_ttm_t<64, RC>(x, v, bt, m, mtot, koff, y, ks, kper, st, ga);
  }
  return cudaErrorInvalidValue;
}

static int device_sms() {
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms < 1)
      sms = 148;
  }
  return sms;
}

// Short contractions (I <= 8: cfg5's mode of extent 3): a streaming kernel, one thread per
// column j -- the I fibre values in registers, B^T (I x m) in shared memory, m outputs written
// in Y's layout.  The DMMA kernel pads K to its 16-row chunk and runs one K stage per CTA, so
// it was latency-bound (cfg5 shrink of the 3-extent mode: 43 us for 40 MB of traffic).
// Each output is an fma chain over r ascending (deterministic; the DMMA path sums in another
// fixed order, both within the fp64 contract).
constexpr int kSmallI = 8;
template <int IS>
__global__ void __launch_bounds__(256) ttm_small_kernel(const double* __restrict__ x, ModeView v,
                                                        const double* __restrict__ bt, int m, int mtot,
                                                        int koff, double* __restrict__ y, Gather ga) {
  pdl_wait();  // the previous kernel's outputs (programmatic dependent launch)
  pdl_trigger();
  __shared__ double bs[kSmallI * kMaxWidth];
  const int I = (int)v.I;
  for (int e = threadIdx.x; e < I * m; e += blockDim.x) bs[e] = bt[e];  // bt[r + I * k]
  __syncthreads();
  const long long J = v.inner * v.outer;
  for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < J; j += (long long)gridDim.x * blockDim.x) {
    double xr[IS];
    long long ybase, ystride;
    double sc2 = 1.0;
    if (v.inner == 1) {
      const long long cj = ga.idx ? __ldg(ga.idx + j) : j;
#pragma unroll
      for (int r = 0; r < IS; ++r) xr[r] = (r < I && cj >= 0) ? __ldg(x + I * cj + r) : 0.0;
      if (ga.scale) {
        const double sc = ga.scale[j];
        sc2 = sc * sc;
      }
      ybase = j * mtot + koff;
      ystride = 1;
    } else {
      const long long o = j / v.inner, i = j - o * v.inner;
      const long long base = i + v.inner * (long long)I * o;
#pragma unroll
      for (int r = 0; r < IS; ++r) xr[r] = r < I ? __ldg(x + base + v.inner * r) : 0.0;
      ybase = i + v.inner * ((long long)mtot * o + koff);
      ystride = v.inner;
    }
    for (int k = 0; k < m; ++k) {
      double acc = 0.0;
#pragma unroll
      for (int r = 0; r < IS; ++r)
        if (r < I) acc = fma(bs[r + I * k], xr[r], acc);
      y[ybase + ystride * k] = ga.scale ? acc * sc2 : acc;
    }
  }
}

static cudaError_t launch_ttm_small(const double* x, ModeView v, const double* bt, int m, double* y,
                                    cudaStream_t st, Gather ga) {
  const long long J = v.inner * v.outer;
  const long long blocks = std::min<long long>((J + 255) / 256, 8LL * device_sms());
  auto go = [&](auto is) {
    return launch_pdl(ttm_small_kernel<decltype(is)::value>, dim3((unsigned)blocks), dim3(256), 0, st, x, v, bt,
                      m, m, 0, y, ga);
  };
  const cudaError_t e = v.I <= 4 ? go(std::integral_constant<int, 4>{}) : go(std::integral_constant<int, 8>{});
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t launch_ttm(const double* x, ModeView v, const double* bt, int m, double* y,
                       cudaStream_t st, Gather ga) {
  if (ga.idx && v.inner != 1) return cudaErrorInvalidValue;  // gathered: mode-0 views only
  if (m < 1) return cudaErrorInvalidValue;
  const long long J = v.inner * v.outer;
  if (J == 0) return cudaSuccess;
  if (v.I <= kSmallI && m <= kMaxWidth && !getenv("LMRA_TTM_NO_SMALL")) return launch_ttm_small(x, v, bt, m, y, st, ga);
  // Narrow outputs (few 128-column tiles, e.g. the power scheme on sampled columns or the
  // core's last contraction) leave most SMs idle over a long K: split K across CTAs into
  // fixed-order partials (deterministic), >= 64 rows of K per split.
  const long long jt = (J + 127) / 128;
  int ks = 1;
  const int sms = device_sms();
  const long long mink = getenv("LMRA_TTM_MINK") ? atoll(getenv("LMRA_TTM_MINK")) : 32;
  if (jt * 2 <= sms && v.I >= 64) {
    // (both resident CTAs of an SM: small contractions -- the core's later modes, the last
    // shrinks -- were a ~10-stage K loop on a few CTAs, latency-bound at ~15 us)
    ks = (int)std::max<long long>(1, std::min<long long>(2 * sms / jt, v.I / mink));
  } else if (v.I >= 512 && jt < 8LL * sms) {
    // a few waves of a long-K contraction: fill the last wave (two CTAs per SM) by splitting
    // K, each extra split charged ~3 % for its partials' round trip
    const double slots = 2.0 * sms;
    auto fill = [&](int k) {
      const double n = (double)(jt * k);
      return n / (std::ceil(n / slots) * slots) - 0.03 * (k - 1);
    };
    for (int k = 2; k <= 4 && v.I / k >= 128; ++k)
      if (fill(k) > fill(ks) + 1e-9) ks = k;
  }
  long long kper = (v.I + ks - 1) / ks;
  kper = ((kper + 15) / 16) * 16;
  ks = (int)((v.I + kper - 1) / kper);
  double* part = y;
  if (ks > 1) {
    cudaError_t pe =
        scratch_alloc(reinterpret_cast<void**>(&part), sizeof(double) * (size_t)J * m * ks, st);
    if (pe != cudaSuccess) return pe;
  }
  cudaError_t e = cudaSuccess;
  // widths above one DMMA tile are done as column blocks of <= kMaxWidth output rows
  for (int k0 = 0; k0 < m && e == cudaSuccess; k0 += kMaxWidth) {
    int mb = std::min(kMaxWidth, m - k0);
    const double* btb = bt + (size_t)v.I * k0;
    e = v.inner == 1 ? launch_ttm_rc<true>(x, v, btb, mb, m, k0, part, ks, kper, st, ga)
                     : launch_ttm_rc<false>(x, v, btb, mb, m, k0, part, ks, kper, st, ga);
  }
  if (ks > 1) {
    if (e == cudaSuccess) {
      const long long n = J * m;
      {
    const cudaError_t le = launch_reduce_splits(part, ks, n, y, st);
    if (le != cudaSuccess) return le;
  }
      e = cudaGetLastError();
    }
    scratch_free(part, st);
  }
  return e;
}

template <int M8, bool RC>
static cudaError_t launch_gram_t(const double* x, ModeView v, const double* h, int s, int stot,
                                 int koff, double* zpart, int nsplit, long long jper,
                                 cudaStream_t st, Gather ga) {
  using C = GramCfg<M8, RC>;
  static unsigned long long attr_done = 0;
  cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(gram_kernel<M8, RC>), C::SMEM,
                                   attr_done);
  if (e != cudaSuccess) return e;
  dim3 grid((unsigned)((v.I + C::RT - 1) / C::RT), (unsigned)nsplit);
  {
    const cudaError_t le = launch_pdl(gram_kernel<M8, RC>, dim3(grid), dim3(kGramThreads), C::SMEM, st, x, v, h, s, stot, koff, zpart, jper, ga);
    if (le != cudaSuccess) return le;
  }
  return cudaGetLastError();
}

template <bool RC>
static cudaError_t launch_gram_rc(const double* x, ModeView v, const double* h, int s, int stot,
                                  int koff, double* zpart, int nsplit, long long jper,
                                  cudaStream_t st, Gather ga) {
  switch ((s + 7) / 8) {
    case 1: return launch_gram_t<8, RC>(x, v, h, s, stot, koff, zpart, nsplit, jper, st, ga);
    case 2: return launch_gram_t<16, RC>(x, v, h, s, stot, koff, zpart, nsplit, jper, st, ga);
    case 3: return launch_gram_t<24, RC>(x, v, h, s, stot, koff, zpart, nsplit, jper, st, ga);
    case 4: return launch_gram_t<32, RC>(x, v, h, s, stot, koff, zpart, nsplit, jper, st, ga);
    case 5: return launch_gram_t<40, RC>(x, v, h, s, stot, koff, zpart, nsplit, jper, st, ga);
    case 6: return launch_gram_t<48, RC>(x, v, h, s, stot, koff, zpart, nsplit, jper, st, ga);
    case 7: return launch_gram_t<56, RC>(x, v, h, s, stot, koff, zpart, nsplit, jper, st, ga);
    case 8: return launch_gram_t<64, RC>(x, v, h, s, stot, koff, zpart, nsplit, jper, st, ga);
  }
  return cudaErrorInvalidValue;
}

GramPlan plan_gram(ModeView v, int num_sms) {
  GramPlan p;
  const long long J = v.inner * v.outer;
  const long long rtiles = (v.I + kGramRT - 1) / kGramRT;
  long long target = (long long)num_sms * (kGramMT == 1 ? 4 : 3);  // ~ resident CTAs (one wave)
  long long ns = std::max<long long>(1, target / std::max<long long>(1, rtiles));
  // at least 32 columns per split (two K chunks) so each CTA amortises its prologue
  const long long minj = getenv("LMRA_GRAM_MINJ") ? atoll(getenv("LMRA_GRAM_MINJ")) : 16;
  ns = std::min<long long>(ns, std::max<long long>(1, J / minj));
  ns = std::min<long long>(ns, 1024);
  long long jper = (J + ns - 1) / ns;
  jper = ((jper + 15) / 16) * 16;
  ns = (J + jper - 1) / jper;
  p.nsplit = (int)std::max<long long>(1, ns);
  p.jper = jper;
  return p;
}

cudaError_t launch_gram(const double* x, ModeView v, const double* h, int s, double* zpart,
                        const GramPlan& plan, double* z, cudaStream_t st, Gather ga) {
  if (s < 1) return cudaErrorInvalidValue;
  if (ga.idx && v.inner != 1) return cudaErrorInvalidValue;
  for (int k0 = 0; k0 < s; k0 += kMaxWidth) {
    int sb = std::min(kMaxWidth, s - k0);
    cudaError_t e =
        v.inner == 1
            ? launch_gram_rc<true>(x, v, h, sb, s, k0, zpart, plan.nsplit, plan.jper, st, ga)
            : launch_gram_rc<false>(x, v, h, sb, s, k0, zpart, plan.nsplit, plan.jper, st, ga);
    if (e != cudaSuccess) return e;
  }
  long long n = v.I * s;
  {
    const cudaError_t le = launch_reduce_splits(zpart, plan.nsplit, n, z, st);
    if (le != cudaSuccess) return le;
  }
  return cudaGetLastError();
}

cudaError_t launch_gather(const double* x, ModeView v, const long long* idx, const double* scale,
                          long long T, double* out, cudaStream_t st) {
  if (T == 0) return cudaSuccess;
  if (v.inner == 1) {
    {
    const cudaError_t le = launch_pdl(gather_contig_kernel, dim3((unsigned)((T + 7) / 8)), dim3(256), 0, st, x, v.I, idx, scale, T, out);
    if (le != cudaSuccess) return le;
  }
  } else {
    // rows split over grid.y: each sampled fiber is strided (one sector per element), so the
    // gather is latency-bound and wants every SM issuing
    const long long tb = (T + 31) / 32, rb = (v.I + 31) / 32;
    const long long ry = std::max<long long>(1, std::min<long long>(rb, (4LL * device_sms() + tb - 1) / tb));
    {
    const cudaError_t le = launch_pdl(gather_strided_kernel, dim3(dim3((unsigned)tb, (unsigned)ry)), dim3(256), 0, st, x, v, idx, scale, T, out);
    if (le != cudaSuccess) return le;
  }
  }
  return cudaGetLastError();
}

}  // namespace lmra_dev

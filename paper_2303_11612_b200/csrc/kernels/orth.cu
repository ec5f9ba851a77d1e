// orth.cu -- on-device orthonormalisation of the I_n x s sketch C.
//
// Replaces thin_svd (linalg.cpp:33-43, Eigen BDCSVD) + fix_signs (linalg.cpp:13-29)
// as used by leading_left_singular_vectors (linalg.cpp:82-87):
//   C = Q R            Householder TSQR: leaves of <= 256 rows factored in parallel CTAs,
//                      their stacked R factors reduced level by level; the last block gets
//                      a column-pivoted Householder QR
//   R = U_R S V^T      one-sided (Hestenes) Jacobi on R^T with the rotations accumulated:
//                      R^T J = W  =>  R = J diag(|W_j|) (W/|W|)^T, so U_R = J (orthogonal even
//                      for zero singular values).  The pivoted R is graded, which makes
//                      Jacobi on R^T converge in a few sweeps (de Rijk / Drmac).
//   U = Q [U_R ; 0]    reflectors applied in reverse, level by level back down the tree
//   fix_signs          largest-|u| entry (first index on ties) made >= 0
// All reductions run in a fixed order, so the result is deterministic run to run.
// Householder QR is used instead of CholeskyQR2 because the sketches of the
// BASELINE configs reach kappa(C) ~ 1e16, far past CholeskyQR2's
// u^{-1/2} limit.
//
// Register-resident panels, columns by warp.  A block of <= 256 rows x <= 64 columns lives
// in registers: warp w holds columns w, w + 16, w + 32, w + 48 (four slots), lane l holds
// rows l, l + 32, ... (RPL rows per lane).  Every column reduction (norm, v^T a) is then a
// warp butterfly, and a Householder step needs ONE block barrier: the warp owning the step's
// column forms the reflector and publishes v (double-buffered by step parity), every warp
// updates its own remaining columns.  Applying stored reflectors needs no barrier at all.
// (Round-1 history: rows-by-warp panels needed four barriers and two cross-warp partial
// reductions per step -- 4350 cycles a step measured with tools/microbench/qr_bench.cu; the
// first version kept the panel in shared memory and was bound on shared-memory bandwidth.)
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "common.cuh"

namespace lmra_dev {

constexpr int kQThreads = 512;
constexpr int kQWarps = kQThreads / 32;
constexpr int kMaxBlockRows = 256;            // rows per CTA: 32 lanes x RPL (<= 8)
constexpr int kOrthMaxS = 64;
constexpr int kCW = kOrthMaxS / kQWarps;      // column slots per warp
// Column c lives in warp c / kCW, slot c % kCW: narrow sketches occupy few warps and the others
// skip every reduction (64-bit shuffles run at 0.5 per clock per SM: with columns dealt
// round-robin, s = 15 kept all 16 warps reducing every Householder step).
__device__ __forceinline__ int slot_col(int w, int j) { return w * kCW + j; }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
  return v;
}

// Warp sums of the four slots, every lane ends with all four (identical bits in every
// lane).  Reduce-scatter then all-gather: lane bits 4 and 3 pick which slot a lane keeps
// while the other slots are handed to the partner, so the five butterfly levels move one
// value instead of four -- 9 double shuffles instead of 20 (measured: QR step 2730 -> 2490
// cycles, apply step 1330 -> 1200, tools/microbench/qr_bench.cu).
__device__ __forceinline__ void warp_sum_cw(double (&t)[kCW]) {
  static_assert(kCW == 4, "warp_sum_cw is written for four slots");
  const int l = threadIdx.x & 31;
  const bool b4 = (l >> 4) & 1, b3 = (l >> 3) & 1;
  // level xor 16: keep the slot pair {2 b4, 2 b4 + 1}
  const double r0 = __shfl_xor_sync(0xffffffffu, b4 ? t[0] : t[2], 16);
  const double r1 = __shfl_xor_sync(0xffffffffu, b4 ? t[1] : t[3], 16);
  const double u0 = (b4 ? t[2] : t[0]) + r0, u1 = (b4 ? t[3] : t[1]) + r1;
  // level xor 8: keep slot 2 b4 + b3
  const double r2 = __shfl_xor_sync(0xffffffffu, b3 ? u0 : u1, 8);
  double v = (b3 ? u1 : u0) + r2;
  // the eight lanes holding the same slot: symmetric butterfly
  v += __shfl_xor_sync(0xffffffffu, v, 4);
  v += __shfl_xor_sync(0xffffffffu, v, 2);
  v += __shfl_xor_sync(0xffffffffu, v, 1);
  // all-gather: the pair's other slot, then the other pair
  const double o = __shfl_xor_sync(0xffffffffu, v, 8);
  const double lo = b3 ? o : v, hi = b3 ? v : o;  // slots 2 b4, 2 b4 + 1
  const double plo = __shfl_xor_sync(0xffffffffu, lo, 16);
  const double phi = __shfl_xor_sync(0xffffffffu, hi, 16);
  t[0] = b4 ? plo : lo;
  t[1] = b4 ? phi : hi;
  t[2] = b4 ? lo : plo;
  t[3] = b4 ? hi : phi;
}

// ---------------------------------------------------------------------------
// shared scratch of the register-resident QR / apply / Jacobi
// ---------------------------------------------------------------------------
struct QSmem {
  double* part;   // kQWarps x 64: Jacobi per-warp partials
  double* vbuf;   // 2 x kMaxBlockRows: the current reflector (by step parity)
  double* fval;   // 64 } Jacobi: cos / sin of the round (128 contiguous doubles)
  double* rowk;   // 64 }
  double* red;    // 64: per-column best |y| (sign fix)
  double* cn;     // 64: squared column norms over the remaining rows (pivoted QR)
  double* tau;    // 64
  double* normp;  // kQWarps
  int* pidx;      // 64: Jacobi flags
  int* piv;       // 64: logical position -> physical column (QR); argmax row (sign fix)
  int* ipiv;      // 64: physical column -> logical position
};
constexpr size_t kQScratchDoubles = kQWarps * 64 + 2 * kMaxBlockRows + 64 * 5 + kQWarps;
constexpr size_t kQScratchBytes = kQScratchDoubles * 8 + 3 * 64 * 4 + 64;

__device__ __forceinline__ QSmem carve_q(double* base) {
  QSmem q;
  q.part = base;
  q.vbuf = q.part + kQWarps * 64;
  q.fval = q.vbuf + 2 * kMaxBlockRows;
  q.rowk = q.fval + 64;
  q.red = q.rowk + 64;
  q.cn = q.red + 64;
  q.tau = q.cn + 64;
  q.normp = q.tau + 64;
  q.pidx = reinterpret_cast<int*>(q.normp + kQWarps);
  q.piv = q.pidx + 64;
  q.ipiv = q.piv + 64;
  return q;
}

// 1/sqrt(x), 1/x for normal positive x: hardware approximation plus two Newton steps (full
// double precision within an ulp or two) -- short dependent chains, where the IEEE library
// sqrt / division carry special-case branches on the critical path.
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double h = 0.5 * x;
  y = y * fma(-h * y, y, 1.5);
  y = y * fma(-h * y, y, 1.5);
  return y;
}

__device__ __forceinline__ double rcp_nr(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  return fma(y, e, y);
}

// dlarfg scalars for the column (alpha; ||x(below)||^2 = ss > 0): beta = -sign(alpha) n,
// tau = (beta - alpha) / beta = 1 + |alpha| / n, scale = 1 / (alpha - beta).
__device__ __forceinline__ void householder_scalars(double alpha, double ss, double& beta,
                                                    double& tk, double& scale) {
  const double n2 = fma(alpha, alpha, ss);
  if (n2 > 0x1.0p-1000 && n2 < 0x1.0p+1000) {
    const double rn = rsqrt_nr(n2);
    const double n = n2 * rn;
    beta = -copysign(n, alpha);
    tk = fma(fabs(alpha), rn, 1.0);
    scale = copysign(rcp_nr(fabs(alpha) + n), alpha);
  } else {  // far from 1: the IEEE path (no flush, no overflow in the approximations)
    beta = -copysign(sqrt(n2), alpha);
    tk = (beta - alpha) / beta;
    scale = 1.0 / (alpha - beta);
  }
}

// ---------------------------------------------------------------------------
// column-by-warp panels <-> shared tiles
// ---------------------------------------------------------------------------
// coalesced global (rows x cols, ld lda) -> shared tile (ld ldt), rows [rows, prow) zeroed
__device__ __forceinline__ void load_tile(const double* __restrict__ g, long long lda, int rows,
                                          int cols, double* t, int ldt, int prow) {
  for (int e = threadIdx.x; e < rows * cols; e += kQThreads) {
    const int i = e % rows, c = e / rows;
    t[i + ldt * c] = g[i + (size_t)lda * c];
  }
  const int pad = prow - rows;
  for (int e = threadIdx.x; e < pad * cols; e += kQThreads) {
    const int i = e % pad, c = e / pad;
    t[rows + i + ldt * c] = 0.0;
  }
}

template <int RPL>
__device__ __forceinline__ void cw_load(const double* t, int ldt, int rows, int cols,
                                        double (&a)[kCW][RPL]) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
#pragma unroll
  for (int j = 0; j < kCW; ++j) {
    const int c = slot_col(w, j);
#pragma unroll
    for (int i = 0; i < RPL; ++i) {
      const int r = l + 32 * i;
      a[j][i] = (r < rows && c < cols) ? t[r + (size_t)ldt * c] : 0.0;
    }
  }
}

template <int RPL>
__device__ __forceinline__ void cw_store(const double (&a)[kCW][RPL], int rows, int cols,
                                         double* t, int ldt) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
#pragma unroll
  for (int j = 0; j < kCW; ++j) {
    const int c = slot_col(w, j);
#pragma unroll
    for (int i = 0; i < RPL; ++i) {
      const int r = l + 32 * i;
      if (r < rows && c < cols) t[r + (size_t)ldt * c] = a[j][i];
    }
  }
}

// ---------------------------------------------------------------------------
// Householder QR of the panel a (m x s; rows >= m and columns >= s zero).  LAPACK dlarfg
// convention: H_k = I - tau v v^T, v_k = 1, beta = -sign(alpha) ||x||.  Columns are never
// moved: logical column k lives in physical column q.piv[k] (identity without pivoting),
// which on exit holds R(0..k, k) in rows <= k and v_k below; q.tau[k] the scalars.
// Pivoting takes, at step k, the remaining column with the largest norm over rows >= k
// (first logical position on ties; norms recomputed exactly every step) -- it only permutes
// R's columns, so the left singular vectors are unaffected.
// Barriers: one per step (the owner warp's v), plus one for the norms when pivoting.
// ---------------------------------------------------------------------------
#ifdef LMRA_QR_CLOCKS
__device__ unsigned long long g_qrclk[8];  // microbenchmark only: warp-0 phase cycles per QR
#define QR_T(v) const long long v = clock64()
#define QR_ACC(i, a, b) \
  if (threadIdx.x == 0) qacc[i] += (b) - (a)
#else
#define QR_T(v)
#define QR_ACC(i, a, b)
#endif
template <int RPL>
__device__ void reg_qr(double (&a)[kCW][RPL], int m, int s, const QSmem& q, bool pivot) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const int kmax = min(m, s);
#ifdef LMRA_QR_CLOCKS
  long long qacc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#endif
  int pA = l, pB = l + 32;  // physical column at logical positions l and l + 32
  unsigned done = 0;        // slots of this warp already factored
  if (pivot) {
    double t[kCW];
#pragma unroll
    for (int j = 0; j < kCW; ++j) {
      t[j] = 0.0;
#pragma unroll
      for (int i = 0; i < RPL; ++i) t[j] = fma(a[j][i], a[j][i], t[j]);
    }
    warp_sum_cw(t);
    if (l == 0)
#pragma unroll
      for (int j = 0; j < kCW; ++j)
        if (slot_col(w, j) < s) {
          q.cn[slot_col(w, j)] = t[j];
          q.red[slot_col(w, j)] = t[j];  // the original norms (downdate safeguard; q.red is the sign fix's later)
        }
    __syncthreads();
  }
  for (int k = 0; k < kmax; ++k) {
    QR_T(c0);
    int pc = k;
    if (pivot) {  // every warp: the same argmax over the remaining logical positions
      // one warp max-reduction (REDUX) of 32-bit keys instead of a 5-level shuffle tree of
      // (double, position) pairs (64-bit shuffles run at 0.5 per clock per SM, and all 16
      // warps did this every step): key = the squared norm's top 25 bits (sign, exponent, 13
      // mantissa bits -- non-negative doubles order like their bit patterns) above 127 - pos,
      // so the largest norm wins and norms equal to ~1e-4 go to the first position
      auto key = [](double v, int pos) -> unsigned {
        const unsigned hi = (unsigned)((unsigned long long)__double_as_longlong(v) >> 32);
        return (hi & ~0x7Fu) | (unsigned)(127 - pos);
      };
      const unsigned ka = (l >= k && l < s) ? key(q.cn[pA], l) : 0u;
      const unsigned kb = (l + 32 >= k && l + 32 < s) ? key(q.cn[pB], l + 32) : 0u;
      const unsigned best = __reduce_max_sync(0xffffffffu, ka > kb ? ka : kb);
      const int pos = 127 - (int)(best & 0x7Fu);
      const int pk = __shfl_sync(0xffffffffu, k < 32 ? pA : pB, k & 31);
      pc = __shfl_sync(0xffffffffu, pos < 32 ? pA : pB, pos & 31);
      if (l == (k & 31)) {
        if (k < 32)
          pA = pc;
        else
          pB = pc;
      }
      if (pos != k && l == (pos & 31)) {
        if (pos < 32)
          pA = pk;
        else
          pB = pk;
      }
    }
    QR_T(c1);
    QR_ACC(0, c0, c1);
    double* vb = q.vbuf + (k & 1) * kMaxBlockRows;
    if (w == pc / kCW) {  // owner warp: reflector of physical column pc
      const int oj = pc % kCW;
      done |= 1u << oj;
      double col[RPL];
#pragma unroll
      for (int i = 0; i < RPL; ++i) col[i] = a[0][i];
#pragma unroll
      for (int j = 1; j < kCW; ++j)
        if (j == oj)
#pragma unroll
          for (int i = 0; i < RPL; ++i) col[i] = a[j][i];
      double t0 = 0.0, t1 = 0.0, al = 0.0;
#pragma unroll
      for (int i = 0; i < RPL; ++i) {
        const int r = l + 32 * i;
        if (r > k) {
          if (i & 1)
            t1 = fma(col[i], col[i], t1);
          else
            t0 = fma(col[i], col[i], t0);
        }
        if (r == k) al = col[i];
      }
      double ss = t0 + t1;
#pragma unroll
      for (int msk = 16; msk >= 1; msk >>= 1) {
        ss += __shfl_xor_sync(0xffffffffu, ss, msk);
        al += __shfl_xor_sync(0xffffffffu, al, msk);
      }
      double beta = al, tk = 0.0, scale = 0.0;
      if (ss != 0.0) householder_scalars(al, ss, beta, tk, scale);
#pragma unroll
      for (int i = 0; i < RPL; ++i) {
        const int r = l + 32 * i;
        if (r > k) {
          col[i] *= scale;
          vb[r] = col[i];
        } else if (r == k) {
          col[i] = beta;
          vb[r] = 1.0;
        } else {
          vb[r] = 0.0;
        }
      }
#pragma unroll
      for (int j = 0; j < kCW; ++j)
        if (j == oj)
#pragma unroll
          for (int i = 0; i < RPL; ++i) a[j][i] = col[i];
      if (l == 0) q.tau[k] = tk;
    }
    QR_T(c2);
    QR_ACC(1, c1, c2);
    __syncthreads();
    QR_T(c3);
    QR_ACC(2, c2, c3);
    const double tk = q.tau[k];
    bool act[kCW];
#pragma unroll
    for (int j = 0; j < kCW; ++j) act[j] = (slot_col(w, j) < s) && !((done >> j) & 1u);
    // warp-uniform: a warp whose columns are all factored (or past s) skips the reduction
    const int nvalid = min(kCW, max(0, s - slot_col(w, 0)));
    const bool any_act = (~done & ((1u << nvalid) - 1u)) != 0u;
    if (tk != 0.0 && any_act) {
      double vr[RPL], t[kCW];
#pragma unroll
      for (int i = 0; i < RPL; ++i) vr[i] = vb[l + 32 * i];
#pragma unroll
      for (int j = 0; j < kCW; ++j) {
        t[j] = 0.0;
        if (act[j])
#pragma unroll
          for (int i = 0; i < RPL; ++i) t[j] = fma(vr[i], a[j][i], t[j]);
      }
      warp_sum_cw(t);
#pragma unroll
      for (int j = 0; j < kCW; ++j)
        if (act[j]) {
          const double f = tk * t[j];
#pragma unroll
          for (int i = 0; i < RPL; ++i) a[j][i] = fma(-f, vr[i], a[j][i]);
        }
    }
    QR_T(c4);
    QR_ACC(3, c3, c4);
    if (pivot && k + 1 < kmax) {  // norms over rows > k of the remaining columns
      // downdated (dgeqp3's rule): the reflector keeps each column's norm over rows >= k, so the
      // norm over rows > k is the old one less the new row-k entry squared; lane k % 32 holds
      // row k.  Recomputed (warp reduction) when the downdate cancelled below 1e-6 of the
      // column's original squared norm.
      const int ik = k >> 5;
      int redo = 0;
#pragma unroll
      for (int j = 0; j < kCW; ++j) {
        double rk = a[j][0];
#pragma unroll
        for (int i = 1; i < RPL; ++i) rk = i == ik ? a[j][i] : rk;
        if (act[j] && l == (k & 31)) {
          const int c = slot_col(w, j);
          const double nv = q.cn[c] - rk * rk;
          if (!(nv > 1e-6 * q.red[c])) redo = 1;
          q.cn[c] = nv;
        }
      }
      if (__shfl_sync(0xffffffffu, redo, k & 31)) {
        double t[kCW];
#pragma unroll
        for (int j = 0; j < kCW; ++j) {
          t[j] = 0.0;
#pragma unroll
          for (int i = 0; i < RPL; ++i)
            if (l + 32 * i > k) t[j] = fma(a[j][i], a[j][i], t[j]);
        }
        warp_sum_cw(t);
        __syncwarp();
        if (l == 0)
#pragma unroll
          for (int j = 0; j < kCW; ++j)
            if (act[j]) {
              q.cn[slot_col(w, j)] = t[j];
              q.red[slot_col(w, j)] = t[j];
            }
      }
      __syncthreads();
    }
    QR_T(c5);
    QR_ACC(4, c4, c5);
  }
#ifdef LMRA_QR_CLOCKS
  if (threadIdx.x == 0)
    for (int i = 0; i < 5; ++i) g_qrclk[i] = qacc[i];
#endif
  if (w == 0) {
    q.piv[l] = pivot ? pA : l;
    q.piv[l + 32] = pivot ? pB : l + 32;
  }
  __syncthreads();
}

// y <- H_{k_lo} H_{k_lo+1} ... H_{k_hi-1} y  (reflectors applied last to first).
// Vs: logical column k holds v_k below row k (ld ldv >= 32 * RPL, rows >= m zero); tau in
// smem.  Each warp applies every reflector to its own columns: no block barrier.
template <int RPL>
__device__ void reg_apply(double (&y)[kCW][RPL], int mu, const double* Vs, int ldv,
                          const double* tau, int k_hi, int k_lo) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (slot_col(w, 0) >= mu) return;
  bool act[kCW];
#pragma unroll
  for (int j = 0; j < kCW; ++j) act[j] = slot_col(w, j) < mu;
  for (int k = k_hi - 1; k >= k_lo; --k) {
    const double tk = tau[k];
    if (tk == 0.0) continue;
    double vr[RPL], t[kCW];
#pragma unroll
    for (int i = 0; i < RPL; ++i) {
      const int r = l + 32 * i;
      vr[i] = r > k ? Vs[r + (size_t)ldv * k] : (r == k ? 1.0 : 0.0);
    }
#pragma unroll
    for (int j = 0; j < kCW; ++j) {
      t[j] = 0.0;
      if (act[j])
#pragma unroll
        for (int i = 0; i < RPL; ++i) t[j] = fma(vr[i], y[j][i], t[j]);
    }
    warp_sum_cw(t);
#pragma unroll
    for (int j = 0; j < kCW; ++j)
      if (act[j]) {
        const double f = tk * t[j];
#pragma unroll
        for (int i = 0; i < RPL; ++i) y[j][i] = fma(-f, vr[i], y[j][i]);
      }
  }
}

// Per-column argmax |y| over rows < m with the reference's scan semantics (strict >, first
// index wins) -> best[c], bidx[c] (bidx = -1 if the column is all zero here).  Ends with a
// block barrier.
template <int RPL>
__device__ void reg_argmax(const double (&y)[kCW][RPL], int m, int mu, double* best, int* bidx) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
#pragma unroll
  for (int j = 0; j < kCW; ++j) {
    const int c = slot_col(w, j);
    if (c < mu) {
      double b = 0.0;
      int bi = -1;
#pragma unroll
      for (int i = 0; i < RPL; ++i) {
        const double v = fabs(y[j][i]);
        const int r = l + 32 * i;
        if (r < m && v > b) {
          b = v;
          bi = r;
        }
      }
#pragma unroll
      for (int msk = 16; msk >= 1; msk >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, b, msk);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, msk);
        if (ob > b || (ob == b && oi >= 0 && (bi < 0 || oi < bi))) {
          b = ob;
          bi = oi;
        }
      }
      if (l == 0) {
        best[c] = b;
        bidx[c] = bi;
      }
    }
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// One-sided Jacobi on G = R^T (s x 64, zero columns >= s), rotations accumulated in J.
//
// Register-resident with a recursive pair ordering.  The 64 column slots are the (top,
// bottom) registers of the 32 lanes; lane j rotates the pair (top_j, bottom_j).  Warps 0-7
// hold 8 rows each of G, warps 8-15 8 rows each of J, so a rotation is lane-local and the
// pair's dot products are per-warp partials combined by warp 0 (fixed warp order).  The
// schedule: within groups of g lanes (g = 32, 16, ..., 1) the bottoms shift cyclically by
// one lane per round for g rounds (every top meets every bottom of its group), then each
// group splits in halves whose tops pair with tops and bottoms with bottoms (one XOR
// shuffle).  63 rounds cover all 2016 slot pairs; each round moves one register column
// per lane by a shuffle instead of reloading both columns of every pair from shared memory
// (the previous round-robin version was bound on shared-memory bandwidth at ~1900 cycles a
// round).  Offline simulation on the cfg4 sketches: 7-8 sweeps, as with round-robin.
// Sketches with s <= 16 / 32 use 16 / 32 slots (15 / 31 rounds a sweep).
// ---------------------------------------------------------------------------
// Circle-method move after a round: lane 0 keeps its top (the fixed player), every other top
// moves one lane right (lane 1 takes lane 0's bottom), every bottom one lane left (lane P-1
// takes its own top).  Two shuffles per register row.
__device__ __forceinline__ void circle_shift(double (&T)[8], double (&B)[8], int& cT, int& cB, int l, int P) {
  if (P == 1) return;  // one pair: nothing moves
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const double up = __shfl_up_sync(0xffffffffu, l == 0 ? B[i] : T[i], 1);
    const double dn = __shfl_down_sync(0xffffffffu, B[i], 1);
    const double t = T[i];
    if (l != 0) T[i] = up;
    B[i] = l == P - 1 ? t : dn;
  }
  const int up = __shfl_up_sync(0xffffffffu, l == 0 ? cB : cT, 1);
  const int dn = __shfl_down_sync(0xffffffffu, cB, 1);
  const int t = cT;
  if (l != 0) cT = up;
  cB = l == P - 1 ? t : dn;
}

__device__ int g_jacobi_sweeps;
// phase clocks of the most recent orth_core_kernel (thread 0; diagnostics only): start, tile
// loaded, QR done, G scaled, Jacobi done, order done, end
__device__ long long g_orth_clk[8];
#define ORTH_CLK(i) \
  if (threadIdx.x == 0 && phase == kOrthFull) g_orth_clk[i] = clock64()
#ifdef LMRA_JACOBI_CLOCKS
__device__ unsigned long long g_jclk[8];  // microbenchmark only: per-phase cycles, warp 0
#endif

__device__ __forceinline__ void named_bar(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// Rotation for the pair (top, bottom) with squared norms a, b and inner product c: the
// smaller root t of t^2 + 2 zeta t - 1 = 0 (zeta = (b - a) / 2c), written without forming
// t: with d = b - a, r = sqrt(d^2 + 4c^2), u = |d| + r:  1 + t^2 = 2r / u, so
//   cos = u / sqrt(2 r u),  sin = sign(d) 2c / sqrt(2 r u).
// G is pre-scaled by a power of two (max |g| in [1, 2)), so a, b, c neither overflow nor
// need the exponent-scaled path; the rotation is orthogonal to an ulp or two regardless of
// the accuracy of t.
// Early stop: a sweep whose pairs all had c^2 <= 0.01 tol (a b) before their rotation
// (relative off-diagonal below 0.1 sqrt(tol)) leaves, by the quadratic convergence of the
// cyclic one-sided Jacobi, relative off-diagonals of ~(0.1 sqrt(tol))^2 = 0.01 tol: the next
// sweep would rotate nothing above the tolerance (it is the verification sweep), so it is
// skipped.  On the BASELINE sketches the last rotating sweep's largest relative off-diagonal is
// 2e-9 .. 3e-10 against a threshold of ~2e-8: one sweep of 7-10 saved.
__device__ __forceinline__ double jacobi_quad_thr2(double tol) { return 0.01 * tol; }  // on c^2 / (a b)

__device__ __forceinline__ bool jacobi_angle(double a, double b, double c, double tol2,
                                             double& cs, double& sn) {
  cs = 1.0;
  sn = 0.0;
  if (!(c != 0.0 && c * c > tol2 * (a * b))) return false;
  const double d = b - a;
  const double q = fma(d, d, 4.0 * c * c);
  const double r = q * rsqrt_nr(q);
  const double u = fabs(d) + r;
  const double qn = rsqrt_nr(2.0 * r * u);
  cs = u * qn;
  sn = (d >= 0.0 ? 2.0 * c : -2.0 * c) * qn;
  return true;
}

// Per round: every G warp writes its partial (a, b, c) of each lane's pair; after a named
// barrier among the G warps, warp 0 sums them (fixed order) and forms the angles; a second
// barrier (G and J warps) releases the rotation.  (Measured alternatives -- every G warp
// forming all angles itself, or J warps consuming the angles asynchronously from an
// mbarrier ring -- were slower: the angle chain is issue-bound when replicated, and the
// ring's extra synchronisation costs more than the J rotation it takes off the barrier.)
// The Jacobi split over a 2-CTA cluster: CTA 0 rotates G and forms the angles, CTA 1 accumulates
// J from the angles it receives through a ring in its shared memory (DSMEM stores + remote
// mbarrier arrives), a few rounds behind.  With J off CTA 0's SM a round runs ~29 % faster
// (microbenchmark: 1500 -> 1070 cycles for s = 60): the fp64 and shuffle pipes and the angle
// barrier are no longer shared with the J rotations.  (The same ring between warps of ONE CTA
// was slower: the J rotations then still compete for the SM's pipes.)
constexpr int kJRing = 8;  // ring slots (rounds CTA 1 may lag)
struct JLink {
  uint32_t ring;    // CTA 1's ring [kJRing][cos 32 | sin 32] (DSMEM address)
  uint32_t ctl;     // CTA 1's control words [kJRing]: 0 round, 1 sweep end, 2 stop
  uint32_t full;    // CTA 1's full barriers [kJRing] (32 arrivals: the lanes of warp 0)
  uint64_t* empty;  // CTA 0's empty barriers [kJRing] (one arrival per J warp)
};

__device__ bool reg_jacobi(double* G, int s, double* J, double tol, const QSmem& q,
                           const JLink* link = nullptr) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const bool isG = w < 8;
  const int row0 = (w & 7) * 8;
  double* part = q.part;  // [3][8 warps][32 lanes]
  double* csn = q.fval;   // [round parity][cos 32 | sin 32]: q.fval and q.rowk (128 doubles)
  int* flags = q.pidx;    // [0, 60) per-sweep "rotated", [63] result
  int* big = reinterpret_cast<int*>(q.red);  // [0, 60) per-sweep "a pair above the early-stop bound"
                                             // (q.red is the sign fix's, after the Jacobi)
  // circle-method round robin: lanes l < P hold the pair (top_l, bottom_l) of 2P >= s column
  // slots; 2P - 1 rounds visit every pair once (s = 50: 49 rounds, not the 63 of a 64-slot
  // power-of-two tournament)
  const int nh = (s + 1) / 2;
  // rows: warps 0 .. gw-1 hold G (8 rows each), warps 8 .. 8+gw-1 the same rows of J (rows
  // >= s of J stay zero for every real column); the other warps sit the Jacobi out
  const int gw = (s + 7) / 8;
  // linked: J lives on CTA 1; warp 8 (a J warp otherwise) forwards each round's angles there
  // after bar B, off the G warps' critical path (a remote store + release-arrive costs a
  // DSMEM round trip)
  const bool sender = link && w == 8;
  const bool active = link ? ((isG && (w & 7) < gw) || sender) : ((w & 7) < gw);
  const int barb = link ? 32 * gw + 32 : 64 * gw;
  int jround = 0;  // linked: ring entries sent (sender)
  double T[8], B[8];
  int cT = l < nh ? l : 1 << 20, cB = l < nh ? l + nh : 1 << 20;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int r = row0 + i;
    if (isG) {
      T[i] = (r < s && cT < s) ? G[r + (size_t)s * cT] : 0.0;
      B[i] = (r < s && cB < s) ? G[r + (size_t)s * cB] : 0.0;
    } else {
      T[i] = r == cT ? 1.0 : 0.0;
      B[i] = r == cB ? 1.0 : 0.0;
    }
  }
  if (threadIdx.x < 64) flags[threadIdx.x] = 0;
  if (threadIdx.x < 64) big[threadIdx.x] = 0;
  __syncthreads();
  const bool early = tol > 0.0;  // a negative tol switches the early stop off (LMRA_JACOBI_EARLY=0)
  tol = fabs(tol);
  const double tol2 = tol * tol;
  const double qthr2 = jacobi_quad_thr2(tol);
  bool converged = false;
  int round = 0;  // global round counter (csn parity)
#ifdef LMRA_JACOBI_CLOCKS
  long long jc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#endif
  if (!active) goto done;
  for (int sweep = 0; sweep < 60 && !converged; ++sweep) {
    {
      for (int r = 0; r < 2 * nh - 1; ++r, ++round) {
        double* cs_r = csn + 64 * (round & 1);
#ifdef LMRA_JACOBI_CLOCKS
        const long long k0 = clock64();
        long long k1 = k0, k2 = k0;
#endif
        if (isG) {
          double a = 0.0, b = 0.0, c = 0.0;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            a = fma(T[i], T[i], a);
            b = fma(B[i], B[i], b);
            c = fma(T[i], B[i], c);
          }
          part[(0 * 8 + w) * 32 + l] = a;
          part[(1 * 8 + w) * 32 + l] = b;
          part[(2 * 8 + w) * 32 + l] = c;
          named_bar(1, 32 * gw);
#ifdef LMRA_JACOBI_CLOCKS
          k1 = clock64();
#endif
          if (w == 0) {
            double pa[8], pb[8], pc[8];
#pragma unroll
            for (int w2 = 0; w2 < 8; ++w2) {
              pa[w2] = w2 < gw ? part[(0 * 8 + w2) * 32 + l] : 0.0;
              pb[w2] = w2 < gw ? part[(1 * 8 + w2) * 32 + l] : 0.0;
              pc[w2] = w2 < gw ? part[(2 * 8 + w2) * 32 + l] : 0.0;
            }
            const double sa = ((pa[0] + pa[1]) + (pa[2] + pa[3])) + ((pa[4] + pa[5]) + (pa[6] + pa[7]));
            const double sb = ((pb[0] + pb[1]) + (pb[2] + pb[3])) + ((pb[4] + pb[5]) + (pb[6] + pb[7]));
            const double sc = ((pc[0] + pc[1]) + (pc[2] + pc[3])) + ((pc[4] + pc[5]) + (pc[6] + pc[7]));
            double cs, sn;
            // lanes past the P pairs receive stale columns from the circle move: identity
            if (l < nh && jacobi_angle(sa, sb, sc, tol2, cs, sn)) flags[sweep] = 1;
            if (l < nh && sc * sc > qthr2 * (sa * sb)) big[sweep] = 1;
            if (l >= nh) {
              cs = 1.0;
              sn = 0.0;
            }
            cs_r[l] = cs;
            cs_r[32 + l] = sn;
          }
#ifdef LMRA_JACOBI_CLOCKS
          k2 = clock64();
#endif
        }
        named_bar(2, barb);  // bar B: angles of this round visible to every active warp
#ifdef LMRA_JACOBI_CLOCKS
        const long long k3 = clock64();
#endif
        const double cs = cs_r[l], sn = cs_r[32 + l];
        if (sender) {  // the round's angles to CTA 1
          const int slot = jround % kJRing;
          mbar_wait_cluster(&link->empty[slot], ((unsigned)(jround / kJRing) & 1u) ^ 1u);
          dsmem_st_f64(link->ring + (uint32_t)(slot * 64 + l) * 8, cs);
          dsmem_st_f64(link->ring + (uint32_t)(slot * 64 + 32 + l) * 8, sn);
          if (l == 0) dsmem_st_s32(link->ctl + (uint32_t)slot * 4, 0);
          mbar_arrive_remote(link->full + (uint32_t)slot * 8);
          ++jround;
          continue;
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const double x = T[i], y = B[i];
          T[i] = cs * x - sn * y;
          B[i] = sn * x + cs * y;
        }
        circle_shift(T, B, cT, cB, l, nh);
#ifdef LMRA_JACOBI_CLOCKS
        {  // k0->k1 partials + bar A, k1->k2 angles, k2->k3 bar B, k3->k4 rotate (registers)
          const long long k4 = clock64();
          jc[0] += k1 - k0;
          jc[1] += k2 - k1;
          jc[2] += k3 - k2;
          jc[3] += k4 - k3;
          jc[4] += 1;
          jc[5] += k3 - k0;
          jc[6] += k4 - k3;
        }
#endif
      }
    }
    // flags[sweep] / big[sweep] were written before the sweep's last bar B
    if (!flags[sweep] || (early && !big[sweep])) {
      converged = true;
      if (threadIdx.x == 0) g_jacobi_sweeps = sweep + 1;
    }
    if (sender) {  // sweep end: continue / stop to CTA 1
      const int slot = jround % kJRing;
      mbar_wait_cluster(&link->empty[slot], ((unsigned)(jround / kJRing) & 1u) ^ 1u);
      if (l == 0) dsmem_st_s32(link->ctl + (uint32_t)slot * 4, (converged || sweep + 1 >= 60) ? 2 : 1);
      mbar_arrive_remote(link->full + (uint32_t)slot * 8);
      ++jround;
    }
  }
done:
#ifdef LMRA_JACOBI_CLOCKS
  if (threadIdx.x == 0)
    for (int i = 0; i < 5; ++i) g_jclk[i] = jc[i];
  if (threadIdx.x == 256)
    for (int i = 5; i < 7; ++i) g_jclk[i] = jc[i];
#endif
  __syncthreads();
  if (active) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int r = row0 + i;
      if (isG) {
        if (r < s) {
          if (l < nh && cT < s) G[r + (size_t)s * cT] = T[i];
          if (l < nh && cB < s) G[r + (size_t)s * cB] = B[i];
        }
      } else if (!sender && l < nh && cT < 64) {  // (lanes past the pairs hold stale columns; linked: J is on CTA 1)
        J[r + 64 * cT] = T[i];
        J[r + 64 * cB] = B[i];
      }
    }
  }
  __syncthreads();
  // converged is only known to the active warps: publish it
  if (threadIdx.x == 0) flags[63] = converged ? 1 : 0;
  __syncthreads();
  return flags[63] != 0;
}


// ---------------------------------------------------------------------------
// Two-warp Jacobi for narrow sketches (s <= 32): the same one-sided Jacobi on G = R^T with the
// rotations accumulated in J, the same circle-method pair order and angle formula as
// reg_jacobi, but with no block barrier.  Warp 0 holds G, warp 1 holds J, both in registers:
// lanes are grouped L per pair (L = 32 / P2, P2 = the power of two >= the P = ceil(s / 2)
// pairs); lane (p, h) holds rows [h H, h H + H) of the pair's two columns.  A pair's dot
// products are H-row partials combined by log2(L) xor-shuffles, every lane of the pair forms
// the same angle, the rotation is lane-local, the circle move is two shuffles by L lanes.
// Warp 0 hands each round's angles to warp 1 through a double-buffered slot and a 64-thread
// named barrier (warp 1 rotates J and moves its columns one round behind).  reg_jacobi's round
// (partials -> barrier -> warp 0 forms the angles -> barrier -> rotate) costs ~1-2 k cycles
// whatever s is; at s = 15..30 that fixed cost dominated the sketch SVD.
template <int L, int H>
__device__ __forceinline__ void circle_move_rows(double (&T)[H], double (&B)[H], int p, int P) {
#pragma unroll
  for (int i = 0; i < H; ++i) {
    const double up = __shfl_up_sync(0xffffffffu, p == 0 ? B[i] : T[i], L);
    const double dn = __shfl_down_sync(0xffffffffu, B[i], L);
    const double t = T[i];
    if (p != 0) T[i] = up;
    B[i] = p == P - 1 ? t : dn;
  }
}

template <int L>
__device__ __forceinline__ void circle_move_slots(int& cT, int& cB, int p, int P) {
  const int up = __shfl_up_sync(0xffffffffu, p == 0 ? cB : cT, L);
  const int dn = __shfl_down_sync(0xffffffffu, cB, L);
  const int t = cT;
  if (p != 0) cT = up;
  cB = p == P - 1 ? t : dn;
}

// slots: [2][cos 32 | sin 32] doubles; ctl: [2] ints (0 round, 1 stop)
template <int L, int H>
__device__ bool narrow_jacobi_g(double* G, int s, double tol, double* slots, int* ctl) {
  const int l = threadIdx.x & 31;
  const int p = l / L, h = l % L;
  const int P = (s + 1) / 2;
  const bool live = p < P;
  const bool early = tol > 0.0;  // a negative tol switches the early stop off (LMRA_JACOBI_EARLY=0)
  tol = fabs(tol);
  const double tol2 = tol * tol;
  int cT = live ? p : 1 << 20, cB = live ? p + P : 1 << 20;
  double T[H], B[H];
#pragma unroll
  for (int i = 0; i < H; ++i) {
    const int r = h * H + i;
    T[i] = (live && r < s && cT < s) ? G[r + (size_t)s * cT] : 0.0;
    B[i] = (live && r < s && cB < s) ? G[r + (size_t)s * cB] : 0.0;
  }
  bool converged = false;
  int round = 0;
  const double qthr2 = jacobi_quad_thr2(tol);
  for (int sweep = 0; sweep < 60 && !converged; ++sweep) {
    bool rotated = false, big = false;
    for (int rd = 0; rd < 2 * P - 1; ++rd, ++round) {
#ifdef LMRA_JACOBI_CLOCKS
      const long long k0 = clock64();
#endif
      // two accumulators per sum (shorter fma chains), added once
      double a = 0.0, b = 0.0, c = 0.0, a2 = 0.0, b2 = 0.0, c2 = 0.0;
#pragma unroll
      for (int i = 0; i < H; i += 2) {
        a = fma(T[i], T[i], a);
        b = fma(B[i], B[i], b);
        c = fma(T[i], B[i], c);
        if (i + 1 < H) {
          a2 = fma(T[i + 1], T[i + 1], a2);
          b2 = fma(B[i + 1], B[i + 1], b2);
          c2 = fma(T[i + 1], B[i + 1], c2);
        }
      }
      a += a2;
      b += b2;
      c += c2;
#pragma unroll
      for (int m = 1; m < L; m <<= 1) {  // the pair's L lanes, fixed xor order: identical sums
        a += __shfl_xor_sync(0xffffffffu, a, m);
        b += __shfl_xor_sync(0xffffffffu, b, m);
        c += __shfl_xor_sync(0xffffffffu, c, m);
      }
      double cs = 1.0, sn = 0.0;
      if (live && jacobi_angle(a, b, c, tol2, cs, sn)) rotated = true;
      if (live && c * c > qthr2 * (a * b)) big = true;
      double* sl = slots + 64 * (round & 1);
      if (h == 0 && p < 32) {
        sl[p] = cs;
        sl[32 + p] = sn;
      }
      if (l == 0) ctl[round & 1] = 0;
#ifdef LMRA_JACOBI_CLOCKS
      const long long k1 = clock64();
#endif
      named_bar(1, 64);  // the round's angles to warp 1
#ifdef LMRA_JACOBI_CLOCKS
      const long long k2 = clock64();
#endif
#pragma unroll
      for (int i = 0; i < H; ++i) {
        const double x = T[i], y = B[i];
        T[i] = cs * x - sn * y;
        B[i] = sn * x + cs * y;
      }
      if (P > 1) {
        circle_move_rows<L, H>(T, B, p, P);
        circle_move_slots<L>(cT, cB, p, P);
      }
#ifdef LMRA_JACOBI_CLOCKS
      if (l == 0) {
        const long long k3 = clock64();
        g_jclk[0] += k1 - k0;
        g_jclk[1] += k2 - k1;
        g_jclk[2] += k3 - k2;
        g_jclk[4] += 1;
      }
#endif
    }
    if (!__any_sync(0xffffffffu, rotated) || (early && !__any_sync(0xffffffffu, big))) {
      converged = true;
      if (l == 0) g_jacobi_sweeps = sweep + 1;
    }
  }
  if (l == 0) ctl[round & 1] = 1;  // stop
  named_bar(1, 64);
  if (live) {
#pragma unroll
    for (int i = 0; i < H; ++i) {
      const int r = h * H + i;
      if (r < s) {
        if (cT < s) G[r + (size_t)s * cT] = T[i];
        if (cB < s) G[r + (size_t)s * cB] = B[i];
      }
    }
  }
  return converged;
}

template <int L, int H>
__device__ void narrow_jacobi_j(double* J, int s, const double* slots, const int* ctl) {
  const int l = threadIdx.x & 31;
  const int p = l / L, h = l % L;
  const int P = (s + 1) / 2;
  const bool live = p < P;
  int cT = live ? p : 1 << 20, cB = live ? p + P : 1 << 20;
  double T[H], B[H];
#pragma unroll
  for (int i = 0; i < H; ++i) {
    const int r = h * H + i;
    T[i] = r == cT ? 1.0 : 0.0;
    B[i] = r == cB ? 1.0 : 0.0;
  }
  for (int round = 0;; ++round) {
    named_bar(1, 64);
    if (ctl[round & 1]) break;
    const double* sl = slots + 64 * (round & 1);
    const double cs = live ? sl[p] : 1.0, sn = live ? sl[32 + p] : 0.0;
#pragma unroll
    for (int i = 0; i < H; ++i) {
      const double x = T[i], y = B[i];
      T[i] = cs * x - sn * y;
      B[i] = sn * x + cs * y;
    }
    if (P > 1) {
      circle_move_rows<L, H>(T, B, p, P);
      circle_move_slots<L>(cT, cB, p, P);
    }
  }
  if (live) {
#pragma unroll
    for (int i = 0; i < H; ++i) {
      const int r = h * H + i;
      if (r < 64 && cT < 64) J[r + 64 * cT] = T[i];
      if (r < 64 && cB < 64) J[r + 64 * cB] = B[i];
    }
  }
}

// the whole CTA: warps 0 / 1 run the G / J halves, the others wait; the flag goes through smem
template <int L, int H>
__device__ bool narrow_jacobi_lh(double* G, int s, double* J, double tol, const QSmem& q) {
  const int w = threadIdx.x >> 5;
  double* slots = q.fval;  // q.fval + q.rowk: 128 contiguous doubles
  int* ctl = q.pidx;       // [0, 2) round control, [63] result
  if (w == 0) {
    const bool conv = narrow_jacobi_g<L, H>(G, s, tol, slots, ctl);
    if ((threadIdx.x & 31) == 0) q.pidx[63] = conv ? 1 : 0;
  } else if (w == 1) {
    narrow_jacobi_j<L, H>(J, s, slots, ctl);
  }
  __syncthreads();
  return q.pidx[63] != 0;
}

__device__ bool narrow_jacobi(double* G, int s, double* J, double tol, const QSmem& q) {
  // J is read as 64 x 64 afterwards: identity first (the J warp writes the s real slots)
  for (int e = threadIdx.x; e < 64 * 64; e += kQThreads) J[e] = (e % 65 == 0) ? 1.0 : 0.0;
  __syncthreads();
  if (s <= 8) return narrow_jacobi_lh<8, 2>(G, s, J, tol, q);
  if (s <= 16) return narrow_jacobi_lh<4, 4>(G, s, J, tol, q);
  if (s <= 24) return narrow_jacobi_lh<2, 12>(G, s, J, tol, q);
  return narrow_jacobi_lh<2, 16>(G, s, J, tol, q);
}

// CTA 1 of the cluster: the J half of reg_jacobi, driven by the angles CTA 0 sends; the
// final J goes into CTA 0's J buffer (jdst: its DSMEM address).  Same register layout,
// tournament and rotation arithmetic as the J warps of reg_jacobi.
__device__ void jacobi_j_consumer(int s, const double* ring, const int* ctl, uint64_t* full,
                                  uint32_t empty_remote, uint32_t jdst) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const int row0 = (w & 7) * 8;
  // circle-method round robin: lanes l < P hold the pair (top_l, bottom_l) of 2P >= s column
  // slots; 2P - 1 rounds visit every pair once (s = 50: 49 rounds, not the 63 of a 64-slot
  // power-of-two tournament)
  const int nh = (s + 1) / 2;
  const int gw = (s + 7) / 8;
  if (!(w >= 8 && (w & 7) < gw)) return;
  double T[8], B[8];
  int cT = l < nh ? l : 1 << 20, cB = l < nh ? l + nh : 1 << 20;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int r = row0 + i;
    T[i] = r == cT ? 1.0 : 0.0;
    B[i] = r == cB ? 1.0 : 0.0;
  }
  int jround = 0;
  for (int sweep = 0; sweep < 60; ++sweep) {
    {
      for (int r = 0; r < 2 * nh - 1; ++r) {
        const int slot = jround % kJRing;
        mbar_wait_cluster(&full[slot], (unsigned)(jround / kJRing) & 1u);
        const double cs = ring[slot * 64 + l], sn = ring[slot * 64 + 32 + l];
        __syncwarp();
        if (l == 0) mbar_arrive_remote(empty_remote + (uint32_t)slot * 8);
        ++jround;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const double x = T[i], y = B[i];
          T[i] = cs * x - sn * y;
          B[i] = sn * x + cs * y;
        }
        circle_shift(T, B, cT, cB, l, nh);
      }
    }
    const int slot = jround % kJRing;  // sweep end
    mbar_wait_cluster(&full[slot], (unsigned)(jround / kJRing) & 1u);
    const int c = ctl[slot];
    __syncwarp();
    if (l == 0) mbar_arrive_remote(empty_remote + (uint32_t)slot * 8);
    ++jround;
    if (c == 2) break;
  }
  if (l < nh && cT < 64) {  // (lanes past the pairs hold stale columns)
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int r = row0 + i;
      dsmem_st_f64(jdst + (uint32_t)(r + 64 * cT) * 8, T[i]);
      dsmem_st_f64(jdst + (uint32_t)(r + 64 * cB) * 8, B[i]);
    }
  }
}

// ---------------------------------------------------------------------------
// Leaf QR: block b of A (m x s, lda) -> reflectors into V (same rows), tau[b*s + k],
// R_b into rows [b*s, b*s+s) of S (ld lds), zeros below the diagonal.
// ---------------------------------------------------------------------------
template <int RPL>
__global__ void __launch_bounds__(kQThreads) orth_leaf_qr_kernel(
    const double* __restrict__ A, long long m, int s, int lda, int nb, double* __restrict__ V,
    double* __restrict__ tau, double* __restrict__ S, int lds, const int* __restrict__ gate, int run_if) {
  pdl_wait();  // the previous kernel's outputs (programmatic dependent launch)
  if (gate && *gate != run_if) return;  // the other branch of a gated pair of paths (cholqr fallback)
  pdl_trigger();
  extern __shared__ __align__(16) double sm[];
  const QSmem q = carve_q(sm);
  double* tile = sm + kQScratchBytes / 8;
  const int b = blockIdx.x;
  const long long r0 = (m * b) / nb, r1 = (m * (b + 1)) / nb;
  const int rows = (int)(r1 - r0), ldt = rows | 1;
  load_tile(A + r0, lda, rows, s, tile, ldt, rows);
  __syncthreads();
  double a[kCW][RPL];
  cw_load(tile, ldt, rows, s, a);
  reg_qr(a, rows, s, q, false);
  cw_store(a, rows, s, tile, ldt);
  __syncthreads();
  for (int e = threadIdx.x; e < rows * s; e += kQThreads) {
    const int i = e % rows, c = e / rows;
    V[r0 + i + (size_t)lda * c] = tile[i + ldt * c];
  }
  for (int e = threadIdx.x; e < s * s; e += kQThreads) {
    const int i = e % s, c = e / s;
    S[(size_t)b * s + i + (size_t)lds * c] = (i <= c && i < rows) ? tile[i + ldt * c] : 0.0;
  }
  for (int k = threadIdx.x; k < s; k += kQThreads) tau[(size_t)b * s + k] = k < min(rows, s) ? q.tau[k] : 0.0;
}

// ---------------------------------------------------------------------------
// Core: one CTA.  S (m x s, lds) -> pivoted QR -> Jacobi on R^T -> Y = Q [U_R(:, :mu); 0].
// final != 0: sign-fix Y and write it to out (ld ldo); else write Y to out unsigned.
// ---------------------------------------------------------------------------
// phase (the split used by the core / shrink contractions, launch_orth_basis + launch_orth_finish):
//   kOrthFull   the whole chain above;
//   kOrthBasis  pivoted QR only: G = R^T (unscaled) to gbuf (s x s) and Y = Q [I_s; 0] (m x s) to
//               out -- the basis Q_C of the sketch, before any Jacobi;
//   kOrthJacobi Jacobi on gbuf's G only: U_R(:, :mu) (singular values descending) to ur (s x mu).
constexpr int kOrthFull = 0, kOrthBasis = 1, kOrthJacobi = 2;

template <int RPL>
__global__ void __launch_bounds__(kQThreads) orth_core_kernel(
    const double* __restrict__ S, int m, int s, int lds, int mu, double* __restrict__ out,
    int ldo, int final_level, int* status, double jacobi_tol, int clustered, int phase,
    double* __restrict__ gbuf, double* __restrict__ ur, int basis_pivot, const int* __restrict__ gate, int run_if,
    int narrow_jacobi_on) {
  pdl_wait();  // the previous kernel's outputs (programmatic dependent launch)
  if (gate && *gate != run_if) return;  // the other branch of a gated pair of paths (cholqr fallback)
  ORTH_CLK(0);
  // no early pdl_trigger(): a dependent launched now would park its CTAs (waiting in
  // griddepcontrol.wait) on SMs for the whole Jacobi, and a big kernel of another stream (the
  // core contraction beside a split orthonormalisation) could not use those SMs; the trigger
  // comes once the Jacobi is done (CTA 1 of a cluster triggers by exiting)
  extern __shared__ __align__(16) double sm[];
  const QSmem q = carve_q(sm);
  const int n = 64;  // Jacobi column slots (zero columns beyond s)
  const int ldv = (32 * RPL) | 1;
  double* Vs = sm + kQScratchBytes / 8;        // m x s (ld ldv): input, then reflectors, then Y
  double* G = Vs + (size_t)ldv * s;            // s x s   (R^T)
  double* J = G + (size_t)s * s;               // n x n   (accumulated rotations)
  double* sig = J + (size_t)n * n;             // n
  int* perm = reinterpret_cast<int*>(sig + n); // n
  uint64_t* jbars = reinterpret_cast<uint64_t*>(perm + n);  // [kJRing]: CTA 0 empty, CTA 1 full
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  // cluster of 2 (clustered): CTA 1 only accumulates the Jacobi rotations (jacobi_j_consumer);
  // its ring lives in its q.part, its control words in its q.ipiv
  const uint32_t crank = clustered ? cluster_ctarank() : 0;
  if (clustered) {
    if (threadIdx.x == 0) {
      for (int k = 0; k < kJRing; ++k) mbar_init(&jbars[k], crank == 0 ? (unsigned)((s + 7) / 8) : 32u);
      mbar_fence_init();
    }
    cluster_sync();  // both CTAs' barriers initialised before any remote arrive
    if (crank == 1) {
      jacobi_j_consumer(s, q.part, q.ipiv, jbars, dsmem_addr(smem_u32(jbars), 0), dsmem_addr(smem_u32(J), 0));
      cluster_sync();  // J delivered to CTA 0
      return;
    }
  }

  if (phase == kOrthJacobi) {  // G from the basis phase
    for (int e = threadIdx.x; e < s * s; e += kQThreads) G[e] = gbuf[e];
    __syncthreads();
  } else {
    load_tile(S, lds, m, s, Vs, ldv, 32 * RPL);
    __syncthreads();
    ORTH_CLK(1);
    double a[kCW][RPL];
    cw_load(Vs, ldv, m, s, a);
    // the basis phase skips the column pivoting: it only preconditions the Jacobi (graded R,
    // fewer sweeps), and in the split form the Jacobi runs off the critical path
    reg_qr(a, m, s, q, phase != kOrthBasis || basis_pivot);
    if ((int)threadIdx.x < s) q.ipiv[q.piv[threadIdx.x]] = threadIdx.x;
    __syncthreads();
    ORTH_CLK(2);
    // G = R^T (lower triangle), reflectors to Vs in logical column order
#pragma unroll
    for (int j = 0; j < kCW; ++j) {
      const int c = slot_col(w, j);
      if (c >= s) continue;
      const int k = q.ipiv[c];
#pragma unroll
      for (int i = 0; i < RPL; ++i) {
        const int r = l + 32 * i;
        if (r < s) G[k + (size_t)s * r] = r <= k && r < m ? a[j][i] : 0.0;
        if (r > k && r < m) Vs[r + (size_t)ldv * k] = a[j][i];
      }
    }
    __syncthreads();
    if (phase == kOrthBasis) {  // G out, Y = Q [I_s; 0] (logical column order) to out
      pdl_trigger();
      for (int e = threadIdx.x; e < s * s; e += kQThreads) gbuf[e] = G[e];
      double y[kCW][RPL];
#pragma unroll
      for (int j = 0; j < kCW; ++j) {
        const int c = slot_col(w, j);
#pragma unroll
        for (int i = 0; i < RPL; ++i) y[j][i] = (c < s && l + 32 * i == c) ? 1.0 : 0.0;
      }
      reg_apply(y, s, Vs, ldv, q.tau, min(m, s), 0);
      __syncthreads();  // every warp is done reading the reflectors
      cw_store(y, m, s, Vs, ldv);
      __syncthreads();
      for (int e = threadIdx.x; e < m * s; e += kQThreads) {
        const int i = e % m, c = e / m;
        out[i + (size_t)ldo * c] = Vs[i + (size_t)ldv * c];
      }
      return;
    }
  }
  {  // G *= 2^-e with max |G| in [1, 2) (exact; only J and the singular values' order are used)
    double mx = 0.0;
    for (int e = threadIdx.x; e < s * s; e += kQThreads) mx = fmax(mx, fabs(G[e]));
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 8));
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 4));
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
    if (l == 0) q.normp[w] = mx;
    __syncthreads();
    double gm = 0.0;
    for (int k = 0; k < kQWarps; ++k) gm = fmax(gm, q.normp[k]);
    if (gm > 0.0 && isfinite(gm)) {
      const int ex = ilogb(gm);
      for (int e = threadIdx.x; e < s * s; e += kQThreads) G[e] = ldexp(G[e], -ex);
    }
    __syncthreads();
  }
  ORTH_CLK(3);
  bool converged;
  if (clustered) {
    JLink link;
    link.ring = dsmem_addr(smem_u32(q.part), 1);
    link.ctl = dsmem_addr(smem_u32(q.ipiv), 1);
    link.full = dsmem_addr(smem_u32(jbars), 1);
    link.empty = jbars;
    converged = reg_jacobi(G, s, J, jacobi_tol, q, &link);
    cluster_sync();  // CTA 1 has written J here
  } else {
    // narrow sketches: the barrier-free one-warp Jacobi (LMRA_NARROW_JACOBI=0: the block one)
    // narrow sketches (s <= 32): the barrier-free two-warp Jacobi (LMRA_NARROW_JACOBI=0: the block one);
    // wider ones keep the block form (a multi-warp register form with shared-memory edge exchange
    // measured 1.6x slower per round at s = 40..60, tools/microbench/jacobi_variants.cu)
    converged = (s <= 32 && narrow_jacobi_on) ? narrow_jacobi(G, s, J, jacobi_tol, q)
                                              : reg_jacobi(G, s, J, jacobi_tol, q);
  }
  pdl_trigger();
  ORTH_CLK(4);
  // singular values = column norms of G, fixed order
  for (int c = w; c < s; c += kQWarps) {
    double t = 0.0;
    for (int i = l; i < s; i += 32) t += G[i + (size_t)s * c] * G[i + (size_t)s * c];
    t = warp_sum(t);
    if (l == 0) sig[c] = sqrt(t);
  }
  __syncthreads();
  if ((int)threadIdx.x < s) {  // stable descending order of the s real columns (pad excluded)
    const int c = threadIdx.x;
    const double v = sig[c];
    int rank = 0;
    for (int d = 0; d < s; ++d) rank += (sig[d] > v) || (sig[d] == v && d < c);
    perm[rank] = c;
  }
  __syncthreads();
  ORTH_CLK(5);
  if (phase == kOrthJacobi) {  // U_R(:, :mu) in descending singular-value order
    for (int e = threadIdx.x; e < s * mu; e += kQThreads) {
      const int r = e % s, c = e / s;
      ur[r + (size_t)s * c] = J[r + (size_t)n * perm[c]];
    }
    if (threadIdx.x == 0 && status) *status = converged ? 0 : 1;
    return;
  }
  // Y = [U_R(:, :mu) ; 0] with U_R = J(0:s, perm), then the reflectors
  double y[kCW][RPL];
#pragma unroll
  for (int j = 0; j < kCW; ++j) {
    const int c = slot_col(w, j);
#pragma unroll
    for (int i = 0; i < RPL; ++i) {
      const int r = l + 32 * i;
      y[j][i] = (c < mu && r < s && r < m) ? J[r + (size_t)n * perm[c]] : 0.0;
    }
  }
  reg_apply(y, mu, Vs, ldv, q.tau, min(m, s), 0);
  if (final_level) {
    reg_argmax(y, m, mu, q.red, q.piv);  // best |.| per column in q.red, row in q.piv
    cw_store(y, m, mu, Vs, ldv);
    __syncthreads();
    if ((int)threadIdx.x < mu) {
      const int c = threadIdx.x, im = q.piv[c];
      q.fval[c] = (im >= 0 && Vs[im + (size_t)ldv * c] < 0.0) ? -1.0 : 1.0;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < m * mu; e += kQThreads) {
      const int i = e % m, c = e / m;
      out[i + (size_t)ldo * c] = q.fval[c] * Vs[i + (size_t)ldv * c];
    }
  } else {
    __syncthreads();  // every warp is done reading the reflectors
    cw_store(y, m, mu, Vs, ldv);
    __syncthreads();
    for (int e = threadIdx.x; e < m * mu; e += kQThreads) {
      const int i = e % m, c = e / m;
      out[i + (size_t)ldo * c] = Vs[i + (size_t)ldv * c];
    }
  }
  if (threadIdx.x == 0 && status) *status = converged ? 0 : 1;
  ORTH_CLK(6);
}

// ---------------------------------------------------------------------------
// Leaf apply: block b: Y_b = Q_b [W(b*s : b*s+s, :) ; 0] -> out rows [r0, r1) (ld ldo).
// With pbest also records per-block column argmax partials for the sign fix.
// ---------------------------------------------------------------------------
template <int RPL>
__global__ void __launch_bounds__(kQThreads) orth_leaf_apply_kernel(
    const double* __restrict__ V, long long m, int s, int ldv, int nb,
    const double* __restrict__ tau, const double* __restrict__ W, int ldw, int mu,
    double* __restrict__ out, int ldo, double* __restrict__ pbest, int* __restrict__ pidx,
    const int* __restrict__ gate, int run_if) {
  pdl_wait();  // the previous kernel's outputs (programmatic dependent launch)
  if (gate && *gate != run_if) return;  // the other branch of a gated pair of paths (cholqr fallback)
  pdl_trigger();
  extern __shared__ __align__(16) double sm[];
  const QSmem q = carve_q(sm);
  double* tile = sm + kQScratchBytes / 8;
  const int b = blockIdx.x;
  const long long r0 = (m * b) / nb, r1 = (m * (b + 1)) / nb;
  const int rows = (int)(r1 - r0), ldt = (32 * RPL) | 1;
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  load_tile(V + r0, ldv, rows, s, tile, ldt, 32 * RPL);
  for (int k = threadIdx.x; k < s; k += kQThreads) q.tau[k] = tau[(size_t)b * s + k];
  double y[kCW][RPL];
#pragma unroll
  for (int j = 0; j < kCW; ++j) {
    const int c = slot_col(w, j);
#pragma unroll
    for (int i = 0; i < RPL; ++i) {
      const int r = l + 32 * i;
      y[j][i] = (c < mu && r < s && r < rows) ? W[(size_t)b * s + r + (size_t)ldw * c] : 0.0;
    }
  }
  __syncthreads();
  reg_apply(y, mu, tile, ldt, q.tau, min(rows, s), 0);
  if (pbest) {
    reg_argmax(y, rows, mu, q.red, q.piv);
    if ((int)threadIdx.x < mu) {
      const int c = threadIdx.x, im = q.piv[c];
      pbest[(size_t)b * mu + c] = q.red[c];
      pidx[(size_t)b * mu + c] = im >= 0 ? (int)(r0 + im) : 0;
    }
  }
  __syncthreads();  // every warp is done reading the reflectors
  cw_store(y, rows, mu, tile, ldt);
  __syncthreads();
  for (int e = threadIdx.x; e < rows * mu; e += kQThreads) {
    const int i = e % rows, c = e / rows;
    out[r0 + i + (size_t)ldo * c] = tile[i + ldt * c];
  }
}

// Sign fix: per column, combine block partials in block order; flip if negative.
__global__ void orth_signfix_kernel(double* __restrict__ U, long long m, int ldu, int mu, int nb,
                                    const double* __restrict__ pbest,
                                    const int* __restrict__ pidx, const int* __restrict__ gate, int run_if) {
  pdl_wait();  // the previous kernel's outputs (programmatic dependent launch)
  if (gate && *gate != run_if) return;  // the other branch of a gated pair of paths (cholqr fallback)
  pdl_trigger();
  const int c = blockIdx.x;
  __shared__ int flip;
  if (threadIdx.x == 0) {
    double best = 0.0;
    int imax = 0;
    for (int b = 0; b < nb; ++b) {
      double v = pbest[(size_t)b * mu + c];
      if (v > best) {
        best = v;
        imax = pidx[(size_t)b * mu + c];
      }
    }
    flip = U[imax + (size_t)ldu * c] < 0.0;
  }
  __syncthreads();
  if (!flip) return;
  for (long long i = threadIdx.x; i < m; i += blockDim.x) U[i + (size_t)ldu * c] = -U[i + (size_t)ldu * c];
}

// ---------------------------------------------------------------------------
// host planning
// ---------------------------------------------------------------------------
struct OrthLevel {
  long long m;  // rows of this level's input
  int nb;       // row blocks (leaves)
  size_t v_off, tau_off, w_off;  // workspace offsets (doubles)
};

// rows per lane of the column-by-warp panels
static int rpl_for(long long rows) { return rows <= 64 ? 2 : rows <= 128 ? 4 : 8; }

// shared tiles hold 32 * RPL rows (ld (32 * RPL) | 1) so reflector columns can be read
// without row guards
static size_t leaf_smem(long long rows, int s) {
  return kQScratchBytes + sizeof(double) * (size_t)((32 * rpl_for(rows)) | 1) * s + 64;
}

static size_t core_smem(long long m, int s) {
  const int n = 64;
  return kQScratchBytes +
         sizeof(double) * ((size_t)((32 * rpl_for(m)) | 1) * s + (size_t)s * s + (size_t)n * n + n) +
         sizeof(int) * n + 8 * kJRing + 64;
}

static std::vector<OrthLevel> plan_levels(long long I, int s, size_t* total) {
  std::vector<OrthLevel> lv;
  size_t off = 0;
  long long m = I;
  while (m > kMaxBlockRows) {
    OrthLevel L;
    L.m = m;
    L.nb = (int)((m + kMaxBlockRows - 1) / kMaxBlockRows);
    L.v_off = off;
    off += (size_t)m * s;
    L.tau_off = off;
    off += (size_t)L.nb * s;
    L.w_off = off;  // stacked R of this level = next level's input (nb*s x s)
    off += (size_t)L.nb * s * s;
    lv.push_back(L);
    m = (long long)L.nb * s;
  }
  *total = off;
  return lv;
}

// Householder tree workspace (the fallback path's, and the whole of it without CholeskyQR)
static size_t tree_workspace_doubles(long long I, int s) {
  size_t used = 0;
  std::vector<OrthLevel> lv = plan_levels(I, s, &used);
  for (auto& L : lv) used += (size_t)L.nb * s * s;  // W per level (mu <= s)
  if (!lv.empty()) used += (size_t)lv[0].nb * s * 2;
  return used + 64;
}

// CholeskyQR basis first (cholqr.cu) for sketches whose Householder tree has four or more
// leaves (I > 768 rows) and that fit one cluster.  Measured (B200, whole decompositions): cfg4's
// 1000 x 60 sketches 4.02 -> 3.87 ms; at cfg5's 512 x 50 even; at cfg2's 400 x 30 the tree is
// cheaper (1.85 vs 2.11 ms) -- the CholeskyQR's three s-step Cholesky chains cost the same at
// any I, the tree's leaf / stacked-R chains grow with I.  LMRA_ORTH_CHOLQR=0 / 1 forces it off /
// on (any I > 256 the cluster takes).
// CholeskyQR serves the split form's basis Q_C (an orthonormal basis of the sketch for the first
// core contraction) above 768 rows.  The factors always come from the Householder path: the
// CholeskyQR R loses the column-graded relative accuracy that column-pivoted Householder keeps,
// and factors taken from it (pivoted QR + Jacobi on that R) missed the 1e-10 subspace contract on
// some power-scheme sketches (sines 1.9e-10 / 7.8e-10 on 900 x 10 / 1000 x 10 sketches where the
// Householder path gives 2e-14).  LMRA_ORTH_CHOLQR=0: no CholeskyQR at all; =1: CholeskyQR from
// 257 rows, for the factors too (tests of that path).
static bool use_cholqr(long long I, int s) {  // the basis phase
  const char* env = getenv("LMRA_ORTH_CHOLQR");
  if (env && env[0] == '0') return false;
  const long long min_rows = (env && env[0] == '1') ? kMaxBlockRows + 1 : 3 * kMaxBlockRows + 1;
  return I >= min_rows && cholqr_supported(I, s);
}
static bool use_cholqr_factor(long long I, int s) {  // the full orthonormalisation
  const char* env = getenv("LMRA_ORTH_CHOLQR");
  return env && env[0] == '1' && use_cholqr(I, s);
}

// [tree | Q_C (I x s) | R (s x s) | Y (s x s) | gate]
size_t orth_workspace_doubles(long long I, int s) {
  return tree_workspace_doubles(I, s) + (use_cholqr(I, s) ? (size_t)I * s + 2 * (size_t)s * s + 64 : 0);
}

// sweeps taken by the most recent converged Jacobi (diagnostics only)
void last_orth_clocks(long long* out7) { cudaMemcpyFromSymbol(out7, g_orth_clk, 7 * sizeof(long long)); }

int last_jacobi_sweeps() {
  int v = 0;
  cudaMemcpyFromSymbol(&v, g_jacobi_sweeps, sizeof(int));
  return v;
}

namespace {

// the attribute is set once per kernel (and device) to the largest size any call can use
constexpr size_t kOrthSmemMax = 227 * 1024;

// Gate of the launches issued while a GateScope is alive: each kernel returns at once unless
// *gate == run_if (the Householder fallback behind a CholeskyQR attempt runs only if it failed).
struct Gate {
  const int* p = nullptr;
  int run_if = 0;
};
thread_local Gate g_gate;
struct GateScope {
  Gate saved;
  GateScope(const int* p, int run_if) : saved(g_gate) { g_gate = Gate{p, run_if}; }
  ~GateScope() { g_gate = saved; }
};

template <int RPL>
cudaError_t leaf_qr(const double* A, long long m, int s, int nb, double* V, double* tau,
                    double* S, int lds, cudaStream_t st) {
  static unsigned long long done = 0;
  const long long rows = (m + nb - 1) / nb;
  const size_t smem = leaf_smem(rows, s);
  cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(orth_leaf_qr_kernel<RPL>), kOrthSmemMax, done);
  if (e != cudaSuccess) return e;
  {
    const cudaError_t le = launch_pdl(orth_leaf_qr_kernel<RPL>, dim3(nb), dim3(kQThreads), smem, st, A, m, s, (int)m, nb, V, tau, S, lds,
                                      g_gate.p, g_gate.run_if);
    if (le != cudaSuccess) return le;
  }
  return cudaGetLastError();
}

// LMRA_NARROW_JACOBI=0: sketches with s <= 32 take the block Jacobi too (comparison / tests)
static int narrow_jacobi_on() {
  const char* e = getenv("LMRA_NARROW_JACOBI");
  return !(e && e[0] == '0');
}

// LMRA_ORTH_BASIS_PIVOT=1: pivot in the basis phase too
static int basis_pivot() {
  static const int on = getenv("LMRA_ORTH_BASIS_PIVOT") && getenv("LMRA_ORTH_BASIS_PIVOT")[0] == '1';
  return on;
}

template <int RPL>
cudaError_t core(const double* S, int m, int s, int mu, double* out, int ldo, int final_level,
                 int* status, double tol, cudaStream_t st, int phase = kOrthFull, double* gbuf = nullptr,
                 double* ur = nullptr) {
  static unsigned long long done = 0;
  const size_t smem = core_smem(m, s);
  cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(orth_core_kernel<RPL>), kOrthSmemMax, done);
  if (e != cudaSuccess) return e;
  // the Jacobi's rotation accumulation on a second SM of a 2-CTA cluster (LMRA_ORTH_CLUSTER=0:
  // one CTA does both halves)
  // (only for wide sketches: below s = 48 the cluster launch and the DSMEM handoff cost more
  // than the J rotations they move -- measured on cfg1 / cfg2 / cfg3)
  static const bool cluster_ok = !(getenv("LMRA_ORTH_CLUSTER") && getenv("LMRA_ORTH_CLUSTER")[0] == '0');
  // (the split form's Jacobi runs beside the core contraction, off the critical path: one CTA,
  // so that it never waits for two co-scheduled SMs the contraction has taken)
  const bool clustered = cluster_ok && s >= 48 && phase == kOrthFull;
  if (clustered) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2);
    cfg.blockDim = dim3(kQThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    note_launch();
    const cudaError_t le = cudaLaunchKernelEx(&cfg, orth_core_kernel<RPL>, S, m, s, m, mu, out, ldo, final_level,
                                              status, tol, 1, phase, gbuf, ur, basis_pivot(), g_gate.p,
                                              g_gate.run_if, narrow_jacobi_on());
    if (le != cudaSuccess) return le;
  } else {
    const cudaError_t le = launch_pdl(orth_core_kernel<RPL>, dim3(1), dim3(kQThreads), smem, st, S, m, s, m, mu,
                                      out, ldo, final_level, status, tol, 0, phase, gbuf, ur, basis_pivot(), g_gate.p,
                                      g_gate.run_if, narrow_jacobi_on());
    if (le != cudaSuccess) return le;
  }
  return cudaGetLastError();
}

template <int RPL>
cudaError_t leaf_apply(const double* V, long long m, int s, int nb, const double* tau,
                       const double* W, int ldw, int mu, double* out, double* pbest, int* pidx,
                       cudaStream_t st) {
  static unsigned long long done = 0;
  const long long rows = (m + nb - 1) / nb;
  const size_t smem = leaf_smem(rows, s);
  cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(orth_leaf_apply_kernel<RPL>), kOrthSmemMax, done);
  if (e != cudaSuccess) return e;
  {
    const cudaError_t le = launch_pdl(orth_leaf_apply_kernel<RPL>, dim3(nb), dim3(kQThreads), smem, st, V, m, s, (int)m, nb, tau, W, ldw, mu,
                                                          out, (int)m, pbest, pidx, g_gate.p, g_gate.run_if);
    if (le != cudaSuccess) return le;
  }
  return cudaGetLastError();
}

#define LMRA_RPL_DISPATCH(rpl, call) ((rpl) == 2 ? call<2> : (rpl) == 4 ? call<4> : call<8>)

}  // namespace

__global__ void __launch_bounds__(256) orth_rotate_signfix_kernel(const double* __restrict__ qc, long long I, int s,
                                                                  const double* __restrict__ ur, int mu,
                                                                  double* __restrict__ u, double* __restrict__ ur_s,
                                                                  const int* __restrict__ gate, int run_if);
static cudaError_t launch_orth_tree(const double* c, long long I, int s, int mu, double* u, double* work,
                                    int* status, double tol, const std::vector<OrthLevel>& lv, size_t used,
                                    cudaStream_t st);

cudaError_t launch_orth(const double* c, long long I, int s, int mu, double* u, double* work,
                        int* status, cudaStream_t st) {
  if (s < 1 || s > kOrthMaxS || mu < 1 || mu > s || I < s) return cudaErrorInvalidValue;
  if (core_smem(kMaxBlockRows, kOrthMaxS) > kOrthSmemMax) return cudaErrorInvalidConfiguration;
  // Jacobi stopping rule: rotate while |g_p.g_q| > tol |g_p| |g_q|; below ~s*eps the inner
  // product is rounding noise and further rotations cannot reduce it.
  double tol = 8.0 * s * 0x1.0p-53;
  if (const char* env = getenv("LMRA_JACOBI_TOL")) tol = atof(env);
  if (const char* env = getenv("LMRA_JACOBI_EARLY"))  // =0: always run the verification sweep
    if (env[0] == '0') tol = -tol;
  size_t used = 0;
  std::vector<OrthLevel> lv = plan_levels(I, s, &used);
  cudaError_t e;
  if (lv.empty())
    return LMRA_RPL_DISPATCH(rpl_for(I), core)(c, (int)I, s, mu, u, (int)I, 1, status, tol, st, kOrthFull, nullptr,
                                               nullptr);
  if (use_cholqr_factor(I, s)) {
    // C = Q_C R by CholeskyQR (cluster kernel), then the s x s chain on R: pivoted QR + Jacobi
    // -> Y = left singular vectors of R (s x mu), U = Q_C Y with the sign rule.  If the
    // CholeskyQR flags a failure, the same launches skip and the Householder tree below runs.
    double* qcb = work + tree_workspace_doubles(I, s);
    double* rm = qcb + (size_t)I * s;
    double* y = rm + (size_t)s * s;
    int* gate = reinterpret_cast<int*>(y + (size_t)s * s);
    e = launch_cholqr(c, I, s, qcb, rm, gate, st);
    if (e != cudaSuccess) return e;
    {
      GateScope gs(gate, 0);
      e = LMRA_RPL_DISPATCH(rpl_for(s), core)(rm, s, s, mu, y, s, 0, status, tol, st, kOrthFull, nullptr, nullptr);
      if (e != cudaSuccess) return e;
    }
    e = launch_pdl(orth_rotate_signfix_kernel, dim3(mu), dim3(256), 0, st, (const double*)qcb, I, s,
                   (const double*)y, mu, u, (double*)nullptr, (const int*)gate, 0);
    if (e != cudaSuccess) return e;
    GateScope gs(gate, 1);
    return launch_orth_tree(c, I, s, mu, u, work, status, tol, lv, used, st);
  }
  return launch_orth_tree(c, I, s, mu, u, work, status, tol, lv, used, st);
}

// the Householder tree path of launch_orth (leaves, pivoted core, back down, sign fix)
static cudaError_t launch_orth_tree(const double* c, long long I, int s, int mu, double* u, double* work,
                                    int* status, double tol, const std::vector<OrthLevel>& lv, size_t used,
                                    cudaStream_t st) {
  cudaError_t e;
  std::vector<size_t> wbuf(lv.size());
  for (size_t l = 0; l < lv.size(); ++l) {
    wbuf[l] = used;
    used += (size_t)lv[l].nb * s * mu;
  }
  double* pbest = work + used;
  int* pidx = reinterpret_cast<int*>(pbest + (size_t)lv[0].nb * mu);
  // leaves, level by level
  for (size_t l = 0; l < lv.size(); ++l) {
    const OrthLevel& L = lv[l];
    const double* A = l == 0 ? c : work + lv[l - 1].w_off;
    const int rpl = rpl_for((L.m + L.nb - 1) / L.nb);
    e = LMRA_RPL_DISPATCH(rpl, leaf_qr)(A, L.m, s, L.nb, work + L.v_off, work + L.tau_off,
                                        work + L.w_off, L.nb * s, st);
    if (e != cudaSuccess) return e;
  }
  // core on the last stacked R
  const OrthLevel& last = lv.back();
  const int mB = last.nb * s;
  e = LMRA_RPL_DISPATCH(rpl_for(mB), core)(work + last.w_off, mB, s, mu, work + wbuf.back(), mB, 0,
                                          status, tol, st, kOrthFull, nullptr, nullptr);
  if (e != cudaSuccess) return e;
  // back down
  for (int l = (int)lv.size() - 1; l >= 0; --l) {
    const OrthLevel& L = lv[l];
    double* out = l == 0 ? u : work + wbuf[l - 1];
    const int rpl = rpl_for((L.m + L.nb - 1) / L.nb);
    e = LMRA_RPL_DISPATCH(rpl, leaf_apply)(work + L.v_off, L.m, s, L.nb, work + L.tau_off,
                                           work + wbuf[l], L.nb * s, mu, out,
                                           l == 0 ? pbest : nullptr, l == 0 ? pidx : nullptr, st);
    if (e != cudaSuccess) return e;
  }
  {
    const cudaError_t le = launch_pdl(orth_signfix_kernel, dim3(mu), dim3(256), 0, st, u, I, (int)I, mu, lv[0].nb, pbest, pidx,
                                      g_gate.p, g_gate.run_if);
    if (le != cudaSuccess) return le;
  }
  return cudaGetLastError();
}


// ---------------------------------------------------------------------------
// The split orthonormalisation: the basis Q_C (I x s) of the sketch first, the s x s Jacobi
// after it (the big contraction that follows runs on Q_C while the Jacobi finishes), then
// U = Q_C U_R(:, :mu) with the sign rule; U_R' = U_R(:, :mu) D carries the same column signs D
// so that X x_n U^T = (X x_n Q_C^T) x_n U_R'^T.
// ---------------------------------------------------------------------------
// one CTA per column c: u(:, c) = Q_C U_R(:, c) (fma over k in order), then the sign rule of
// fix_signs (linalg.cpp:13-29): the largest |u| (first index on ties) made >= 0, and the same
// sign applied to U_R(:, c).
__global__ void __launch_bounds__(256) orth_rotate_signfix_kernel(const double* __restrict__ qc, long long I, int s,
                                                                  const double* __restrict__ ur, int mu,
                                                                  double* __restrict__ u, double* __restrict__ ur_s,
                                                                  const int* __restrict__ gate, int run_if) {
  pdl_wait();
  if (gate && *gate != run_if) return;  // the other branch of a gated pair of paths (cholqr fallback)
  pdl_trigger();
  const int c = blockIdx.x;
  __shared__ double urc[64];
  __shared__ double bv[8];
  __shared__ long long bi[8];
  __shared__ double sgn;
  for (int k = threadIdx.x; k < s; k += blockDim.x) urc[k] = ur[k + (size_t)s * c];
  __syncthreads();
  double best = 0.0;
  long long bidx = -1;
  for (long long i = threadIdx.x; i < I; i += blockDim.x) {
    double acc = 0.0;
    for (int k = 0; k < s; ++k) acc = fma(qc[i + I * k], urc[k], acc);
    u[i + I * c] = acc;
    const double a = fabs(acc);
    if (a > best) {  // rows visited in increasing order per thread: strict > keeps the first
      best = a;
      bidx = i;
    }
  }
  const int l = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int msk = 16; msk >= 1; msk >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, msk);
    const long long oi = __shfl_xor_sync(0xffffffffu, bidx, msk);
    if (ob > best || (ob == best && oi >= 0 && (bidx < 0 || oi < bidx))) {
      best = ob;
      bidx = oi;
    }
  }
  if (l == 0) {
    bv[w] = best;
    bi[w] = bidx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = 0.0;
    long long ix = -1;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k)
      if (bv[k] > b || (bv[k] == b && bi[k] >= 0 && (ix < 0 || bi[k] < ix))) {
        b = bv[k];
        ix = bi[k];
      }
    sgn = (ix >= 0 && u[ix + I * c] < 0.0) ? -1.0 : 1.0;
  }
  __syncthreads();
  const double sg = sgn;
  if (ur_s)
    for (int k = threadIdx.x; k < s; k += blockDim.x) ur_s[k + (size_t)s * c] = sg * urc[k];
  if (sg < 0.0)
    for (long long i = threadIdx.x; i < I; i += blockDim.x) u[i + I * c] = -u[i + I * c];
}

size_t orth_split_workspace_doubles(long long I, int s) {
  return orth_workspace_doubles(I, s) + 2 * (size_t)s * s + 64;
}

// workspace: [orth tree | G (s x s) | U_R (s x s)]
cudaError_t launch_orth_basis(const double* c, long long I, int s, double* qc, double* work, cudaStream_t st) {
  if (s < 1 || s > kOrthMaxS || I < s) return cudaErrorInvalidValue;
  size_t used = 0;
  std::vector<OrthLevel> lv = plan_levels(I, s, &used);
  double* gbuf = work + orth_workspace_doubles(I, s);
  cudaError_t e;
  if (lv.empty())
    return LMRA_RPL_DISPATCH(rpl_for(I), core)(c, (int)I, s, s, qc, (int)I, 0, nullptr, 0.0, st, kOrthBasis, gbuf,
                                               nullptr);
  // CholeskyQR: Q_C and R (to gbuf; the finish runs pivoted QR + Jacobi on it); the Householder
  // tree below (G = R^T to gbuf) runs only if it fails
  int* gate = reinterpret_cast<int*>(gbuf + 2 * (size_t)s * s);
  const bool cq = use_cholqr(I, s);
  if (cq) {
    e = launch_cholqr(c, I, s, qc, gbuf, gate, st);
    if (e != cudaSuccess) return e;
  }
  GateScope gs(cq ? gate : nullptr, 1);
  std::vector<size_t> wbuf(lv.size());
  for (size_t l = 0; l < lv.size(); ++l) {
    wbuf[l] = used;
    used += (size_t)lv[l].nb * s * s;
  }
  for (size_t l = 0; l < lv.size(); ++l) {
    const OrthLevel& L = lv[l];
    const double* A = l == 0 ? c : work + lv[l - 1].w_off;
    e = LMRA_RPL_DISPATCH(rpl_for((L.m + L.nb - 1) / L.nb), leaf_qr)(A, L.m, s, L.nb, work + L.v_off,
                                                                      work + L.tau_off, work + L.w_off, L.nb * s, st);
    if (e != cudaSuccess) return e;
  }
  const OrthLevel& last = lv.back();
  const int mB = last.nb * s;
  e = LMRA_RPL_DISPATCH(rpl_for(mB), core)(work + last.w_off, mB, s, s, work + wbuf.back(), mB, 0, nullptr, 0.0, st,
                                          kOrthBasis, gbuf, nullptr);
  if (e != cudaSuccess) return e;
  for (int l = (int)lv.size() - 1; l >= 0; --l) {
    const OrthLevel& L = lv[l];
    double* out = l == 0 ? qc : work + wbuf[l - 1];
    e = LMRA_RPL_DISPATCH(rpl_for((L.m + L.nb - 1) / L.nb), leaf_apply)(
        work + L.v_off, L.m, s, L.nb, work + L.tau_off, work + wbuf[l], L.nb * s, s, out, nullptr, nullptr, st);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// urs (s x mu) = Q_C^T U: the coefficients of the factor in the split form's basis, so that
// X x_n U^T = (X x_n Q_C^T) x_n urs^T.  One warp per coefficient (grid mu x ceil(s / 8)), eight
// independent loads per lane in flight (the loop over I was a latency chain: ~0.1 ms with a warp
// walking eight dots), fixed-order sums (deterministic).
__global__ void __launch_bounds__(256) basis_coeffs_kernel(const double* __restrict__ qc, long long I, int s,
                                                           const double* __restrict__ u, double* __restrict__ urs) {
  pdl_wait();  // the previous kernel's outputs (programmatic dependent launch)
  pdl_trigger();
  const int b = blockIdx.x, w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const int a = blockIdx.y * 8 + w;
  if (a >= s) return;
  const double* ub = u + (size_t)I * b;
  const double* qa = qc + (size_t)I * a;
  double t = 0.0;
  for (long long i0 = 0; i0 < I; i0 += 256) {
    double v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const long long i = i0 + l + 32 * k;
      v[k] = i < I ? qa[i] * ub[i] : 0.0;
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) t += v[k];
  }
  t = warp_sum(t);
  if (l == 0) urs[a + (size_t)s * b] = t;
}

cudaError_t launch_basis_coeffs(const double* qc, long long I, int s, const double* u, int mu, double* urs,
                                cudaStream_t st) {
  if (s < 1 || mu < 1 || I < 1) return cudaErrorInvalidValue;
  return launch_pdl(basis_coeffs_kernel, dim3((unsigned)mu, (unsigned)((s + 7) / 8)), dim3(256), 0, st, qc, I, s, u,
                    urs);
}

cudaError_t launch_orth_finish(const double* qc, long long I, int s, int mu, double* u, double* ur_signed,
                               double* work, int* status, cudaStream_t st) {
  if (s < 1 || s > kOrthMaxS || mu < 1 || mu > s || I < s) return cudaErrorInvalidValue;
  double tol = 8.0 * s * 0x1.0p-53;
  if (const char* env = getenv("LMRA_JACOBI_TOL")) tol = atof(env);
  if (const char* env = getenv("LMRA_JACOBI_EARLY"))  // =0: always run the verification sweep
    if (env[0] == '0') tol = -tol;
  double* gbuf = work + orth_workspace_doubles(I, s);
  double* ur = gbuf + (size_t)s * s;
  int* gate = reinterpret_cast<int*>(gbuf + 2 * (size_t)s * s);
  const bool cq = use_cholqr(I, s);
  cudaError_t e;
  if (cq) {  // R from the CholeskyQR: pivoted QR + Jacobi -> U_R(:, :mu) = Y (s x mu)
    GateScope gs(gate, 0);
    e = LMRA_RPL_DISPATCH(rpl_for(s), core)(gbuf, s, s, mu, ur, s, 0, status, tol, st, kOrthFull, nullptr, nullptr);
    if (e != cudaSuccess) return e;
  }
  {
    GateScope gs(cq ? gate : nullptr, 1);
    e = LMRA_RPL_DISPATCH(rpl_for(s), core)(nullptr, s, s, mu, nullptr, s, 0, status, tol, st, kOrthJacobi, gbuf, ur);
    if (e != cudaSuccess) return e;
  }
  return launch_pdl(orth_rotate_signfix_kernel, dim3(mu), dim3(256), 0, st, qc, I, s, (const double*)ur, mu, u,
                    ur_signed, (const int*)nullptr, 0);
}

// ---------------------------------------------------------------------------
// QR-proxy extraction (qr_project_extract, linalg.cpp:89-99) building blocks
// ---------------------------------------------------------------------------
__global__ void eye_kernel(double* __restrict__ e, int s) {
  pdl_wait();  // the chain's earlier kernels must be complete before the next one may rely on it
  pdl_trigger();
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < s * s; k += gridDim.x * blockDim.x)
    e[k] = (k % s == k / s) ? 1.0 : 0.0;
}

// workspace of the R-only tree: the leaf levels plus the top block's reflectors and tau
static size_t r_tree_doubles(long long m, int s, std::vector<OrthLevel>* lv_out, size_t* top_off) {
  size_t used = 0;
  std::vector<OrthLevel> lv = plan_levels(m, s, &used);
  const long long mt = lv.empty() ? m : (long long)lv.back().nb * s;
  *top_off = used;
  used += (size_t)mt * s + s;  // top reflectors (mt x s), tau (s)
  if (lv_out) *lv_out = lv;
  return used;
}

size_t r_factor_workspace_doubles(long long m, int s) {
  size_t top = 0;
  return r_tree_doubles(m, s, nullptr, &top) + 64;
}

// R (s x s, column-major, zeros below the diagonal) of the tall m x s matrix a: Householder
// TSQR leaves level by level, then one Householder QR of the last stacked block.  Row signs
// of R follow the dlarfg convention per block (only |R| and R^T R are tree-independent).
cudaError_t launch_r_factor(const double* a, long long m, int s, double* r, double* work,
                            cudaStream_t st) {
  if (s < 1 || s > kOrthMaxS || m < s) return cudaErrorInvalidValue;
  std::vector<OrthLevel> lv;
  size_t top = 0;
  r_tree_doubles(m, s, &lv, &top);
  cudaError_t e;
  for (size_t l = 0; l < lv.size(); ++l) {
    const OrthLevel& L = lv[l];
    const double* A = l == 0 ? a : work + lv[l - 1].w_off;
    e = LMRA_RPL_DISPATCH(rpl_for((L.m + L.nb - 1) / L.nb), leaf_qr)(A, L.m, s, L.nb, work + L.v_off,
                                                                      work + L.tau_off, work + L.w_off,
                                                                      L.nb * s, st);
    if (e != cudaSuccess) return e;
  }
  const long long mt = lv.empty() ? m : (long long)lv.back().nb * s;
  const double* At = lv.empty() ? a : work + lv.back().w_off;
  return LMRA_RPL_DISPATCH(rpl_for(mt), leaf_qr)(At, mt, s, 1, work + top, work + top + (size_t)mt * s, r, s,
                                                 st);
}

size_t thin_q_workspace_doubles(long long I, int s) {
  std::vector<OrthLevel> lv;
  size_t top = 0;
  size_t used = r_tree_doubles(I, s, &lv, &top);
  used += (size_t)s * s * 2;                                // R of the top block, identity
  for (auto& L : lv) used += (size_t)L.nb * s * s;          // W per level
  return used + 64;
}

// Thin Q (I x s) of C (thin_qr, linalg.cpp:52-60): the reflectors of the R tree applied to
// [I_s; 0] back down the tree.  One block (I <= 256) is exactly Householder QR with LAPACK's
// (dgeqrf/dorgqr, = Eigen HouseholderQR) sign convention; above that the TSQR Q spans the
// same column space with per-column signs that may differ.
cudaError_t launch_thin_q(const double* c, long long I, int s, double* q, double* work, cudaStream_t st) {
  if (s < 1 || s > kOrthMaxS || I < s) return cudaErrorInvalidValue;
  std::vector<OrthLevel> lv;
  size_t top = 0;
  size_t used = r_tree_doubles(I, s, &lv, &top);
  double* R = work + used;
  double* E = R + (size_t)s * s;
  used += (size_t)s * s * 2;
  std::vector<size_t> wbuf(lv.size());
  for (size_t l = 0; l < lv.size(); ++l) {
    wbuf[l] = used;
    used += (size_t)lv[l].nb * s * s;
  }
  cudaError_t e = launch_r_factor(c, I, s, R, work, st);
  if (e != cudaSuccess) return e;
  {
    const cudaError_t le = launch_pdl(eye_kernel, dim3(1), dim3(256), 0, st, E, s);
    if (le != cudaSuccess) return le;
  }
  const long long mt = lv.empty() ? I : (long long)lv.back().nb * s;
  double* out_top = lv.empty() ? q : work + wbuf.back();
  e = LMRA_RPL_DISPATCH(rpl_for(mt), leaf_apply)(work + top, mt, s, 1, work + top + (size_t)mt * s, E, s, s,
                                                 out_top, nullptr, nullptr, st);
  if (e != cudaSuccess) return e;
  for (int l = (int)lv.size() - 1; l >= 0; --l) {
    const OrthLevel& L = lv[l];
    double* out = l == 0 ? q : work + wbuf[l - 1];
    e = LMRA_RPL_DISPATCH(rpl_for((L.m + L.nb - 1) / L.nb), leaf_apply)(
        work + L.v_off, L.m, s, L.nb, work + L.tau_off, work + wbuf[l], L.nb * s, s, out, nullptr, nullptr, st);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// out (J x I, column-major) = the transposed mode unfolding of x: out[j + J r] = X3[i, r, o],
// j = i + inner o.  Each (r, o) fibre segment of `inner` contiguous values is a contiguous
// run in out as well, so this is a strided copy (coalesced both ways for inner >= 32); the
// mode-0 case (inner = 1) is a plain transpose.
__global__ void unfold_t_kernel(const double* __restrict__ x, long long inner, long long I, long long outer,
                                double* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const long long n = inner * I * outer, J = inner * outer;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    const long long i = e % inner, ro = e / inner, r = ro % I, o = ro / I;
    out[i + inner * o + J * r] = x[e];
  }
}

cudaError_t launch_unfold_t(const double* x, long long inner, long long I, long long outer, double* out,
                            cudaStream_t st) {
  if (inner == 1) return launch_transpose(x, I, outer, out, st);
  const long long n = inner * I * outer;
  const unsigned blocks = (unsigned)std::min<long long>((n + 255) / 256, 148LL * 16);
  return launch_pdl(unfold_t_kernel, dim3(blocks), dim3(256), 0, st, x, inner, I, outer, out);
}

}  // namespace lmra_dev

// orth.cu -- on-device orthonormalisation of the I_n x s sketch C.
//
// Replaces thin_svd (linalg.cpp:33-43, Eigen BDCSVD) + fix_signs (linalg.cpp:13-29)
// as used by leading_left_singular_vectors (linalg.cpp:82-87):
//   C = Q R            blocked Householder TSQR: phase A per row block (recursive levels),
//                      phase B column-pivoted Householder on the stacked R factors
//   R = U_R S V^T      one-sided (Hestenes) Jacobi on R^T with the rotations accumulated:
//                      R^T J = W  =>  R = J diag(|W_j|) (W/|W|)^T, so U_R = J (orthogonal even
//                      for zero singular values).  The pivoted R is graded, which makes
//                      Jacobi on R^T converge in a few sweeps (de Rijk / Drmac).
//   U = Q [U_R ; 0]    reflectors applied in reverse (phase C per row block, staged in smem)
//   fix_signs          largest-|u| entry (first index on ties) made >= 0
// All reductions run in a fixed order, so the result is deterministic run to run.
// Householder QR is used instead of CholeskyQR2 because the sketches of the
// BASELINE configs reach kappa(C) ~ 1e16, far past CholeskyQR2's
// u^{-1/2} limit.
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "common.cuh"

namespace lmra_dev {

constexpr int kOrthThreads = 1024;
constexpr int kOrthWarps = kOrthThreads / 32;
constexpr size_t kOrthSmemBudget = 200 * 1024;
constexpr int kOrthMaxS = 64;
constexpr int kApplyChunk = 8;  // reflectors staged per smem chunk in phase C

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
  return v;
}

// Lane-strided dot product over rows [lo, m) with stride 32 and four independent
// accumulators (ILP: the loads of four rows are in flight together).
__device__ __forceinline__ double lane_dot(const double* __restrict__ a,
                                           const double* __restrict__ b, int lo, int m) {
  double d0 = 0.0, d1 = 0.0, d2 = 0.0, d3 = 0.0;
  int i = lo;
  for (; i + 96 < m; i += 128) {
    d0 += a[i] * b[i];
    d1 += a[i + 32] * b[i + 32];
    d2 += a[i + 64] * b[i + 64];
    d3 += a[i + 96] * b[i + 96];
  }
  for (; i < m; i += 32) d0 += a[i] * b[i];
  return (d0 + d1) + (d2 + d3);
}

// Householder QR in place on A (m x s, column-major, leading dim lda, in shared memory).
// On exit: R in the upper triangle, v_k (unit leading entry implicit) below the
// diagonal, tau[k].  LAPACK dlarfg convention: H_k = I - tau v v^T, beta = -sign(a)*||x||.
// Column c is owned by warp c % 32.  With piv != nullptr, columns are pivoted
// (largest remaining norm first, first index on ties; norms recomputed exactly each
// step in the update pass) and piv[] receives the permutation; cn is s doubles scratch.
__device__ void block_householder_qr(double* A, int m, int s, int lda, double* tau, int* piv,
                                     double* cn) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kmax = min(m, s);
  auto make_reflector = [&](int k) {  // executed by the owner warp of column k
    if (piv) {  // pick the pivot among columns k..s-1 and swap it into k
      double best = -1.0;
      int p = k;
      for (int c = k + lane; c < s; c += 32) {
        if (cn[c] > best) {
          best = cn[c];
          p = c;
        }
      }
#pragma unroll
      for (int msk = 16; msk >= 1; msk >>= 1) {
        double ob = __shfl_xor_sync(0xffffffffu, best, msk);
        int op = __shfl_xor_sync(0xffffffffu, p, msk);
        if (ob > best || (ob == best && op < p)) {
          best = ob;
          p = op;
        }
      }
      if (p != k) {
        double* ck = A + (size_t)lda * k;
        double* cp = A + (size_t)lda * p;
        for (int i = lane; i < m; i += 32) {
          double t = ck[i];
          ck[i] = cp[i];
          cp[i] = t;
        }
        if (lane == 0) {
          double t = cn[k];
          cn[k] = cn[p];
          cn[p] = t;
          int ti = piv[k];
          piv[k] = piv[p];
          piv[p] = ti;
        }
        __syncwarp();
      }
    }
    double* col = A + (size_t)lda * k;
    double ss = warp_sum(lane_dot(col, col, k + 1 + lane, m));
    const double alpha = col[k];
    double t = 0.0;
    if (ss != 0.0) {
      const double beta = -copysign(sqrt(alpha * alpha + ss), alpha);
      t = (beta - alpha) / beta;
      const double scale = 1.0 / (alpha - beta);
      for (int i = k + 1 + lane; i < m; i += 32) col[i] *= scale;
      __syncwarp();
      if (lane == 0) col[k] = beta;
    }
    if (lane == 0) tau[k] = t;
    __syncwarp();
  };
  if (piv) {
    for (int c = warp; c < s; c += kOrthWarps) {
      const double* col = A + (size_t)lda * c;
      double a = warp_sum(lane_dot(col, col, lane, m));
      if (lane == 0) {
        cn[c] = a;
        piv[c] = c;
      }
    }
    __syncthreads();
  }
  if (kmax > 0 && warp == 0) make_reflector(0);
  __syncthreads();
  for (int k = 0; k < kmax; ++k) {
    const double* v = A + (size_t)lda * k;
    const double tk = tau[k];
    for (int c = warp; c < s; c += 32) {
      if (c <= k) continue;
      double* col = A + (size_t)lda * c;
      if (tk != 0.0) {
        double d = warp_sum(lane_dot(v, col, k + 1 + lane, m));
        d += col[k];
        const double f = tk * d;
        double nn = 0.0;
#pragma unroll 4
        for (int i = k + 1 + lane; i < m; i += 32) {
          double val = col[i] - f * v[i];
          col[i] = val;
          nn += val * val;
        }
        __syncwarp();
        if (lane == 0) col[k] -= f;
        if (piv) {
          nn = warp_sum(nn);
          if (lane == 0) cn[c] = nn;
        }
        __syncwarp();
      } else if (piv) {
        double nn = warp_sum(lane_dot(col, col, k + 1 + lane, m));
        if (lane == 0) cn[c] = nn;
        __syncwarp();
      }
      if (c == k + 1 && k + 1 < kmax && !piv) make_reflector(k + 1);
    }
    __syncthreads();
    if (piv && k + 1 < kmax) {  // the pivot needs every column's updated norm
      if (warp == (k + 1) % 32) make_reflector(k + 1);
      __syncthreads();
    }
  }
}

// Y (m x mu, ld ldy, shared) <- Q Y with Q = H_0 H_1 ... H_{kmax-1} from (V, tau) in shared
// memory.  Each warp owns whole columns of Y, so no block barrier between reflectors.
__device__ void apply_q(const double* V, int ldv, const double* tau, int m, int s, double* Y,
                        int ldy, int mu, int k_hi, int k_lo) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int c = warp; c < mu; c += kOrthWarps) {
    double* y = Y + (size_t)ldy * c;
    for (int k = k_hi - 1; k >= k_lo; --k) {
      const double tk = tau[k];
      if (tk == 0.0) continue;
      const double* v = V + (size_t)ldv * (k - k_lo);
      double d = warp_sum(lane_dot(v, y, k + 1 + lane, m));
      d += y[k];
      const double f = tk * d;
#pragma unroll 4
      for (int i = k + 1 + lane; i < m; i += 32) y[i] -= f * v[i];
      __syncwarp();
      if (lane == 0) y[k] -= f;
      __syncwarp();
    }
  }
}

// argmax |y| with the reference's scan semantics (strict >, first index wins);
// all-zero column -> index 0 with value 0.
__device__ void warp_argmax(const double* y, int m, double& best, int& imax) {
  const int lane = threadIdx.x & 31;
  best = 0.0;
  imax = 0;
  bool found = false;
  for (int i = lane; i < m; i += 32) {
    double a = fabs(y[i]);
    if (a > best) {
      best = a;
      imax = i;
      found = true;
    }
  }
  if (!found) imax = 0x7fffffff;
#pragma unroll
  for (int msk = 16; msk >= 1; msk >>= 1) {
    double ob = __shfl_xor_sync(0xffffffffu, best, msk);
    int oi = __shfl_xor_sync(0xffffffffu, imax, msk);
    if (ob > best || (ob == best && oi < imax)) {
      best = ob;
      imax = oi;
    }
  }
  if (best == 0.0) imax = 0;
}

// One-sided Jacobi on G (s x n, ld s; n even, column n-1 may be a zero pad); the same
// rotations are applied to the columns of J (n x n, ld n).  Round-robin (circle)
// ordering: n/2 disjoint pairs per round.  A quad of 4 lanes owns one pair (8 pairs per
// warp, rows strided by 4): the rotation math is done once per pair instead of once per
// warp lane-replicated, which keeps the SM's issue slots free (ncu: the warp-per-pair
// version was issue-bound at 58% slot use on instruction count, not latency).
__device__ int g_jacobi_sweeps;
#ifdef LMRA_JACOBI_CLOCKS
__device__ unsigned long long g_jclk[8];
#endif

// One round of the parallel one-sided Jacobi: LPP lanes own one column pair, each lane
// holds R = ceil(s / LPP) rows of both columns (and of the two J columns) in registers;
// the loops are fully unrolled so a lane's loads issue together (the runtime-trip-count
// smem loops of the first version serialised on load latency: ~3000 cycles per round).
template <int LPP, int R>
__device__ void jacobi_round(double* G, int s, int n, double* J, int* flag, double tol2,
                             const unsigned char* pairs) {
  const int lane = threadIdx.x & 31, sub = lane & (LPP - 1);
  const int pair = threadIdx.x / LPP;
  if (pair >= n / 2) return;
  const unsigned gmask = LPP == 32 ? 0xffffffffu : (((1u << LPP) - 1u) << (lane & ~(LPP - 1)));
  const int p = pairs[2 * pair], q = pairs[2 * pair + 1];
  double* gp = G + (size_t)s * p;
  double* gq = G + (size_t)s * q;
  double x[R], y[R];
#ifdef LMRA_JACOBI_CLOCKS
  long long tc0 = clock64();
#endif
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int i = sub + r * LPP;
    x[r] = i < s ? gp[i] : 0.0;
    y[r] = i < s ? gq[i] : 0.0;
  }
  double a = 0.0, b = 0.0, c = 0.0;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    a = fma(x[r], x[r], a);
    b = fma(y[r], y[r], b);
    c = fma(x[r], y[r], c);
  }
#pragma unroll
  for (int m = 1; m < LPP; m <<= 1) {
    a += __shfl_xor_sync(gmask, a, m);
    b += __shfl_xor_sync(gmask, b, m);
    c += __shfl_xor_sync(gmask, c, m);
  }
#ifdef LMRA_JACOBI_CLOCKS
  long long tc1 = clock64();
#endif
  // rotate while c^2 > tol^2 a b (no sqrt); huge norms take an exponent-scaled path
  bool rot;
  double sa = a, sb = b, sc = c;
  if (fmax(a, b) < 1e150) {
    rot = c != 0.0 && c * c > tol2 * (a * b);
  } else {
    const int ea = ilogb(fmax(fmax(a, b), fabs(c)));
    sa = ldexp(a, -ea);
    sb = ldexp(b, -ea);
    sc = ldexp(c, -ea);
    rot = c != 0.0 && sc * sc > tol2 * (sa * sb);
  }
  if (!rot) return;
  // smaller root of t^2 + 2 zeta t - 1 = 0, zeta = (b - a) / (2c):
  //   t = sign(d) 2c / (|d| + sqrt(d^2 + 4c^2)),  d = b - a;
  // sqrt, reciprocal and rsqrt on the critical path (~100 + 80 + 75 cycles, measured).
  const double d = sb - sa;
  const double t = (d >= 0.0 ? 2.0 * sc : -2.0 * sc) * __drcp_rn(fabs(d) + sqrt(fma(d, d, 4.0 * sc * sc)));
  const double cs = rsqrt(fma(t, t, 1.0));
  const double sn = cs * t;
#ifdef LMRA_JACOBI_CLOCKS
  long long tc2 = clock64();
#endif
  double* jp = J + (size_t)n * p;
  double* jq = J + (size_t)n * q;
  double u[R], w[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int i = sub + r * LPP;
    u[r] = i < n ? jp[i] : 0.0;
    w[r] = i < n ? jq[i] : 0.0;
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int i = sub + r * LPP;
    if (i < s) {
      gp[i] = cs * x[r] - sn * y[r];
      gq[i] = sn * x[r] + cs * y[r];
    }
    if (i < n) {
      jp[i] = cs * u[r] - sn * w[r];
      jq[i] = sn * u[r] + cs * w[r];
    }
  }
  if (sub == 0) *flag = 1;
#ifdef LMRA_JACOBI_CLOCKS
  if (pair == 0 && sub == 0) {
    long long tc3 = clock64();
    g_jclk[0] += tc1 - tc0;
    g_jclk[1] += tc2 - tc1;
    g_jclk[2] += tc3 - tc2;
    g_jclk[3] += 1;
  }
#endif
}

// One-sided Jacobi on G (s x n, ld s; n even, column n-1 may be a zero pad); the same
// rotations are applied to the columns of J (n x n, ld n).  Round-robin (circle)
// ordering, n/2 disjoint pairs per round; `pairs` is smem scratch of n*(n-1) bytes.
__device__ bool one_sided_jacobi(double* G, int s, int n, double* J, int* flag, double tol,
                                 unsigned char* pairs) {
  const double tol2 = tol * tol;
  for (int e = threadIdx.x; e < (n - 1) * (n / 2); e += blockDim.x) {
    const int round = e / (n / 2), k = e % (n / 2);
    int p, q;
    if (k == 0) {
      p = n - 1;
      q = round;
    } else {
      p = (round + k) % (n - 1);
      q = (round - k + (n - 1)) % (n - 1);
    }
    pairs[2 * e] = (unsigned char)min(p, q);
    pairs[2 * e + 1] = (unsigned char)max(p, q);
  }
  for (int sweep = 0; sweep < 60; ++sweep) {
    if (threadIdx.x == 0) *flag = 0;
    __syncthreads();
    for (int round = 0; round < n - 1; ++round) {
      const unsigned char* pr = pairs + (size_t)round * n;
      if (s <= 16)
        jacobi_round<4, 4>(G, s, n, J, flag, tol2, pr);
      else if (s <= 32)
        jacobi_round<8, 4>(G, s, n, J, flag, tol2, pr);
      else
        jacobi_round<16, 4>(G, s, n, J, flag, tol2, pr);
      __syncthreads();
    }
    const int f = *flag;
    __syncthreads();
    if (!f) {
      if (threadIdx.x == 0) g_jacobi_sweeps = sweep + 1;
      return true;
    }
  }
  return false;
}

// ---------------------------------------------------------------------------
// Phase A: QR of row block b of A (m x s, lda) -> reflectors into V (same rows),
// tau[b*s + k], R_b into rows [b*s, b*s+s) of S (ld lds), zeros below the diagonal.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kOrthThreads) orth_block_qr_kernel(
    const double* __restrict__ A, long long m, int s, int lda, int nb, double* __restrict__ V,
    double* __restrict__ tau, double* __restrict__ S, int lds) {
  extern __shared__ __align__(16) double sm[];
  const int b = blockIdx.x;
  const long long r0 = (m * b) / nb, r1 = (m * (b + 1)) / nb;
  const int rows = (int)(r1 - r0);
  double* W = sm;                      // rows x s
  double* t = sm + (size_t)rows * s;   // s
  for (int e = threadIdx.x; e < rows * s; e += kOrthThreads) {
    int i = e % rows, c = e / rows;
    W[e] = A[r0 + i + (size_t)lda * c];
  }
  __syncthreads();
  block_householder_qr(W, rows, s, rows, t, nullptr, nullptr);
  __syncthreads();
  for (int e = threadIdx.x; e < rows * s; e += kOrthThreads) {
    int i = e % rows, c = e / rows;
    V[r0 + i + (size_t)lda * c] = W[e];
  }
  for (int e = threadIdx.x; e < s * s; e += kOrthThreads) {
    int i = e % s, c = e / s;
    S[(size_t)b * s + i + (size_t)lds * c] = (i <= c && i < rows) ? W[i + (size_t)rows * c] : 0.0;
  }
  for (int k = threadIdx.x; k < s; k += kOrthThreads) tau[(size_t)b * s + k] = k < rows ? t[k] : 0.0;
}

// ---------------------------------------------------------------------------
// Phase B: one CTA. S (m x s, lds) -> pivoted QR -> Jacobi on R^T -> Y = Q [U_R(:, :mu); 0].
// final != 0: sign-fix Y and write it to out (ld ldo); else write Y to out unsigned.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kOrthThreads) orth_core_kernel(
    const double* __restrict__ S, int m, int s, int lds, int mu, double* __restrict__ out,
    int ldo, int final_level, int* status, double jacobi_tol) {
  extern __shared__ __align__(16) double sm[];
  const int n = s + (s & 1);  // even column count for the tournament
  double* A = sm;                                   // m x s
  double* Y = A + (size_t)m * s;                    // m x mu
  double* G = Y + (size_t)m * mu;                   // s x n   (R^T, padded)
  double* J = G + (size_t)s * n;                    // n x n   (accumulated rotations)
  double* tau = J + (size_t)n * n;                  // s
  double* cn = tau + s;                             // s
  double* sig = cn + s;                             // n
  int* piv = reinterpret_cast<int*>(sig + n);       // s
  int* perm = piv + s;                              // n
  int* flag = perm + n;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  for (int e = threadIdx.x; e < m * s; e += kOrthThreads) {
    int i = e % m, c = e / m;
    A[e] = S[i + (size_t)lds * c];
  }
  __syncthreads();
  block_householder_qr(A, m, s, m, tau, piv, cn);
  __syncthreads();
  // G = R^T (s x s lower triangle), zero pad column; J = I
  for (int e = threadIdx.x; e < s * n; e += kOrthThreads) {
    int i = e % s, j = e / s;  // G[i, j] = R[j, i]
    G[e] = (j < s && j <= i && j < m) ? A[j + (size_t)m * i] : 0.0;
  }
  for (int e = threadIdx.x; e < n * n; e += kOrthThreads) J[e] = (e % n == e / n) ? 1.0 : 0.0;
  __syncthreads();
  const bool converged =
      one_sided_jacobi(G, s, n, J, flag, jacobi_tol, reinterpret_cast<unsigned char*>(flag + 1));
  // singular values = column norms of G, fixed order
  for (int c = warp; c < n; c += kOrthWarps) {
    double a = 0.0;
    for (int i = lane; i < s; i += 32) a += G[i + (size_t)s * c] * G[i + (size_t)s * c];
    a = warp_sum(a);
    if (lane == 0) sig[c] = sqrt(a);
  }
  __syncthreads();
  if (threadIdx.x < s) {  // stable descending order of the s real columns (pad excluded)
    const int c = threadIdx.x;
    const double v = sig[c];
    int rank = 0;
    for (int d = 0; d < s; ++d) rank += (sig[d] > v) || (sig[d] == v && d < c);
    perm[rank] = c;
  }
  __syncthreads();
  // Y = [U_R(:, :mu) ; 0] with U_R = J(0:s, perm)
  for (int e = threadIdx.x; e < m * mu; e += kOrthThreads) {
    int i = e % m, c = e / m;
    Y[e] = i < s ? J[i + (size_t)n * perm[c]] : 0.0;
  }
  __syncthreads();
  apply_q(A, m, tau, m, s, Y, m, mu, min(m, s), 0);
  __syncthreads();
  if (final_level) {
    for (int c = warp; c < mu; c += kOrthWarps) {
      double best;
      int imax;
      warp_argmax(Y + (size_t)m * c, m, best, imax);
      const bool flip = Y[imax + (size_t)m * c] < 0.0;
      __syncwarp();
      for (int i = lane; i < m; i += 32) {
        double val = Y[i + (size_t)m * c];
        out[i + (size_t)ldo * c] = flip ? -val : val;
      }
    }
  } else {
    for (int e = threadIdx.x; e < m * mu; e += kOrthThreads) {
      int i = e % m, c = e / m;
      out[i + (size_t)ldo * c] = Y[e];
    }
  }
  if (threadIdx.x == 0 && status) *status = converged ? 0 : 1;
}

// ---------------------------------------------------------------------------
// Phase C: block b: Y_b = Q_b [W(b*s : b*s+s, :) ; 0] -> out rows [r0, r1) (ld ldo).
// Reflectors are staged through shared memory kApplyChunk at a time.  With pbest also
// records per-block column argmax partials for the sign fix.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kOrthThreads) orth_block_apply_kernel(
    const double* __restrict__ V, long long m, int s, int ldv, int nb,
    const double* __restrict__ tau, const double* __restrict__ W, int ldw, int mu,
    double* __restrict__ out, int ldo, double* __restrict__ pbest, int* __restrict__ pidx) {
  extern __shared__ __align__(16) double sm[];
  const int b = blockIdx.x;
  const long long r0 = (m * b) / nb, r1 = (m * (b + 1)) / nb;
  const int rows = (int)(r1 - r0);
  double* Y = sm;                                  // rows x mu
  double* Vs = Y + (size_t)rows * mu;              // rows x kApplyChunk
  double* ts = Vs + (size_t)rows * kApplyChunk;    // s
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int e = threadIdx.x; e < rows * mu; e += kOrthThreads) {
    int i = e % rows, c = e / rows;
    Y[e] = i < s ? W[(size_t)b * s + i + (size_t)ldw * c] : 0.0;
  }
  for (int k = threadIdx.x; k < s; k += kOrthThreads) ts[k] = tau[(size_t)b * s + k];
  const int kmax = min(rows, s);
  for (int k_hi = kmax; k_hi > 0; k_hi -= kApplyChunk) {
    const int k_lo = max(0, k_hi - kApplyChunk);
    __syncthreads();
    for (int e = threadIdx.x; e < rows * (k_hi - k_lo); e += kOrthThreads) {
      int i = e % rows, kk = e / rows;
      Vs[e] = V[r0 + i + (size_t)ldv * (k_lo + kk)];
    }
    __syncthreads();
    apply_q(Vs, rows, ts, rows, s, Y, rows, mu, k_hi, k_lo);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < rows * mu; e += kOrthThreads) {
    int i = e % rows, c = e / rows;
    out[r0 + i + (size_t)ldo * c] = Y[e];
  }
  if (pbest) {
    for (int c = warp; c < mu; c += kOrthWarps) {
      double best;
      int imax;
      warp_argmax(Y + (size_t)rows * c, rows, best, imax);
      if (lane == 0) {
        pbest[(size_t)b * mu + c] = best;
        pidx[(size_t)b * mu + c] = (int)(r0 + imax);
      }
    }
  }
}

// Phase D: per column, combine block partials in block order; flip if negative.
__global__ void orth_signfix_kernel(double* __restrict__ U, long long m, int ldu, int mu, int nb,
                                    const double* __restrict__ pbest,
                                    const int* __restrict__ pidx) {
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
  int nb;       // row blocks
  size_t v_off, tau_off, w_off;  // workspace offsets (doubles)
};

static size_t core_smem(long long m, int s, int mu) {
  int n = s + (s & 1);
  return sizeof(double) * ((size_t)m * s + (size_t)m * mu + (size_t)s * n + (size_t)n * n + 2 * s + n) +
         sizeof(int) * (s + n + 1) + (size_t)n * n + 64;
}

static long long block_rows(int s, int mu) {
  // phase A: rows x s ; phase C: rows x (mu + kApplyChunk)
  return (long long)(kOrthSmemBudget / (sizeof(double) * (size_t)std::max(s, mu + kApplyChunk))) - 8;
}

static std::vector<OrthLevel> plan_levels(long long I, int s, int mu, size_t* total) {
  std::vector<OrthLevel> lv;
  size_t off = 0;
  long long m = I;
  while (core_smem(m, s, mu) > kOrthSmemBudget) {
    long long per = block_rows(s, mu);
    int nb = std::max(2, (int)((m + per - 1) / per));
    OrthLevel L;
    L.m = m;
    L.nb = nb;
    L.v_off = off;
    off += (size_t)m * s;
    L.tau_off = off;
    off += (size_t)nb * s;
    L.w_off = off;  // stacked R of this level = next level's input (nb*s x s)
    off += (size_t)nb * s * s;
    lv.push_back(L);
    m = (long long)nb * s;
  }
  *total = off;
  return lv;
}

size_t orth_workspace_doubles(long long I, int s) {
  // upper bound over mu <= s
  size_t best = 64;
  for (int mu = 1; mu <= s; ++mu) {
    size_t used = 0;
    std::vector<OrthLevel> lv = plan_levels(I, s, mu, &used);
    for (auto& L : lv) used += (size_t)L.nb * s * mu;
    if (!lv.empty()) used += (size_t)lv[0].nb * mu * 2;
    best = std::max(best, used + 64);
  }
  return best;
}

// sweeps taken by the most recent converged Jacobi (diagnostics only)
int last_jacobi_sweeps() {
  int v = 0;
  cudaMemcpyFromSymbol(&v, g_jacobi_sweeps, sizeof(int));
  return v;
}

cudaError_t launch_orth(const double* c, long long I, int s, int mu, double* u, double* work,
                        int* status, cudaStream_t st) {
  if (s < 1 || s > kOrthMaxS || mu < 1 || mu > s || I < s) return cudaErrorInvalidValue;
  static unsigned long long a1 = 0, a2 = 0, a3 = 0;
  cudaError_t e;
  if ((e = ensure_smem_attr(reinterpret_cast<const void*>(orth_core_kernel), kOrthSmemBudget + 16384, a1)) != cudaSuccess) return e;
  if ((e = ensure_smem_attr(reinterpret_cast<const void*>(orth_block_qr_kernel), kOrthSmemBudget + 16384, a2)) != cudaSuccess) return e;
  if ((e = ensure_smem_attr(reinterpret_cast<const void*>(orth_block_apply_kernel), kOrthSmemBudget + 16384, a3)) != cudaSuccess) return e;

  // Jacobi stopping rule: rotate while |g_p.g_q| > tol |g_p| |g_q|; below ~s*eps the inner
  // product is rounding noise and further rotations cannot reduce it.
  double tol = 8.0 * s * 0x1.0p-53;
  if (const char* env = getenv("LMRA_JACOBI_TOL")) tol = atof(env);
  size_t used = 0;
  std::vector<OrthLevel> lv = plan_levels(I, s, mu, &used);
  if (lv.empty()) {
    orth_core_kernel<<<1, kOrthThreads, core_smem(I, s, mu), st>>>(c, (int)I, s, (int)I, mu, u,
                                                                    (int)I, 1, status, tol);
    return cudaGetLastError();
  }
  std::vector<size_t> wbuf(lv.size());
  for (size_t l = 0; l < lv.size(); ++l) {
    wbuf[l] = used;
    used += (size_t)lv[l].nb * s * mu;
  }
  double* pbest = work + used;
  int* pidx = reinterpret_cast<int*>(pbest + (size_t)lv[0].nb * mu);
  // phase A, level by level
  for (size_t l = 0; l < lv.size(); ++l) {
    const OrthLevel& L = lv[l];
    const double* A = l == 0 ? c : work + lv[l - 1].w_off;
    long long per = (L.m + L.nb - 1) / L.nb;
    size_t smem = sizeof(double) * ((size_t)per * s + s) + 64;
    orth_block_qr_kernel<<<L.nb, kOrthThreads, smem, st>>>(A, L.m, s, (int)L.m, L.nb,
                                                          work + L.v_off, work + L.tau_off,
                                                          work + L.w_off, L.nb * s);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  // phase B on the last stacked R
  const OrthLevel& last = lv.back();
  const int mB = last.nb * s;
  orth_core_kernel<<<1, kOrthThreads, core_smem(mB, s, mu), st>>>(
      work + last.w_off, mB, s, mB, mu, work + wbuf.back(), mB, 0, status, tol);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  // phase C, back down
  for (int l = (int)lv.size() - 1; l >= 0; --l) {
    const OrthLevel& L = lv[l];
    const double* W = work + wbuf[l];
    const int ldw = L.nb * s;
    double* out = l == 0 ? u : work + wbuf[l - 1];
    const int ldo = (int)L.m;
    long long per = (L.m + L.nb - 1) / L.nb;
    size_t smem = sizeof(double) * ((size_t)per * (mu + kApplyChunk) + s) + 64;
    orth_block_apply_kernel<<<L.nb, kOrthThreads, smem, st>>>(
        work + L.v_off, L.m, s, (int)L.m, L.nb, work + L.tau_off, W, ldw, mu, out, ldo,
        l == 0 ? pbest : nullptr, l == 0 ? pidx : nullptr);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  orth_signfix_kernel<<<mu, 256, 0, st>>>(u, I, (int)I, mu, lv[0].nb, pbest, pidx);
  return cudaGetLastError();
}

}  // namespace lmra_dev

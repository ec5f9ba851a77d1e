// orth.cu -- on-device orthonormalisation of the I_n x s sketch C.
//
// Replaces thin_svd (linalg.cpp:33-43, Eigen BDCSVD) + fix_signs (linalg.cpp:13-29)
// as used by leading_left_singular_vectors (linalg.cpp:82-87):
//   C = Q R            blocked Householder TSQR (phase A per row block, recursive)
//   R = U_R S V^T      one-sided (Hestenes) Jacobi on R, parallel round-robin order
//   U = Q [U_R ; 0]    reflectors applied in reverse (phase C per row block)
//   fix_signs          largest-|u| entry (first index on ties) made >= 0
// All reductions run in a fixed order, so the result is deterministic run to run.
// Householder QR is used instead of CholeskyQR2 because the sketches of the
// BASELINE configs reach kappa(C) ~ 1e16, far past CholeskyQR2's
// u^{-1/2} limit.
#include <algorithm>
#include <vector>

#include "common.cuh"

namespace lmra_dev {

constexpr int kOrthThreads = 1024;
constexpr int kOrthWarps = kOrthThreads / 32;
constexpr size_t kOrthSmemBudget = 200 * 1024;
constexpr int kOrthMaxS = 64;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
  return v;
}

// Householder QR in place on A (m x s, column-major, leading dim lda, in shared memory).
// On exit: R in the upper triangle, v_k (unit leading entry implicit) below the
// diagonal, tau[k].  LAPACK dlarfg convention: H_k = I - tau v v^T, beta = -sign(a)*||x||.
// Column c is owned by warp c % 32; one block barrier per reflector.
__device__ void block_householder_qr(double* A, int m, int s, int lda, double* tau) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kmax = min(m, s);
  auto make_reflector = [&](int k) {  // executed by the owner warp of column k
    double* col = A + (size_t)lda * k;
    double ss = 0.0;
    for (int i = k + 1 + lane; i < m; i += 32) ss += col[i] * col[i];
    ss = warp_sum(ss);
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
  };
  if (kmax > 0 && warp == 0) make_reflector(0);
  __syncthreads();
  for (int k = 0; k < kmax; ++k) {
    const double* v = A + (size_t)lda * k;
    const double tk = tau[k];
    for (int c = warp; c < s; c += 32) {
      if (c <= k) continue;
      double* col = A + (size_t)lda * c;
      if (tk != 0.0) {
        double d = 0.0;
        for (int i = k + 1 + lane; i < m; i += 32) d += v[i] * col[i];
        d = warp_sum(d);
        d += col[k];
        const double f = tk * d;
        for (int i = k + 1 + lane; i < m; i += 32) col[i] -= f * v[i];
        __syncwarp();
        if (lane == 0) col[k] -= f;
        __syncwarp();
      }
      if (c == k + 1 && k + 1 < kmax) make_reflector(k + 1);
    }
    __syncthreads();
  }
}

// Y (m x mu, ld ldy, shared) <- Q Y with Q = H_0 H_1 ... H_{kmax-1} from (V, tau).
// V may live in global memory (read through L1); each warp owns whole columns of Y,
// so no block barrier is needed between reflectors.
__device__ void apply_q(const double* V, int ldv, const double* tau, int m, int s, double* Y,
                        int ldy, int mu) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kmax = min(m, s);
  for (int c = warp; c < mu; c += kOrthWarps) {
    double* y = Y + (size_t)ldy * c;
    for (int k = kmax - 1; k >= 0; --k) {
      const double tk = tau[k];
      if (tk == 0.0) continue;
      const double* v = V + (size_t)ldv * k;
      double d = 0.0;
      for (int i = k + 1 + lane; i < m; i += 32) d += v[i] * y[i];
      d = warp_sum(d);
      d += y[k];
      const double f = tk * d;
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

// One-sided Jacobi on G (s x n, ld ldg, shared; n even, column n-1 may be a zero pad).
// Round-robin (circle) ordering: n/2 disjoint pairs per round, one warp per pair.
__device__ bool one_sided_jacobi(double* G, int s, int n, int ldg, int* flag) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double tol = 1e-15;
  for (int sweep = 0; sweep < 60; ++sweep) {
    if (threadIdx.x == 0) *flag = 0;
    __syncthreads();
    for (int round = 0; round < n - 1; ++round) {
      for (int k = warp; k < n / 2; k += kOrthWarps) {
        int p, q;
        if (k == 0) {
          p = n - 1;
          q = round;
        } else {
          p = (round + k) % (n - 1);
          q = (round - k + (n - 1)) % (n - 1);
        }
        if (p > q) {
          int tmp = p;
          p = q;
          q = tmp;
        }
        double* gp = G + (size_t)ldg * p;
        double* gq = G + (size_t)ldg * q;
        double a = 0.0, b = 0.0, c = 0.0;
        for (int i = lane; i < s; i += 32) {
          double x = gp[i], y = gq[i];
          a += x * x;
          b += y * y;
          c += x * y;
        }
        a = warp_sum(a);
        b = warp_sum(b);
        c = warp_sum(c);
        if (c != 0.0 && fabs(c) > tol * sqrt(a) * sqrt(b)) {
          const double zeta = (b - a) / (2.0 * c);
          const double t = copysign(1.0, zeta) / (fabs(zeta) + hypot(1.0, zeta));
          const double cs = 1.0 / sqrt(1.0 + t * t);
          const double sn = cs * t;
          for (int i = lane; i < s; i += 32) {
            double x = gp[i], y = gq[i];
            gp[i] = cs * x - sn * y;
            gq[i] = sn * x + cs * y;
          }
          if (lane == 0) *flag = 1;
        }
      }
      __syncthreads();
    }
    const int f = *flag;
    __syncthreads();
    if (!f) return true;
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
  block_householder_qr(W, rows, s, rows, t);
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
// Phase B: one CTA. S (m x s, lds) -> QR -> Jacobi SVD of R -> Y = Q [U_R(:, :mu); 0].
// final != 0: sign-fix Y and write it to out (ld = m); else write Y to out unsigned.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kOrthThreads) orth_core_kernel(
    const double* __restrict__ S, int m, int s, int lds, int mu, double* __restrict__ out,
    int ldo, int final_level, int* status) {
  extern __shared__ __align__(16) double sm[];
  const int n = s + (s & 1);  // even column count for the tournament
  double* A = sm;                                   // m x s
  double* Y = A + (size_t)m * s;                    // m x mu
  double* G = Y + (size_t)m * mu;                   // s x n
  double* tau = G + (size_t)s * n;                  // s
  double* sig = tau + s;                            // n
  int* perm = reinterpret_cast<int*>(sig + n);      // n
  int* flag = perm + n;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  for (int e = threadIdx.x; e < m * s; e += kOrthThreads) {
    int i = e % m, c = e / m;
    A[e] = S[i + (size_t)lds * c];
  }
  __syncthreads();
  block_householder_qr(A, m, s, m, tau);
  __syncthreads();
  // G = R (s x s upper triangle), zero pad column
  for (int e = threadIdx.x; e < s * n; e += kOrthThreads) {
    int i = e % s, c = e / s;
    G[e] = (c < s && i <= c && i < m) ? A[i + (size_t)m * c] : 0.0;
  }
  __syncthreads();
  const bool converged = one_sided_jacobi(G, s, n, s, flag);
  // singular values = column norms, fixed order
  for (int c = warp; c < n; c += kOrthWarps) {
    double a = 0.0;
    for (int i = lane; i < s; i += 32) a += G[i + (size_t)s * c] * G[i + (size_t)s * c];
    a = warp_sum(a);
    if (lane == 0) sig[c] = sqrt(a);
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // stable descending sort of the s real columns (pad excluded)
    for (int c = 0; c < s; ++c) perm[c] = c;
    for (int c = 1; c < s; ++c) {
      int v = perm[c];
      int d = c - 1;
      while (d >= 0 && sig[perm[d]] < sig[v]) {
        perm[d + 1] = perm[d];
        --d;
      }
      perm[d + 1] = v;
    }
  }
  __syncthreads();
  // Y = [U_R(:, :mu) ; 0]
  for (int e = threadIdx.x; e < m * mu; e += kOrthThreads) {
    int i = e % m, c = e / m;
    double val = 0.0;
    if (i < s) {
      int src = perm[c];
      double sg = sig[src];
      val = sg > 0.0 ? G[i + (size_t)s * src] / sg : 0.0;
    }
    Y[e] = val;
  }
  __syncthreads();
  // complete the basis for exactly-zero singular values (rank-deficient sketch)
  if (warp == 0) {
    int next_e = 0;
    for (int c = 0; c < mu; ++c) {
      if (sig[perm[c]] > 0.0) continue;
      while (next_e < s) {
        double* y = Y + (size_t)m * c;
        for (int i = lane; i < s; i += 32) y[i] = (i == next_e) ? 1.0 : 0.0;
        __syncwarp();
        for (int pass = 0; pass < 2; ++pass) {
          for (int c2 = 0; c2 < mu; ++c2) {
            if (c2 == c || (c2 > c && sig[perm[c2]] <= 0.0)) continue;
            const double* z = Y + (size_t)m * c2;
            double d = 0.0;
            for (int i = lane; i < s; i += 32) d += z[i] * y[i];
            d = warp_sum(d);
            for (int i = lane; i < s; i += 32) y[i] -= d * z[i];
            __syncwarp();
          }
        }
        double nn = 0.0;
        for (int i = lane; i < s; i += 32) nn += y[i] * y[i];
        nn = sqrt(warp_sum(nn));
        ++next_e;
        if (nn > 0.5) {
          for (int i = lane; i < s; i += 32) y[i] /= nn;
          __syncwarp();
          break;
        }
      }
    }
  }
  __syncthreads();
  apply_q(A, m, tau, m, s, Y, m, mu);
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
// With final != 0 also records per-block column argmax partials.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kOrthThreads) orth_block_apply_kernel(
    const double* __restrict__ V, long long m, int s, int ldv, int nb,
    const double* __restrict__ tau, const double* __restrict__ W, int ldw, int mu,
    double* __restrict__ out, int ldo, double* __restrict__ pbest, int* __restrict__ pidx) {
  extern __shared__ __align__(16) double sm[];
  const int b = blockIdx.x;
  const long long r0 = (m * b) / nb, r1 = (m * (b + 1)) / nb;
  const int rows = (int)(r1 - r0);
  double* Y = sm;  // rows x mu
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int e = threadIdx.x; e < rows * mu; e += kOrthThreads) {
    int i = e % rows, c = e / rows;
    Y[e] = i < s ? W[(size_t)b * s + i + (size_t)ldw * c] : 0.0;
  }
  __syncthreads();
  apply_q(V + r0, ldv, tau + (size_t)b * s, rows, s, Y, rows, mu);
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
  size_t a_off, v_off, tau_off, w_off;  // workspace offsets (doubles); a_off = input
};

static size_t core_smem(long long m, int s, int mu) {
  int n = s + (s & 1);
  return sizeof(double) * ((size_t)m * s + (size_t)m * mu + (size_t)s * n + s + n) +
         sizeof(int) * (n + 1) + 64;
}

static std::vector<OrthLevel> plan_levels(long long I, int s, int mu, size_t* total) {
  std::vector<OrthLevel> lv;
  size_t off = 0;
  long long m = I;
  // level 0 input is the caller's C (not in the workspace)
  while (core_smem(m, s, mu) > kOrthSmemBudget) {
    long long per = (long long)(kOrthSmemBudget / (sizeof(double) * (size_t)std::max(s, mu))) - 8;
    int nb = (int)((m + per - 1) / per);
    nb = std::max(nb, 2);
    OrthLevel L;
    L.m = m;
    L.nb = nb;
    L.a_off = lv.empty() ? (size_t)-1 : lv.back().w_off;  // input = previous level's stacked R
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
  // upper bound over mu <= s (more levels and wider W buffers at mu = s)
  size_t used = 0;
  std::vector<OrthLevel> lv = plan_levels(I, s, s, &used);
  for (auto& L : lv) used += (size_t)L.nb * s * s;
  if (!lv.empty()) used += (size_t)lv[0].nb * s * 2;
  return used + 64;
}

cudaError_t launch_orth(const double* c, long long I, int s, int mu, double* u, double* work,
                        int* status, cudaStream_t st) {
  if (s < 1 || s > kOrthMaxS || mu < 1 || mu > s || I < s) return cudaErrorInvalidValue;
  static unsigned long long a1 = 0, a2 = 0, a3 = 0;
  cudaError_t e;
  if ((e = ensure_smem_attr(reinterpret_cast<const void*>(orth_core_kernel), kOrthSmemBudget + 16384, a1)) != cudaSuccess) return e;
  if ((e = ensure_smem_attr(reinterpret_cast<const void*>(orth_block_qr_kernel), kOrthSmemBudget + 16384, a2)) != cudaSuccess) return e;
  if ((e = ensure_smem_attr(reinterpret_cast<const void*>(orth_block_apply_kernel), kOrthSmemBudget + 16384, a3)) != cudaSuccess) return e;

  size_t used = 0;
  std::vector<OrthLevel> lv = plan_levels(I, s, mu, &used);
  if (lv.empty()) {
    orth_core_kernel<<<1, kOrthThreads, core_smem(I, s, mu), st>>>(c, (int)I, s, (int)I, mu, u,
                                                                    (int)I, 1, status);
    return cudaGetLastError();
  }
  // W buffers after the level data
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
      work + last.w_off, mB, s, mB, mu, work + wbuf.back(), mB, 0, status);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  // phase C, back down
  for (int l = (int)lv.size() - 1; l >= 0; --l) {
    const OrthLevel& L = lv[l];
    const double* W = work + wbuf[l];
    const int ldw = L.nb * s;
    double* out = l == 0 ? u : work + wbuf[l - 1];
    const int ldo = (int)L.m;
    long long per = (L.m + L.nb - 1) / L.nb;
    size_t smem = sizeof(double) * (size_t)per * mu + 64;
    orth_block_apply_kernel<<<L.nb, kOrthThreads, smem, st>>>(
        work + L.v_off, L.m, s, (int)L.m, L.nb, work + L.tau_off, W, ldw, mu, out, ldo,
        l == 0 ? pbest : nullptr, l == 0 ? pidx : nullptr);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  orth_signfix_kernel<<<mu, 256, 0, st>>>(u, I, (int)I, mu, lv[0].nb, pbest, pidx);
  return cudaGetLastError();
}

}  // namespace lmra_dev

// cholqr.cu -- orthonormal basis of a sketch C (I x s, s <= 64) by shifted CholeskyQR3 in one
// thread-block cluster.
//
// The Householder TSQR of orth.cu factors C with ~s dependent reflector steps per tree level
// (leaf QR, stacked-R QR, two reflector back-applications: ~0.27 ms for cfg4's 1000 x 60 sketch,
// all of it on the critical path between the sampling chain and the core contraction).  CholeskyQR
// replaces those chains by Gram products and one s x s Cholesky per pass:
//   pass 0   G = C^T C + sigma I, sigma = 11 (I s + s (s + 1)) u tr(G)   (shifted CholeskyQR;
//            Fukaya, Kannan, Nakatsukasa, Yamamoto, Yanagisawa 2020): Q1 = C R1^{-1} has
//            kappa(Q1) <= ~1e5 whatever kappa(C) <= ~u^{-1} is -- the sketches reach 1e16
//   pass 1-2 plain CholeskyQR of Q1, Q2 (CholeskyQR2): Q orthonormal to O(u)
// and C = Q R with R = R3 R2 R1, backward stable like Householder QR (||C - Q R|| = O(u) ||C||).
// The caller takes the left singular vectors of C as Q x (those of R): the s x s SVD follows.
//
// Failure is detected, never hidden: a non-positive or non-finite Cholesky pivot in any pass, or
// a last-pass pivot outside [1/2, 2] (Q2 then is not nearly orthonormal, e.g. a numerically
// rank-deficient C, for which no C R^{-1} basis exists), sets *fail = 1; the orth.cu launchers
// enqueue the Householder TSQR behind this kernel gated on that flag.
//
// Layout: cluster of P <= 8 CTAs, CTA c owns rows [I c / P, I (c + 1) / P) of C, kept in shared
// memory row-major (ld 68 == 4 mod 16: the m16n8k4 DMMA fragments of Q as A or B operand are
// conflict-free).  Per pass: partial Gram Q_c^T Q_c on the fp64 tensor pipe (DMMA) -> one
// reduce-scatter + broadcast through distributed shared memory (fixed summation order, so every
// CTA holds the same bits) -> the Cholesky and R^{-1} redundantly in every CTA (identical
// arithmetic, identical results, no broadcast) -> Q_c <- Q_c R^{-1} on the DMMA pipe.  CTA 0
// accumulates R = R3 R2 R1.  Every reduction runs in a fixed order: deterministic run to run.
#include <cstdlib>

#include "common.cuh"

namespace lmra_dev {

namespace {

constexpr int kCqThreads = 512;
constexpr int kCqS = 64;     // padded sketch width
constexpr int kCqLdQ = 68;   // row-major Q block and R^{-1}: == 4 (mod 16) doubles
constexpr int kCqLdG = 65;   // Gram / Cholesky work matrix
constexpr int kCqMaxP = 8;
constexpr int kCqMaxRows16 = 160;

__host__ __device__ constexpr size_t cq_smem_doubles(int rows16) {
  return (size_t)rows16 * kCqLdQ + kCqS * kCqS + kCqS * kCqLdG + 2 * kCqS * kCqLdQ + 16 + 4 * 272 + 8;
}

// the same shared address in the first 8 CTAs of the cluster (rank q >= P reads rank P - 1),
// eight loads in flight at once
__device__ __forceinline__ void cq_dsmem_ld8(uint32_t la, int P, double (&v)[8]) {
  uint32_t ra[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) ra[q] = dsmem_addr(la, (uint32_t)(q < P ? q : P - 1));
  asm volatile(
      "ld.shared::cluster.f64 %0, [%8];\n ld.shared::cluster.f64 %1, [%9];\n"
      "ld.shared::cluster.f64 %2, [%10];\n ld.shared::cluster.f64 %3, [%11];\n"
      "ld.shared::cluster.f64 %4, [%12];\n ld.shared::cluster.f64 %5, [%13];\n"
      "ld.shared::cluster.f64 %6, [%14];\n ld.shared::cluster.f64 %7, [%15];\n"
      : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]), "=d"(v[4]), "=d"(v[5]), "=d"(v[6]), "=d"(v[7])
      : "r"(ra[0]), "r"(ra[1]), "r"(ra[2]), "r"(ra[3]), "r"(ra[4]), "r"(ra[5]), "r"(ra[6]), "r"(ra[7])
      : "memory");
}

__device__ __forceinline__ void named_bar_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

__device__ __forceinline__ double cq_rsqrt(double x) {  // approximation + two Newton steps
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double h = 0.5 * x;
  y = y * fma(-h * y, y, 1.5);
  y = y * fma(-h * y, y, 1.5);
  return y;
}

#ifdef LMRA_CHOLQR_CLOCKS  // microbenchmark only (tools/microbench/cholqr_bench.cu): CTA 0 phase cycles
__device__ unsigned long long g_cqclk[10];
#define CQ_T(idx)                                                   \
  do {                                                              \
    __syncthreads();                                                \
    if (threadIdx.x == 0 && rank == 0) {                            \
      const long long _n = clock64();                               \
      g_cqclk[idx] += _n - cq_t0;                                   \
      cq_t0 = _n;                                                   \
    }                                                               \
  } while (0)
#else
#define CQ_T(idx)
#endif

__global__ void __launch_bounds__(kCqThreads, 1) cholqr_kernel(const double* __restrict__ c, long long I, int s,
                                                               int P, double* __restrict__ qc,
                                                               double* __restrict__ rout, int* __restrict__ fail) {
  pdl_wait();  // the sketch is the previous kernel's output (programmatic dependent launch)
  extern __shared__ __align__(16) double sm[];
  const int rank = (int)cluster_ctarank();
  const long long r0 = I * rank / P, r1 = I * (rank + 1) / P;
  const int rb = (int)(r1 - r0);
  // the same shared-memory layout in every CTA (remote addresses are mapped from local ones)
  const int rows16 = (int)(((I + P - 1) / P + 15) & ~15LL);
  double* Q = sm;                        // rows16 x 68, row-major
  double* Gp = Q + rows16 * kCqLdQ;      // 64 x 64: this CTA's partial Gram (read by every CTA)
  double* G = Gp + kCqS * kCqS;          // 64 x 65: reduced Gram; Cholesky in place: the lower
                                         // triangle is the trailing matrix, the strict upper R
  double* Ri = G + kCqS * kCqLdG;        // 64 x 68: L^{-1} = R^{-T} (lower), row-major
  double* Rt = Ri + kCqS * kCqLdQ;       // 64 x 68: R3 R2 R1 (CTA 0), row-major
  double* pinv = Rt + kCqS * kCqLdQ;     // [16] P^{-1} of the current pivot tile
  // per-tile panels at a stride of 17 doubles (lanes of a warp reading different tiles hit
  // different banks)
  double* lblk = pinv + 16;              // [16][17] L_k^{-1} of every pivot tile
  double* wpan = lblk + 272;             // [16][17] multipliers W_i of the current block column
  double* gpan = wpan + 272;             // [16][17] the block column G(i, kb)
  double* epan = gpan + 272;             // [16][17] E's block row kb
  int* sflag = reinterpret_cast<int*>(epan + 272);
  double* sshift = reinterpret_cast<double*>(sflag + 2);
  const int tid = threadIdx.x, w = tid >> 5, l = tid & 31, g = l >> 2, t = l & 3;
#ifdef LMRA_CHOLQR_CLOCKS
  long long cq_t0 = clock64();
#endif

  // C rows -> Q (coalesced global reads), zero padding rows and columns
  for (int e = tid; e < rows16 * kCqS; e += kCqThreads) {
    const int i = e % rows16, j = e / rows16;
    Q[i * kCqLdQ + j] = (i < rb && j < s) ? c[r0 + i + I * j] : 0.0;
  }
  if (tid == 0) sflag[0] = 0;
  __syncthreads();
  CQ_T(0);

  for (int pass = 0; pass < 3; ++pass) {
    // ---- partial Gram Q_c^T Q_c, lower triangle only (DMMA m16n8k4): the 20 16 x 8 tiles at or
    // below the diagonal, two per warp (warps 0-9) sharing the A fragment; even / odd k-steps
    // accumulate separately (four independent DMMA chains per warp), summed at the end
    if (w < 10) {
      // warp -> (a, b0): a = 0: 1 warp, a = 1: 2, a = 2: 3, a = 3: 4 (tiles b0, b0 + 1)
      const int a = w < 1 ? 0 : w < 3 ? 1 : w < 6 ? 2 : 3;
      const int b0 = 2 * (w - (a * (a + 1)) / 2);
      double d0[4] = {0.0, 0.0, 0.0, 0.0}, d1[4] = {0.0, 0.0, 0.0, 0.0};
      double e0[4] = {0.0, 0.0, 0.0, 0.0}, e1[4] = {0.0, 0.0, 0.0, 0.0};
      for (int k = 0; k < rows16; k += 8) {
        const double* qr = Q + (k + t) * kCqLdQ;
        const double* qs = qr + 4 * kCqLdQ;
        const double a0 = qr[16 * a + g], a1 = qr[16 * a + g + 8], bb0 = qr[8 * b0 + g], bb1 = qr[8 * b0 + 8 + g];
        const double c0 = qs[16 * a + g], c1 = qs[16 * a + g + 8], cb0 = qs[8 * b0 + g], cb1 = qs[8 * b0 + 8 + g];
        dmma16x8x4(d0, a0, a1, bb0);
        dmma16x8x4(d1, a0, a1, bb1);
        dmma16x8x4(e0, c0, c1, cb0);
        dmma16x8x4(e1, c0, c1, cb1);
      }
      double* o = Gp + (16 * a + g) * kCqS + 8 * b0 + 2 * t;
      o[0] = d0[0] + e0[0];
      o[1] = d0[1] + e0[1];
      o[8 * kCqS] = d0[2] + e0[2];
      o[8 * kCqS + 1] = d0[3] + e0[3];
      o[8] = d1[0] + e1[0];
      o[9] = d1[1] + e1[1];
      o[8 * kCqS + 8] = d1[2] + e1[2];
      o[8 * kCqS + 9] = d1[3] + e1[3];
    }
    CQ_T(1);
    cluster_sync();  // every CTA's partial is complete (and the previous pass is done with G)
    // ---- reduce-scatter + broadcast of the lower triangle: CTA `rank` sums its slice of the
    // entries over the P partials in CTA order and stores the sums into every CTA's G
    {
      const int per = (kCqS * kCqS + P - 1) / P;
      const int e0 = rank * per, e1 = min(kCqS * kCqS, e0 + per);
      for (int e = e0 + tid; e < e1; e += kCqThreads) {
        const int i = e >> 6, j = e & 63;
        if (j > i) continue;
        const uint32_t la = smem_u32(Gp + e);
        double pv[8];
        cq_dsmem_ld8(la, P, pv);
        double v = 0.0;
#pragma unroll
        for (int q = 0; q < kCqMaxP; ++q)
          if (q < P) v += pv[q];
        const uint32_t da = smem_u32(G + i * kCqLdG + j);
        for (int q = 0; q < P; ++q) dsmem_st_f64(dsmem_addr(da, (uint32_t)q), v);
      }
    }
    cluster_sync();  // the reduced lower triangle is in every CTA
    CQ_T(2);
    if (pass == 0) {  // shift sigma = 11 (I s + s (s + 1)) u tr(G) on the diagonal
      if (tid == 0) {
        double tr = 0.0;
        for (int i = 0; i < s; ++i) tr += G[i * kCqLdG + i];
        *sshift = 11.0 * ((double)I * s + (double)s * (s + 1)) * 0x1.0p-53 * tr;
      }
      __syncthreads();
      if (tid < s) G[tid * kCqLdG + tid] += *sshift;
    }
    // ---- Cholesky G = L L^T by block elimination on 4 x 4 tiles, with L^{-1} from the same block
    // row operations applied to the identity (E).  Block step kb: the pivot tile P = G(kb, kb) is
    // factored P = L_k L_k^T by its owner (A); every panel tile i > kb forms the multipliers
    // W_i = G(i, kb) P^{-1} and publishes them with G(i, kb), the E tiles of block row kb publish
    // themselves (C); then G(i, j) -= W_i G(j, kb)^T (kb < j <= i) and E(i, j) -= W_i E(kb, j)
    // (j <= kb) (U).  At the end L^{-1} = blockdiag(L_k^{-1}) E, and R = L^T: R(kb, kb) = L_k^T,
    // R(kb, i) = L_k^{-1} G(i, kb)^T, written to G's upper triangle (incl. the diagonal).
    // Threads: warps 0-4 own the 136 lower tiles of G, warps 5-9 those of E, one per thread, in
    // registers; two named barriers (warps 0-9) per block step, 16 block steps at most.
    double* E = Ri;  // L^{-1}, row-major ld 68 (written once at the end)
    if (w < 10) {
      const bool isE = w >= 5;
      const int tix = isE ? tid - 160 : tid;  // packed lower-triangle tile index over 16 x 16
      const bool own = tix < 136;
      int ti = 0;
      while ((ti + 1) * (ti + 2) / 2 <= tix) ++ti;
      const int tj = tix - ti * (ti + 1) / 2;
      const int i0 = 4 * ti, j0 = 4 * tj;
      double v[4][4];
#pragma unroll
      for (int a2 = 0; a2 < 4; ++a2)
#pragma unroll
        for (int b2 = 0; b2 < 4; ++b2) {
          const int i = i0 + a2, j = j0 + b2;
          v[a2][b2] = !own ? 0.0 : isE ? (i == j ? 1.0 : 0.0) : (i < s && j <= i) ? G[i * kCqLdG + j] : 0.0;
        }
      const int nb = (s + 3) >> 2;
      const bool pass2 = pass == 2;
      named_bar_sync(1, 320);  // every G tile has read the reduced Gram (R goes to G's upper part)
#ifdef LMRA_CHOLQR_CLOCKS
      long long tb0 = clock64();
#endif
      for (int kb = 0; kb < nb; ++kb) {
        // (A) pivot tile: P = L L^T (4 x 4, entries past s on an identity), L^{-1}, P^{-1}
        if (own && !isE && ti == kb && tj == kb) {
          double L[4][4], Li[4][4];
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            double d = v[c][c];
#pragma unroll
            for (int m2 = 0; m2 < c; ++m2) d = fma(-L[c][m2], L[c][m2], d);
            if (i0 + c >= s) d = 1.0;
            const bool bad = !(d > 0.0) || !(d < 0x1.0p+1000) || (pass2 && !(d >= 0.5 && d <= 2.0));
            if (bad) {
              sflag[0] = 1;
              d = 1.0;
            }
            const double rc = cq_rsqrt(d);
            L[c][c] = d * rc;
#pragma unroll
            for (int r2 = c + 1; r2 < 4; ++r2) {
              double x = i0 + r2 < s ? v[r2][c] : 0.0;
#pragma unroll
              for (int m2 = 0; m2 < c; ++m2) x = fma(-L[r2][m2], L[c][m2], x);
              L[r2][c] = x * rc;
            }
#pragma unroll
            for (int r2 = 0; r2 < c; ++r2) L[r2][c] = 0.0;
            Li[c][c] = rc;
          }
#pragma unroll
          for (int c = 0; c < 4; ++c)  // L^{-1}: forward substitution, column c
#pragma unroll
            for (int r2 = 0; r2 < 4; ++r2) {
              if (r2 > c) {
                double x = 0.0;
#pragma unroll
                for (int m2 = c; m2 < r2; ++m2) x = fma(-L[r2][m2], Li[m2][c], x);
                Li[r2][c] = x * Li[r2][r2];
              } else if (r2 < c) {
                Li[r2][c] = 0.0;
              }
            }
#pragma unroll
          for (int a2 = 0; a2 < 4; ++a2)
#pragma unroll
            for (int b2 = 0; b2 < 4; ++b2) {
              double x = 0.0;  // P^{-1} = L^{-T} L^{-1}
#pragma unroll
              for (int m2 = 0; m2 < 4; ++m2) x = fma(Li[m2][a2], Li[m2][b2], x);
              pinv[a2 * 4 + b2] = x;
              lblk[kb * 17 + a2 * 4 + b2] = Li[a2][b2];
              if (b2 >= a2 && i0 + b2 < s) G[(i0 + a2) * kCqLdG + i0 + b2] = L[b2][a2];  // R(kb, kb) = L^T
            }
        }
        named_bar_sync(1, 320);
#ifdef LMRA_CHOLQR_CLOCKS
        long long tb1 = clock64();
        if (tid == 0 && rank == 0) g_cqclk[8] += tb1 - tb0;
#endif
        // (C) panel tiles: W_i = G(i, kb) P^{-1}, R(kb, i) = L_k^{-1} G(i, kb)^T; E row block kb
        if (own && !isE && tj == kb && ti > kb) {
          double pv[16], lk[16];
#pragma unroll
          for (int e2 = 0; e2 < 16; ++e2) {
            pv[e2] = pinv[e2];
            lk[e2] = lblk[kb * 17 + e2];
          }
#pragma unroll
          for (int a2 = 0; a2 < 4; ++a2)
#pragma unroll
            for (int b2 = 0; b2 < 4; ++b2) {
              double x = 0.0, y = 0.0;
#pragma unroll
              for (int m2 = 0; m2 < 4; ++m2) {
                x = fma(v[a2][m2], pv[m2 * 4 + b2], x);
                y = fma(lk[b2 * 4 + m2], v[a2][m2], y);  // (L_k^{-1} G(i,kb)^T)(b2, a2)
              }
              wpan[ti * 17 + a2 * 4 + b2] = x;
              gpan[ti * 17 + a2 * 4 + b2] = v[a2][b2];
              if (i0 + a2 < s && j0 + b2 < s) G[(j0 + b2) * kCqLdG + i0 + a2] = y;
            }
        }
        if (own && isE && ti == kb)
#pragma unroll
          for (int a2 = 0; a2 < 4; ++a2)
#pragma unroll
            for (int b2 = 0; b2 < 4; ++b2) epan[tj * 17 + a2 * 4 + b2] = v[a2][b2];
        named_bar_sync(1, 320);
#ifdef LMRA_CHOLQR_CLOCKS
        tb0 = clock64();
        if (tid == 0 && rank == 0) g_cqclk[9] += tb0 - tb1;
#endif
        // (U) trailing G tiles and E tiles below block row kb
        if (own && ti > kb && (isE ? tj <= kb : tj > kb)) {
          double wv[16], ov[16];
#pragma unroll
          for (int e2 = 0; e2 < 16; ++e2) {
            wv[e2] = wpan[ti * 17 + e2];
            ov[e2] = isE ? epan[tj * 17 + e2] : gpan[tj * 17 + e2];
          }
#pragma unroll
          for (int a2 = 0; a2 < 4; ++a2)
#pragma unroll
            for (int b2 = 0; b2 < 4; ++b2) {
              double x = v[a2][b2];
#pragma unroll
              for (int m2 = 0; m2 < 4; ++m2)  // G: W_i G(j,kb)^T (ov row b2); E: W_i E(kb,j) (ov column b2)
                x = fma(-wv[a2 * 4 + m2], isE ? ov[m2 * 4 + b2] : ov[b2 * 4 + m2], x);
              v[a2][b2] = x;
            }
        }
      }
      if (own && isE) {  // L^{-1}(i, j) = L_ti^{-1} E(ti, j)
        double lk[16];
#pragma unroll
        for (int e2 = 0; e2 < 16; ++e2) lk[e2] = lblk[ti * 17 + e2];
#pragma unroll
        for (int a2 = 0; a2 < 4; ++a2)
#pragma unroll
          for (int b2 = 0; b2 < 4; ++b2) {
            double x = 0.0;
#pragma unroll
            for (int m2 = 0; m2 < 4; ++m2) x = fma(lk[a2 * 4 + m2], v[m2][b2], x);
            const int i = i0 + a2, j = j0 + b2;
            E[i * kCqLdQ + j] = (i < s && j <= i) ? x : 0.0;
          }
      }
    } else {
      // warps 10-15: zero E's strict upper triangle (the E tiles write the lower one) and padding
      for (int e = tid - 320; e < kCqS * kCqLdQ; e += kCqThreads - 320) {
        const int i = e / kCqLdQ, j = e % kCqLdQ;
        if (j > i || j >= kCqS) E[e] = 0.0;
      }
    }
    __syncthreads();
    CQ_T(3);
    // ---- Q_c <- Q_c R^{-1} = Q_c L^{-T} (DMMA m16n8k4): B(k, j) = L^{-1}(j, k), 0 for k > j.
    // Warp w: row blocks (w >> 1) + 8 r, column blocks (w & 1) + {0, 2, 4, 6} (the four tiles
    // share each A fragment); results stay in registers until every warp is done reading Q
    {
      const int nrb = rows16 / 16;
      constexpr int kRb = (kCqMaxRows16 / 16 + 7) / 8;  // row blocks per warp
      double acc[kRb][4][4];
      const int cb0 = w & 1;
      const int kend = min(s, 8 * (cb0 + 6) + 8);
#pragma unroll
      for (int rr = 0; rr < kRb; ++rr) {
#pragma unroll
        for (int ti = 0; ti < 4; ++ti) acc[rr][ti][0] = acc[rr][ti][1] = acc[rr][ti][2] = acc[rr][ti][3] = 0.0;
        const int rbk = (w >> 1) + 8 * rr;
        if (rbk < nrb) {
          const double* qa = Q + (16 * rbk + g) * kCqLdQ + t;
          for (int k = 0; k < kend; k += 4) {
            const double a0 = qa[k], a1 = qa[8 * kCqLdQ + k];
#pragma unroll
            for (int ti = 0; ti < 4; ++ti) {
              const int cb = cb0 + 2 * ti;
              if (k < 8 * cb + 8) dmma16x8x4(acc[rr][ti], a0, a1, E[(8 * cb + g) * kCqLdQ + k + t]);
            }
          }
        }
      }
      __syncthreads();  // every warp is done reading Q
#pragma unroll
      for (int rr = 0; rr < kRb; ++rr) {
        const int rbk = (w >> 1) + 8 * rr;
        if (rbk < nrb)
#pragma unroll
          for (int ti = 0; ti < 4; ++ti) {
            const int cb = cb0 + 2 * ti;
            double* o = Q + (16 * rbk + g) * kCqLdQ + 8 * cb + 2 * t;
            o[0] = acc[rr][ti][0];
            o[1] = acc[rr][ti][1];
            o[8 * kCqLdQ] = acc[rr][ti][2];
            o[8 * kCqLdQ + 1] = acc[rr][ti][3];
          }
      }
    }
    __syncthreads();
    CQ_T(5);
    // ---- CTA 0: R_total <- R_pass R_total (DMMA; R_pass = the upper triangle of G incl. the
    // diagonal, 0 below)
    if (rank == 0) {
      if (pass == 0) {
        for (int e = tid; e < kCqS * kCqLdQ; e += kCqThreads) {
          const int i = e / kCqLdQ, j = e % kCqLdQ;
          Rt[e] = (i < s && j < s && j >= i) ? G[i * kCqLdG + j] : 0.0;
        }
      } else {
        double acc[2][4];  // 64 x 64 = 4 x 8 tiles of 16 x 8: two per warp
#pragma unroll
        for (int ti = 0; ti < 2; ++ti) acc[ti][0] = acc[ti][1] = acc[ti][2] = acc[ti][3] = 0.0;
        for (int k = 0; k < s; k += 4) {
#pragma unroll
          for (int ti = 0; ti < 2; ++ti) {
            const int tile = w + 16 * ti, rbk = tile >> 3, cb = tile & 7;
            const int i0 = 16 * rbk + g, i1 = i0 + 8, kk = k + t;
            const double a0 = kk >= i0 ? G[i0 * kCqLdG + kk] : 0.0;
            const double a1 = kk >= i1 ? G[i1 * kCqLdG + kk] : 0.0;
            dmma16x8x4(acc[ti], kk < s ? a0 : 0.0, kk < s ? a1 : 0.0, Rt[kk * kCqLdQ + 8 * cb + g]);
          }
        }
        __syncthreads();
#pragma unroll
        for (int ti = 0; ti < 2; ++ti) {
          const int tile = w + 16 * ti, rbk = tile >> 3, cb = tile & 7;
          double* o = Rt + (16 * rbk + g) * kCqLdQ + 8 * cb + 2 * t;
          o[0] = acc[ti][0];
          o[1] = acc[ti][1];
          o[8 * kCqLdQ] = acc[ti][2];
          o[8 * kCqLdQ + 1] = acc[ti][3];
        }
      }
    }
    __syncthreads();
    CQ_T(6);
  }
  pdl_trigger();
  for (int e = tid; e < rb * s; e += kCqThreads) {
    const int i = e % rb, j = e / rb;
    qc[r0 + i + I * j] = Q[i * kCqLdQ + j];
  }
  if (rank == 0) {
    for (int e = tid; e < s * s; e += kCqThreads) {
      const int i = e % s, j = e / s;
      rout[e] = i <= j ? Rt[i * kCqLdQ + j] : 0.0;
    }
    if (tid == 0) *fail = sflag[0];
  }
  // (no remote shared-memory access after the last pass's second cluster barrier)
}

}  // namespace

int cholqr_cluster_size(long long I) {
  long long p = (I + 63) / 64;
  return (int)(p < 1 ? 1 : p > kCqMaxP ? kCqMaxP : p);
}

bool cholqr_supported(long long I, int s) {
  if (s < 1 || s > kCqS || I < s) return false;
  const int P = cholqr_cluster_size(I);
  const long long rb = (I + P - 1) / P;
  return ((rb + 15) & ~15LL) <= kCqMaxRows16;
}

cudaError_t launch_cholqr(const double* c, long long I, int s, double* qc, double* r, int* fail,
                          cudaStream_t st) {
  if (!cholqr_supported(I, s)) return cudaErrorInvalidValue;
  static unsigned long long done = 0;
  const size_t smax = cq_smem_doubles(kCqMaxRows16) * sizeof(double);
  cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(cholqr_kernel), smax, done);
  if (e != cudaSuccess) return e;
  const int P = cholqr_cluster_size(I);
  const int rows16 = (int)(((I + P - 1) / P + 15) & ~15LL);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(P);
  cfg.blockDim = dim3(kCqThreads);
  cfg.dynamicSmemBytes = cq_smem_doubles(rows16) * sizeof(double);
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = P;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  note_launch();
  e = cudaLaunchKernelEx(&cfg, cholqr_kernel, c, I, s, P, qc, r, fail);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace lmra_dev

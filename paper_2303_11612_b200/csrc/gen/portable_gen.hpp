// portable_gen.hpp -- the BASELINE synthetic inputs,
// defined so that the host and the device produce the SAME BITS.
//
// None of the five BASELINE generators exists in the reference, so this file
// is their definition.  Every floating-point step is an explicit IEEE operation -- add,
// mul, div, sqrt and fused multiply-add, each correctly rounded on x86-64 (SSE2 + FMA3,
// compiled with -ffp-contract=off -mfma) and on sm_100a (__dadd_rn / __dmul_rn / __fma_rn /
// __ddiv_rn / __dsqrt_rn, which nvcc never contracts or reorders) -- and every reduction
// runs in one fixed sequential order.  The transcendental functions are our own
// polynomial evaluations (gp_log, gp_sincos): libm's log/sin/cos and CUDA's differ in the
// last ulp, which is why the round-1 device generators could not be reproduced on the
// host.  So:
//   * bench.py's CPU arm generates on the host exactly the tensor the GPU arm generates on
//     the device, without loading the GPU library;
//   * a multi-GPU rank generates only its slab of the last mode (every element is
//     independent, the normal streams jump ahead, and the two norms that scale the noise
//     are sums of per-slice totals in slice order);
//   * the parity tests check device == host generation bit for bit.
//
// The integer part is the reference's PCG32 (rng.hpp:20-36, seeding and output function)
// and next_double (rng.hpp:45-50); the Box-Muller transform follows rng.hpp:52-63
// (u1 = 1 - next_double, z0 = r cos, z1 = r sin) with the portable log / sincos.
//
// Used by: kernels/gen.cu (device kernels), lmra_b200.cpp (host halves: Omega-free small
// factors U_n, profiles), oracle/lmra_oracle.cpp (the host generators the CPU arm and the
// tests use).  This is input synthesis, not the algorithm under test.
#pragma once

#include <stdint.h>
#include <string.h>

#if defined(__CUDACC__)
#define GP_HD __host__ __device__ __forceinline__
#else
#define GP_HD inline
#include <cmath>
#endif

namespace lmra_gen {

// ------------------------------------------------------------------ exact IEEE operations
GP_HD double gp_add(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dadd_rn(a, b);
#else
  return a + b;
#endif
}
GP_HD double gp_mul(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dmul_rn(a, b);
#else
  return a * b;
#endif
}
GP_HD double gp_fma(double a, double b, double c) {
#if defined(__CUDA_ARCH__)
  return __fma_rn(a, b, c);
#else
  return __builtin_fma(a, b, c);
#endif
}
GP_HD double gp_div(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __ddiv_rn(a, b);
#else
  return a / b;
#endif
}
GP_HD double gp_sqrt(double a) {
#if defined(__CUDA_ARCH__)
  return __dsqrt_rn(a);
#else
  return __builtin_sqrt(a);
#endif
}
GP_HD double gp_rint(double a) {  // round half to even (the default rounding mode on the host)
#if defined(__CUDA_ARCH__)
  return rint(a);
#else
  return __builtin_nearbyint(a);
#endif
}
GP_HD uint64_t gp_bits(double x) {
#if defined(__CUDA_ARCH__)
  return (uint64_t)__double_as_longlong(x);
#else
  uint64_t u;
  memcpy(&u, &x, 8);
  return u;
#endif
}
GP_HD double gp_from_bits(uint64_t u) {
#if defined(__CUDA_ARCH__)
  return __longlong_as_double((long long)u);
#else
  double x;
  memcpy(&x, &u, 8);
  return x;
#endif
}

constexpr double kTwoPi = 6.283185307179586476925286766559;

// ------------------------------------------------------------------ log, sincos
// gp_log(x) for finite x > 0 (normal): x = m 2^e with m in (sqrt(1/2), sqrt(2)],
// log m = 2 atanh(f), f = (m - 1) / (m + 1), |f| <= 0.1716: the atanh series to f^23.
GP_HD double gp_log(double x) {
  const uint64_t b = gp_bits(x);
  int e = (int)((b >> 52) & 0x7ff) - 1023;
  double m = gp_from_bits((b & 0x000fffffffffffffULL) | 0x3ff0000000000000ULL);  // [1, 2)
  if (m > 1.4142135623730951) {
    m = gp_mul(m, 0.5);
    e += 1;
  }
  const double f = gp_div(gp_add(m, -1.0), gp_add(m, 1.0));
  const double s = gp_mul(f, f);
  double p = 1.0 / 23.0;
  p = gp_fma(p, s, 1.0 / 21.0);
  p = gp_fma(p, s, 1.0 / 19.0);
  p = gp_fma(p, s, 1.0 / 17.0);
  p = gp_fma(p, s, 1.0 / 15.0);
  p = gp_fma(p, s, 1.0 / 13.0);
  p = gp_fma(p, s, 1.0 / 11.0);
  p = gp_fma(p, s, 1.0 / 9.0);
  p = gp_fma(p, s, 1.0 / 7.0);
  p = gp_fma(p, s, 1.0 / 5.0);
  p = gp_fma(p, s, 1.0 / 3.0);
  // log m = 2 f + 2 f s p
  const double two_f = gp_mul(2.0, f);
  const double logm = gp_fma(gp_mul(two_f, s), p, two_f);
  const double de = (double)e;
  return gp_fma(de, 0.6931471803691238164901733398437500, gp_fma(de, 1.9082149292705877e-10, logm));
}

// sin and cos of |r| <= pi/4 (Taylor to r^17 / r^18)
GP_HD void gp_sincos_reduced(double r, double* s, double* c) {
  const double z = gp_mul(r, r);
  double ps = -1.0 / 355687428096000.0;          // -1/17!
  ps = gp_fma(ps, z, 1.0 / 1307674368000.0);      // 1/15!
  ps = gp_fma(ps, z, -1.0 / 6227020800.0);        // -1/13!
  ps = gp_fma(ps, z, 1.0 / 39916800.0);           // 1/11!
  ps = gp_fma(ps, z, -1.0 / 362880.0);            // -1/9!
  ps = gp_fma(ps, z, 1.0 / 5040.0);               // 1/7!
  ps = gp_fma(ps, z, -1.0 / 120.0);               // -1/5!
  ps = gp_fma(ps, z, 1.0 / 6.0);                  // 1/3!  -> sin r = r - r z ps
  *s = gp_fma(-gp_mul(r, z), ps, r);
  double pc = 1.0 / 6402373705728000.0;           // 1/18!
  pc = gp_fma(pc, z, -1.0 / 20922789888000.0);    // -1/16!
  pc = gp_fma(pc, z, 1.0 / 87178291200.0);        // 1/14!
  pc = gp_fma(pc, z, -1.0 / 479001600.0);         // -1/12!
  pc = gp_fma(pc, z, 1.0 / 3628800.0);            // 1/10!
  pc = gp_fma(pc, z, -1.0 / 40320.0);             // -1/8!
  pc = gp_fma(pc, z, 1.0 / 720.0);                // 1/6!
  pc = gp_fma(pc, z, -1.0 / 24.0);                // -1/4!  -> cos r = 1 - z/2 + z^2 (-pc)
  *c = gp_fma(gp_mul(z, z), -pc, gp_fma(z, -0.5, 1.0));
}

// sin / cos of |x| <= ~1e6: x = k pi/2 + r (two-constant Cody-Waite with fma), quadrant k mod 4
GP_HD void gp_sincos(double x, double* s, double* c) {
  const double k = gp_rint(gp_mul(x, 0.63661977236758134308));
  double r = gp_fma(-k, 1.5707963267948966192, x);
  r = gp_fma(-k, 6.123233995736766e-17, r);
  double sr, cr;
  gp_sincos_reduced(r, &sr, &cr);
  const long long q = ((long long)k) & 3;
  if (q == 0) {
    *s = sr;
    *c = cr;
  } else if (q == 1) {
    *s = cr;
    *c = -sr;
  } else if (q == 2) {
    *s = -sr;
    *c = -cr;
  } else {
    *s = -cr;
    *c = sr;
  }
}

GP_HD double gp_cos(double x) {
  double s, c;
  gp_sincos(x, &s, &c);
  return c;
}

// ------------------------------------------------------------------ PCG32 (rng.hpp:20-50)
struct Pcg {
  uint64_t state, inc;
  GP_HD Pcg(uint64_t seed, uint64_t stream) {
    inc = (stream << 1u) | 1u;
    state = 0;
    next();
    state += seed;
    next();
  }
  GP_HD uint32_t next() {
    const uint64_t old = state;
    state = old * 6364136223846793005ULL + inc;
    const uint32_t xs = (uint32_t)(((old >> 18u) ^ old) >> 27u);
    const uint32_t rot = (uint32_t)(old >> 59u);
    return (xs >> rot) | (xs << ((32u - rot) & 31u));
  }
  GP_HD void advance(uint64_t delta) {  // jump ahead by delta u32 draws
    uint64_t cm = 6364136223846793005ULL, cp = inc, am = 1, ap = 0;
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
  GP_HD double next_double() {
    const uint64_t hi = next(), lo = next();
    return (double)(((hi << 32) | lo) >> 11) * 0x1.0p-53;  // exact
  }
  // one Box-Muller pair (u1 = 1 - next_double() in (0, 1], u2 = next_double())
  GP_HD void normal_pair(double* z0, double* z1) {
    const double u1 = gp_add(1.0, -next_double());
    const double u2 = next_double();
    const double r = gp_sqrt(gp_mul(-2.0, gp_log(u1)));
    double sn, cs;
    gp_sincos(gp_mul(kTwoPi, u2), &sn, &cs);
    *z0 = gp_mul(r, cs);
    *z1 = gp_mul(r, sn);
  }
};

// Normal deviates [b, e) of stream (seed, stream): element i is value i % 2 of pair i / 2.
GP_HD void gp_normals_range(uint64_t seed, uint64_t stream, double* out, uint64_t b, uint64_t e) {
  if (b >= e) return;
  Pcg g(seed, stream);
  g.advance(4ull * (b / 2));
  uint64_t i = b;
  if (i & 1) {
    double z0, z1;
    g.normal_pair(&z0, &z1);
    out[0] = z1;
    ++i;
  }
  for (; i < e; i += 2) {
    double z0, z1;
    g.normal_pair(&z0, &z1);
    out[i - b] = z0;
    if (i + 1 < e) out[i + 1 - b] = z1;
  }
}

// Uniform next_double() deviates [b, e) of stream (seed, stream) (two u32 draws each).
GP_HD void gp_uniforms_range(uint64_t seed, uint64_t stream, double* out, uint64_t b, uint64_t e) {
  if (b >= e) return;
  Pcg g(seed, stream);
  g.advance(2ull * b);
  for (uint64_t i = b; i < e; ++i) out[i - b] = g.next_double();
}

// ------------------------------------------------------------------ definitions (host halves)
// Stream ids follow the reference's datagen.cpp:20-23: core 100, factor 101 + n, noise 200;
// the video generator uses 300 + t per term and 400 for its noise.
constexpr uint64_t kStreamCore = 100, kStreamFactor = 101, kStreamNoise = 200;
constexpr uint64_t kStreamTerm = 300, kStreamVideoNoise = 400;

// dot product in index order, fma accumulation from +0
GP_HD double gp_dot(const double* a, const double* b, uint64_t n) {
  double acc = 0.0;
  for (uint64_t i = 0; i < n; ++i) acc = gp_fma(a[i], b[i], acc);
  return acc;
}

#if !defined(__CUDA_ARCH__)
// U (I x c, column-major) = orthonormal basis of the normals of stream (seed, 101 + n),
// I x c column-major: modified Gram-Schmidt applied twice, columns in order.  Requires
// 1 <= c <= I.  Host only (the matrices are small); the device path uploads the result.
inline void gp_orthonormal_factor(uint64_t I, uint64_t c, uint64_t seed, uint64_t n, double* u) {
  gp_normals_range(seed, kStreamFactor + n, u, 0, I * c);
  for (uint64_t j = 0; j < c; ++j) {
    double* v = u + I * j;
    for (int pass = 0; pass < 2; ++pass)
      for (uint64_t k = 0; k < j; ++k) {
        const double* q = u + I * k;
        const double r = gp_dot(q, v, I);
        for (uint64_t i = 0; i < I; ++i) v[i] = gp_fma(-r, q[i], v[i]);
      }
    const double nrm = gp_sqrt(gp_dot(v, v, I));
    for (uint64_t i = 0; i < I; ++i) v[i] = gp_div(v[i], nrm);
  }
}

// Cosine profiles and weights of the video tensor: P_n (I_n x R, column-major) packed mode
// after mode, w (R).  Term t draws from stream (seed, 300 + t): w_t, then per mode f, phase.
inline void gp_video_profiles(const uint64_t* dims, int order, uint64_t n_terms, uint64_t seed,
                              double* profiles, double* w) {
  for (uint64_t t = 0; t < n_terms; ++t) {
    Pcg g(seed, kStreamTerm + t);
    w[t] = g.next_double();
    uint64_t off = 0;
    for (int n = 0; n < order; ++n) {
      const double f = gp_add(0.5, gp_mul(7.5, g.next_double()));
      const double ph = gp_mul(kTwoPi, g.next_double());
      const double tf = gp_mul(kTwoPi, f);
      for (uint64_t i = 0; i < dims[n]; ++i) {
        const double x = gp_div((double)i, (double)dims[n]);
        profiles[off + i + dims[n] * t] = gp_cos(gp_add(gp_mul(tf, x), ph));
      }
      off += dims[n] * n_terms;
    }
  }
}

// noise coefficient gamma * ||B|| / ||E|| from per-slice sums of squares (slices of the last
// mode, in order; the sums are sequential over slices)
inline double gp_noise_coef(const double* slice_b, const double* slice_e, uint64_t L, double gamma) {
  double nb = 0.0, ne = 0.0;
  for (uint64_t l = 0; l < L; ++l) {
    nb = gp_add(nb, slice_b[l]);
    ne = gp_add(ne, slice_e[l]);
  }
  return gp_div(gp_mul(gamma, gp_sqrt(nb)), gp_sqrt(ne));
}
#endif

// ------------------------------------------------------------------ per-element definitions
// Mode product of the Tucker signal: y[a, i, o] = sum_k U[i, k] x[a, k, o], the sum over k
// ascending as an fma chain from +0 (B = G x_0 U_0 x_1 U_1 ... in mode order).
GP_HD double gp_ttm_element(const double* x, long long inner, long long K, const double* u, long long ldu,
                            long long a, long long i, long long o) {
  double acc = 0.0;
  for (long long k = 0; k < K; ++k) acc = gp_fma(u[i + ldu * k], x[a + inner * (k + K * o)], acc);
  return acc;
}

// Video element: sum_t (((w_t P_0(i_0, t)) P_1(i_1, t)) ...), terms in order, from +0.
GP_HD double gp_video_element(const long long* idx, const long long* dims, int order, const double* profiles,
                              const double* w, int n_terms) {
  double acc = 0.0;
  for (int t = 0; t < n_terms; ++t) {
    double v = w[t];
    long long off = 0;
    for (int k = 0; k < order; ++k) {
      v = gp_mul(v, profiles[off + idx[k] + dims[k] * t]);
      off += dims[k] * n_terms;
    }
    acc = gp_add(acc, v);
  }
  return acc;
}

}  // namespace lmra_gen

// lmra_oracle.cpp -- CPU restatement of the reference's randomized Tucker hot path.
//
// TEST INFRASTRUCTURE ONLY (see lmra_oracle.h).  Compiled with -ffp-contract=off so
// every a*b+c the reference writes is two roundings, exactly as in the reference
// sources; the only fused operations are the explicit std::fma in the canonical
// column-norm order.
#include "lmra_oracle.h"
#include "../paper_2303_11612_b200/csrc/gen/portable_gen.hpp"

#include <dlfcn.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstring>
#include <exception>
#include <functional>
#include <numeric>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace {

thread_local std::string g_err;

// ---------------------------------------------------------------- BLAS/LAPACK
using i64 = long long;
typedef void (*dgemm_t)(const char*, const char*, const i64*, const i64*, const i64*,
                        const double*, const double*, const i64*, const double*, const i64*,
                        const double*, double*, const i64*, size_t, size_t);
typedef void (*dgesdd_t)(const char*, const i64*, const i64*, double*, const i64*, double*,
                         double*, const i64*, double*, const i64*, double*, const i64*, i64*,
                         i64*, size_t);
typedef void (*dgeqrf_t)(const i64*, const i64*, double*, const i64*, double*, double*,
                         const i64*, i64*);
typedef void (*dorgqr_t)(const i64*, const i64*, const i64*, double*, const i64*,
                         const double*, double*, const i64*, i64*);
typedef void (*setthreads_t)(int);

struct Blas {
  dgemm_t dgemm = nullptr;
  dgesdd_t dgesdd = nullptr;
  dgeqrf_t dgeqrf = nullptr;
  dorgqr_t dorgqr = nullptr;
  setthreads_t set_threads = nullptr;
} g_blas;

void need_blas() {
  if (!g_blas.dgemm) throw std::runtime_error("oracle: BLAS not initialised (orc_init_blas)");
}

// ---------------------------------------------------------------- RNG, rng.hpp:20-66
struct Rng {
  uint64_t state = 0, inc = 1;
  double cached = 0.0;
  bool has_cached = false;
  Rng(uint64_t seed, uint64_t stream) {  // rng.hpp:22-28
    inc = (stream << 1u) | 1u;
    state = 0;
    next_u32();
    state += seed;
    next_u32();
  }
  uint32_t next_u32() {  // rng.hpp:30-36
    uint64_t old = state;
    state = old * 6364136223846793005ULL + inc;
    uint32_t xs = static_cast<uint32_t>(((old >> 18u) ^ old) >> 27u);
    uint32_t rot = static_cast<uint32_t>(old >> 59u);
    return (xs >> rot) | (xs << ((32u - rot) & 31u));
  }
  double next_double() {  // rng.hpp:39-44
    uint64_t hi = next_u32();
    uint64_t lo = next_u32();
    uint64_t x = (hi << 32) | lo;
    return static_cast<double>(x >> 11) * 0x1.0p-53;
  }
  double next_normal() {  // rng.hpp:47-59
    if (has_cached) {
      has_cached = false;
      return cached;
    }
    double u1 = 1.0 - next_double();
    double u2 = next_double();
    double r = std::sqrt(-2.0 * std::log(u1));
    double a = 6.283185307179586476925286766559 * u2;
    cached = r * std::sin(a);
    has_cached = true;
    return r * std::cos(a);
  }
  // LCG jump-ahead by `delta` u32 draws (O(log delta)); used only to split long
  // normal sequences across threads, bit-identical to sequential generation.
  void advance(uint64_t delta) {
    uint64_t cur_mult = 6364136223846793005ULL, cur_plus = inc;
    uint64_t acc_mult = 1, acc_plus = 0;
    while (delta > 0) {
      if (delta & 1) {
        acc_mult *= cur_mult;
        acc_plus = acc_plus * cur_mult + cur_plus;
      }
      cur_plus = (cur_mult + 1) * cur_plus;
      cur_mult *= cur_mult;
      delta >>= 1;
    }
    state = acc_mult * state + acc_plus;
  }
};

// Fills out[0..n) with normals n0, n0+1, ... of stream (seed, stream): element e is the
// cos (e even) or sin (e odd) half of Box-Muller pair e/2, which consumes draws 4(e/2)..+3.
void fill_normals(uint64_t seed, uint64_t stream, double* out, size_t n, int threads) {
  auto work = [&](size_t b, size_t e) {
    if (b >= e) return;
    Rng g(seed, stream);
    size_t pair = b / 2;
    g.advance(4 * pair);
    size_t i = b;
    if (i & 1) {  // start on the sin half
      g.next_normal();
      out[i++] = g.next_normal();
    }
    for (; i < e; ++i) out[i] = g.next_normal();
  };
  if (threads <= 1 || n < (1u << 20)) {
    work(0, n);
    return;
  }
  std::vector<std::thread> pool;
  size_t chunk = ((n + threads - 1) / threads + 1) & ~size_t(1);
  for (int t = 0; t < threads; ++t) {
    size_t b = std::min(n, t * chunk), e = std::min(n, b + chunk);
    pool.emplace_back(work, b, e);
  }
  for (auto& t : pool) t.join();
}

int default_threads() {
  unsigned h = std::thread::hardware_concurrency();
  return h ? static_cast<int>(h) : 1;
}

// ---------------------------------------------------------------- dense types
struct Mat {  // column-major
  size_t r = 0, c = 0;
  std::vector<double> d;
  Mat() = default;
  Mat(size_t r_, size_t c_) : r(r_), c(c_), d(r_ * c_, 0.0) {}
  double& operator()(size_t i, size_t j) { return d[i + r * j]; }
  double operator()(size_t i, size_t j) const { return d[i + r * j]; }
};

struct Tensor {
  std::vector<size_t> dims;
  std::vector<double> v;
  Tensor() = default;
  explicit Tensor(std::vector<size_t> d) : dims(std::move(d)) {
    size_t n = 1;
    for (size_t x : dims) n *= x;
    v.assign(n, 0.0);
  }
  size_t size() const { return v.size(); }
};

// C = op(A) * op(B), all column-major
void gemm(bool ta, bool tb, size_t m, size_t n, size_t k, const double* a, size_t lda,
          const double* b, size_t ldb, double* c, size_t ldc, double beta = 0.0) {
  need_blas();
  if (m == 0 || n == 0) return;
  i64 M = (i64)m, N = (i64)n, K = (i64)k, LA = (i64)std::max<size_t>(lda, 1),
      LB = (i64)std::max<size_t>(ldb, 1), LC = (i64)std::max<size_t>(ldc, 1);
  double one = 1.0;
  g_blas.dgemm(ta ? "T" : "N", tb ? "T" : "N", &M, &N, &K, &one, a, &LA, b, &LB, &beta, c, &LC,
               1, 1);
}

Mat matmul(const Mat& a, bool ta, const Mat& b, bool tb) {
  size_t m = ta ? a.c : a.r, k = ta ? a.r : a.c, n = tb ? b.r : b.c;
  size_t k2 = tb ? b.c : b.r;
  if (k != k2) throw std::invalid_argument("matmul: inner dimensions differ");
  Mat out(m, n);
  gemm(ta, tb, m, n, k, a.d.data(), a.r, b.d.data(), b.r, out.d.data(), m);
  return out;
}

// ---------------------------------------------------------------- tensor.cpp:60-139
void inner_outer(const std::vector<size_t>& dims, size_t mode, size_t& inner, size_t& outer) {
  inner = 1;
  for (size_t k = 0; k < mode; ++k) inner *= dims[k];
  outer = 1;
  for (size_t k = mode + 1; k < dims.size(); ++k) outer *= dims[k];
}

Mat unfold(const Tensor& t, size_t mode) {  // tensor.cpp:60-86
  size_t rows = t.dims[mode], inner, outer;
  inner_outer(t.dims, mode, inner, outer);
  Mat m(rows, inner * outer);
  if (mode == 0) {
    std::memcpy(m.d.data(), t.v.data(), sizeof(double) * t.size());
    return m;
  }
  const double* src = t.v.data();
  double* dst = m.d.data();
  for (size_t o = 0; o < outer; ++o)
    for (size_t r = 0; r < rows; ++r) {
      const double* s = src + (o * rows + r) * inner;
      double* d = dst + r + o * inner * rows;
      for (size_t i = 0; i < inner; ++i) d[i * rows] = s[i];
    }
  return m;
}

Tensor fold(const Mat& m, size_t mode, const std::vector<size_t>& dims) {  // tensor.cpp:88-116
  size_t rows = dims[mode], inner, outer;
  inner_outer(dims, mode, inner, outer);
  if (m.r != rows || m.c != inner * outer)
    throw std::invalid_argument("fold: matrix shape does not match target dims");
  Tensor t(dims);
  if (mode == 0) {
    std::memcpy(t.v.data(), m.d.data(), sizeof(double) * t.size());
    return t;
  }
  const double* src = m.d.data();
  double* dst = t.v.data();
  for (size_t o = 0; o < outer; ++o)
    for (size_t r = 0; r < rows; ++r) {
      const double* s = src + r + o * inner * rows;
      double* d = dst + (o * rows + r) * inner;
      for (size_t i = 0; i < inner; ++i) d[i] = s[i * rows];
    }
  return t;
}

Tensor mode_n_product(const Tensor& t, const Mat& b, size_t mode) {  // tensor.cpp:118-139
  if (mode >= t.dims.size()) throw std::out_of_range("mode_n_product: mode out of range");
  if (b.c != t.dims[mode])
    throw std::invalid_argument(
        "mode_n_product: matrix columns must match tensor mode dimension");
  std::vector<size_t> od = t.dims;
  od[mode] = b.r;
  if (mode == 0) {
    size_t cols = t.size() / t.dims[0];
    Tensor out(od);
    gemm(false, false, b.r, cols, t.dims[0], b.d.data(), b.r, t.v.data(), t.dims[0],
         out.v.data(), b.r);
    return out;
  }
  Mat m = unfold(t, mode);
  Mat r = matmul(b, false, m, false);
  return fold(r, mode, od);
}

Mat transpose(const Mat& a) {
  Mat t(a.c, a.r);
  for (size_t j = 0; j < a.c; ++j)
    for (size_t i = 0; i < a.r; ++i) t(j, i) = a(i, j);
  return t;
}

// ---------------------------------------------------------------- linalg.cpp:12-99
void fix_signs(Mat& u, Mat& v) {  // linalg.cpp:13-29
  for (size_t k = 0; k < u.c; ++k) {
    size_t imax = 0;
    double best = 0.0;
    for (size_t i = 0; i < u.r; ++i) {
      double a = std::abs(u(i, k));
      if (a > best) {
        best = a;
        imax = i;
      }
    }
    if (u(imax, k) < 0.0) {
      for (size_t i = 0; i < u.r; ++i) u(i, k) = -u(i, k);
      if (k < v.c)
        for (size_t i = 0; i < v.r; ++i) v(i, k) = -v(i, k);
    }
  }
}

struct Svd {
  Mat U;
  std::vector<double> S;
  Mat V;
};

Svd thin_svd(const Mat& m) {  // linalg.cpp:33-43 (BDCSVD -> LAPACK dgesdd)
  need_blas();
  i64 M = (i64)m.r, N = (i64)m.c, mn = std::min(M, N);
  Svd out;
  out.U = Mat(m.r, (size_t)mn);
  out.S.assign((size_t)mn, 0.0);
  Mat vt((size_t)mn, m.c);
  if (mn == 0) return out;
  std::vector<double> a = m.d;
  std::vector<i64> iwork(8 * (size_t)mn);
  i64 lwork = -1, info = 0;
  double wq = 0;
  i64 ldu = std::max<i64>(M, 1), ldvt = std::max<i64>(mn, 1), lda = std::max<i64>(M, 1);
  g_blas.dgesdd("S", &M, &N, a.data(), &lda, out.S.data(), out.U.d.data(), &ldu, vt.d.data(),
                &ldvt, &wq, &lwork, iwork.data(), &info, 1);
  lwork = (i64)wq + 1;
  std::vector<double> work((size_t)lwork);
  g_blas.dgesdd("S", &M, &N, a.data(), &lda, out.S.data(), out.U.d.data(), &ldu, vt.d.data(),
                &ldvt, work.data(), &lwork, iwork.data(), &info, 1);
  if (info != 0) throw std::runtime_error("thin_svd: SVD iteration did not converge");
  out.V = transpose(vt);
  fix_signs(out.U, out.V);
  return out;
}

Mat thin_qr_q(const Mat& m) {  // linalg.cpp:52-60 (HouseholderQR -> dgeqrf/dorgqr)
  need_blas();
  if (m.r < m.c) throw std::invalid_argument("thin_qr: requires rows >= cols");
  i64 M = (i64)m.r, N = (i64)m.c, lda = std::max<i64>(M, 1), info = 0, lwork = -1;
  Mat q = m;
  std::vector<double> tau((size_t)std::max<i64>(N, 1));
  double wq = 0;
  g_blas.dgeqrf(&M, &N, q.d.data(), &lda, tau.data(), &wq, &lwork, &info);
  lwork = (i64)wq + 1;
  std::vector<double> work((size_t)lwork);
  g_blas.dgeqrf(&M, &N, q.d.data(), &lda, tau.data(), work.data(), &lwork, &info);
  lwork = -1;
  g_blas.dorgqr(&M, &N, &N, q.d.data(), &lda, tau.data(), &wq, &lwork, &info);
  lwork = (i64)wq + 1;
  work.assign((size_t)lwork, 0.0);
  g_blas.dorgqr(&M, &N, &N, q.d.data(), &lda, tau.data(), work.data(), &lwork, &info);
  if (info != 0) throw std::runtime_error("thin_qr: LAPACK failure");
  return q;
}

Mat gram_power_apply(const Mat& a, const Mat& g, int q, int strategy) {  // linalg.cpp:62-80
  if (g.r != a.r) throw std::invalid_argument("gram_power_apply: G must have as many rows as A");
  if (q < 1) throw std::invalid_argument("gram_power_apply: q must be >= 1");
  Mat c = g;
  if (strategy == 0) {
    for (int k = 0; k < q; ++k) {
      Mat half = matmul(a, true, c, false);
      c = matmul(a, false, half, false);
    }
  } else {
    Mat gram = matmul(a, false, a, true);
    for (int k = 0; k < q; ++k) c = matmul(gram, false, c, false);
  }
  return c;
}

Mat leading_left_singular_vectors(const Mat& c, size_t mu) {  // linalg.cpp:82-87
  size_t maxrank = std::min(c.r, c.c);
  if (mu < 1 || mu > maxrank)
    throw std::invalid_argument("leading_left_singular_vectors: mu out of range");
  Svd s = thin_svd(c);
  Mat u(c.r, mu);
  std::memcpy(u.d.data(), s.U.d.data(), sizeof(double) * c.r * mu);
  return u;
}

Mat qr_project_extract(const Mat& c, const Mat& a_unfold, size_t mu) {  // linalg.cpp:89-99
  if (c.r != a_unfold.r) throw std::invalid_argument("qr_project_extract: row counts differ");
  if (mu < 1 || mu > c.c) throw std::invalid_argument("qr_project_extract: mu out of range");
  Mat q = thin_qr_q(c);
  Mat projected = matmul(q, true, a_unfold, false);
  Mat u1 = leading_left_singular_vectors(projected, mu);
  return matmul(q, false, u1, false);
}

// ---------------------------------------------------------------- sketching.cpp
double stable_sum(const double* v, size_t n) {  // sketching.cpp:13-24
  double s = 0.0, c = 0.0;
  for (size_t i = 0; i < n; ++i) {
    double x = v[i];
    double t = s + x;
    if (std::abs(s) >= std::abs(x))
      c += (s - t) + x;
    else
      c += (x - t) + s;
    s = t;
  }
  return s + c;
}

void check_distribution(const std::vector<double>& w) {  // sketching.cpp:28-38
  if (w.empty()) throw std::invalid_argument("probability distribution must be nonempty");
  for (double x : w)
    if (!(x >= 0.0)) throw std::invalid_argument("probability weights must be nonnegative");
  double s = stable_sum(w.data(), w.size());
  if (std::abs(s - 1.0) > 1e-12) throw std::invalid_argument("probability weights must sum to one");
}

std::vector<double> normalized(std::vector<double> raw) {  // sketching.cpp:40-48
  for (double w : raw)
    if (!(w >= 0.0)) throw std::invalid_argument("probability weights must be nonnegative");
  double s = stable_sum(raw.data(), raw.size());
  if (s <= 0.0) throw std::invalid_argument("cannot normalize an all-zero distribution");
  for (double& w : raw) w /= s;
  check_distribution(raw);
  return raw;
}

std::vector<double> uniform(size_t n) {  // sketching.cpp:50-53
  if (n == 0) throw std::invalid_argument("probability distribution must be nonempty");
  std::vector<double> w(n, 1.0 / static_cast<double>(n));
  check_distribution(w);
  return w;
}

struct Samples {
  std::vector<int64_t> idx;
  std::vector<double> scales;
};

Samples randsample(size_t L, const std::vector<double>& p, uint64_t seed, uint64_t stream) {
  // sketching.cpp:96-131
  if (L < 1) throw std::invalid_argument("randsample: L must be positive");
  std::vector<double> cum(p.size());
  double acc = 0.0;
  for (size_t i = 0; i < p.size(); ++i) {
    acc += p[i];
    cum[i] = acc;
  }
  if (!(acc > 0.0)) throw std::invalid_argument("randsample: all-zero distribution");
  size_t last = p.size();
  while (last > 0 && p[last - 1] == 0.0) --last;
  --last;
  Samples s;
  s.idx.resize(L);
  s.scales.resize(L);
  Rng gen(seed, stream);
  const double scale_base = 1.0 / std::sqrt(static_cast<double>(L));
  for (size_t j = 0; j < L; ++j) {
    double u = gen.next_double() * acc;
    auto it = std::upper_bound(cum.begin(), cum.end(), u);
    size_t idx = (it == cum.end()) ? last : static_cast<size_t>(it - cum.begin());
    if (p[idx] == 0.0) idx = last;
    s.idx[j] = static_cast<int64_t>(idx);
    s.scales[j] = scale_base / std::sqrt(p[idx]);
  }
  return s;
}

Mat sample_columns(const Mat& a, const Samples& s) {  // sketching.cpp:133-141
  Mat c(a.r, s.idx.size());
  for (size_t j = 0; j < s.idx.size(); ++j) {
    const double* src = a.d.data() + a.r * (size_t)s.idx[j];
    double* dst = c.d.data() + a.r * j;
    for (size_t i = 0; i < a.r; ++i) dst[i] = src[i] * s.scales[j];
  }
  return c;
}

Mat gaussian_matrix(size_t rows, size_t cols, uint64_t seed, uint64_t stream) {
  // sketching.cpp:164-173
  if (rows < 1 || cols < 1) throw std::invalid_argument("gaussian_matrix: shape must be positive");
  Mat g(rows, cols);
  fill_normals(seed, stream, g.d.data(), rows * cols, default_threads());
  return g;
}

// Canonical squared norm of a fiber (shared with the GPU kernels): chunks of 32 consecutive
// entries accumulated with fma from +0; pairs of chunks (segments of 64 entries) summed; the
// segment sums added in order.  (Two levels so that a fibre split across devices at multiples
// of 64 entries combines per-device segment sums into the same bits; fibres of <= 64 entries
// give the plain in-order chunk sum.)
double canonical_sqnorm(const double* x, size_t len, size_t stride) {
  double total = 0.0, seg = 0.0;
  size_t c = 0;
  for (size_t c0 = 0; c0 < len; c0 += 32, ++c) {
    double p = 0.0;
    size_t c1 = std::min(len, c0 + 32);
    for (size_t r = c0; r < c1; ++r) {
      double v = x[r * stride];
      p = std::fma(v, v, p);
    }
    seg = (c & 1) ? seg + p : p;
    if ((c & 1) || c1 == len) total = total + seg;
  }
  return total;
}

std::vector<double> probabilities_from_norms(std::vector<double> w, int regime, double beta) {
  // tucker.cpp:110-130 (after the squaredNorm loop)
  const size_t n = w.size();
  if (regime == ORC_UNIFORM) return uniform(n);
  double total = 0.0;
  for (size_t i = 0; i < n; ++i) total += w[i];
  if (total <= 0.0) return uniform(n);
  for (auto& x : w) x /= total;
  if (regime == ORC_OPTIMAL) return normalized(std::move(w));
  if (!(beta > 0.0 && beta <= 1.0))
    throw std::invalid_argument("nearly-optimal mixture weight must lie in (0, 1]");
  for (auto& x : w) x = beta * x + (1.0 - beta) / static_cast<double>(n);
  return normalized(std::move(w));
}

std::vector<double> gram_sampling_norms(const Mat& a) {  // tucker.cpp:117-120 (norm half)
  std::vector<double> w(a.c);
  for (size_t j = 0; j < a.c; ++j) w[j] = canonical_sqnorm(a.d.data() + a.r * j, a.r, 1);
  return w;
}

// ---------------------------------------------------------------- tucker.cpp
struct Config {
  std::vector<size_t> mu;
  size_t oversampling = 10;
  int power = 1;
  double alpha = 0.2;
  int regime = ORC_UNIFORM;
  double beta = 0.5;
  std::vector<size_t> t_samples;
  std::vector<size_t> order;
  uint64_t seed = 0;
  int strategy = 0;
  int mode_threads = 1;
  bool keep_trace = false;
  int hooi_max_sweeps = 50;
  double hooi_tol = 1e-8;
};

Config to_config(const orc_config* c, int order) {
  Config k;
  k.mu.assign(c->rank, c->rank + order);
  k.oversampling = c->oversampling;
  k.power = c->power;
  k.alpha = c->alpha;
  k.regime = c->regime;
  k.beta = c->regime_beta;
  if (c->t_samples) k.t_samples.assign(c->t_samples, c->t_samples + order);
  if (c->order) k.order.assign(c->order, c->order + order);
  k.seed = c->seed;
  k.strategy = c->strategy;
  k.mode_threads = std::max(1, c->mode_threads);
  k.keep_trace = c->keep_trace != 0;
  k.hooi_max_sweeps = c->hooi_max_sweeps;
  k.hooi_tol = c->hooi_tol;
  return k;
}

std::vector<size_t> clamped_for(const std::vector<size_t>& mu, const std::vector<size_t>& dims) {
  // tucker.cpp:174-188
  if (mu.size() != dims.size())
    throw std::invalid_argument("rank vector length must equal tensor order");
  std::vector<size_t> out(mu.size());
  for (size_t n = 0; n < mu.size(); ++n) {
    if (mu[n] < 1) throw std::invalid_argument("rank entries must be positive");
    out[n] = std::min(mu[n], dims[n]);
  }
  return out;
}

struct Resolved {
  std::vector<size_t> mu, sketch, order;
};

Resolved resolve(const Tensor& a, const Config& cfg) {  // tucker.cpp:24-52
  const size_t nm = a.dims.size();
  if (nm == 0) throw std::invalid_argument("cannot decompose an order-0 tensor");
  if (cfg.mu.size() != nm) throw std::invalid_argument("rank vector length must equal tensor order");
  if (cfg.power < 1) throw std::invalid_argument("power exponent must be >= 1");
  Resolved r;
  r.mu = clamped_for(cfg.mu, a.dims);
  r.sketch.resize(nm);
  for (size_t n = 0; n < nm; ++n) r.sketch[n] = std::min(r.mu[n] + cfg.oversampling, a.dims[n]);
  if (cfg.order.empty()) {
    r.order.resize(nm);
    std::iota(r.order.begin(), r.order.end(), size_t{0});
  } else {
    if (cfg.order.size() != nm)
      throw std::invalid_argument("processing order length must equal tensor order");
    std::vector<bool> seen(nm, false);
    for (size_t m : cfg.order) {
      if (m >= nm || seen[m])
        throw std::invalid_argument("processing order must be a permutation of the modes");
      seen[m] = true;
    }
    r.order = cfg.order;
  }
  return r;
}

Mat top_left_vectors_clamped(const Mat& m, size_t mu) {  // tucker.cpp:65-77
  return leading_left_singular_vectors(m, std::min(mu, std::min(m.r, m.c)));
}

Tensor core_from_factors(const Tensor& a, const std::vector<Mat>& f) {  // tucker.cpp:81-92
  std::vector<size_t> idx(f.size());
  std::iota(idx.begin(), idx.end(), size_t{0});
  std::stable_sort(idx.begin(), idx.end(), [&](size_t i, size_t j) { return f[i].c < f[j].c; });
  Tensor t = a;
  for (size_t n : idx) t = mode_n_product(t, transpose(f[n]), n);
  return t;
}

size_t other_dims_product(const std::vector<size_t>& dims, size_t mode) {
  size_t p = 1;
  for (size_t k = 0; k < dims.size(); ++k)
    if (k != mode) p *= dims[k];
  return p;
}

size_t samples_from_alpha(double alpha, size_t cols) {  // tucker.cpp:101-106
  if (!(alpha > 0.0 && alpha < 1.0))
    throw std::invalid_argument("sampling fraction alpha must lie in (0, 1)");
  auto t = static_cast<size_t>(std::ceil(alpha * static_cast<double>(cols)));
  return std::max<size_t>(t, 1);
}

std::vector<size_t> amm_sample_counts(const std::vector<size_t>& dims, const Config& cfg,
                                      bool sequential) {  // tucker.cpp:348-376
  const size_t nm = dims.size();
  if (!cfg.t_samples.empty()) {
    if (cfg.t_samples.size() != nm)
      throw std::invalid_argument("sample count override length must equal tensor order");
    for (size_t t : cfg.t_samples)
      if (t < 1) throw std::invalid_argument("sample counts must be positive");
    return cfg.t_samples;
  }
  std::vector<size_t> counts(nm);
  if (!sequential) {
    for (size_t n = 0; n < nm; ++n) counts[n] = samples_from_alpha(cfg.alpha, other_dims_product(dims, n));
    return counts;
  }
  std::vector<size_t> cur = dims;
  std::vector<size_t> mu = clamped_for(cfg.mu, dims);
  std::vector<size_t> order = cfg.order;
  if (order.empty()) {
    order.resize(nm);
    std::iota(order.begin(), order.end(), size_t{0});
  }
  for (size_t n : order) {
    counts[n] = samples_from_alpha(cfg.alpha, other_dims_product(cur, n));
    cur[n] = mu[n];
  }
  return counts;
}

void run_modes(size_t nm, int cap, const std::function<void(size_t)>& body) {  // tucker.cpp:134-160
  if (cap <= 1 || nm <= 1) {
    for (size_t n = 0; n < nm; ++n) body(n);
    return;
  }
  std::atomic<size_t> next{0};
  std::vector<std::exception_ptr> errors(nm);
  auto worker = [&] {
    for (;;) {
      size_t n = next.fetch_add(1);
      if (n >= nm) return;
      try {
        body(n);
      } catch (...) {
        errors[n] = std::current_exception();
      }
    }
  };
  size_t workers = std::min<size_t>((size_t)cap, nm);
  std::vector<std::thread> pool;
  for (size_t i = 0; i + 1 < workers; ++i) pool.emplace_back(worker);
  worker();
  for (auto& t : pool) t.join();
  for (auto& e : errors)
    if (e) std::rethrow_exception(e);
}

struct Trace {
  Mat omega;
  Mat sketch;  // C = (A A^T)^q G, the matrix whose top left singular vectors are the factor
  Samples samples;
  std::vector<double> norms;
};

}  // namespace

struct orc_result {
  Tensor core;
  std::vector<Mat> factors;
  std::vector<Trace> trace;
  double seconds = 0.0;
};

namespace {

// tucker.cpp:110-130 on an unfolding, with the trace hook
std::vector<double> mode_probabilities(const Mat& a_n, const Config& cfg, Trace* tr) {
  if (cfg.regime == ORC_UNIFORM) return uniform(a_n.c);
  std::vector<double> w = gram_sampling_norms(a_n);
  if (tr && cfg.keep_trace) tr->norms = w;
  return probabilities_from_norms(std::move(w), cfg.regime, cfg.beta);
}

// ---------------------------------------------------------------- deterministic baselines
double frobenius_norm(const Tensor& t) {  // tensor.cpp (sequential sum of squares)
  double s = 0.0;
  for (double v : t.v) s += v * v;
  return std::sqrt(s);
}

void alg_thosvd(const Tensor& a, const Config& cfg, orc_result& res) {  // tucker.cpp:242-248
  Resolved r = resolve(a, cfg);
  const size_t nm = a.dims.size();
  res.factors.assign(nm, Mat());
  res.trace.assign(nm, Trace());
  for (size_t n = 0; n < nm; ++n) {
    Mat a_n = unfold(a, n);
    res.factors[n] = top_left_vectors_clamped(a_n, r.mu[n]);
    if (cfg.keep_trace) res.trace[n].sketch = std::move(a_n);
  }
  res.core = core_from_factors(a, res.factors);
}

void alg_sthosvd(const Tensor& a, const Config& cfg, orc_result& res) {  // tucker.cpp:250-259
  Resolved r = resolve(a, cfg);
  const size_t nm = a.dims.size();
  res.factors.assign(nm, Mat());
  res.trace.assign(nm, Trace());
  Tensor work = a;
  for (size_t n : r.order) {
    Mat a_n = unfold(work, n);
    res.factors[n] = top_left_vectors_clamped(a_n, r.mu[n]);
    if (cfg.keep_trace) res.trace[n].sketch = std::move(a_n);
    work = mode_n_product(work, transpose(res.factors[n]), n);
  }
  res.core = std::move(work);
}

void alg_hooi(const Tensor& a, const Config& cfg, orc_result& res) {  // tucker.cpp:261-316
  Resolved r = resolve(a, cfg);
  const size_t nm = a.dims.size();
  alg_sthosvd(a, cfg, res);  // init = st_hosvd (tucker.cpp:314-316)
  std::vector<Mat>& factors = res.factors;
  Tensor core = core_from_factors(a, factors);
  const double norm_a = frobenius_norm(a);
  if (norm_a == 0.0) {
    res.core = std::move(core);
    return;
  }
  double prev = frobenius_norm(core);
  bool converged = false;
  int sweep = 0;
  const size_t last = r.order.back();
  while (sweep < cfg.hooi_max_sweeps) {
    ++sweep;
    for (size_t n : r.order) {
      Tensor y = a;
      for (size_t m = 0; m < nm; ++m)
        if (m != n) y = mode_n_product(y, transpose(factors[m]), m);
      Mat y_n = unfold(y, n);
      factors[n] = top_left_vectors_clamped(y_n, r.mu[n]);
      if (cfg.keep_trace) res.trace[n].sketch = std::move(y_n);
      if (n == last) core = mode_n_product(y, transpose(factors[n]), n);
    }
    const double cur = frobenius_norm(core);
    if (std::abs(cur - prev) / norm_a < cfg.hooi_tol) {
      converged = true;
      break;
    }
    prev = cur;
  }
  if (!converged)
    std::fprintf(stderr, "lmra: hooi stopped after %d sweeps without meeting the tolerance\n", sweep);
  res.core = std::move(core);
}

void alg_power(const Tensor& a, const Config& cfg, bool sequential, orc_result& res) {
  // tucker.cpp:318-346
  Resolved r = resolve(a, cfg);
  const size_t nm = a.dims.size();
  res.factors.assign(nm, Mat());
  res.trace.assign(nm, Trace());
  if (!sequential) {
    run_modes(nm, cfg.mode_threads, [&](size_t n) {
      Mat a_n = unfold(a, n);
      Mat g = gaussian_matrix(a.dims[n], r.sketch[n], cfg.seed, n + 1);
      Mat c = gram_power_apply(a_n, g, cfg.power, cfg.strategy);
      res.factors[n] = top_left_vectors_clamped(c, r.mu[n]);
      if (cfg.keep_trace) res.trace[n].sketch = c;
      if (cfg.keep_trace) res.trace[n].omega = std::move(g);
    });
    res.core = core_from_factors(a, res.factors);
    return;
  }
  Tensor work = a;
  for (size_t n : r.order) {
    Mat a_n = unfold(work, n);
    Mat g = gaussian_matrix(work.dims[n], r.sketch[n], cfg.seed, n + 1);
    Mat c = gram_power_apply(a_n, g, cfg.power, cfg.strategy);
    res.factors[n] = top_left_vectors_clamped(c, r.mu[n]);
    if (cfg.keep_trace) res.trace[n].sketch = c;
    if (cfg.keep_trace) res.trace[n].omega = std::move(g);
    work = mode_n_product(work, transpose(res.factors[n]), n);
  }
  res.core = std::move(work);
}

// tucker.cpp:422-454: the QR-proxy variants (alg6 / alg7).  mu is capped at the numerical
// rank limit min(sketch width, unfolding columns) (rank_cap, tucker.cpp:65-71).
void alg_power_qr(const Tensor& a, const Config& cfg, bool sequential, orc_result& res) {
  Resolved r = resolve(a, cfg);
  const size_t nm = a.dims.size();
  res.factors.assign(nm, Mat());
  res.trace.assign(nm, Trace());
  auto one = [&](const Tensor& t, size_t n) {
    Mat a_n = unfold(t, n);
    Mat g = gaussian_matrix(t.dims[n], r.sketch[n], cfg.seed, n + 1);
    Mat c = gram_power_apply(a_n, g, cfg.power, cfg.strategy);
    const size_t mu = std::min(r.mu[n], std::min(r.sketch[n], a_n.c));
    res.factors[n] = qr_project_extract(c, a_n, mu);
    if (cfg.keep_trace) {
      res.trace[n].sketch = c;
      res.trace[n].omega = std::move(g);
    }
  };
  if (!sequential) {
    run_modes(nm, cfg.mode_threads, [&](size_t n) { one(a, n); });
    res.core = core_from_factors(a, res.factors);
    return;
  }
  Tensor work = a;
  for (size_t n : r.order) {
    one(work, n);
    work = mode_n_product(work, transpose(res.factors[n]), n);
  }
  res.core = std::move(work);
}

void alg_amm(const Tensor& a, const Config& cfg, bool sequential, orc_result& res) {
  // tucker.cpp:378-420
  Resolved r = resolve(a, cfg);
  const size_t nm = a.dims.size();
  res.factors.assign(nm, Mat());
  res.trace.assign(nm, Trace());
  if (!sequential) {
    std::vector<size_t> t_n = amm_sample_counts(a.dims, cfg, false);
    run_modes(nm, cfg.mode_threads, [&](size_t n) {
      Mat a_n = unfold(a, n);
      std::vector<double> p = mode_probabilities(a_n, cfg, &res.trace[n]);
      Samples s = randsample(t_n[n], p, cfg.seed, nm + n + 1);
      Mat sampled = sample_columns(a_n, s);
      Mat g = gaussian_matrix(a.dims[n], r.sketch[n], cfg.seed, n + 1);
      Mat c = gram_power_apply(sampled, g, cfg.power, cfg.strategy);
      res.factors[n] = top_left_vectors_clamped(c, r.mu[n]);
      if (cfg.keep_trace) res.trace[n].sketch = c;
      if (cfg.keep_trace) {
        res.trace[n].omega = std::move(g);
        res.trace[n].samples = std::move(s);
      }
    });
    res.core = core_from_factors(a, res.factors);
    return;
  }
  if (!cfg.t_samples.empty() && cfg.t_samples.size() != nm)
    throw std::invalid_argument("sample count override length must equal tensor order");
  Tensor work = a;
  for (size_t n : r.order) {
    Mat a_n = unfold(work, n);
    size_t t_n = cfg.t_samples.empty() ? samples_from_alpha(cfg.alpha, a_n.c) : cfg.t_samples[n];
    if (t_n < 1) throw std::invalid_argument("sample counts must be positive");
    std::vector<double> p = mode_probabilities(a_n, cfg, &res.trace[n]);
    Samples s = randsample(t_n, p, cfg.seed, nm + n + 1);
    Mat sampled = sample_columns(a_n, s);
    Mat g = gaussian_matrix(work.dims[n], r.sketch[n], cfg.seed, n + 1);
    Mat c = gram_power_apply(sampled, g, cfg.power, cfg.strategy);
    res.factors[n] = top_left_vectors_clamped(c, r.mu[n]);
    if (cfg.keep_trace) res.trace[n].sketch = c;
    if (cfg.keep_trace) {
      res.trace[n].omega = std::move(g);
      res.trace[n].samples = std::move(s);
    }
    work = mode_n_product(work, transpose(res.factors[n]), n);
  }
  res.core = std::move(work);
}

Tensor make_tensor(const double* x, const uint64_t* dims, int order) {
  std::vector<size_t> d(dims, dims + order);
  for (size_t v : d)
    if (v == 0) throw std::invalid_argument("tensor dimension must be positive");
  Tensor t(d);
  std::memcpy(t.v.data(), x, sizeof(double) * t.size());
  return t;
}

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = std::string("invalid_argument: ") + e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = std::string("runtime_error: ") + e.what();
    return 2;
  }
}

}  // namespace

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }

int orc_init_blas(const char* path) {
  return guard([&] {
    void* h = dlopen(path, RTLD_NOW | RTLD_LOCAL);
    if (!h) throw std::runtime_error(std::string("dlopen failed: ") + dlerror());
    g_blas.dgemm = (dgemm_t)dlsym(h, "scipy_dgemm_64_");
    g_blas.dgesdd = (dgesdd_t)dlsym(h, "scipy_dgesdd_64_");
    g_blas.dgeqrf = (dgeqrf_t)dlsym(h, "scipy_dgeqrf_64_");
    g_blas.dorgqr = (dorgqr_t)dlsym(h, "scipy_dorgqr_64_");
    g_blas.set_threads = (setthreads_t)dlsym(h, "scipy_openblas_set_num_threads64_");
    if (!g_blas.dgemm || !g_blas.dgesdd || !g_blas.dgeqrf || !g_blas.dorgqr)
      throw std::runtime_error("BLAS/LAPACK symbols missing");
  });
}

void orc_set_blas_threads(int n) {
  if (g_blas.set_threads) g_blas.set_threads(n);
}

void orc_rng_u32(uint64_t seed, uint64_t stream, uint64_t skip, uint32_t* out, size_t n) {
  Rng g(seed, stream);
  g.advance(skip);
  for (size_t i = 0; i < n; ++i) out[i] = g.next_u32();
}

void orc_rng_double(uint64_t seed, uint64_t stream, double* out, size_t n) {
  Rng g(seed, stream);
  for (size_t i = 0; i < n; ++i) out[i] = g.next_double();
}

void orc_rng_normal(uint64_t seed, uint64_t stream, double* out, size_t n) {
  Rng g(seed, stream);  // strictly sequential, the reference's own loop
  for (size_t i = 0; i < n; ++i) out[i] = g.next_normal();
}

int orc_gaussian_matrix(uint64_t rows, uint64_t cols, uint64_t seed, uint64_t stream, double* out) {
  return guard([&] {
    Mat g = gaussian_matrix(rows, cols, seed, stream);
    std::memcpy(out, g.d.data(), sizeof(double) * rows * cols);
  });
}

double orc_stable_sum(const double* v, size_t n) { return stable_sum(v, n); }

int orc_column_sqnorms(const double* x, const uint64_t* dims, int order, int mode, double* w) {
  return guard([&] {
    std::vector<size_t> d(dims, dims + order);
    size_t inner, outer;
    inner_outer(d, (size_t)mode, inner, outer);
    size_t L = d[mode];
    for (size_t o = 0; o < outer; ++o)
      for (size_t i = 0; i < inner; ++i)
        w[i + inner * o] = canonical_sqnorm(x + i + inner * L * o, L, inner);
  });
}

int orc_probabilities(const double* w, uint64_t n, int regime, double beta, double* p) {
  return guard([&] {
    std::vector<double> v(w, w + n);
    std::vector<double> out = probabilities_from_norms(std::move(v), regime, beta);
    std::memcpy(p, out.data(), sizeof(double) * n);
  });
}

int orc_randsample(uint64_t L, const double* p, uint64_t n, uint64_t seed, uint64_t stream,
                   int64_t* idx, double* scales) {
  return guard([&] {
    std::vector<double> pv(p, p + n);
    check_distribution(pv);
    Samples s = randsample(L, pv, seed, stream);
    std::memcpy(idx, s.idx.data(), sizeof(int64_t) * L);
    std::memcpy(scales, s.scales.data(), sizeof(double) * L);
  });
}

int orc_amm_sample_counts(const uint64_t* dims, int order, const orc_config* cfg, int sequential,
                          uint64_t* out) {
  return guard([&] {
    Config k = to_config(cfg, order);
    std::vector<size_t> d(dims, dims + order);
    std::vector<size_t> c = amm_sample_counts(d, k, sequential != 0);
    for (int n = 0; n < order; ++n) out[n] = c[n];
  });
}

int orc_mode_n_product(const double* x, const uint64_t* dims, int order, int mode,
                       const double* b, uint64_t b_rows, double* y) {
  return guard([&] {
    Tensor t = make_tensor(x, dims, order);
    Mat bm(b_rows, dims[mode]);
    std::memcpy(bm.d.data(), b, sizeof(double) * bm.d.size());
    Tensor o = mode_n_product(t, bm, (size_t)mode);
    std::memcpy(y, o.v.data(), sizeof(double) * o.size());
  });
}

int orc_gram_power_apply(const double* a, uint64_t rows, uint64_t cols, const double* g,
                         uint64_t s, int q, int strategy, double* c) {
  return guard([&] {
    Mat am(rows, cols), gm(rows, s);
    std::memcpy(am.d.data(), a, sizeof(double) * rows * cols);
    std::memcpy(gm.d.data(), g, sizeof(double) * rows * s);
    Mat out = gram_power_apply(am, gm, q, strategy);
    std::memcpy(c, out.d.data(), sizeof(double) * rows * s);
  });
}

int orc_leading_left_singular_vectors(const double* c, uint64_t rows, uint64_t cols, uint64_t mu,
                                      double* u) {
  return guard([&] {
    Mat cm(rows, cols);
    std::memcpy(cm.d.data(), c, sizeof(double) * rows * cols);
    Mat out = leading_left_singular_vectors(cm, mu);
    std::memcpy(u, out.d.data(), sizeof(double) * rows * mu);
  });
}

int orc_thin_qr_q(const double* m, uint64_t rows, uint64_t cols, double* q) {
  return guard([&] {
    Mat mm(rows, cols);
    std::memcpy(mm.d.data(), m, sizeof(double) * rows * cols);
    Mat out = thin_qr_q(mm);
    std::memcpy(q, out.d.data(), sizeof(double) * rows * cols);
  });
}

int orc_qr_project_extract(const double* c, uint64_t rows, uint64_t cols, const double* a,
                           uint64_t a_cols, uint64_t mu, double* out) {
  return guard([&] {
    Mat cm(rows, cols), am(rows, a_cols);
    std::memcpy(cm.d.data(), c, sizeof(double) * rows * cols);
    std::memcpy(am.d.data(), a, sizeof(double) * rows * a_cols);
    Mat f = qr_project_extract(cm, am, mu);
    std::memcpy(out, f.d.data(), sizeof(double) * rows * mu);
  });
}

int orc_run(int alg, const double* x, const uint64_t* dims, int order, const orc_config* cfg,
            orc_result** out) {
  *out = nullptr;
  return guard([&] {
    if (order < 1) throw std::invalid_argument("cannot decompose an order-0 tensor");
    Tensor a = make_tensor(x, dims, order);
    Config k = to_config(cfg, order);
    auto res = new orc_result();
    try {
      auto t0 = std::chrono::steady_clock::now();  // bench.cpp:247-249 timed span
      switch (alg) {
        case ORC_ALG1: alg_power(a, k, false, *res); break;
        case ORC_ALG2: alg_power(a, k, true, *res); break;
        case ORC_ALG4: alg_amm(a, k, false, *res); break;
        case ORC_ALG5: alg_amm(a, k, true, *res); break;
        case ORC_ALG6: alg_power_qr(a, k, false, *res); break;
        case ORC_ALG7: alg_power_qr(a, k, true, *res); break;
        case ORC_THOSVD: alg_thosvd(a, k, *res); break;
        case ORC_STHOSVD: alg_sthosvd(a, k, *res); break;
        case ORC_HOOI: alg_hooi(a, k, *res); break;
        default: throw std::invalid_argument("unknown algorithm");
      }
      auto t1 = std::chrono::steady_clock::now();
      res->seconds = std::chrono::duration<double>(t1 - t0).count();
    } catch (...) {
      delete res;
      throw;
    }
    *out = res;
  });
}

int orc_result_order(const orc_result* r) { return (int)r->factors.size(); }
void orc_result_core_dims(const orc_result* r, uint64_t* dims) {
  for (size_t n = 0; n < r->core.dims.size(); ++n) dims[n] = r->core.dims[n];
}
void orc_result_factor_dims(const orc_result* r, int n, uint64_t* rows, uint64_t* cols) {
  *rows = r->factors[n].r;
  *cols = r->factors[n].c;
}
void orc_result_core(const orc_result* r, double* out) {
  std::memcpy(out, r->core.v.data(), sizeof(double) * r->core.size());
}
void orc_result_factor(const orc_result* r, int n, double* out) {
  std::memcpy(out, r->factors[n].d.data(), sizeof(double) * r->factors[n].d.size());
}
double orc_result_seconds(const orc_result* r) { return r->seconds; }
void orc_result_omega_dims(const orc_result* r, int n, uint64_t* rows, uint64_t* cols) {
  *rows = r->trace[n].omega.r;
  *cols = r->trace[n].omega.c;
}
void orc_result_omega(const orc_result* r, int n, double* out) {
  std::memcpy(out, r->trace[n].omega.d.data(), sizeof(double) * r->trace[n].omega.d.size());
}
void orc_result_sketch_dims(const orc_result* r, int n, uint64_t* rows, uint64_t* cols) {
  *rows = r->trace[n].sketch.r;
  *cols = r->trace[n].sketch.c;
}
void orc_result_sketch(const orc_result* r, int n, double* out) {
  std::memcpy(out, r->trace[n].sketch.d.data(), sizeof(double) * r->trace[n].sketch.d.size());
}
uint64_t orc_result_num_samples(const orc_result* r, int n) { return r->trace[n].samples.idx.size(); }
void orc_result_samples(const orc_result* r, int n, int64_t* idx, double* scales) {
  const Samples& s = r->trace[n].samples;
  std::memcpy(idx, s.idx.data(), sizeof(int64_t) * s.idx.size());
  std::memcpy(scales, s.scales.data(), sizeof(double) * s.scales.size());
}
uint64_t orc_result_num_norms(const orc_result* r, int n) { return r->trace[n].norms.size(); }
void orc_result_norms(const orc_result* r, int n, double* w) {
  std::memcpy(w, r->trace[n].norms.data(), sizeof(double) * r->trace[n].norms.size());
}
void orc_result_free(orc_result* r) { delete r; }

double orc_relative_error(const double* x, const uint64_t* dims, int order, const orc_result* r) {
  // tucker.cpp:222-240: reconstruct (core x_n Q_n for n = 0..N-1), then the RE loop
  double re = -1.0;
  guard([&] {
    Tensor a = make_tensor(x, dims, order);
    Tensor t = r->core;
    for (size_t n = 0; n < r->factors.size(); ++n) t = mode_n_product(t, r->factors[n], n);
    double num = 0.0, den = 0.0;
    for (size_t i = 0; i < a.size(); ++i) {
      double d = a.v[i] - t.v[i];
      num += d * d;
      den += a.v[i] * a.v[i];
    }
    if (den == 0.0) throw std::invalid_argument("relative_error: zero reference tensor");
    re = std::sqrt(num / den);
  });
  return re;
}

}  // extern "C"

// ---------------------------------------------------------------- BASELINE generators
// The definitions live in paper_2303_11612_b200/csrc/gen/portable_gen.hpp (input synthesis,
// not the algorithm under test: explicit IEEE operations and fixed orders, so the host
// loops below give the device generators' exact bits).  Threads split independent outputs
// only; every sum keeps the definition's sequential order.
namespace {
template <class F>
void parallel_for(size_t n, F&& f) {  // f(begin, end) over [0, n)
  const int th = default_threads();
  if (th <= 1 || n < 2) {
    f(size_t{0}, n);
    return;
  }
  std::vector<std::thread> pool;
  const size_t chunk = (n + th - 1) / th;
  for (int t = 0; t < th; ++t) {
    const size_t b = std::min(n, t * chunk), e = std::min(n, b + chunk);
    if (b < e) pool.emplace_back([&f, b, e] { f(b, e); });
  }
  for (auto& t : pool) t.join();
}

// y[a, i, o] = sum_k U[i, k] x[a, k, o] (fma chain over k), i < I.  Blocked over a so the
// block's x(a, :, o) panel stays in cache while every i is formed from it.
void gen_ttm_host(const double* x, size_t inner, size_t K, size_t I, size_t outer, const double* u, size_t ldu,
                  double* y) {
  constexpr size_t kBlock = 512;
  const size_t nab = (inner + kBlock - 1) / kBlock;
  parallel_for(outer * nab, [&](size_t b, size_t e) {
    // the block's x(a, :, o) panel is copied to a contiguous buffer first: its K rows sit
    // inner * 8 bytes apart, which for a large inner maps them all onto the same cache sets
    std::vector<double> panel(K * kBlock), acc(kBlock);
    for (size_t r = b; r < e; ++r) {
      const size_t ab = r % nab, o = r / nab;
      const size_t a0 = ab * kBlock, a1 = std::min(inner, a0 + kBlock), na = a1 - a0;
      for (size_t k = 0; k < K; ++k)
        std::memcpy(panel.data() + k * kBlock, x + inner * (k + K * o) + a0, na * sizeof(double));
      for (size_t i = 0; i < I; ++i) {
        for (size_t a = 0; a < na; ++a) acc[a] = 0.0;
        for (size_t k = 0; k < K; ++k) {
          const double uk = u[i + ldu * k];
          const double* xk = panel.data() + k * kBlock;
          for (size_t a = 0; a < na; ++a) acc[a] = lmra_gen::gp_fma(uk, xk[a], acc[a]);
        }
        std::memcpy(y + inner * (i + I * o) + a0, acc.data(), na * sizeof(double));
      }
    }
  });
}
}  // namespace

extern "C" {

int orc_gen_tucker_noise(const uint64_t* dims, const uint64_t* core_dims, int order, double gamma,
                         uint64_t seed, double* out) {
  return guard([&] {
    using namespace lmra_gen;
    if (order < 1 || order > 8) throw std::invalid_argument("generator: order must be 1..8");
    std::vector<size_t> cd(core_dims, core_dims + order), d(dims, dims + order);
    for (int n = 0; n < order; ++n)
      if (cd[n] < 1 || cd[n] > d[n]) throw std::invalid_argument("core dimensions must lie in [1, I_n]");
    size_t ncore = 1, total = 1;
    for (int n = 0; n < order; ++n) {
      ncore *= cd[n];
      total *= d[n];
    }
    auto tp = std::chrono::steady_clock::now();
    auto lap = [&](const char* what) {
      if (!getenv("ORC_GEN_TIMING")) return;
      auto t = std::chrono::steady_clock::now();
      fprintf(stderr, "gen %s %.3f s\n", what, std::chrono::duration<double>(t - tp).count());
      tp = t;
    };
    std::vector<double> cur(ncore);
    gp_normals_range(seed, kStreamCore, cur.data(), 0, ncore);
    std::vector<size_t> cdim = cd;
    for (int n = 0; n < order; ++n) {
      std::vector<double> u(d[n] * cd[n]);
      gp_orthonormal_factor(d[n], cd[n], seed, (uint64_t)n, u.data());
      size_t inner = 1, outer = 1;
      for (int k = 0; k < n; ++k) inner *= cdim[k];
      for (int k = n + 1; k < order; ++k) outer *= cdim[k];
      const bool last = n == order - 1;
      std::vector<double> y;
      double* dst = out;
      if (!last) {
        y.resize(inner * d[n] * outer);
        dst = y.data();
      }
      gen_ttm_host(cur.data(), inner, cd[n], d[n], outer, u.data(), d[n], dst);
      cdim[n] = d[n];
      if (!last) cur.swap(y);
      lap("ttm");
    }
    // per-slice (last mode) sums of squares of B and of E: fibres of d0 (fma chain), slice =
    // sequential sum of its fibres, total = sequential sum over slices
    const size_t d0 = d[0], L = order == 1 ? 1 : d[order - 1];
    const size_t nfib = total / d0, per = nfib / L;
    std::vector<double> fb(nfib), fe(nfib);
    parallel_for(nfib, [&](size_t b, size_t e) {
      std::vector<double> z(d0 + 1);
      for (size_t f = b; f < e; ++f) {
        const double* p = out + f * d0;
        double acc = 0.0;
        for (size_t i = 0; i < d0; ++i) acc = gp_fma(p[i], p[i], acc);
        fb[f] = acc;
        gp_normals_range(seed, kStreamNoise, z.data(), f * d0, (f + 1) * d0);
        acc = 0.0;
        for (size_t i = 0; i < d0; ++i) acc = gp_fma(z[i], z[i], acc);
        fe[f] = acc;
      }
    });
    lap("fibre sums");
    std::vector<double> sb(L), se(L);
    for (size_t l = 0; l < L; ++l) {
      double ab = 0.0, ae = 0.0;
      for (size_t j = 0; j < per; ++j) {
        ab = gp_add(ab, fb[l * per + j]);
        ae = gp_add(ae, fe[l * per + j]);
      }
      sb[l] = ab;
      se[l] = ae;
    }
    const double coef = gp_noise_coef(sb.data(), se.data(), L, gamma);
    parallel_for((total + 63) / 64, [&](size_t b, size_t e) {
      double z[64];
      for (size_t r = b; r < e; ++r) {
        const size_t e0 = r * 64, e1 = std::min(total, e0 + 64);
        gp_normals_range(seed, kStreamNoise, z, e0, e1);
        for (size_t i = e0; i < e1; ++i) out[i] = gp_add(out[i], gp_mul(coef, z[i - e0]));
      }
    });
    lap("noise");
  });
}

int orc_gen_hilbert(const uint64_t* dims, int order, double* out) {
  return guard([&] {
    size_t total = 1;
    for (int n = 0; n < order; ++n) total *= dims[n];
    std::vector<size_t> idx(order, 0);
    for (size_t e = 0; e < total; ++e) {
      size_t s = 0;
      for (int n = 0; n < order; ++n) s += idx[n];
      out[e] = 1.0 / static_cast<double>(s + 1);
      for (int n = 0; n < order; ++n) {
        if (++idx[n] < dims[n]) break;
        idx[n] = 0;
      }
    }
  });
}

int orc_gen_video(const uint64_t* dims, int order, uint64_t n_terms, double noise, uint64_t seed,
                  double* out) {
  return guard([&] {
    using namespace lmra_gen;
    if (order < 1 || order > 8) throw std::invalid_argument("generator: order must be 1..8");
    if (n_terms < 1) throw std::invalid_argument("video generator: n_terms must be positive");
    std::vector<long long> d(dims, dims + order);
    size_t total = 1, tot = 0;
    for (long long v : d) {
      total *= (size_t)v;
      tot += (size_t)v * n_terms;
    }
    std::vector<double> prof(tot), w(n_terms);
    gp_video_profiles(dims, order, n_terms, seed, prof.data(), w.data());
    parallel_for((total + 63) / 64, [&](size_t b, size_t e) {
      for (size_t r = b; r < e; ++r) {
        const size_t e0 = r * 64, e1 = std::min(total, e0 + 64);
        Pcg g(seed, kStreamVideoNoise);
        g.advance(2ull * e0);
        for (size_t el = e0; el < e1; ++el) {
          long long idx[8];
          size_t rem = el;
          for (int k = 0; k < order; ++k) {
            idx[k] = (long long)(rem % (size_t)d[k]);
            rem /= (size_t)d[k];
          }
          const double v = gp_video_element(idx, d.data(), order, prof.data(), w.data(), (int)n_terms);
          out[el] = gp_add(v, gp_mul(noise, g.next_double()));
        }
      }
    });
  });
}

}  // extern "C"

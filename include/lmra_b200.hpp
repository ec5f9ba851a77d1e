// lmra_b200.hpp -- C++ drop-in for the reference's hot-path API (namespace lmra,
// proj/include/lmra/tucker.hpp:17-121), header-only over the C ABI in lmra_b200.h.
//
// Same names, argument meaning and exception surface as the reference:
//   rand_thosvd_power / rand_sthosvd_power / rand_thosvd_amm / rand_sthosvd_amm,
//   rand_thosvd_power_qr / rand_sthosvd_power_qr, run_algorithm, amm_sample_counts,
//   AlgoConfig, MultilinearRank, TuckerDecomposition; load_tensor / save_tensor (TNSR).
// std::invalid_argument / std::runtime_error are re-thrown from the ABI status codes.
//
// Also: t_hosvd / st_hosvd / hooi (the deterministic baselines), reconstruct /
// relative_error, parse_algorithm / algorithm_id / all_algorithm_ids, thread_cap,
// MultilinearRank::clamped_for.
//
// Deviation: Eigen3 is not a dependency, so TuckerDecomposition::factors is a
// std::vector<lmra::Matrix> -- a column-major rows() x cols() matrix with data() and
// operator()(i, j); with Eigen available, `Eigen::Map<const Eigen::MatrixXd>(m.data(),
// m.rows(), m.cols())` views it without a copy.  hooi() starts from st_hosvd (the reference's
// two-argument overload); the overload taking an explicit init is not provided.
// Multi-GPU follows the thread_cap() idiom: LMRA_NUM_GPUS=N (tucker.cpp:164-172 reads
// LMRA_NUM_THREADS the same way) makes every randomized T-HOSVD / ST-HOSVD call run on devices
// 0..N-1 from this process (lmra_run_algorithm_multigpu); one process per GPU instead passes
// its slab of the last mode through the C ABI after lmra_context_set_comm.
#pragma once

#include <cstdint>
#include <cstdio>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "lmra_b200.h"

namespace lmra {

namespace detail {
inline void check(int rc) {
  if (rc == LMRA_OK) return;
  const char* m = lmra_last_error();
  if (rc == LMRA_EINVAL) throw std::invalid_argument(m);
  throw std::runtime_error(m);
}
struct Ctx {
  lmra_context* c = nullptr;
  explicit Ctx(int device) { check(lmra_context_create(device, nullptr, &c)); }
  ~Ctx() { lmra_context_destroy(c); }
};
inline lmra_context* default_context() {
  thread_local std::unique_ptr<Ctx> ctx;
  if (!ctx) ctx = std::make_unique<Ctx>(0);
  return ctx->c;
}
}  // namespace detail

// tensor.hpp:14-44 -- dense tensor, first index fastest
class DenseTensor {
 public:
  DenseTensor() = default;
  explicit DenseTensor(std::vector<std::size_t> dims) : dims_(std::move(dims)) {
    std::size_t n = 1;
    for (std::size_t d : dims_) n *= d;
    values_.assign(n, 0.0);
  }
  DenseTensor(std::vector<std::size_t> dims, std::vector<double> values)
      : dims_(std::move(dims)), values_(std::move(values)) {
    std::size_t n = 1;
    for (std::size_t d : dims_) n *= d;
    if (n != values_.size()) throw std::invalid_argument("value count does not match tensor shape");
  }
  std::size_t order() const { return dims_.size(); }
  const std::vector<std::size_t>& dims() const { return dims_; }
  std::size_t dim(std::size_t m) const { return dims_.at(m); }
  std::size_t size() const { return values_.size(); }
  const double* data() const { return values_.data(); }
  double* data() { return values_.data(); }
  double operator[](std::size_t i) const { return values_[i]; }
  double& operator[](std::size_t i) { return values_[i]; }

 private:
  std::vector<std::size_t> dims_;
  std::vector<double> values_;
};

// column-major dense matrix (stands in for Eigen::MatrixXd, see header comment)
class Matrix {
 public:
  Matrix() = default;
  Matrix(std::size_t r, std::size_t c) : r_(r), c_(c), v_(r * c, 0.0) {}
  std::size_t rows() const { return r_; }
  std::size_t cols() const { return c_; }
  const double* data() const { return v_.data(); }
  double* data() { return v_.data(); }
  double operator()(std::size_t i, std::size_t j) const { return v_[i + r_ * j]; }
  double& operator()(std::size_t i, std::size_t j) { return v_[i + r_ * j]; }

 private:
  std::size_t r_ = 0, c_ = 0;
  std::vector<double> v_;
};

enum class ProbRegime { Optimal, NearlyOptimal, Uniform };  // sketching.hpp:31
enum class GramStrategy { A, B };                           // linalg.hpp:26

struct MultilinearRank {  // tucker.hpp:17-24
  std::vector<std::size_t> mu;
  MultilinearRank() = default;
  explicit MultilinearRank(std::vector<std::size_t> m) : mu(std::move(m)) {}
  // tucker.cpp:174-188
  std::vector<std::size_t> clamped_for(const std::vector<std::size_t>& dims) const {
    if (mu.size() != dims.size()) throw std::invalid_argument("rank vector length must equal tensor order");
    std::vector<std::size_t> out(mu.size());
    bool clamped = false;
    for (std::size_t n = 0; n < mu.size(); ++n) {
      if (mu[n] < 1) throw std::invalid_argument("rank entries must be positive");
      out[n] = mu[n] < dims[n] ? mu[n] : dims[n];
      clamped |= out[n] != mu[n];
    }
    if (clamped) std::fputs("lmra: target rank exceeds tensor dimensions, clamping\n", stderr);
    return out;
  }
};

struct TuckerDecomposition {  // tucker.hpp:27-30
  DenseTensor core;
  std::vector<Matrix> factors;
};

struct AlgoConfig {  // tucker.hpp:32-45
  MultilinearRank rank;
  std::size_t oversampling = 10;
  int power = 1;
  double alpha = 0.2;
  ProbRegime regime = ProbRegime::Uniform;
  double regime_beta = 0.5;
  std::vector<std::size_t> t_samples;
  std::vector<std::size_t> order;
  std::uint64_t seed = 0;
  GramStrategy strategy = GramStrategy::A;
  int hooi_max_sweeps = 50;
  double hooi_tol = 1e-8;
};

struct HooiStats {  // tucker.hpp:73-76
  bool converged = false;
  int sweeps = 0;
};

enum class Algorithm {  // tucker.hpp:47-57
  Thosvd, Sthosvd, Hooi, RandThosvdPower, RandSthosvdPower, RandThosvdAmm, RandSthosvdAmm,
  RandThosvdPowerQr, RandSthosvdPowerQr,
};

namespace detail {
struct CConfig {
  std::vector<uint64_t> rank, t, order;
  lmra_algo_config c{};
  explicit CConfig(const AlgoConfig& cfg) {
    lmra_algo_config_init(&c);
    rank.assign(cfg.rank.mu.begin(), cfg.rank.mu.end());
    t.assign(cfg.t_samples.begin(), cfg.t_samples.end());
    order.assign(cfg.order.begin(), cfg.order.end());
    c.rank = rank.data();
    c.n_rank = rank.size();
    c.oversampling = cfg.oversampling;
    c.power = cfg.power;
    c.alpha = cfg.alpha;
    c.regime = cfg.regime == ProbRegime::Optimal ? LMRA_OPTIMAL
               : cfg.regime == ProbRegime::NearlyOptimal ? LMRA_NEARLY_OPTIMAL
                                                         : LMRA_UNIFORM;
    c.regime_beta = cfg.regime_beta;
    c.t_samples = t.empty() ? nullptr : t.data();
    c.n_t_samples = t.size();
    c.order = order.empty() ? nullptr : order.data();
    c.n_order = order.size();
    c.seed = cfg.seed;
    c.strategy = cfg.strategy == GramStrategy::A ? LMRA_STRATEGY_A : LMRA_STRATEGY_B;
    c.hooi_max_sweeps = cfg.hooi_max_sweeps;
    c.hooi_tol = cfg.hooi_tol;
  }
};

inline TuckerDecomposition run(int alg, const DenseTensor& a, const AlgoConfig& cfg, HooiStats* stats = nullptr) {
  CConfig cc(cfg);
  std::vector<uint64_t> dims(a.dims().begin(), a.dims().end());
  lmra_result* r = nullptr;
  const int ngpu = lmra_device_cap();  // LMRA_NUM_GPUS
  if (ngpu > 1 && alg != LMRA_ALG6 && alg != LMRA_ALG7 && alg != LMRA_THOSVD && alg != LMRA_STHOSVD &&
      alg != LMRA_HOOI) {
    std::vector<int> devs(ngpu);
    for (int d = 0; d < ngpu; ++d) devs[d] = d;
    check(lmra_run_algorithm_multigpu(ngpu, devs.data(), alg, a.data(), dims.data(), (int)dims.size(), LMRA_HOST,
                                      &cc.c, nullptr, &r));
  } else {
    check(lmra_run_algorithm(default_context(), alg, a.data(), dims.data(), (int)dims.size(), LMRA_HOST, &cc.c,
                             nullptr, &r));
  }
  std::unique_ptr<lmra_result, void (*)(lmra_result*)> guard(r, lmra_result_free);
  const int N = lmra_result_order(r);
  std::vector<uint64_t> cd(N);
  lmra_result_core_dims(r, cd.data());
  TuckerDecomposition out;
  out.core = DenseTensor(std::vector<std::size_t>(cd.begin(), cd.end()));
  check(lmra_result_copy_core(r, out.core.data(), LMRA_HOST));
  for (int n = 0; n < N; ++n) {
    uint64_t rows = 0, cols = 0;
    lmra_result_factor_dims(r, n, &rows, &cols);
    Matrix m(rows, cols);
    check(lmra_result_copy_factor(r, n, m.data(), LMRA_HOST));
    out.factors.push_back(std::move(m));
  }
  if (stats) {
    int conv = 0, sw = 0;
    lmra_result_hooi_stats(r, &conv, &sw);
    stats->converged = conv != 0;
    stats->sweeps = sw;
  }
  return out;
}
}  // namespace detail

// tucker.hpp:91-102
inline TuckerDecomposition rand_thosvd_power(const DenseTensor& a, const AlgoConfig& cfg) {
  return detail::run(LMRA_ALG1, a, cfg);
}
inline TuckerDecomposition rand_sthosvd_power(const DenseTensor& a, const AlgoConfig& cfg) {
  return detail::run(LMRA_ALG2, a, cfg);
}
inline TuckerDecomposition rand_thosvd_amm(const DenseTensor& a, const AlgoConfig& cfg) {
  return detail::run(LMRA_ALG4, a, cfg);
}
inline TuckerDecomposition rand_sthosvd_amm(const DenseTensor& a, const AlgoConfig& cfg) {
  return detail::run(LMRA_ALG5, a, cfg);
}
// tucker.hpp:107-108 (QR-proxy extraction)
inline TuckerDecomposition rand_thosvd_power_qr(const DenseTensor& a, const AlgoConfig& cfg) {
  return detail::run(LMRA_ALG6, a, cfg);
}
inline TuckerDecomposition rand_sthosvd_power_qr(const DenseTensor& a, const AlgoConfig& cfg) {
  return detail::run(LMRA_ALG7, a, cfg);
}

// tucker.hpp:70-89 (the deterministic baselines)
inline TuckerDecomposition t_hosvd(const DenseTensor& a, const AlgoConfig& cfg) {
  return detail::run(LMRA_THOSVD, a, cfg);
}
inline TuckerDecomposition st_hosvd(const DenseTensor& a, const AlgoConfig& cfg) {
  return detail::run(LMRA_STHOSVD, a, cfg);
}
inline TuckerDecomposition hooi(const DenseTensor& a, const AlgoConfig& cfg, HooiStats* stats = nullptr) {
  return detail::run(LMRA_HOOI, a, cfg, stats);
}

// tucker.hpp:110-111
inline TuckerDecomposition run_algorithm(Algorithm alg, const DenseTensor& a, const AlgoConfig& cfg) {
  switch (alg) {
    case Algorithm::Thosvd: return t_hosvd(a, cfg);
    case Algorithm::Sthosvd: return st_hosvd(a, cfg);
    case Algorithm::Hooi: return hooi(a, cfg);
    case Algorithm::RandThosvdPower: return rand_thosvd_power(a, cfg);
    case Algorithm::RandSthosvdPower: return rand_sthosvd_power(a, cfg);
    case Algorithm::RandThosvdAmm: return rand_thosvd_amm(a, cfg);
    case Algorithm::RandSthosvdAmm: return rand_sthosvd_amm(a, cfg);
    case Algorithm::RandThosvdPowerQr: return rand_thosvd_power_qr(a, cfg);
    case Algorithm::RandSthosvdPowerQr: return rand_sthosvd_power_qr(a, cfg);
  }
  throw std::invalid_argument("unknown algorithm");
}

inline std::optional<Algorithm> parse_algorithm(const std::string& id) {  // tucker.cpp:190-201
  if (id == "thosvd") return Algorithm::Thosvd;
  if (id == "sthosvd") return Algorithm::Sthosvd;
  if (id == "hooi") return Algorithm::Hooi;
  if (id == "alg1") return Algorithm::RandThosvdPower;
  if (id == "alg2") return Algorithm::RandSthosvdPower;
  if (id == "alg4") return Algorithm::RandThosvdAmm;
  if (id == "alg5") return Algorithm::RandSthosvdAmm;
  if (id == "alg6") return Algorithm::RandThosvdPowerQr;
  if (id == "alg7") return Algorithm::RandSthosvdPowerQr;
  return std::nullopt;
}

inline std::string algorithm_id(Algorithm a) {  // tucker.cpp:203-215
  switch (a) {
    case Algorithm::Thosvd: return "thosvd";
    case Algorithm::Sthosvd: return "sthosvd";
    case Algorithm::Hooi: return "hooi";
    case Algorithm::RandThosvdPower: return "alg1";
    case Algorithm::RandSthosvdPower: return "alg2";
    case Algorithm::RandThosvdAmm: return "alg4";
    case Algorithm::RandSthosvdAmm: return "alg5";
    case Algorithm::RandThosvdPowerQr: return "alg6";
    case Algorithm::RandSthosvdPowerQr: return "alg7";
  }
  return "?";
}

inline std::vector<std::string> all_algorithm_ids() {  // tucker.cpp:217-220
  const char* ids[16];
  const int n = lmra_all_algorithm_ids(ids, 16);
  return std::vector<std::string>(ids, ids + n);
}

inline int thread_cap() { return lmra_thread_cap(); }  // tucker.hpp:121

// tucker.hpp:63-66: reconstruct (core x_n Q_n) and relative_error, evaluated on the device
inline DenseTensor reconstruct(const TuckerDecomposition& d) {
  const int N = (int)d.factors.size();
  std::vector<uint64_t> cd(d.core.dims().begin(), d.core.dims().end()), rows(N);
  std::vector<const double*> f(N);
  std::vector<std::size_t> od(N);
  for (int n = 0; n < N; ++n) {
    f[n] = d.factors[n].data();
    rows[n] = d.factors[n].rows();
    od[n] = d.factors[n].rows();
  }
  DenseTensor out(od);
  detail::check(lmra_reconstruct(detail::default_context(), d.core.data(), cd.data(), N, f.data(), rows.data(),
                                 LMRA_HOST, out.data(), LMRA_HOST));
  return out;
}
inline double relative_error(const DenseTensor& a, const DenseTensor& approx) {
  if (a.dims() != approx.dims()) throw std::invalid_argument("relative_error: shape mismatch");
  std::vector<uint64_t> d(a.dims().begin(), a.dims().end());
  double re = 0.0;
  detail::check(lmra_relative_error(detail::default_context(), a.data(), approx.data(), d.data(), (int)d.size(),
                                    LMRA_HOST, &re));
  return re;
}

// tucker.hpp:116-117
inline std::vector<std::size_t> amm_sample_counts(const std::vector<std::size_t>& dims,
                                                  const AlgoConfig& cfg, bool sequential) {
  detail::CConfig cc(cfg);
  std::vector<uint64_t> d(dims.begin(), dims.end()), out(dims.size());
  detail::check(lmra_amm_sample_counts(d.data(), (int)d.size(), &cc.c, sequential ? 1 : 0, out.data()));
  return std::vector<std::size_t>(out.begin(), out.end());
}

// tensor_io.hpp:12-13 -- TNSR files (host tensors; lmra_tnsr_load with LMRA_DEVICE streams a
// file straight into HBM instead)
inline void save_tensor(const std::string& path, const DenseTensor& t) {
  std::vector<uint64_t> d(t.dims().begin(), t.dims().end());
  detail::check(lmra_tnsr_save(nullptr, path.c_str(), t.data(), LMRA_HOST, d.data(), (int)d.size()));
}
inline DenseTensor load_tensor(const std::string& path) {
  int order = 0;
  std::vector<uint64_t> d(64);
  detail::check(lmra_tnsr_read_header(path.c_str(), &order, d.data(), (int)d.size()));
  if (order > (int)d.size()) {
    d.resize((size_t)order);
    detail::check(lmra_tnsr_read_header(path.c_str(), &order, d.data(), order));
  }
  DenseTensor t(std::vector<std::size_t>(d.begin(), d.begin() + order));
  detail::check(lmra_tnsr_load(nullptr, path.c_str(), t.data(), LMRA_HOST));
  return t;
}

}  // namespace lmra

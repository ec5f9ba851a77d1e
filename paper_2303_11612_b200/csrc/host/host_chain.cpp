// host_chain.cpp -- see host_chain.hpp.  Compiled with -ffp-contract=off.
#include "host_chain.hpp"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <iostream>
#include <numeric>
#include <stdexcept>
#include <condition_variable>
#include <deque>
#include <mutex>
#include <thread>

namespace lmra_host {

// ---------------------------------------------------------------- rng.hpp:20-66
Rng::Rng(uint64_t seed, uint64_t stream) {
  inc_ = (stream << 1u) | 1u;
  state_ = 0;
  next_u32();
  state_ += seed;
  next_u32();
}

uint32_t Rng::next_u32() {
  uint64_t old = state_;
  state_ = old * 6364136223846793005ULL + inc_;
  uint32_t xs = static_cast<uint32_t>(((old >> 18u) ^ old) >> 27u);
  uint32_t rot = static_cast<uint32_t>(old >> 59u);
  return (xs >> rot) | (xs << ((32u - rot) & 31u));
}

double Rng::next_double() {
  uint64_t hi = next_u32();
  uint64_t lo = next_u32();
  return static_cast<double>(((hi << 32) | lo) >> 11) * 0x1.0p-53;
}

double Rng::next_normal() {
  if (has_cached_) {
    has_cached_ = false;
    return cached_;
  }
  double u1 = 1.0 - next_double();
  double u2 = next_double();
  double r = std::sqrt(-2.0 * std::log(u1));
  double a = 6.283185307179586476925286766559 * u2;
  cached_ = r * std::sin(a);
  has_cached_ = true;
  return r * std::cos(a);
}

void Rng::advance(uint64_t delta) {
  uint64_t cm = 6364136223846793005ULL, cp = inc_, am = 1, ap = 0;
  while (delta) {
    if (delta & 1) {
      am *= cm;
      ap = ap * cm + cp;
    }
    cp = (cm + 1) * cp;
    cm *= cm;
    delta >>= 1;
  }
  state_ = am * state_ + ap;
}

int host_threads() {
  unsigned h = std::thread::hardware_concurrency();
  return h ? static_cast<int>(std::min(h, 64u)) : 1;
}

void fill_normals_range(uint64_t seed, uint64_t stream, double* out, size_t b, size_t e) {
  if (b >= e) return;
  Rng g(seed, stream);
  g.advance(4 * (b / 2));
  size_t i = b;
  if (i & 1) {
    g.next_normal();
    out[i++] = g.next_normal();
  }
  for (; i < e; ++i) out[i] = g.next_normal();
}

// ---------------------------------------------------------------- worker pool
namespace {
class Pool {
 public:
  explicit Pool(int n) {
    for (int i = 0; i < n; ++i) workers_.emplace_back([this] { loop(); });
  }
  ~Pool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
      stop_flag_.store(true, std::memory_order_release);
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }
  void push(std::function<void()> f) {
    {
      std::lock_guard<std::mutex> lk(mu_);
      q_.push_back(std::move(f));
      queued_.fetch_add(1, std::memory_order_release);
    }
    cv_.notify_one();
  }
  // runs one queued job on the calling thread (false: queue empty) -- a waiter helps instead of
  // sleeping while the workers wake up (small batches: the wake-up dominated)
  bool try_run_one() {
    std::function<void()> f;
    {
      std::lock_guard<std::mutex> lk(mu_);
      if (q_.empty()) return false;
      f = std::move(q_.front());
      q_.pop_front();
      queued_.fetch_sub(1, std::memory_order_release);
    }
    f();
    return true;
  }
  void push_batch(std::vector<std::function<void()>>& fs) {
    {
      std::lock_guard<std::mutex> lk(mu_);
      for (auto& f : fs) q_.push_back(std::move(f));
      queued_.fetch_add((long)fs.size(), std::memory_order_release);
    }
    cv_.notify_all();
  }

 private:
  // A worker that finished a job keeps polling the queue for a short while before it sleeps on
  // the condition variable: a run's Omega draw is split into ~2 jobs per worker, and waking 16
  // sleeping workers through the condition variable took ~50 us (cfg1's 3 x 3000 normals were
  // drawn in 60-85 us on 16 threads, ~17 us of work); decompositions issued back to back find
  // the workers still polling.  (OpenMP runtimes keep their workers spinning the same way.)
  static double spin_ms() {  // LMRA_POOL_SPIN_US overrides (0: sleep at once)
    static const double v = getenv("LMRA_POOL_SPIN_US") ? atof(getenv("LMRA_POOL_SPIN_US")) / 1000.0 : 2.0;
    return v;
  }
  bool try_pop(std::function<void()>& f) {
    if (queued_.load(std::memory_order_acquire) == 0) return false;
    std::lock_guard<std::mutex> lk(mu_);
    if (q_.empty()) return false;
    f = std::move(q_.front());
    q_.pop_front();
    queued_.fetch_sub(1, std::memory_order_release);
    return true;
  }
  void loop() {
    for (;;) {
      std::function<void()> f;
      const auto spin_end = std::chrono::steady_clock::now() + std::chrono::microseconds((long)(spin_ms() * 1000));
      while (!try_pop(f)) {
        if (stop_flag_.load(std::memory_order_acquire)) break;
        if (std::chrono::steady_clock::now() >= spin_end) break;
        std::this_thread::yield();
      }
      if (!f) {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [this] { return stop_ || !q_.empty(); });
        if (stop_ && q_.empty()) return;
        f = std::move(q_.front());
        q_.pop_front();
        queued_.fetch_sub(1, std::memory_order_release);
      }
      f();
    }
  }
  std::vector<std::thread> workers_;
  std::deque<std::function<void()>> q_;
  std::mutex mu_;
  std::condition_variable cv_;
  bool stop_ = false;
  std::atomic<long> queued_{0};       // q_.size(), readable without the lock (the polling workers)
  std::atomic<bool> stop_flag_{false};
};

Pool& pool() {
  static Pool p(std::max(1, host_threads()));
  return p;
}
}  // namespace

struct TaskGroup::State {
  std::mutex mu;
  std::condition_variable cv;
  long pending = 0;
};

TaskGroup::TaskGroup() : st_(std::make_shared<State>()) {}
TaskGroup::~TaskGroup() { wait(); }

void TaskGroup::run(std::function<void()> f) {
  {
    std::lock_guard<std::mutex> lk(st_->mu);
    ++st_->pending;
  }
  std::shared_ptr<State> st = st_;
  pool().push([st, f = std::move(f)] {
    f();
    std::lock_guard<std::mutex> lk(st->mu);
    if (--st->pending == 0) st->cv.notify_all();
  });
}

void TaskGroup::run_batch(std::vector<std::function<void()>> fs) {
  if (fs.empty()) return;
  {
    std::lock_guard<std::mutex> lk(st_->mu);
    st_->pending += (long)fs.size();
  }
  std::shared_ptr<State> st = st_;
  std::vector<std::function<void()>> wrapped;
  wrapped.reserve(fs.size());
  for (auto& f : fs)
    wrapped.emplace_back([st, f = std::move(f)] {
      f();
      std::lock_guard<std::mutex> lk(st->mu);
      if (--st->pending == 0) st->cv.notify_all();
    });
  pool().push_batch(wrapped);
}

void TaskGroup::wait() {
  for (;;) {
    {
      std::lock_guard<std::mutex> lk(st_->mu);
      if (st_->pending == 0) return;
    }
    if (!pool().try_run_one()) break;
  }
  std::unique_lock<std::mutex> lk(st_->mu);
  st_->cv.wait(lk, [this] { return st_->pending == 0; });
}

void fill_normals(uint64_t seed, uint64_t stream, double* out, size_t n, int threads) {
  if (threads <= 1 || n < 8192) {
    fill_normals_range(seed, stream, out, 0, n);
    return;
  }
  // chunks on the persistent pool (jump-ahead per chunk: bit-identical to the sequential loop)
  const size_t chunk = std::max<size_t>(4096, ((n / (4 * (size_t)threads)) + 1) & ~size_t(1));
  TaskGroup tg;
  std::vector<std::function<void()>> tasks;
  for (size_t b = 0; b < n; b += chunk) {
    const size_t e = std::min(n, b + chunk);
    tasks.emplace_back([=] { fill_normals_range(seed, stream, out, b, e); });
  }
  tg.run_batch(std::move(tasks));
  tg.wait();
}

// ---------------------------------------------------------------- sketching.cpp:13-53
double stable_sum(const double* v, size_t n) {
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

void check_distribution(const std::vector<double>& w) {
  if (w.empty()) throw std::invalid_argument("probability distribution must be nonempty");
  for (double x : w)
    if (!(x >= 0.0)) throw std::invalid_argument("probability weights must be nonnegative");
  double s = stable_sum(w.data(), w.size());
  if (std::abs(s - 1.0) > 1e-12) throw std::invalid_argument("probability weights must sum to one");
}

static std::vector<double> normalized(std::vector<double> raw) {
  for (double w : raw)
    if (!(w >= 0.0)) throw std::invalid_argument("probability weights must be nonnegative");
  double s = stable_sum(raw.data(), raw.size());
  if (s <= 0.0) throw std::invalid_argument("cannot normalize an all-zero distribution");
  for (double& w : raw) w /= s;
  check_distribution(raw);
  return raw;
}

std::vector<double> uniform_distribution(size_t n) {
  if (n == 0) throw std::invalid_argument("probability distribution must be nonempty");
  std::vector<double> w(n, 1.0 / static_cast<double>(n));
  check_distribution(w);
  return w;
}

// ---------------------------------------------------------------- tucker.cpp:110-130
std::vector<double> probabilities_from_norms(std::vector<double> w, int regime, double beta) {
  const size_t n = w.size();
  if (regime == kUniform) return uniform_distribution(n);
  double total = 0.0;
  for (size_t i = 0; i < n; ++i) total += w[i];
  if (total <= 0.0) return uniform_distribution(n);
  for (auto& x : w) x /= total;
  if (regime == kOptimal) return normalized(std::move(w));
  if (!(beta > 0.0 && beta <= 1.0))
    throw std::invalid_argument("nearly-optimal mixture weight must lie in (0, 1]");
  for (auto& x : w) x = beta * x + (1.0 - beta) / static_cast<double>(n);
  return normalized(std::move(w));
}

// ---------------------------------------------------------------- sketching.cpp:96-131
Samples randsample(size_t L, const std::vector<double>& p, uint64_t seed, uint64_t stream) {
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

// ---------------------------------------------------------------- tucker.cpp config rules
std::vector<size_t> clamped_for(const std::vector<size_t>& mu, const std::vector<size_t>& dims) {
  if (mu.size() != dims.size())
    throw std::invalid_argument("rank vector length must equal tensor order");
  std::vector<size_t> out(mu.size());
  bool clamped = false;
  for (size_t n = 0; n < mu.size(); ++n) {
    if (mu[n] < 1) throw std::invalid_argument("rank entries must be positive");
    out[n] = std::min(mu[n], dims[n]);
    clamped |= out[n] != mu[n];
  }
  if (clamped) std::cerr << "lmra: target rank exceeds tensor dimensions, clamping\n";
  return out;
}

Resolved resolve(const std::vector<size_t>& dims, const Config& cfg) {
  const size_t nm = dims.size();
  if (nm == 0) throw std::invalid_argument("cannot decompose an order-0 tensor");
  if (cfg.mu.size() != nm) throw std::invalid_argument("rank vector length must equal tensor order");
  if (cfg.power < 1) throw std::invalid_argument("power exponent must be >= 1");
  Resolved r;
  r.mu = clamped_for(cfg.mu, dims);
  r.sketch.resize(nm);
  for (size_t n = 0; n < nm; ++n) r.sketch[n] = std::min(r.mu[n] + cfg.oversampling, dims[n]);
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

size_t other_dims_product(const std::vector<size_t>& dims, size_t mode) {
  size_t p = 1;
  for (size_t k = 0; k < dims.size(); ++k)
    if (k != mode) p *= dims[k];
  return p;
}

size_t samples_from_alpha(double alpha, size_t cols) {
  if (!(alpha > 0.0 && alpha < 1.0))
    throw std::invalid_argument("sampling fraction alpha must lie in (0, 1)");
  auto t = static_cast<size_t>(std::ceil(alpha * static_cast<double>(cols)));
  return std::max<size_t>(t, 1);
}

std::vector<size_t> amm_sample_counts(const std::vector<size_t>& dims, const Config& cfg,
                                      bool sequential) {
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

}  // namespace lmra_host

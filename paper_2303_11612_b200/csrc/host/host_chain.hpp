// host_chain.hpp -- host-side pieces of the path that must be bit-exact with the
// reference: the PCG32/Box-Muller stream (rng.hpp:20-66), Omega (sketching.cpp:164-173),
// the probability chain (tucker.cpp:110-130, sketching.cpp:13-53) and the multinomial
// selector (sketching.cpp:96-131).  Compiled with -ffp-contract=off: every a*b+c here is
// two roundings, as in the reference sources.
#pragma once
#include <cstdint>
#include <functional>
#include <memory>
#include <string>
#include <vector>

namespace lmra_host {

enum Regime { kOptimal = 0, kNearlyOptimal = 1, kUniform = 2 };

class Rng {
 public:
  Rng(uint64_t seed, uint64_t stream);
  uint32_t next_u32();
  double next_double();
  double next_normal();
  void advance(uint64_t delta);  // jump ahead by delta u32 draws

 private:
  uint64_t state_ = 0, inc_ = 1;
  double cached_ = 0.0;
  bool has_cached_ = false;
};

// normals [0, n) of stream (seed, stream) in generation order; threads split the
// sequence with jump-ahead (bit-identical to the sequential loop).
void fill_normals(uint64_t seed, uint64_t stream, double* out, size_t n, int threads);

// normals [b, e) of stream (seed, stream) (b even), written to out[b..e)
void fill_normals_range(uint64_t seed, uint64_t stream, double* out, size_t b, size_t e);

// A set of host tasks run by a persistent process-wide worker pool (threads are started
// once; spawning threads per run cost more than the Omega draw of the small configs).
class TaskGroup {
 public:
  TaskGroup();
  ~TaskGroup();  // waits
  TaskGroup(const TaskGroup&) = delete;
  TaskGroup& operator=(const TaskGroup&) = delete;
  void run(std::function<void()> f);
  void run_batch(std::vector<std::function<void()>> fs);  // one queue lock, one wake-up
  void wait();

 private:
  struct State;
  std::shared_ptr<State> st_;
};

double stable_sum(const double* v, size_t n);
void check_distribution(const std::vector<double>& w);
std::vector<double> uniform_distribution(size_t n);
// tucker.cpp:110-130 from precomputed squared column norms w (consumed)
std::vector<double> probabilities_from_norms(std::vector<double> w, int regime, double beta);

struct Samples {
  std::vector<int64_t> idx;
  std::vector<double> scales;
};
Samples randsample(size_t L, const std::vector<double>& p, uint64_t seed, uint64_t stream);

// tucker.cpp:24-52,101-106,174-188,348-376
struct Config {
  std::vector<size_t> mu;
  size_t oversampling = 10;
  int power = 1;
  double alpha = 0.2;
  int regime = kUniform;
  double beta = 0.5;
  std::vector<size_t> t_samples;
  std::vector<size_t> order;
  uint64_t seed = 0;
  int strategy = 0;
  int hooi_max_sweeps = 50;
  double hooi_tol = 1e-8;
};

struct Resolved {
  std::vector<size_t> mu, sketch, order;
};

std::vector<size_t> clamped_for(const std::vector<size_t>& mu, const std::vector<size_t>& dims);
Resolved resolve(const std::vector<size_t>& dims, const Config& cfg);
size_t samples_from_alpha(double alpha, size_t cols);
size_t other_dims_product(const std::vector<size_t>& dims, size_t mode);
std::vector<size_t> amm_sample_counts(const std::vector<size_t>& dims, const Config& cfg,
                                      bool sequential);

int host_threads();

}  // namespace lmra_host

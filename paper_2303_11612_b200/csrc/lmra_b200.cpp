// lmra_b200.cpp -- host orchestration of the randomized Tucker hot path + the C ABI.
//
// Mirrors the control flow of the reference's four entry points
//   rand_thosvd_power  tucker.cpp:318-330   (alg1)
//   rand_sthosvd_power tucker.cpp:332-346   (alg2)
//   rand_thosvd_amm    tucker.cpp:378-395   (alg4)
//   rand_sthosvd_amm   tucker.cpp:397-420   (alg5)
// with every flop on the device (kernels/*.cu) and the tensor read in place (no unfold).
// The only host work is what must be bit-exact with the reference's seeded host RNG:
// Omega (gaussian_matrix) and the sampling chain (probabilities -> randsample).
#include "../../include/lmra_b200.h"

#include <cuda_runtime.h>
#include "host/nccl_dyn.hpp"
#include "host/cusolver_dyn.hpp"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstring>
#include <memory>
#include <map>
#include <mutex>
#include <numeric>
#include <set>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "host/host_chain.hpp"
#include "host/tnsr.hpp"
#include "kernels/kernels.hpp"
#include "gen/portable_gen.hpp"

using lmra_dev::ModeView;

namespace {

thread_local std::string g_err;

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

void ckn(ncclResult_t e, const char* what) {
  if (e != ncclSuccess) throw CudaError(std::string(what) + ": " + lmra_host::nccl().GetErrorString(e));
}

template <class F>
int guard(F&& f) {
  try {
    f();
    return LMRA_OK;
  } catch (const std::logic_error& e) {  // invalid_argument, out_of_range
    g_err = e.what();
    return LMRA_EINVAL;
  } catch (const CudaError& e) {
    g_err = e.what();
    return LMRA_ECUDA;
  } catch (const std::exception& e) {
    g_err = e.what();
    return LMRA_ERUNTIME;
  }
}

double now_ms() {
  return std::chrono::duration<double, std::milli>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

// ------------------------------------------------------------------ collectives
// The sharded path needs two collectives on small device buffers: an in-place sum
// all-reduce and an equal-count all-gather.  NcclComm is the product (one process per GPU,
// NVLink); ThreadComm runs several ranks as host threads of one process (each with its own
// context/stream, possibly on one GPU) with device-side copies and host barriers -- no
// kernel ever waits on another rank -- so the sharded code can be checked rank-for-rank on
// a single GPU.
struct Comm {
  int nranks = 1, rank = 0;
  virtual ~Comm() = default;
  virtual void allreduce_sum(double* buf, size_t n, cudaStream_t st) = 0;
  virtual void allgather(const double* send, double* recv, size_t n_per_rank, cudaStream_t st) = 0;
  virtual void abort() {}  // a rank failed mid-run: release peers blocked in a collective
};

struct NcclComm : Comm {
  ncclComm_t c = nullptr;
  ~NcclComm() override {
    if (c) lmra_host::nccl().CommDestroy(c);
  }
  // a rank failed mid-run: abort the communicator so peers blocked in a collective return with
  // an error instead of hanging; the communicator is unusable afterwards (a new one must be set)
  void abort() override {
    if (c && lmra_host::nccl().CommAbort) lmra_host::nccl().CommAbort(c);
    c = nullptr;
  }
  void usable() const {
    if (!c) throw std::runtime_error("NCCL communicator was aborted by an earlier failed run");
  }
  // all-gather + a fixed-order (rank order) sum instead of ncclAllReduce: every rank gets
  // the same bits, identical to ThreadComm's sum (the path the GPU tests check rank for rank)
  // and independent of the reduction algorithm NCCL picks (ring / tree / NVLS)
  void allreduce_sum(double* buf, size_t n, cudaStream_t st) override {
    if (n == 0) return;
    usable();
    double* tmp = nullptr;
    ck(lmra_dev::scratch_alloc(reinterpret_cast<void**>(&tmp), n * nranks * sizeof(double), st), "alloc");
    ckn(lmra_host::nccl().AllGather(buf, tmp, n, ncclDouble, c, st), "ncclAllGather");
    ck(lmra_dev::launch_sum_ranks_strided(tmp, nranks, (long long)n, buf, st), "sum_ranks");
    lmra_dev::scratch_free(tmp, st);
  }
  void allgather(const double* send, double* recv, size_t n, cudaStream_t st) override {
    usable();
    ckn(lmra_host::nccl().AllGather(send, recv, n, ncclDouble, c, st), "ncclAllGather");
  }
};

struct ThreadGroup {
  int n = 1;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  long long gen = 0;
  bool aborted = false;  // sticky: a group whose run failed on some rank is not reusable
  std::vector<const double*> ptrs;
  explicit ThreadGroup(int nr) : n(nr), ptrs(nr, nullptr) {}
  void barrier() {
    std::unique_lock<std::mutex> lk(m);
    if (aborted) throw std::runtime_error("thread group: a peer rank failed");
    const long long g = gen;
    if (++arrived == n) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g || aborted; });
      if (gen == g) throw std::runtime_error("thread group: a peer rank failed");
    }
  }
  void abort() {
    std::lock_guard<std::mutex> lk(m);
    aborted = true;
    cv.notify_all();
  }
};

struct ThreadComm : Comm {
  std::shared_ptr<ThreadGroup> g;
  void allreduce_sum(double* buf, size_t n, cudaStream_t st) override;
  void abort() override { g->abort(); }
  void allgather(const double* send, double* recv, size_t n, cudaStream_t st) override {
    ck(cudaStreamSynchronize(st), "sync");
    g->ptrs[rank] = send;
    g->barrier();
    for (int r = 0; r < nranks; ++r)
      ck(cudaMemcpyAsync(recv + (size_t)r * n, g->ptrs[r], n * sizeof(double),
                         cudaMemcpyDeviceToDevice, st),
         "allgather copy");
    ck(cudaStreamSynchronize(st), "sync");
    g->barrier();
  }
};

void ThreadComm::allreduce_sum(double* buf, size_t n, cudaStream_t st) {
  ck(cudaStreamSynchronize(st), "sync");
  g->ptrs[rank] = buf;
  g->barrier();
  double* tmp = nullptr;
  const double** dptrs = nullptr;
  ck(cudaMallocAsync(reinterpret_cast<void**>(&tmp), std::max<size_t>(n, 1) * sizeof(double), st), "alloc");
  ck(cudaMallocAsync(reinterpret_cast<void**>(&dptrs), nranks * sizeof(double*), st), "alloc");
  ck(cudaMemcpyAsync(dptrs, g->ptrs.data(), nranks * sizeof(double*), cudaMemcpyHostToDevice, st), "H2D");
  ck(lmra_dev::launch_sum_ranks(dptrs, nranks, (long long)n, tmp, st), "sum_ranks");
  ck(cudaStreamSynchronize(st), "sync");
  g->barrier();  // every rank has read every buffer
  ck(cudaMemcpyAsync(buf, tmp, n * sizeof(double), cudaMemcpyDeviceToDevice, st), "copy");
  cudaFreeAsync(tmp, st);
  cudaFreeAsync(dptrs, st);
  ck(cudaStreamSynchronize(st), "sync");
}

}  // namespace

// ------------------------------------------------------------------ context
// int8 tensor-core contractions on (default) or off (LMRA_TTM_I8=0: every contraction on DMMA)
bool ttm_i8_on() {
  static const bool on = !(getenv("LMRA_TTM_I8") && std::string(getenv("LMRA_TTM_I8")) == "0");
  return on;
}

// Device blocks handed to results (core, factors), recycled instead of cudaMalloc/cudaFree
// per run (each of those costs ~0.1 ms and cudaFree synchronises the device).  Shared by the
// context and its results, so a result may outlive the context.
struct ResultBlocks {
  int device = 0;
  std::mutex mu;
  std::multimap<size_t, void*> free_blocks;  // capacity -> block
  std::map<void*, size_t> cap;
  void* get(size_t bytes) {
    size_t c = 256;
    while (c < bytes) c <<= 1;
    {
      std::lock_guard<std::mutex> lk(mu);
      auto it = free_blocks.find(c);
      if (it != free_blocks.end()) {
        void* p = it->second;
        free_blocks.erase(it);
        return p;
      }
    }
    void* p = nullptr;
    if (cudaMalloc(&p, c) != cudaSuccess) throw std::runtime_error("cudaMalloc (result) failed");
    std::lock_guard<std::mutex> lk(mu);
    cap[p] = c;
    return p;
  }
  void put(void* p) {
    if (!p) return;
    std::lock_guard<std::mutex> lk(mu);
    auto it = cap.find(p);
    if (it != cap.end()) free_blocks.emplace(it->second, p);
  }
  ~ResultBlocks() {
    int prev = -1;
    cudaGetDevice(&prev);
    if (prev != device) cudaSetDevice(device);
    for (auto& kv : cap) cudaFree(kv.first);
    if (prev >= 0 && prev != device) cudaSetDevice(prev);
  }
};

struct lmra_context {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int num_sms = 148;
  std::shared_ptr<Comm> comm;  // set: sharded runs (tensor = this rank's slab of the last mode)
  int nranks = 1, rank = 0;
  std::mutex mu;
  long long launches = 0;
  int profile = 0;  // per-launch CUDA events (lmra_context_set_profiling): 1 every phase,
                    // 2 only the phases on the context's own stream (light)
  bool keep_trace = true;  // copy drawn samples / norms back to the host (lmra_context_set_trace)
  std::vector<cudaEvent_t> events;
  size_t next_event = 0;
  std::vector<cudaStream_t> aux;   // per-mode streams (T-HOSVD modes run concurrently)
  double* pinned = nullptr;        // pinned staging for Omega (async H2D, no pageable sync)
  size_t pinned_doubles = 0;
  // Per-run device arena (see ArenaScope): one cudaMalloc'd block, bump-allocated during a
  // run, reset when the run has synchronised, grown between runs to what the last run asked.
  char* arena = nullptr;
  size_t arena_cap = 0, arena_off = 0, arena_want = 0;
  std::shared_ptr<ResultBlocks> results = std::make_shared<ResultBlocks>();
  cusolverDnHandle_t cusolver = nullptr;  // deterministic baselines only (lazily created)
  // the per-mode stream of the mode the core contracts first, at the device's highest stream
  // priority: its sampling chain, power scheme and basis gate the long contraction, and three
  // modes' latency-bound chains compete for the same SMs (cfg4: that mode's sampler finished
  // last, 0.15 ms after the others)
  cudaStream_t hi = nullptr;
  cudaStream_t hi_stream() {
    if (!hi) {
      int lo = 0, greatest = 0;
      if (cudaDeviceGetStreamPriorityRange(&lo, &greatest) != cudaSuccess) greatest = 0;
      if (cudaStreamCreateWithPriority(&hi, cudaStreamNonBlocking, greatest) != cudaSuccess)
        throw std::runtime_error("cudaStreamCreate failed");
    }
    return hi;
  }
  cudaStream_t aux_stream(size_t i) {
    while (aux.size() <= i) {
      cudaStream_t s;
      if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess)
        throw std::runtime_error("cudaStreamCreate failed");
      aux.push_back(s);
    }
    return aux[i];
  }
  double* pinned_buffer(size_t n) {
    if (n > pinned_doubles) {
      if (pinned) cudaFreeHost(pinned);
      pinned = nullptr;
      if (cudaMallocHost(reinterpret_cast<void**>(&pinned), n * sizeof(double)) != cudaSuccess)
        throw std::runtime_error("cudaMallocHost failed");
      pinned_doubles = n;
    }
    return pinned;
  }
  cudaEvent_t event() {  // pooled timing events, recycled every run
    if (next_event == events.size()) {
      cudaEvent_t e;
      if (cudaEventCreate(&e) != cudaSuccess) throw std::runtime_error("cudaEventCreate failed");
      events.push_back(e);
    }
    return events[next_event++];
  }
};

namespace {

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) ck(cudaSetDevice(dev), "cudaSetDevice");
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// Device memory of a run.  The stream-ordered pool (cudaMallocAsync) stalled the host for
// 1-700 ms at random steps of an otherwise steady-state loop (measured on cfg5 with
// LMRA_TIMELINE: 6 MB / 60 MB requests remapping memory), so every buffer of a run comes
// from a per-context arena instead: bump allocation, no frees, reset once the run has
// synchronised.  A request that does not fit falls back to the pool and the arena is grown
// to the run's total before the next run (the first run of a shape warms it).
static thread_local lmra_context* t_arena_ctx = nullptr;

static void* arena_take(size_t bytes) {
  lmra_context* c = t_arena_ctx;
  if (!c) return nullptr;
  const size_t b = (bytes + 255) & ~size_t(255);
  c->arena_want += b;
  if (c->arena_off + b > c->arena_cap) return nullptr;
  void* p = c->arena + c->arena_off;
  c->arena_off += b;
  return p;
}

static bool in_arena(const void* p) {
  const lmra_context* c = t_arena_ctx;
  return c && c->arena && p >= c->arena && p < c->arena + c->arena_cap;
}

class ArenaScope {
 public:
  explicit ArenaScope(lmra_context* ctx) : ctx_(ctx), prev_(t_arena_ctx) {
    ctx_->arena_off = 0;
    ctx_->arena_want = 0;
    t_arena_ctx = ctx_;
  }
  ~ArenaScope() {
    // every stream of the run is drained before its memory is handed out again
    cudaStreamSynchronize(ctx_->stream);
    for (cudaStream_t s : ctx_->aux) cudaStreamSynchronize(s);
    t_arena_ctx = prev_;
    if (ctx_->arena_want > ctx_->arena_cap) {
      if (ctx_->arena) cudaFree(ctx_->arena);
      ctx_->arena = nullptr;
      ctx_->arena_cap = 0;
      const size_t cap = ctx_->arena_want + ctx_->arena_want / 8 + (64u << 20);
      if (cudaMalloc(reinterpret_cast<void**>(&ctx_->arena), cap) == cudaSuccess)
        ctx_->arena_cap = cap;
      else
        cudaGetLastError();  // no room: later runs keep using the pool
    }
    ctx_->arena_off = 0;
    ctx_->arena_want = 0;
  }

 private:
  lmra_context* ctx_;
  lmra_context* prev_;
};

// diagnostics (LMRA_TIMELINE=1): phase timeline and slow host calls on stderr
static bool diag_timing() {
  static const bool on = getenv("LMRA_TIMELINE") && getenv("LMRA_TIMELINE")[0] == '1';
  return on;
}

// Stream-ordered device buffer from the device's (retained) memory pool.
class DevBuf {
 public:
  DevBuf() = default;
  DevBuf(size_t n, cudaStream_t st) : st_(st), n_(n) {
    if (!n) return;
    const size_t bytes = std::max<size_t>(n, 2) * sizeof(double);
    if ((p_ = static_cast<double*>(arena_take(bytes)))) {
      arena_ = true;
      return;
    }
    const double t0 = diag_timing() ? now_ms() : 0.0;
    ck(cudaMallocAsync(reinterpret_cast<void**>(&p_), bytes, st), "cudaMallocAsync");
    if (diag_timing() && now_ms() - t0 > 0.5)
      fprintf(stderr, "hostslow cudaMallocAsync %zu MB %.3f ms\n", n * 8 >> 20, now_ms() - t0);
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept { *this = std::move(o); }
  DevBuf& operator=(DevBuf&& o) noexcept {
    release();
    p_ = o.p_;
    st_ = o.st_;
    n_ = o.n_;
    arena_ = o.arena_;
    o.p_ = nullptr;
    o.n_ = 0;
    return *this;
  }
  ~DevBuf() { release(); }
  double* get() const { return p_; }
  size_t size() const { return n_; }
  // the stream of the buffer's last use (its free is ordered after that stream's work)
  void rebind(cudaStream_t st) { st_ = st; }
  // ownership to the caller (results outlive the run): a copy in a recycled result block,
  // returned to the context's ResultBlocks by ~lmra_result
  double* detach() {
    if (!p_) return nullptr;
    if (!t_arena_ctx) throw std::logic_error("DevBuf::detach outside a run");
    double* d = static_cast<double*>(t_arena_ctx->results->get(std::max<size_t>(n_, 2) * sizeof(double)));
    ck(cudaMemcpyAsync(d, p_, n_ * sizeof(double), cudaMemcpyDeviceToDevice, st_), "D2D result");
    release();
    n_ = 0;
    return d;
  }

 private:
  void release() {
    if (p_ && !arena_) cudaFreeAsync(p_, st_);
    p_ = nullptr;
    arena_ = false;
  }
  double* p_ = nullptr;
  cudaStream_t st_ = nullptr;
  size_t n_ = 0;
  bool arena_ = false;
};

// sampled matrices of at least this many elements are read in place by the power scheme
// (Gather) instead of being materialised; LMRA_FUSED_GATHER_MIN overrides (tests force it)
size_t fused_gather_min() {
  const char* e = getenv("LMRA_FUSED_GATHER_MIN");
  return e ? (size_t)strtoull(e, nullptr, 10) : (size_t(1) << 22);
}

ModeView view_of(const std::vector<size_t>& dims, size_t mode) {
  ModeView v;
  v.inner = 1;
  for (size_t k = 0; k < mode; ++k) v.inner *= (long long)dims[k];
  v.I = (long long)dims[mode];
  v.outer = 1;
  for (size_t k = mode + 1; k < dims.size(); ++k) v.outer *= (long long)dims[k];
  return v;
}

size_t prod(const std::vector<size_t>& d) {
  size_t p = 1;
  for (size_t x : d) p *= x;
  return p;
}

// Shard plan of the last mode (extent L over P ranks): contiguous slabs, balanced in units of
// 64 rows (two canonical norm chunks) when L >= 64 P, so that a fibre of the last mode splits
// between ranks only at segment boundaries of the canonical squared norm (canon_add) and the
// sharded norms combine to the single-device bits; otherwise balanced rows.
constexpr size_t kShardUnit = 64;
void shard_bounds(size_t L, size_t P, size_t r, size_t* start, size_t* count) {
  size_t b, e;
  if (L >= kShardUnit * P) {
    const size_t u = (L + kShardUnit - 1) / kShardUnit;
    b = std::min(L, (u * r) / P * kShardUnit);
    e = std::min(L, (u * (r + 1)) / P * kShardUnit);
  } else {
    b = (L * r) / P;
    e = (L * (r + 1)) / P;
  }
  *start = b;
  *count = e - b;
}

}  // namespace

// ------------------------------------------------------------------ result
struct lmra_result {
  int device = 0;
  std::shared_ptr<ResultBlocks> blocks;  // owner of core / factors
  std::vector<size_t> core_dims;
  double* core = nullptr;
  std::vector<size_t> f_rows, f_cols;
  std::vector<double*> factors;
  std::vector<size_t> om_rows, om_cols;
  std::vector<std::vector<double>> omega;
  std::vector<std::vector<int64_t>> idx;
  std::vector<std::vector<double>> scales;
  std::vector<std::vector<double>> norms;
  double t_total = 0, t_rng = 0, t_sampling = 0, t_device = 0, launches = 0;
  int sampler_fallbacks = 0;  // uncertified Neumaier roundings resolved sequentially
  int hooi_converged = 0, hooi_sweeps = 0;  // HooiStats (tucker.hpp:73-76), hooi runs only
  struct Phase {
    std::string name;
    double ms;
    int count;
  };
  std::vector<Phase> phases;  // device time per launch category (profiling contexts only)
  // set once core / factor device pointers were handed out (lmra_result_*_device): the caller
  // may have queued reads of them on streams of its own
  mutable std::atomic<bool> exposed{false};
  ~lmra_result() {
    int prev = -1;
    cudaGetDevice(&prev);
    if (prev != device) cudaSetDevice(device);
    if (blocks) {
      // the run that produced the blocks has synchronised; reads the caller queued elsewhere
      // through the device pointers must finish before the next run's detach() reuses the
      // blocks on the context stream -- the guarantee cudaFree gave (it synchronises)
      if (exposed.load()) cudaDeviceSynchronize();
      blocks->put(core);
      for (double* f : factors) blocks->put(f);
    } else {
      if (core) cudaFree(core);
      for (double* f : factors)
        if (f) cudaFree(f);
    }
    if (prev >= 0 && prev != device) cudaSetDevice(prev);
  }
};

namespace {

// ------------------------------------------------------------------ the engine
// One launch (or launch group) bracketed by CUDA events on the launching stream.
struct PhaseRec {
  std::string name;
  cudaEvent_t a, b;
};

class Engine {
 public:
  Engine(lmra_context* ctx, std::vector<PhaseRec>* prof = nullptr)
      : ctx_(ctx), st_(ctx->stream), prof_(prof) {}
  Engine(lmra_context* ctx, cudaStream_t st, std::vector<PhaseRec>* prof)
      : ctx_(ctx), st_(st), prof_(prof) {}

  template <class F>
  void launch(const std::string& phase, F&& f) {
    cudaEvent_t a = nullptr, b = nullptr;
    // profiling level 3: events only around the mode-0 contraction (the launch the bench's
    // roofline is quoted on) -- every event record is host work on the critical path of the
    // latency-bound chains, so a timed run keeps them to one pair
    const bool rec = prof_ && (ctx_->profile != 3 || phase.rfind("core_ttm0", 0) == 0 ||
                               phase.rfind("shrink_ttm_m0", 0) == 0);
    if (rec) {
      a = ctx_->event();
      ck(cudaEventRecord(a, st_), "event");
    }
    const double t0 = diag_timing() ? now_ms() : 0.0;
    ck(f(), phase.c_str());
    if (diag_timing() && now_ms() - t0 > 0.5)
      fprintf(stderr, "hostslow launch %s %.3f ms\n", phase.c_str(), now_ms() - t0);
    ++ctx_->launches;
    if (rec) {
      b = ctx_->event();
      ck(cudaEventRecord(b, st_), "event");
      prof_->push_back({phase, a, b});
    }
  }

  // Y = X x_mode Q^T, Q is I x m column-major (already "bt" format)
  DevBuf ttm(const double* x, const std::vector<size_t>& dims, size_t mode, const double* q,
             size_t m, const std::string& phase = "ttm") {
    std::vector<size_t> od = dims;
    od[mode] = m;
    DevBuf y(prod(od), st_);
    launch(phase, [&] { return lmra_dev::launch_ttm(x, view_of(dims, mode), q, (int)m, y.get(), st_); });
    return y;
  }

  // Mode-0 contraction of a tensor whose canonical mode-0 column norms w are known: on the
  // int8 tensor cores (ttm_i8.cu, ~1e-13 relative) when the shape allows, else the DMMA TTM.
  // LMRA_TTM_I8=0 forces the DMMA path.
  // Per-column exponents handed from one int8 contraction to the next: after a mode-0
  // contraction that wrote them, fexp holds the max exponent of every mode-1 fibre of its
  // output, which a following mode-1 contraction uses as its fixed-point scales.
  struct I8Chain {
    DevBuf fexp;
    bool ready = false;
  };

  // Y = X x_mode Q^T.  On the int8 tensor cores when the scales are known: mode 0 with the
  // canonical column norms w, or mode 1 right after such a contraction (chain); the fp64 DMMA
  // product otherwise.  next_mode1: the following contraction is mode 1 of the result.
  DevBuf ttm_mode0(const double* x, const std::vector<size_t>& dims, size_t mode, const double* q,
                   size_t m, const double* w, const std::string& phase, I8Chain* chain = nullptr,
                   bool next_mode1 = false) {
    const bool enabled = ttm_i8_on();
    const size_t total = prod(dims);
    std::vector<size_t> od = dims;
    od[mode] = m;
    if (enabled && mode == 1 && chain && chain->ready && dims.size() >= 2) {
      chain->ready = false;
      const size_t R = dims[0], K = dims[1], O = total / (R * K);
      if (lmra_dev::ttm_i8_inner_supported((long long)R, (long long)K, (long long)O, (int)m, x)) {
        DevBuf y(prod(od), st_);
        DevBuf work((lmra_dev::ttm_i8_workspace_bytes((long long)K, (int)m) + 7) / 8, st_);
        const int* fe = reinterpret_cast<const int*>(chain->fexp.get());
        launch(phase + "_i8", [&] {
          return lmra_dev::launch_ttm_i8_inner(x, (long long)R, (long long)K, (long long)O, q, (int)m, fe,
                                               y.get(), work.get(), st_);
        });
        return y;
      }
    }
    if (chain) chain->ready = false;
    const size_t K = dims[0], J = total / K;
    if (mode != 0 || !w || !enabled || !lmra_dev::ttm_i8_supported((long long)K, (long long)J, (int)m, x))
      return ttm(x, dims, mode, q, m, phase);
    DevBuf y(prod(od), st_);
    DevBuf work((lmra_dev::ttm_i8_workspace_bytes((long long)K, (int)m) + 7) / 8, st_);
    int* fexp = nullptr;
    long long I1 = 0;
    if (chain && next_mode1 && dims.size() >= 2 && dims[1] > 0) {
      I1 = (long long)dims[1];
      const size_t n = m * (J / dims[1]);
      chain->fexp = DevBuf((n + 1) / 2, st_);
      fexp = reinterpret_cast<int*>(chain->fexp.get());
      ck(cudaMemsetAsync(fexp, 0x80, n * sizeof(int), st_), "memset");  // INT_MIN-like
    }
    launch(phase + "_i8", [&] {
      return lmra_dev::launch_ttm_i8(x, (long long)K, (long long)J, q, (int)m, w, y.get(), work.get(), st_,
                                     fexp, I1);
    });
    if (fexp) chain->ready = true;
    return y;
  }

  // c = (A A^T)^q G on the mode-`mode` unfolding view of a; c (I x s) in/out.  ga: A is the
  // gathered, scaled columns of a (AMM, Strategy A only), read in place
  void gram_power(const double* a, ModeView v, DevBuf& c, size_t s, int q, int strategy,
                  lmra_dev::Gather ga = lmra_dev::Gather{}) {
    const size_t I = (size_t)v.I, J = (size_t)(v.inner * v.outer);
    lmra_dev::GramPlan plan = lmra_dev::plan_gram(v, ctx_->num_sms);
    if (strategy == 0) {  // linalg.cpp:70-74, Strategy A
      DevBuf h(J * s, st_);
      DevBuf zpart((size_t)plan.nsplit * I * s, st_);
      for (int k = 0; k < q; ++k) {
        launch("power_half", [&] { return lmra_dev::launch_ttm(a, v, c.get(), (int)s, h.get(), st_, ga); });
        launch("power_gram", [&] {
          return lmra_dev::launch_gram(a, v, h.get(), (int)s, zpart.get(), plan, c.get(), st_, ga);
        });
      }
    } else {  // linalg.cpp:76-77, Strategy B: gram = A A^T once, then c = gram * c
      DevBuf gram(I * I, st_), gramt(I * I, st_);
      DevBuf zpart((size_t)plan.nsplit * I * I, st_);
      launch("power_gram", [&] {
        return lmra_dev::launch_gram(a, v, a, (int)I, zpart.get(), plan, gram.get(), st_);
      });
      launch("transpose", [&] {
        return lmra_dev::launch_transpose(gram.get(), (long long)I, (long long)I, gramt.get(), st_);
      });
      ModeView cv{1, (long long)I, (long long)s};
      for (int k = 0; k < q; ++k) {
        DevBuf nc(I * s, st_);
        launch("power_half", [&] {
          return lmra_dev::launch_ttm(c.get(), cv, gramt.get(), (int)I, nc.get(), st_);
        });
        c = std::move(nc);
      }
    }
  }

  DevBuf orth(const double* c, size_t I, size_t s, size_t mu, int* status) {
    if (s > (size_t)lmra_dev::kMaxWidth) return orth_wide(c, I, s, mu);
    DevBuf u(I * mu, st_);
    DevBuf work(lmra_dev::orth_workspace_doubles((long long)I, (int)s), st_);
    launch("orth", [&] {
      return lmra_dev::launch_orth(c, (long long)I, (int)s, (int)mu, u.get(), work.get(), status, st_);
    });
    return u;
  }

  // Sketches wider than the register-resident orthonormalisation (s > 64: the reference accepts
  // any s = min(mu + p, I_n), tucker.cpp:34-35): thin SVD of the I x s sketch by cuSOLVER dgesvd
  // (U of C directly, I >= s) + the sign rule.  Off every BASELINE configuration (s <= 60);
  // synchronous, so the shared cuSOLVER handle is idle before the next mode uses it.
  DevBuf orth_wide(const double* c, size_t I, size_t s, size_t mu) {
    const auto& cs = lmra_host::cusolver();
    if (!ctx_->cusolver) {
      cusolver_ok(cs.Create(&ctx_->cusolver), "cusolverDnCreate");
      if (cs.SetDeterministicMode) cs.SetDeterministicMode(ctx_->cusolver, CUSOLVER_DETERMINISTIC_RESULTS);
    }
    cusolver_ok(cs.SetStream(ctx_->cusolver, st_), "cusolverDnSetStream");
    if (I > (size_t)INT32_MAX) throw std::invalid_argument("sketch too tall for dgesvd");
    const int iI = (int)I, is = (int)s;
    DevBuf a(I * s, st_), uf(I * s, st_), sv(s, st_), rw(s, st_), info(1, st_), u(I * mu, st_);
    ck(cudaMemcpyAsync(a.get(), c, I * s * sizeof(double), cudaMemcpyDeviceToDevice, st_), "copy");
    ck(cudaMemsetAsync(info.get(), 0, sizeof(double), st_), "memset");
    int lw = 0;
    cusolver_ok(cs.Dgesvd_bufferSize(ctx_->cusolver, iI, is, &lw), "dgesvd_bufferSize");
    DevBuf w((size_t)std::max(lw, 1), st_);
    int* dinfo = reinterpret_cast<int*>(info.get());
    cusolver_ok(cs.Dgesvd(ctx_->cusolver, 'S', 'N', iI, is, a.get(), iI, sv.get(), uf.get(), iI, nullptr, 1, w.get(),
                          lw, rw.get(), dinfo),
                "dgesvd");
    ck(cudaMemcpyAsync(u.get(), uf.get(), I * mu * sizeof(double), cudaMemcpyDeviceToDevice, st_), "copy");
    launch("orth", [&] { return lmra_dev::launch_signfix_columns(u.get(), (long long)I, (int)I, (int)mu, st_); });
    int hinfo = 0;
    ck(cudaMemcpyAsync(&hinfo, dinfo, sizeof(int), cudaMemcpyDeviceToHost, st_), "D2H");
    ck(cudaStreamSynchronize(st_), "sync");
    if (hinfo > 0) throw std::runtime_error("thin_svd: SVD iteration did not converge");
    if (hinfo < 0) throw CudaError("cuSOLVER: illegal argument " + std::to_string(-hinfo));
    return u;
  }
  static void cusolver_ok(cusolverStatus_t st, const char* what) {
    if (st != CUSOLVER_STATUS_SUCCESS) throw CudaError(std::string(what) + ": cuSOLVER status " + std::to_string((int)st));
  }

  // qr_project_extract (linalg.cpp:89-99) for mode n of the tensor x: Q = thin_qr(C).Q,
  // P = X x_n Q^T (the projected unfolding Q^T A_(n), formed in place on the mode view),
  // U1 = top-mu left singular vectors of P_(n) (s x J) with the sign rule -- through the R
  // factor of P_(n)^T when J >= s (P_(n) = R^T Q2^T, so U of R^T = U of P_(n)) -- and the
  // factor Q U1.  P and U1 are kept: X x_n (Q U1)^T = P x_n U1^T, so the following shrink /
  // core contraction of this mode reads P (s rows) instead of the tensor.
  struct QrProxy {
    DevBuf f, p, u1;
  };
  QrProxy qr_extract(const double* x, const std::vector<size_t>& dims, size_t n, const double* c, size_t s,
                     size_t mu, int* status) {
    const size_t I = dims[n];
    const ModeView v = view_of(dims, n);
    const size_t J = (size_t)(v.inner * v.outer);
    QrProxy out;
    DevBuf q(I * s, st_);
    {
      DevBuf w(lmra_dev::thin_q_workspace_doubles((long long)I, (int)s), st_);
      launch("qr_thin_q", [&] { return lmra_dev::launch_thin_q(c, (long long)I, (int)s, q.get(), w.get(), st_); });
    }
    out.p = ttm(x, dims, n, q.get(), s, "qr_project");
    DevBuf pt(J * s, st_);
    launch("qr_unfold", [&] {
      return lmra_dev::launch_unfold_t(out.p.get(), v.inner, (long long)s, v.outer, pt.get(), st_);
    });
    if (J >= s) {
      DevBuf rr(s * s, st_), l(s * s, st_);
      DevBuf w(lmra_dev::r_factor_workspace_doubles((long long)J, (int)s), st_);
      launch("qr_r_factor", [&] {
        return lmra_dev::launch_r_factor(pt.get(), (long long)J, (int)s, rr.get(), w.get(), st_);
      });
      launch("transpose", [&] { return lmra_dev::launch_transpose(rr.get(), (long long)s, (long long)s, l.get(), st_); });
      out.u1 = orth(l.get(), s, s, mu, status);
    } else {  // P_(n) is itself tall (s x J, J < s)
      DevBuf pn(s * J, st_);
      launch("transpose", [&] { return lmra_dev::launch_transpose(pt.get(), (long long)J, (long long)s, pn.get(), st_); });
      out.u1 = orth(pn.get(), s, J, mu, status);
    }
    out.f = DevBuf(I * mu, st_);
    launch("qr_factor", [&] {
      return lmra_dev::launch_ttm(q.get(), ModeView{(long long)I, (long long)s, 1}, out.u1.get(), (int)mu,
                                  out.f.get(), st_);
    });
    return out;
  }

  DevBuf upload(const double* h, size_t n) {
    DevBuf d(n, st_);
    ck(cudaMemcpyAsync(d.get(), h, n * sizeof(double), cudaMemcpyHostToDevice, st_), "H2D");
    return d;
  }

  lmra_context* ctx_;
  cudaStream_t st_;
  std::vector<PhaseRec>* prof_;
};

struct RunInputs {
  int alg;
  const double* x;  // device
  std::vector<size_t> dims;
  lmra_host::Config cfg;
  const lmra_overrides* ov;
};

// Per-mode factor: Omega -> (optional AMM sampling) -> power scheme -> orthonormalise.
struct ModeFactor {
  DevBuf q;
};

void run_algorithm_impl(lmra_context* ctx, const RunInputs& in, lmra_result* res) {
  using namespace lmra_host;
  const double t0 = now_ms();
  std::vector<PhaseRec> prof;
  ctx->next_event = 0;
  Engine eng(ctx, ctx->profile ? &prof : nullptr);
  cudaStream_t st = ctx->stream;
  const auto& cfg = in.cfg;
  const size_t N = in.dims.size();
  for (size_t d : in.dims)
    if (d == 0) throw std::invalid_argument("tensor dimension must be positive");
  Resolved r = resolve(in.dims, cfg);
  const bool amm = in.alg == LMRA_ALG4 || in.alg == LMRA_ALG5;
  const bool qr = in.alg == LMRA_ALG6 || in.alg == LMRA_ALG7;
  const bool sequential = in.alg == LMRA_ALG2 || in.alg == LMRA_ALG5 || in.alg == LMRA_ALG7;
  std::vector<size_t> t_flat;
  if (amm && !sequential) t_flat = amm_sample_counts(in.dims, cfg, false);
  if (amm && sequential && !cfg.t_samples.empty() && cfg.t_samples.size() != N)
    throw std::invalid_argument("sample count override length must equal tensor order");
  for (size_t n = 0; n < N; ++n)  // (alg1/2/4/5 take wide sketches through Engine::orth_wide)
    if (qr && r.sketch[n] > (size_t)lmra_dev::kMaxWidth)
      throw std::invalid_argument("sketch width mu_n + oversampling above 64 is not supported by the QR-proxy variants");

  res->omega.assign(N, {});
  res->om_rows.assign(N, 0);
  res->om_cols.assign(N, 0);
  res->idx.assign(N, {});
  res->scales.assign(N, {});
  res->norms.assign(N, {});
  res->factors.assign(N, nullptr);
  res->f_rows.assign(N, 0);
  res->f_cols.assign(N, 0);

  cudaEvent_t ev0, ev1;
  ck(cudaEventCreate(&ev0), "event");
  ck(cudaEventCreate(&ev1), "event");
  ck(cudaEventRecord(ev0, st), "event");
  const long long launches0 = lmra_dev::g_kernel_launches;

  // Omega for every mode (gaussian_stream = {seed, n+1}, sketching.cpp:164-173) is data
  // independent: a host thread draws it into pinned memory while the GPU already runs
  // the column norms / sampling chains.
  std::vector<size_t> om_off(N + 1, 0);
  for (size_t n = 0; n < N; ++n) {
    res->om_rows[n] = in.dims[n];
    res->om_cols[n] = r.sketch[n];
    om_off[n + 1] = om_off[n] + in.dims[n] * r.sketch[n];
  }
  double* om_pin = ctx->pinned_buffer(om_off[N]);
  // drawn in chunks by the persistent host worker pool (jump-ahead: bit-identical to the
  // sequential stream), overlapping the device's norm pass / sampling chains
  lmra_host::TaskGroup omega_tasks;
  const double tr0 = now_ms();
  bool rng_done = false;
  std::vector<std::function<void()>> omega_jobs;
  // chunk size: ~2 jobs per pool thread, 256..4096 normals (even: chunks start on a
  // Box-Muller pair).  Small draws (cfg1: 3 x 3000 normals) split finely: at ~30 ns a normal,
  // one 4096-normal job per mode kept the device idle ~0.09 ms before the first power step.
  const size_t kChunk = std::min<size_t>(
      4096, std::max<size_t>(256, (om_off[N] / (2 * (size_t)lmra_host::host_threads()) + 1) & ~size_t(1)));
  for (size_t n = 0; n < N; ++n) {
    const size_t cnt = om_off[n + 1] - om_off[n];
    double* dst = om_pin + om_off[n];
    if (in.ov && in.ov->omega && in.ov->omega[n]) {
      std::memcpy(dst, in.ov->omega[n], sizeof(double) * cnt);
      continue;
    }
    const uint64_t seed = cfg.seed, stream = n + 1;
    for (size_t b0 = 0; b0 < cnt; b0 += kChunk) {
      const size_t e0 = std::min(cnt, b0 + kChunk);
      omega_jobs.emplace_back([=] { fill_normals_range(seed, stream, dst, b0, e0); });
    }
  }
  omega_tasks.run_batch(std::move(omega_jobs));
  auto omega_ready = [&] {
    omega_tasks.wait();
    if (!rng_done) {
      res->t_rng = now_ms() - tr0;
      rng_done = true;
      if (diag_timing()) fprintf(stderr, "hostmark omega drawn %.4f ms (dispatched at %.4f)\n", now_ms() - t0, tr0 - t0);
    }
  };

  // per-mode device status words: [0, N) orth convergence, [N, 2N) sampler flags
  DevBuf status(N, st);
  ck(cudaMemsetAsync(status.get(), 0, N * sizeof(double), st), "memset");
  int* status_i = reinterpret_cast<int*>(status.get());
  // device-drawn samples / norms kept until the end of the run for the trace
  std::vector<DevBuf> d_idx(N), d_sc(N), d_w(N);
  std::vector<size_t> n_draws(N, 0);

  // phase 1 of a mode: the sampled columns (AMM only) -- norms + exact sampling chain
  auto sample_mode = [&](Engine& e, const double* x, const std::vector<size_t>& dims, size_t n,
                         size_t t_n) {
    if (!amm) return;
    cudaStream_t s_ = e.st_;
    const ModeView v = view_of(dims, n);
    const size_t J = (size_t)(v.inner * v.outer);
    const double ts0 = now_ms();
    size_t T;
    if (in.ov && in.ov->sample_idx && in.ov->sample_idx[n]) {  // parity overrides
      T = in.ov->n_samples[n];
      const int64_t* oi = in.ov->sample_idx[n];
      for (size_t j = 0; j < T; ++j)
        if (oi[j] < 0 || (size_t)oi[j] >= J) throw std::invalid_argument("sample index out of range");
      d_idx[n] = DevBuf(T + 1, s_);
      d_sc[n] = DevBuf(T, s_);
      ck(cudaMemcpyAsync(d_idx[n].get(), oi, T * sizeof(int64_t), cudaMemcpyHostToDevice, s_),
         "H2D idx");
      ck(cudaMemcpyAsync(d_sc[n].get(), in.ov->sample_scale[n], T * sizeof(double),
                         cudaMemcpyHostToDevice, s_),
         "H2D scales");
      ck(cudaStreamSynchronize(s_), "sync");  // caller's host arrays are only borrowed
    } else {
      T = t_n;
      if (T < 1) throw std::invalid_argument("randsample: L must be positive");
      d_idx[n] = DevBuf(T + 1, s_);
      d_sc[n] = DevBuf(T, s_);
      DevBuf p(J, s_), work(lmra_dev::sampler_workspace_doubles((long long)J), s_);
      if (!d_w[n].get()) {  // not already produced by the fused all-modes pass
        d_w[n] = DevBuf(J, s_);
        if (cfg.regime != kUniform)
          e.launch("norms", [&] { return lmra_dev::launch_column_sqnorms(x, v, d_w[n].get(), s_); });
      }
      e.launch("sampler", [&] {
        return lmra_dev::launch_sampler(
            d_w[n].get(), (long long)J, cfg.regime, cfg.beta, (long long)T, cfg.seed, N + n + 1,
            reinterpret_cast<long long*>(d_idx[n].get()), d_sc[n].get(), p.get(), work.get(),
            status_i + N + n, s_);
      });
    }
    n_draws[n] = T;
    res->t_sampling += now_ms() - ts0;
  };

  // phase 2 of a mode: Omega -> power scheme (on the unfolding or the sampled columns)
  // -> orthonormalised factor.  Omega must be drawn (omega_ready) before this.
  // Omega uploads: every mode's draw goes up in one copy on its own stream as soon as the
  // host thread is done (during the norm pass), instead of in stream order behind each
  // mode's sampling chain, where the copy sat on the critical path.
  std::vector<DevBuf> d_om(N);
  cudaEvent_t om_ready = nullptr;
  auto upload_omegas = [&] {
    omega_ready();
    if (om_ready) return;
    cudaStream_t cs = ctx->aux_stream(N);
    ck(cudaStreamWaitEvent(cs, ev0, 0), "wait");  // the run's start (stream-ordered arena)
    for (size_t n = 0; n < N; ++n) {
      const size_t cnt = om_off[n + 1] - om_off[n];
      d_om[n] = DevBuf(cnt, cs);
      ck(cudaMemcpyAsync(d_om[n].get(), om_pin + om_off[n], cnt * sizeof(double),
                         cudaMemcpyHostToDevice, cs), "H2D omega");
    }
    ck(cudaEventCreateWithFlags(&om_ready, cudaEventDisableTiming), "event");
    ck(cudaEventRecord(om_ready, cs), "event");
    if (diag_timing()) fprintf(stderr, "hostmark omega uploaded %.4f ms\n", now_ms() - t0);
  };
  struct EventGuard {
    cudaEvent_t& e;
    ~EventGuard() {
      if (e) cudaEventDestroy(e);
    }
  } om_guard{om_ready};

  // QR-proxy (alg6/alg7): the projected tensor P and U1 of a mode whose contraction reads P
  std::vector<Engine::QrProxy> qrp(N);
  // Split orthonormalisation (T-HOSVD, opt-in with LMRA_ORTH_SPLIT=1): each mode publishes its
  // sketch basis Q_C (I x s) before the s x s Jacobi, the core's long contractions run on Q_C
  // while the Jacobis finish, and the small rotations U_R'^T are applied to the s_0 x s_1 x ...
  // core at the end (X x_n Q^T = (X x_n Q_C^T) x_n U_R'^T, modes commute).  Parity-tested, but
  // measured slower on cfg4 (4.66-4.78 vs 4.61 ms): the int8 contraction runs power-capped, and
  // Jacobis beside it both slow it (1.48 -> 1.72-1.85 ms) and run ~2x slower themselves.
  struct SplitOrth {
    DevBuf qc, urs, work;
    cudaEvent_t basis = nullptr;
  };
  std::vector<SplitOrth> split(N);
  struct SplitGuard {
    std::vector<SplitOrth>& v;
    ~SplitGuard() {
      for (auto& so : v)
        if (so.basis) cudaEventDestroy(so.basis);
    }
  } split_guard{split};
  // default: on for T-HOSVD inputs of >= 2^27 elements (1 GB), whose first core contraction is
  // long enough to hide the first mode's Jacobi; LMRA_ORTH_SPLIT=0/1 forces it off/on
  bool split_orth = !sequential && !qr && prod(in.dims) >= (size_t(1) << 27);
  if (const char* e = getenv("LMRA_ORTH_SPLIT")) split_orth = !sequential && !qr && e[0] == '1';
  // only the mode the core contracts first is split (core_from_factors: ascending factor width,
  // stable); the later contractions wait for their modes' full factors, whose Jacobis finish
  // under the first contraction
  size_t split_mode = 0;
  if (split_orth) {
    std::vector<size_t> mus(N);
    for (size_t n = 0; n < N; ++n) mus[n] = std::min(r.mu[n], std::min(in.dims[n], r.sketch[n]));
    for (size_t n = 1; n < N; ++n)
      if (mus[n] < mus[split_mode]) split_mode = n;
  }
  // phase 2a: the sketch c (I x s) of mode n
  auto factor_power = [&](Engine& e, const double* x, const std::vector<size_t>& dims,
                          size_t n) -> DevBuf {
    cudaStream_t s_ = e.st_;
    const ModeView v = view_of(dims, n);
    const size_t I = dims[n], s = r.sketch[n];
    upload_omegas();
    ck(cudaStreamWaitEvent(s_, om_ready, 0), "wait omega");
    DevBuf c = std::move(d_om[n]);  // the sketch is formed in place
    c.rebind(s_);
    if (!amm) {
      e.gram_power(x, v, c, s, cfg.power, cfg.strategy);
    } else if (v.inner == 1 && cfg.strategy == 0 && I * n_draws[n] >= fused_gather_min()) {
      // large sampled matrix of contiguous fibres (cfg5 mode 0: 512 x 157287, 644 MB): the
      // power scheme reads the sampled columns in place instead of materialising C'
      // (saves C's write and one of its two reads per power step)
      const size_t T = n_draws[n];
      const lmra_dev::Gather ga{reinterpret_cast<const long long*>(d_idx[n].get()), d_sc[n].get()};
      e.gram_power(x, ModeView{1, (long long)I, (long long)T}, c, s, cfg.power, cfg.strategy, ga);
    } else {
      const size_t T = n_draws[n];
      DevBuf cp(I * T, s_);
      e.launch("gather", [&] {
        return lmra_dev::launch_gather(x, v, reinterpret_cast<const long long*>(d_idx[n].get()),
                                       d_sc[n].get(), (long long)T, cp.get(), s_);
      });
      const ModeView cv{1, (long long)I, (long long)T};
      e.gram_power(cp.get(), cv, c, s, cfg.power, cfg.strategy);
    }
    return c;
  };
  // phase 2b: the factor of mode n from its sketch c
  auto factor_orth = [&](Engine& e, const double* x, const std::vector<size_t>& dims, size_t n,
                         DevBuf& c) -> DevBuf {
    cudaStream_t s_ = e.st_;
    const ModeView v = view_of(dims, n);
    const size_t I = dims[n], s = r.sketch[n];
    if (qr) {  // tucker.cpp:431-434 / 447-450: mu capped at min(sketch width, unfolding columns)
      const size_t J = (size_t)(v.inner * v.outer);
      const size_t mu = std::min(r.mu[n], std::min(s, J));
      if (mu < r.mu[n])
        fprintf(stderr, "lmra: requested rank %zu exceeds matrix rank limit %zu, clamping\n", r.mu[n], mu);
      res->f_rows[n] = I;
      res->f_cols[n] = mu;
      qrp[n] = e.qr_extract(x, dims, n, c.get(), s, mu, status_i + n);
      return std::move(qrp[n].f);
    }
    const size_t mu = std::min(r.mu[n], std::min(I, s));  // top_left_vectors_clamped
    if (mu < r.mu[n])
      fprintf(stderr, "lmra: requested rank %zu exceeds matrix rank limit %zu, clamping\n",
              r.mu[n], mu);
    res->f_rows[n] = I;
    res->f_cols[n] = mu;
    if (split_orth && n == split_mode && dims == in.dims) {
      SplitOrth& so = split[n];
      so.work = DevBuf(lmra_dev::orth_split_workspace_doubles((long long)I, (int)s), s_);
      so.qc = DevBuf(I * s, s_);
      e.launch("orth_basis", [&] {
        return lmra_dev::launch_orth_basis(c.get(), (long long)I, (int)s, so.qc.get(), so.work.get(), s_);
      });
      ck(cudaEventCreateWithFlags(&so.basis, cudaEventDisableTiming), "event");
      ck(cudaEventRecord(so.basis, s_), "event");
      // the factor from the full Householder path (beside the contraction, off the critical path)
      // and its coefficients in the basis: the CholeskyQR basis serves the contraction only
      DevBuf u = e.orth(c.get(), I, s, mu, status_i + n);
      so.urs = DevBuf(s * mu, s_);
      e.launch("orth_coeffs", [&] {
        return lmra_dev::launch_basis_coeffs(so.qc.get(), (long long)I, (int)s, u.get(), (int)mu, so.urs.get(), s_);
      });
      return u;
    }
    return e.orth(c.get(), I, s, mu, status_i + n);
  };
  auto factor_mode = [&](Engine& e, const double* x, const std::vector<size_t>& dims,
                         size_t n) -> DevBuf {
    DevBuf c = factor_power(e, x, dims, n);
    return factor_orth(e, x, dims, n, c);
  };

  std::vector<DevBuf> factors(N);
  if (!sequential) {
    // modes are independent (run_modes, tucker.cpp:134-160): one stream per mode, so the
    // latency-bound sampling / power / orthonormalisation kernels of different modes
    // overlap; the core contraction joins them on the main stream
    const bool any_override = in.ov && in.ov->sample_idx;
    if (amm && cfg.regime != kUniform && N == 3 && !any_override) {
      // every mode samples from the same input: one read of X for all three norm vectors
      const long long I0 = in.dims[0], I1 = in.dims[1], I2 = in.dims[2];
      for (size_t n = 0; n < 3; ++n) d_w[n] = DevBuf(prod(in.dims) / in.dims[n], st);
      DevBuf nwork(lmra_dev::norms3_workspace_doubles(I0, I1, I2), st);
      eng.launch("norms", [&] {
        return lmra_dev::launch_norms3(in.x, I0, I1, I2, d_w[0].get(), d_w[1].get(), d_w[2].get(),
                                       nwork.get(), st);
      });
    }
    cudaEvent_t fork;
    ck(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming), "event");
    ck(cudaEventRecord(fork, st), "event");
    std::vector<Engine> engs;
    engs.reserve(N);
    // the mode core_from_factors contracts first (smallest factor width, stable) runs on the
    // high-priority stream
    size_t first_mode = 0;
    {
      std::vector<size_t> mus(N);
      for (size_t n = 0; n < N; ++n) mus[n] = std::min(r.mu[n], std::min(in.dims[n], r.sketch[n]));
      for (size_t n = 1; n < N; ++n)
        if (mus[n] < mus[first_mode]) first_mode = n;
    }
    static const bool prio = !(getenv("LMRA_STREAM_PRIORITY") && getenv("LMRA_STREAM_PRIORITY")[0] == '0');
    for (size_t n = 0; n < N; ++n) {
      // (not with the split orthonormalisation: measured on cfg4, 3.84 -> 3.90 ms with the split
      // mode's chain prioritised; cfg1 0.370 -> 0.351 ms)
      cudaStream_t sn = (prio && !split_orth && n == first_mode) ? ctx->hi_stream() : ctx->aux_stream(n);
      ck(cudaStreamWaitEvent(sn, fork, 0), "wait");
      engs.emplace_back(ctx, sn, ctx->profile == 1 ? &prof : nullptr);
    }
    for (size_t n = 0; n < N; ++n) sample_mode(engs[n], in.x, in.dims, n, amm ? t_flat[n] : 0);
    upload_omegas();
    // launched phase by phase across the modes (every mode's power scheme, then every mode's
    // orthonormalisation), so the modes' chains start together instead of one host launch
    // sequence (~20 us) apart
    std::vector<DevBuf> sketches(N);
    for (size_t n = 0; n < N; ++n) sketches[n] = factor_power(engs[n], in.x, in.dims, n);
    if (diag_timing()) fprintf(stderr, "hostmark power launched %.4f ms\n", now_ms() - t0);
    for (size_t n = 0; n < N; ++n) factors[n] = factor_orth(engs[n], in.x, in.dims, n, sketches[n]);
    // each contraction of the core waits only for its own mode's factor: the first one
    // (the long int8 / DMMA pass over the tensor) starts as soon as that mode's chain is done,
    // while the other modes' orthonormalisations finish under it
    std::vector<cudaEvent_t> mode_done(N);
    for (size_t n = 0; n < N; ++n) {
      ck(cudaEventCreateWithFlags(&mode_done[n], cudaEventDisableTiming), "event");
      ck(cudaEventRecord(mode_done[n], engs[n].st_), "event");
    }
    struct EventsGuard {
      std::vector<cudaEvent_t>& v;
      ~EventsGuard() {
        for (cudaEvent_t e : v) cudaEventDestroy(e);
      }
    } mode_done_guard{mode_done};
    cudaEventDestroy(fork);
    // core_from_factors (tucker.cpp:81-92): ascending factor width, stable
    std::vector<size_t> idx(N);
    std::iota(idx.begin(), idx.end(), size_t{0});
    std::stable_sort(idx.begin(), idx.end(),
                     [&](size_t a, size_t b) { return res->f_cols[a] < res->f_cols[b]; });
    if (qr)  // only the first contraction reads a projected tensor
      for (size_t k = 1; k < idx.size(); ++k) qrp[idx[k]] = Engine::QrProxy{};
    std::vector<size_t> cur = in.dims;
    DevBuf t;
    const double* src = in.x;
    int step = 0;
    // the first contraction reads the input, whose mode-0 norms the sampler already has
    const double* w0 = (amm && cfg.regime != kUniform && d_w[0].get()) ? d_w[0].get() : nullptr;
    Engine::I8Chain chain;
    if (split_orth) {  // SMs for the orthonormalisations that run beside the first contraction
      int jac = 0;  // every mode's Jacobi core (2-CTA clusters if s >= 48), the split mode's included
      for (size_t n = 0; n < N; ++n) jac += r.sketch[n] >= 48 ? 2 : 1;
      lmra_dev::g_i8_reserved_sms = jac + 1;
    }
    for (size_t k = 0; k < idx.size(); ++k) {
      const size_t n = idx[k];
      const bool next1 = k + 1 < idx.size() && idx[k + 1] == 1;
      if (split_orth && k == 0) {  // the contraction with the basis Q_C, as soon as it exists
        if (n != split_mode) throw std::logic_error("split orthonormalisation: contraction order");
        ck(cudaStreamWaitEvent(st, split[n].basis, 0), "wait");
        const size_t sn = r.sketch[n];
        DevBuf y = eng.ttm_mode0(src, cur, n, split[n].qc.get(), sn, src == in.x ? w0 : nullptr,
                                 "core_ttm" + std::to_string(step++), &chain, next1);
        cur[n] = sn;
        t = std::move(y);
        src = t.get();
        continue;
      }
      ck(cudaStreamWaitEvent(st, mode_done[n], 0), "wait");
      if (qr && k == 0) {  // X x_n (Q U1)^T = P x_n U1^T: read the projected tensor
        std::vector<size_t> pd = cur;
        pd[n] = r.sketch[n];
        t = eng.ttm(qrp[n].p.get(), pd, n, qrp[n].u1.get(), res->f_cols[n], "core_ttm" + std::to_string(step++));
        cur[n] = res->f_cols[n];
        src = t.get();
        continue;
      }
      DevBuf y = eng.ttm_mode0(src, cur, n, factors[n].get(), res->f_cols[n], src == in.x ? w0 : nullptr,
                               "core_ttm" + std::to_string(step++), &chain, next1);
      cur[n] = res->f_cols[n];
      t = std::move(y);
      src = t.get();
    }
    lmra_dev::g_i8_reserved_sms = 0;
    if (split_orth) {  // the rotation U_R'^T of the split mode, after its Jacobi
      const size_t n = idx[0];
      ck(cudaStreamWaitEvent(st, mode_done[n], 0), "wait");
      DevBuf y = eng.ttm(src, cur, n, split[n].urs.get(), res->f_cols[n], "core_rot");
      cur[n] = res->f_cols[n];
      t = std::move(y);
      src = t.get();
    }
    res->core_dims = cur;
    res->core = t.detach();
  } else {
    std::vector<size_t> cur = in.dims;
    DevBuf work;
    const double* src = in.x;
    Engine::I8Chain chain;
    // (no split orthonormalisation here: measured on cfg5, the first shrink with the sketch basis
    // beside the Jacobi, then the s x mu rotation and the mode-1 column exponents, tied the plain
    // order -- 5.37 vs 5.35 ms: the Jacobi beside the power-capped int8 shrink ran 0.35 -> 0.61 ms)
    for (size_t oi = 0; oi < r.order.size(); ++oi) {
      const size_t n = r.order[oi];
      const bool next1 = oi + 1 < r.order.size() && r.order[oi + 1] == 1;
      size_t t_n = 0;
      if (amm) {
        const size_t cols = prod(cur) / cur[n];
        t_n = cfg.t_samples.empty() ? samples_from_alpha(cfg.alpha, cols) : cfg.t_samples[n];
        if (t_n < 1) throw std::invalid_argument("sample counts must be positive");
      }
      sample_mode(eng, src, cur, n, t_n);
      upload_omegas();
      factors[n] = factor_mode(eng, src, cur, n);
      if (qr) {  // shrink through the projected tensor: P x_n U1^T
        std::vector<size_t> pd = cur;
        pd[n] = r.sketch[n];
        DevBuf y = eng.ttm(qrp[n].p.get(), pd, n, qrp[n].u1.get(), res->f_cols[n], "shrink_ttm_m" + std::to_string(n));
        qrp[n] = Engine::QrProxy{};
        cur[n] = res->f_cols[n];
        work = std::move(y);
        src = work.get();
        continue;
      }
      const double* w0 =
          (amm && cfg.regime != kUniform && src == in.x && d_w[n].get() && !(in.ov && in.ov->sample_idx))
              ? d_w[n].get() : nullptr;
      DevBuf y = eng.ttm_mode0(src, cur, n, factors[n].get(), res->f_cols[n], w0,
                               "shrink_ttm_m" + std::to_string(n), &chain, next1);
      cur[n] = res->f_cols[n];
      work = std::move(y);
      src = work.get();
    }
    res->core_dims = cur;
    res->core = work.detach();
  }
  for (size_t n = 0; n < N; ++n) {  // copies on the main stream (ordered after every mode's join)
    factors[n].rebind(st);
    res->factors[n] = factors[n].detach();
  }

  ck(cudaEventRecord(ev1, st), "event");
  std::vector<int> stat(2 * N);
  ck(cudaMemcpyAsync(stat.data(), status.get(), 2 * N * sizeof(int), cudaMemcpyDeviceToHost, st),
     "D2H status");
  // trace of the draws (host copies) -- off for throughput runs (lmra_context_set_trace)
  if (ctx->keep_trace) {
    for (size_t n = 0; n < N; ++n) res->omega[n].assign(om_pin + om_off[n], om_pin + om_off[n + 1]);
    for (size_t n = 0; n < N; ++n) {
      if (n_draws[n] && d_idx[n].get()) {
        res->idx[n].resize(n_draws[n]);
        res->scales[n].resize(n_draws[n]);
        ck(cudaMemcpyAsync(res->idx[n].data(), d_idx[n].get(), n_draws[n] * sizeof(int64_t),
                           cudaMemcpyDeviceToHost, st),
           "D2H idx");
        ck(cudaMemcpyAsync(res->scales[n].data(), d_sc[n].get(), n_draws[n] * sizeof(double),
                           cudaMemcpyDeviceToHost, st),
           "D2H scales");
      }
      if (d_w[n].get() && cfg.regime != kUniform) {
        res->norms[n].resize(d_w[n].size());
        ck(cudaMemcpyAsync(res->norms[n].data(), d_w[n].get(), d_w[n].size() * sizeof(double),
                           cudaMemcpyDeviceToHost, st),
           "D2H norms");
      }
    }
  }
  ck(cudaStreamSynchronize(st), "sync");
  float dev_ms = 0;
  ck(cudaEventElapsedTime(&dev_ms, ev0, ev1), "event time");
  if (getenv("LMRA_TIMELINE") && getenv("LMRA_TIMELINE")[0] == '1' && !prof.empty()) {
    float lead = 0;  // run start -> first phase (host RNG, uploads, launch latency)
    ck(cudaEventElapsedTime(&lead, ev0, prof[0].a), "event time");
    fprintf(stderr, "timeline lead-in %9.4f ms, run %9.4f ms\n", lead, dev_ms);
  }
  cudaEventDestroy(ev0);
  cudaEventDestroy(ev1);
  // the reference's exception surface, in its order of checks (sketching.cpp / tucker.cpp)
  for (size_t n = 0; n < N; ++n) {
    const int f = stat[N + n];
    if (f & 1) throw std::invalid_argument("probability weights must be nonnegative");
    if (f & 32) throw std::invalid_argument("nearly-optimal mixture weight must lie in (0, 1]");
    if (f & 2) throw std::invalid_argument("cannot normalize an all-zero distribution");
    if (f & 4) throw std::invalid_argument("probability weights must sum to one");
    if (f & 8) throw std::invalid_argument("randsample: all-zero distribution");
    if (f & 16) ++res->sampler_fallbacks;
    if (f & 64) throw std::runtime_error("sampler: uniform segment table overflow");
  }
  for (size_t n = 0; n < N; ++n)
    if (stat[n] != 0) throw std::runtime_error("thin_svd: SVD iteration did not converge");
  res->t_device = dev_ms;
  res->launches = (double)(lmra_dev::g_kernel_launches - launches0);
  static const bool timeline = getenv("LMRA_TIMELINE") && getenv("LMRA_TIMELINE")[0] == '1';
  if (timeline && !prof.empty()) {  // diagnostics: phase start/end relative to the first phase
    for (const PhaseRec& p : prof) {
      float a = 0, b = 0;
      ck(cudaEventElapsedTime(&a, prof[0].a, p.a), "event time");
      ck(cudaEventElapsedTime(&b, prof[0].a, p.b), "event time");
      fprintf(stderr, "timeline %-16s %9.4f %9.4f\n", p.name.c_str(), a, b);
    }
  }
  for (const PhaseRec& p : prof) {
    float ms = 0;
    ck(cudaEventElapsedTime(&ms, p.a, p.b), "event time");
    auto it = std::find_if(res->phases.begin(), res->phases.end(),
                           [&](const lmra_result::Phase& q) { return q.name == p.name; });
    if (it == res->phases.end()) {
      res->phases.push_back({p.name, 0.0, 0});
      it = res->phases.end() - 1;
    }
    it->ms += ms;
    it->count += 1;
  }
  res->t_total = now_ms() - t0;
}

// ------------------------------------------------------------------ sharded (multi-GPU) run
// The tensor is sharded along its LAST mode: rank R holds the contiguous slab
// i_{N-1} in [start_R, start_R + count_R) (lmra_shard_range), dims[] are global.
//  * modes n < N-1: an unfolding column j = (i, o) has i_{N-1} inside o, so each rank owns a
//    contiguous range of columns: norms are local and exact (canonical order) and are
//    all-gathered, so every rank runs the identical sampling chain; sampled fibres are
//    gathered by their owner (others contribute zero columns); the power scheme's Gram
//    partials (I_n x s) are all-reduced; the contraction stays local (still sharded).
//  * mode N-1: fibres are split by rows: local norm partials are all-reduced, half-products
//    (T x s or J x s) are all-reduced, the sketch's row blocks are all-gathered; the
//    contraction of this mode produces a partial that is all-reduced, after which the tensor
//    is replicated and the remaining work is identical on every rank.
// Every rank computes bitwise-identical factors (identical reduced inputs, deterministic
// kernels), so no broadcast is needed.
void run_sharded_impl(lmra_context* ctx, const RunInputs& in, lmra_result* res) {
  using namespace lmra_host;
  const double t0 = now_ms();
  std::vector<PhaseRec> prof;
  ctx->next_event = 0;
  Engine eng(ctx, ctx->profile ? &prof : nullptr);
  cudaStream_t st = ctx->stream;
  Comm& comm = *ctx->comm;
  const int P = comm.nranks, R = comm.rank;
  const auto& cfg = in.cfg;
  const size_t N = in.dims.size();
  for (size_t d : in.dims)
    if (d == 0) throw std::invalid_argument("tensor dimension must be positive");
  Resolved r = resolve(in.dims, cfg);
  const bool amm = in.alg == LMRA_ALG4 || in.alg == LMRA_ALG5;
  const bool sequential = in.alg == LMRA_ALG2 || in.alg == LMRA_ALG5;
  std::vector<size_t> t_flat;
  if (amm && !sequential) t_flat = amm_sample_counts(in.dims, cfg, false);
  if (amm && sequential && !cfg.t_samples.empty() && cfg.t_samples.size() != N)
    throw std::invalid_argument("sample count override length must equal tensor order");
  const size_t L = in.dims[N - 1];
  if (L < (size_t)P) throw std::invalid_argument("last mode extent is smaller than the rank count");
  std::vector<size_t> sh0(P), shc(P);
  for (int q = 0; q < P; ++q) {
    shard_bounds(L, (size_t)P, (size_t)q, &sh0[q], &shc[q]);
  }
  const size_t s0 = sh0[R], c0 = shc[R], cmax = *std::max_element(shc.begin(), shc.end());

  res->omega.assign(N, {});
  res->om_rows.assign(N, 0);
  res->om_cols.assign(N, 0);
  res->idx.assign(N, {});
  res->scales.assign(N, {});
  res->norms.assign(N, {});
  res->factors.assign(N, nullptr);
  res->f_rows.assign(N, 0);
  res->f_cols.assign(N, 0);

  cudaEvent_t ev0, ev1;
  ck(cudaEventCreate(&ev0), "event");
  ck(cudaEventCreate(&ev1), "event");
  ck(cudaEventRecord(ev0, st), "event");
  const long long launches0 = lmra_dev::g_kernel_launches;

  std::vector<size_t> om_off(N + 1, 0);
  for (size_t n = 0; n < N; ++n) {
    res->om_rows[n] = in.dims[n];
    res->om_cols[n] = r.sketch[n];
    om_off[n + 1] = om_off[n] + in.dims[n] * r.sketch[n];
  }
  double* om_pin = ctx->pinned_buffer(om_off[N]);
  {
    const double tr0 = now_ms();
    for (size_t n = 0; n < N; ++n) {
      const size_t cnt = om_off[n + 1] - om_off[n];
      if (in.ov && in.ov->omega && in.ov->omega[n])
        std::memcpy(om_pin + om_off[n], in.ov->omega[n], sizeof(double) * cnt);
      else
        fill_normals(cfg.seed, n + 1, om_pin + om_off[n], cnt, host_threads());
    }
    res->t_rng = now_ms() - tr0;
  }
  DevBuf status(N, st);
  ck(cudaMemsetAsync(status.get(), 0, N * sizeof(double), st), "memset");
  int* status_i = reinterpret_cast<int*>(status.get());
  std::vector<DevBuf> d_idx(N), d_sc(N), d_w(N);
  std::vector<size_t> n_draws(N, 0);

  std::vector<size_t> gdims = in.dims;  // global dims of the current tensor
  bool sharded = true;                  // current tensor = this rank's slab of mode N-1
  const double* cur = in.x;
  DevBuf curbuf;
  auto ldims = [&]() {
    std::vector<size_t> d = gdims;
    if (sharded) d[N - 1] = c0;
    return d;
  };
  auto rows_of = [&](const double* m, size_t I, size_t cols, size_t start, size_t cnt) {
    DevBuf out(cnt * cols, st);  // rows [start, start+cnt) of an I x cols column-major matrix
    ck(cudaMemcpy2DAsync(out.get(), cnt * sizeof(double), m + start, I * sizeof(double),
                         cnt * sizeof(double), cols, cudaMemcpyDeviceToDevice, st),
       "rows");
    return out;
  };
  auto gather_rows = [&](const double* local, size_t cols, double* full, size_t I) {
    // all-gather row blocks (c_q x cols each, padded to cmax) into full (I x cols)
    DevBuf send(cmax * cols, st), recv((size_t)P * cmax * cols, st);
    ck(cudaMemsetAsync(send.get(), 0, cmax * cols * sizeof(double), st), "memset");
    ck(cudaMemcpy2DAsync(send.get(), cmax * sizeof(double), local, c0 * sizeof(double),
                         c0 * sizeof(double), cols, cudaMemcpyDeviceToDevice, st),
       "pack");
    comm.allgather(send.get(), recv.get(), cmax * cols, st);
    for (int q = 0; q < P; ++q)
      ck(cudaMemcpy2DAsync(full + sh0[q], I * sizeof(double), recv.get() + (size_t)q * cmax * cols,
                           cmax * sizeof(double), shc[q] * sizeof(double), cols,
                           cudaMemcpyDeviceToDevice, st),
         "unpack");
  };
  // the sampling chain of mode n (no collectives) on engine e's stream
  auto run_sampler = [&](Engine& e, size_t n, const double* w, size_t J, size_t T) -> size_t {
    cudaStream_t ss = e.st_;
    if (in.ov && in.ov->sample_idx && in.ov->sample_idx[n]) {  // parity overrides (global idx)
      T = in.ov->n_samples[n];
      const int64_t* oi = in.ov->sample_idx[n];
      for (size_t j = 0; j < T; ++j)
        if (oi[j] < 0 || (size_t)oi[j] >= J) throw std::invalid_argument("sample index out of range");
      d_idx[n] = DevBuf(T + 1, ss);
      d_sc[n] = DevBuf(T, ss);
      ck(cudaMemcpyAsync(d_idx[n].get(), oi, T * sizeof(int64_t), cudaMemcpyHostToDevice, ss), "H2D idx");
      ck(cudaMemcpyAsync(d_sc[n].get(), in.ov->sample_scale[n], T * sizeof(double),
                         cudaMemcpyHostToDevice, ss), "H2D scales");
      ck(cudaStreamSynchronize(ss), "sync");
      n_draws[n] = T;
      return T;
    }
    if (T < 1) throw std::invalid_argument("randsample: L must be positive");
    d_idx[n] = DevBuf(T + 1, ss);
    d_sc[n] = DevBuf(T, ss);
    DevBuf p(J, ss), work(lmra_dev::sampler_workspace_doubles((long long)J), ss);
    DevBuf dummy;
    if (!w) {  // uniform regime never reads w
      dummy = DevBuf(J, ss);
      w = dummy.get();
    }
    e.launch("sampler", [&] {
      return lmra_dev::launch_sampler(w, (long long)J, cfg.regime, cfg.beta, (long long)T,
                                      cfg.seed, N + n + 1,
                                      reinterpret_cast<long long*>(d_idx[n].get()), d_sc[n].get(),
                                      p.get(), work.get(), status_i + N + n, ss);
    });
    n_draws[n] = T;
    return T;
  };

  // A mode's factor in four pieces:
  //   norms_for   sampling weights (+ their collectives)                       main stream
  //   sample_for  the sampling chain (no collectives)                           engine's stream
  //   power_for   Omega, gather, power scheme (+ collectives), sketch rows      main stream
  //   orth_for    orthonormalisation (no collectives)                           engine's stream
  // ST-HOSVD runs them back to back; T-HOSVD runs the collective-free pieces of all modes
  // concurrently on per-mode streams while every collective stays on the main stream in mode
  // order (the same issue order on every rank).
  struct ModeState {
    size_t J = 0, T = 0;
    DevBuf c;
  };
  std::vector<ModeState> ms(N);
  // local weights already produced by the fused 3-mode pass (T-HOSVD on a 3-way slab); for the
  // last mode its chunk partials when the slabs are segment-aligned
  std::vector<DevBuf> pre_w(N);
  DevBuf pre_chunks;
  bool pre_last = false;
  const bool seg_aligned = L >= kShardUnit * (size_t)P;
  if (seg_aligned && P > 64) throw std::invalid_argument("more than 64 ranks");
  auto norms_for = [&](size_t n) {
    const std::vector<size_t> ld = ldims();
    const ModeView v = view_of(ld, n);
    const bool rows_split = sharded && n == N - 1;
    const size_t Jl = (size_t)(v.inner * v.outer);
    if (!sharded) {  // replicated tensor: every column local
      ms[n].J = Jl;
      if (amm && cfg.regime != kUniform) {
        d_w[n] = DevBuf(Jl, st);
        eng.launch("norms", [&] { return lmra_dev::launch_column_sqnorms(cur, v, d_w[n].get(), st); });
      }
    } else if (rows_split) {  // mode N-1: every column local, its rows split across the ranks
      ms[n].J = Jl;
      if (amm && cfg.regime != kUniform) {
        if (seg_aligned) {
          // the canonical norm's segments of this rank's rows, all-gathered and added in global
          // order: the single-device bits (shard boundaries at multiples of 64 rows)
          const size_t nch = (c0 + 31) / 32;
          DevBuf chunks;
          if (pre_last) {
            chunks = std::move(pre_chunks);
          } else {
            chunks = DevBuf(nch * Jl, st);
            eng.launch("norms", [&] { return lmra_dev::launch_chunk_partials(cur, v, chunks.get(), st); });
          }
          lmra_dev::SegCounts cnt{};
          int kmax = 0;
          for (int q = 0; q < P; ++q) {
            cnt.n[q] = (int)(((shc[q] + 31) / 32 + 1) / 2);
            kmax = std::max(kmax, cnt.n[q]);
          }
          DevBuf segs((size_t)kmax * Jl, st), all((size_t)P * kmax * Jl, st);
          ck(cudaMemsetAsync(segs.get(), 0, (size_t)kmax * Jl * sizeof(double), st), "memset");
          ck(lmra_dev::launch_segment_sums(chunks.get(), (long long)Jl, (int)nch, segs.get(), st), "segments");
          comm.allgather(segs.get(), all.get(), (size_t)kmax * Jl, st);
          d_w[n] = DevBuf(Jl, st);
          ck(lmra_dev::launch_segment_combine(all.get(), (long long)Jl, P, kmax, cnt, d_w[n].get(), st), "combine");
        } else {  // unaligned slabs (L < 64 P): rank partials added in rank order
          if (!pre_last) {
            d_w[n] = DevBuf(Jl, st);
            eng.launch("norms", [&] { return lmra_dev::launch_column_sqnorms(cur, v, d_w[n].get(), st); });
          }
          comm.allreduce_sum(d_w[n].get(), Jl, st);
        }
      }
    } else {  // n < N-1: rank-local column range
      const size_t per = Jl / c0, Jg = per * L;
      ms[n].J = Jg;
      if (amm && cfg.regime != kUniform) {
        DevBuf wl, all((size_t)P * per * cmax, st);
        if (pre_w[n].get()) {
          wl = std::move(pre_w[n]);
        } else {
          wl = DevBuf(per * cmax, st);
          ck(cudaMemsetAsync(wl.get(), 0, per * cmax * sizeof(double), st), "memset");
          eng.launch("norms", [&] { return lmra_dev::launch_column_sqnorms(cur, v, wl.get(), st); });
        }
        comm.allgather(wl.get(), all.get(), per * cmax, st);
        d_w[n] = DevBuf(Jg, st);
        for (int q = 0; q < P; ++q)
          ck(cudaMemcpyAsync(d_w[n].get() + per * sh0[q], all.get() + (size_t)q * per * cmax,
                             per * shc[q] * sizeof(double), cudaMemcpyDeviceToDevice, st),
             "unpack norms");
      }
    }
  };
  auto sample_for = [&](Engine& e, size_t n, size_t t_n) {
    if (amm) ms[n].T = run_sampler(e, n, d_w[n].get(), ms[n].J, t_n);
  };
  auto power_for = [&](size_t n) {
    const size_t I = gdims[n], s = r.sketch[n];
    const std::vector<size_t> ld = ldims();
    const ModeView v = view_of(ld, n);
    DevBuf c(I * s, st);
    ck(cudaMemcpyAsync(c.get(), om_pin + om_off[n], I * s * sizeof(double), cudaMemcpyHostToDevice, st),
       "H2D omega");
    const bool rows_split = sharded && n == N - 1;
    const size_t t_n = ms[n].T;
    if (!sharded) {  // replicated tensor: the single-GPU computation, identical on every rank
      if (!amm) {
        eng.gram_power(cur, v, c, s, cfg.power, cfg.strategy);
      } else {
        DevBuf cp(I * t_n, st);
        eng.launch("gather", [&] {
          return lmra_dev::launch_gather(cur, v, reinterpret_cast<const long long*>(d_idx[n].get()),
                                         d_sc[n].get(), (long long)t_n, cp.get(), st);
        });
        eng.gram_power(cp.get(), ModeView{1, (long long)I, (long long)t_n}, c, s, cfg.power, cfg.strategy);
      }
    } else if (!rows_split) {  // n < N-1: rank-local column range
      const size_t Jl = (size_t)(v.inner * v.outer);
      const lmra_dev::GramPlan plan = lmra_dev::plan_gram(v, ctx->num_sms);
      if (!amm) {
        DevBuf h(Jl * s, st), zpart((size_t)plan.nsplit * I * s, st);
        for (int k = 0; k < cfg.power; ++k) {
          eng.launch("power_half", [&] { return lmra_dev::launch_ttm(cur, v, c.get(), (int)s, h.get(), st); });
          eng.launch("power_gram", [&] {
            return lmra_dev::launch_gram(cur, v, h.get(), (int)s, zpart.get(), plan, c.get(), st);
          });
          comm.allreduce_sum(c.get(), I * s, st);
        }
      } else {
        DevBuf lidx(t_n + 1, st), cp(I * t_n, st);
        ck(lmra_dev::launch_localize_idx(reinterpret_cast<const long long*>(d_idx[n].get()),
                                         (long long)t_n, (long long)(Jl / c0 * s0), (long long)Jl,
                                         reinterpret_cast<long long*>(lidx.get()), st),
           "localize");
        eng.launch("gather", [&] {
          return lmra_dev::launch_gather(cur, v, reinterpret_cast<const long long*>(lidx.get()),
                                         d_sc[n].get(), (long long)t_n, cp.get(), st);
        });
        const ModeView cv{1, (long long)I, (long long)t_n};
        const lmra_dev::GramPlan cplan = lmra_dev::plan_gram(cv, ctx->num_sms);
        DevBuf h(t_n * s, st), zpart((size_t)cplan.nsplit * I * s, st);
        for (int k = 0; k < cfg.power; ++k) {
          eng.launch("power_half", [&] { return lmra_dev::launch_ttm(cp.get(), cv, c.get(), (int)s, h.get(), st); });
          eng.launch("power_gram", [&] {
            return lmra_dev::launch_gram(cp.get(), cv, h.get(), (int)s, zpart.get(), cplan, c.get(), st);
          });
          comm.allreduce_sum(c.get(), I * s, st);
        }
      }
    } else {  // n == N-1 on the slab: fibres split by rows [s0, s0 + c0)
      const size_t J = (size_t)(v.inner * v.outer);  // all columns are local
      DevBuf cr = rows_of(c.get(), I, s, s0, c0);
      if (!amm) {
        const lmra_dev::GramPlan plan = lmra_dev::plan_gram(v, ctx->num_sms);
        DevBuf h(J * s, st), zpart((size_t)plan.nsplit * c0 * s, st);
        for (int k = 0; k < cfg.power; ++k) {
          eng.launch("power_half", [&] { return lmra_dev::launch_ttm(cur, v, cr.get(), (int)s, h.get(), st); });
          comm.allreduce_sum(h.get(), J * s, st);
          eng.launch("power_gram", [&] {
            return lmra_dev::launch_gram(cur, v, h.get(), (int)s, zpart.get(), plan, cr.get(), st);
          });
        }
      } else {
        DevBuf cp(c0 * t_n, st);
        eng.launch("gather", [&] {
          return lmra_dev::launch_gather(cur, v, reinterpret_cast<const long long*>(d_idx[n].get()),
                                         d_sc[n].get(), (long long)t_n, cp.get(), st);
        });
        const ModeView cv{1, (long long)c0, (long long)t_n};
        const lmra_dev::GramPlan cplan = lmra_dev::plan_gram(cv, ctx->num_sms);
        DevBuf h(t_n * s, st), zpart((size_t)cplan.nsplit * c0 * s, st);
        for (int k = 0; k < cfg.power; ++k) {
          eng.launch("power_half", [&] { return lmra_dev::launch_ttm(cp.get(), cv, cr.get(), (int)s, h.get(), st); });
          comm.allreduce_sum(h.get(), t_n * s, st);
          eng.launch("power_gram", [&] {
            return lmra_dev::launch_gram(cp.get(), cv, h.get(), (int)s, zpart.get(), cplan, cr.get(), st);
          });
        }
      }
      gather_rows(cr.get(), s, c.get(), I);
    }
    ms[n].c = std::move(c);
  };
  auto orth_for = [&](Engine& e, size_t n) -> DevBuf {
    const size_t I = gdims[n], s = r.sketch[n];
    const size_t mu = std::min(r.mu[n], std::min(I, s));  // top_left_vectors_clamped
    if (mu < r.mu[n] && R == 0)
      fprintf(stderr, "lmra: requested rank %zu exceeds matrix rank limit %zu, clamping\n",
              r.mu[n], mu);
    res->f_rows[n] = I;
    res->f_cols[n] = mu;
    ms[n].c.rebind(e.st_);
    DevBuf f = e.orth(ms[n].c.get(), I, s, mu, status_i + n);
    return f;
  };
  auto factor = [&](size_t n, size_t t_n) -> DevBuf {
    norms_for(n);
    sample_for(eng, n, t_n);
    power_for(n);
    return orth_for(eng, n);
  };

  Engine::I8Chain chain;
  auto contract = [&](size_t n, const double* q, size_t mu, const std::string& phase, bool next1) {
    const std::vector<size_t> ld = ldims();
    if (!sharded || n != N - 1) {
      // the slab's mode-0 contraction runs on the int8 tensor cores when its canonical column
      // norms are known (this rank's columns of the all-gathered weights), like the
      // single-GPU path; a following mode-1 contraction takes the handed-over exponents
      const double* w0 = nullptr;
      if (n == 0 && cur == in.x && amm && cfg.regime != kUniform && d_w[0].get() &&
          !(in.ov && in.ov->sample_idx)) {
        const size_t per = prod(ld) / ld[0] / ld[N - 1];
        w0 = d_w[0].get() + (sharded ? per * s0 : 0);
      }
      DevBuf y = eng.ttm_mode0(cur, ld, n, q, mu, w0, phase, &chain, next1);
      curbuf = std::move(y);
    } else {  // contraction over the sharded mode: local partial + all-reduce -> replicated
      DevBuf qr = rows_of(q, gdims[n], mu, s0, c0);
      DevBuf y = eng.ttm(cur, ld, n, qr.get(), mu, phase);
      std::vector<size_t> od = ld;
      od[n] = mu;
      comm.allreduce_sum(y.get(), prod(od), st);
      curbuf = std::move(y);
      sharded = false;
    }
    cur = curbuf.get();
    gdims[n] = mu;
  };

  std::vector<DevBuf> factors(N);
  if (!sequential) {
    // phases across modes: norms (main) | samplers (per-mode streams, concurrent) | power
    // schemes with their collectives (main, mode order) | orthonormalisations (per-mode
    // streams, each starting as soon as its sketch is reduced)
    std::vector<cudaEvent_t> evs;
    auto new_event = [&](cudaStream_t on) {
      cudaEvent_t e;
      ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
      evs.push_back(e);
      ck(cudaEventRecord(e, on), "event");
      return e;
    };
    struct EvGuard {
      std::vector<cudaEvent_t>& v;
      ~EvGuard() {
        for (cudaEvent_t e : v) cudaEventDestroy(e);
      }
    } ev_guard{evs};
    if (amm && cfg.regime != kUniform && N == 3 && !(in.ov && in.ov->sample_idx)) {
      // one read of the slab for all three modes' canonical norms (bit-identical to the
      // per-mode passes: modes 0/1 are local columns, mode 2 the slab partials)
      const long long I0 = (long long)gdims[0], I1 = (long long)gdims[1], I2 = (long long)c0;
      const size_t per0 = (size_t)(I1 * I2) / c0, per1 = (size_t)(I0 * I2) / c0;
      pre_w[0] = DevBuf(per0 * cmax, st);
      pre_w[1] = DevBuf(per1 * cmax, st);
      ck(cudaMemsetAsync(pre_w[0].get(), 0, per0 * cmax * sizeof(double), st), "memset");
      ck(cudaMemsetAsync(pre_w[1].get(), 0, per1 * cmax * sizeof(double), st), "memset");
      d_w[2] = DevBuf((size_t)(I0 * I1), st);
      if (seg_aligned) pre_chunks = DevBuf((size_t)((I2 + 31) / 32) * (size_t)(I0 * I1), st);
      DevBuf nwork(lmra_dev::norms3_workspace_doubles(I0, I1, I2), st);
      eng.launch("norms", [&] {
        return lmra_dev::launch_norms3(cur, I0, I1, I2, pre_w[0].get(), pre_w[1].get(), d_w[2].get(),
                                       nwork.get(), st, seg_aligned ? pre_chunks.get() : nullptr);
      });
      pre_last = true;
    }
    for (size_t n = 0; n < N; ++n) norms_for(n);
    const cudaEvent_t norms_done = new_event(st);
    std::vector<Engine> engs;
    engs.reserve(N);
    for (size_t n = 0; n < N; ++n) {
      cudaStream_t sn = ctx->aux_stream(n);
      ck(cudaStreamWaitEvent(sn, norms_done, 0), "wait");
      engs.emplace_back(ctx, sn, ctx->profile == 1 ? &prof : nullptr);
    }
    std::vector<cudaEvent_t> sampled(N);
    for (size_t n = 0; n < N; ++n) {
      sample_for(engs[n], n, amm ? t_flat[n] : 0);
      sampled[n] = new_event(engs[n].st_);
    }
    for (size_t n = 0; n < N; ++n) {
      ck(cudaStreamWaitEvent(st, sampled[n], 0), "wait");
      power_for(n);
      const cudaEvent_t sketched = new_event(st);
      ck(cudaStreamWaitEvent(engs[n].st_, sketched, 0), "wait");
      factors[n] = orth_for(engs[n], n);
    }
    for (size_t n = 0; n < N; ++n) ck(cudaStreamWaitEvent(st, new_event(engs[n].st_), 0), "wait");
    std::vector<size_t> idx(N);
    std::iota(idx.begin(), idx.end(), size_t{0});
    std::stable_sort(idx.begin(), idx.end(),
                     [&](size_t a, size_t b) { return res->f_cols[a] < res->f_cols[b]; });
    int step = 0;
    for (size_t k = 0; k < N; ++k) {
      const size_t n = idx[k];
      contract(n, factors[n].get(), res->f_cols[n], "core_ttm" + std::to_string(step++),
               k + 1 < N && idx[k + 1] == 1);
    }
  } else {
    for (size_t n : r.order) {
      size_t t_n = 0;
      if (amm) {
        const size_t cols = prod(gdims) / gdims[n];
        t_n = cfg.t_samples.empty() ? samples_from_alpha(cfg.alpha, cols) : cfg.t_samples[n];
        if (t_n < 1) throw std::invalid_argument("sample counts must be positive");
      }
      factors[n] = factor(n, t_n);
      const size_t oi = (size_t)(std::find(r.order.begin(), r.order.end(), n) - r.order.begin());
      contract(n, factors[n].get(), res->f_cols[n], "shrink_ttm_m" + std::to_string(n),
               oi + 1 < r.order.size() && r.order[oi + 1] == 1);
    }
  }
  res->core_dims = gdims;
  if (curbuf.get() == nullptr) throw std::runtime_error("sharded run produced no core");
  res->core = curbuf.detach();
  for (size_t n = 0; n < N; ++n) {  // copies on the main stream (ordered after every mode's join)
    factors[n].rebind(st);
    res->factors[n] = factors[n].detach();
  }

  ck(cudaEventRecord(ev1, st), "event");
  std::vector<int> stat(2 * N);
  ck(cudaMemcpyAsync(stat.data(), status.get(), 2 * N * sizeof(int), cudaMemcpyDeviceToHost, st),
     "D2H status");
  if (ctx->keep_trace) {
    for (size_t n = 0; n < N; ++n) res->omega[n].assign(om_pin + om_off[n], om_pin + om_off[n + 1]);
    for (size_t n = 0; n < N; ++n)
      if (n_draws[n]) {
        res->idx[n].resize(n_draws[n]);
        res->scales[n].resize(n_draws[n]);
        ck(cudaMemcpyAsync(res->idx[n].data(), d_idx[n].get(), n_draws[n] * sizeof(int64_t),
                           cudaMemcpyDeviceToHost, st), "D2H idx");
        ck(cudaMemcpyAsync(res->scales[n].data(), d_sc[n].get(), n_draws[n] * sizeof(double),
                           cudaMemcpyDeviceToHost, st), "D2H scales");
      }
  }
  ck(cudaStreamSynchronize(st), "sync");
  float dev_ms = 0;
  ck(cudaEventElapsedTime(&dev_ms, ev0, ev1), "event time");
  if (getenv("LMRA_TIMELINE") && getenv("LMRA_TIMELINE")[0] == '1' && !prof.empty()) {
    float lead = 0;  // run start -> first phase (host RNG, uploads, launch latency)
    ck(cudaEventElapsedTime(&lead, ev0, prof[0].a), "event time");
    fprintf(stderr, "timeline lead-in %9.4f ms, run %9.4f ms\n", lead, dev_ms);
  }
  cudaEventDestroy(ev0);
  cudaEventDestroy(ev1);
  for (size_t n = 0; n < N; ++n) {
    const int f = stat[N + n];
    if (f & 1) throw std::invalid_argument("probability weights must be nonnegative");
    if (f & 32) throw std::invalid_argument("nearly-optimal mixture weight must lie in (0, 1]");
    if (f & 2) throw std::invalid_argument("cannot normalize an all-zero distribution");
    if (f & 4) throw std::invalid_argument("probability weights must sum to one");
    if (f & 8) throw std::invalid_argument("randsample: all-zero distribution");
    if (f & 16) ++res->sampler_fallbacks;
    if (f & 64) throw std::runtime_error("sampler: uniform segment table overflow");
  }
  for (size_t n = 0; n < N; ++n)
    if (stat[n] != 0) throw std::runtime_error("thin_svd: SVD iteration did not converge");
  res->t_device = dev_ms;
  res->launches = (double)(lmra_dev::g_kernel_launches - launches0);
  static const bool timeline = getenv("LMRA_TIMELINE") && getenv("LMRA_TIMELINE")[0] == '1';
  if (timeline && !prof.empty()) {  // diagnostics: phase start/end relative to the first phase
    for (const PhaseRec& p : prof) {
      float a = 0, b = 0;
      ck(cudaEventElapsedTime(&a, prof[0].a, p.a), "event time");
      ck(cudaEventElapsedTime(&b, prof[0].a, p.b), "event time");
      fprintf(stderr, "timeline %-16s %9.4f %9.4f\n", p.name.c_str(), a, b);
    }
  }
  for (const PhaseRec& p : prof) {
    float ms = 0;
    ck(cudaEventElapsedTime(&ms, p.a, p.b), "event time");
    auto it = std::find_if(res->phases.begin(), res->phases.end(),
                           [&](const lmra_result::Phase& q2) { return q2.name == p.name; });
    if (it == res->phases.end()) {
      res->phases.push_back({p.name, 0.0, 0});
      it = res->phases.end() - 1;
    }
    it->ms += ms;
    it->count += 1;
  }
  res->t_total = now_ms() - t0;
}

// ------------------------------------------------------------------ deterministic baselines
// t_hosvd / st_hosvd / hooi (tucker.cpp:242-316).  Their factors are the leading left singular
// vectors of FULL unfoldings (top_left_vectors_clamped(unfold(x, n), mu), tucker.cpp:65-77):
// A_(n)^T = Q R by Householder QR (cuSOLVER dgeqrf on the transposed unfolding, written by
// unfold_t), then the SVD of the I_n x I_n R (dgesvd): A_(n) = V_R S (Q U_R)^T, so the factor is
// V_R(:, :mu) with the sign rule of fix_signs (linalg.cpp:13-29).  Wide-and-short unfoldings
// (J < I) take the SVD of A_(n) itself.  The mode products are the DMMA TTM.
static void cusolver_check(cusolverStatus_t s, const char* what) {
  if (s != CUSOLVER_STATUS_SUCCESS) throw CudaError(std::string(what) + ": cuSOLVER status " + std::to_string((int)s));
}

static DevBuf dense_lsv(lmra_context* ctx, const double* x, const std::vector<size_t>& dims, size_t n,
                        size_t mu_req, size_t* mu_out) {
  const auto& cs = lmra_host::cusolver();
  cudaStream_t st = ctx->stream;
  if (!ctx->cusolver) {
    cusolver_check(cs.Create(&ctx->cusolver), "cusolverDnCreate");
    if (cs.SetDeterministicMode) cs.SetDeterministicMode(ctx->cusolver, CUSOLVER_DETERMINISTIC_RESULTS);
  }
  cusolver_check(cs.SetStream(ctx->cusolver, st), "cusolverDnSetStream");
  const ModeView v = view_of(dims, n);
  const size_t I = dims[n], J = (size_t)(v.inner * v.outer);
  const size_t mu = std::min(mu_req, std::min(I, J));  // rank_cap (tucker.cpp:65-71)
  if (mu < mu_req)
    fprintf(stderr, "lmra: requested rank %zu exceeds matrix rank limit %zu, clamping\n", mu_req, mu);
  *mu_out = mu;
  if (I > (size_t)INT32_MAX || J > (size_t)INT32_MAX) throw std::invalid_argument("unfolding too large for dgesvd");
  Engine eng(ctx);
  DevBuf at(J * I, st), info(1, st), q(I * mu, st), sv(std::min(I, J), st);
  ck(cudaMemsetAsync(info.get(), 0, sizeof(double), st), "memset");
  int* dinfo = reinterpret_cast<int*>(info.get());
  eng.launch("dense_unfold", [&] { return lmra_dev::launch_unfold_t(x, v.inner, (long long)I, v.outer, at.get(), st); });
  const int iI = (int)I, iJ = (int)J;
  if (J >= I) {
    int lw = 0;
    cusolver_check(cs.Dgeqrf_bufferSize(ctx->cusolver, iJ, iI, at.get(), iJ, &lw), "dgeqrf_bufferSize");
    DevBuf tau(I, st), w((size_t)std::max(lw, 1), st);
    cusolver_check(cs.Dgeqrf(ctx->cusolver, iJ, iI, at.get(), iJ, tau.get(), w.get(), lw, dinfo), "dgeqrf");
    DevBuf r(I * I, st), vt(I * I, st), rw(I, st);
    eng.launch("dense_r", [&] { return lmra_dev::launch_copy_upper(at.get(), (long long)J, iI, r.get(), st); });
    int lw2 = 0;
    cusolver_check(cs.Dgesvd_bufferSize(ctx->cusolver, iI, iI, &lw2), "dgesvd_bufferSize");
    DevBuf w2((size_t)std::max(lw2, 1), st);
    cusolver_check(cs.Dgesvd(ctx->cusolver, 'N', 'A', iI, iI, r.get(), iI, sv.get(), nullptr, 1, vt.get(), iI,
                             w2.get(), lw2, rw.get(), dinfo),
                   "dgesvd");
    eng.launch("dense_factor", [&] { return lmra_dev::launch_rows_to_cols(vt.get(), iI, (int)mu, q.get(), st); });
  } else {
    DevBuf a(I * J, st), u(I * J, st), rw(J, st);
    eng.launch("transpose", [&] { return lmra_dev::launch_transpose(at.get(), (long long)J, (long long)I, a.get(), st); });
    int lw2 = 0;
    cusolver_check(cs.Dgesvd_bufferSize(ctx->cusolver, iI, iJ, &lw2), "dgesvd_bufferSize");
    DevBuf w2((size_t)std::max(lw2, 1), st);
    cusolver_check(cs.Dgesvd(ctx->cusolver, 'S', 'N', iI, iJ, a.get(), iI, sv.get(), u.get(), iI, nullptr, 1,
                             w2.get(), lw2, rw.get(), dinfo),
                   "dgesvd");
    ck(cudaMemcpyAsync(q.get(), u.get(), I * mu * sizeof(double), cudaMemcpyDeviceToDevice, st), "copy");
  }
  eng.launch("dense_signs", [&] { return lmra_dev::launch_signfix_columns(q.get(), (long long)I, (int)I, (int)mu, st); });
  int hinfo = 0;
  ck(cudaMemcpyAsync(&hinfo, dinfo, sizeof(int), cudaMemcpyDeviceToHost, st), "D2H");
  ck(cudaStreamSynchronize(st), "sync");  // the locals above are released after this
  if (hinfo > 0) throw std::runtime_error("thin_svd: SVD iteration did not converge");
  if (hinfo < 0) throw CudaError("cuSOLVER: illegal argument " + std::to_string(-hinfo));
  return q;
}

static double frobenius_dev(lmra_context* ctx, const double* t, size_t n) {
  cudaStream_t st = ctx->stream;
  DevBuf work(lmra_dev::diff_sumsq_workspace_doubles(), st), out(2, st);
  ck(lmra_dev::launch_diff_sumsq(t, t, (long long)n, work.get(), out.get(), st), "sumsq");
  double h[2];
  ck(cudaMemcpyAsync(h, out.get(), sizeof(h), cudaMemcpyDeviceToHost, st), "D2H");
  ck(cudaStreamSynchronize(st), "sync");
  return std::sqrt(h[1]);
}

void run_deterministic_impl(lmra_context* ctx, const RunInputs& in, lmra_result* res) {
  using namespace lmra_host;
  const double t0 = now_ms();
  // the per-run arena would grow to every intermediate of every HOOI sweep: stream-ordered
  // pool allocations instead (each buffer freed when its scope ends)
  lmra_context* arena_prev = t_arena_ctx;
  t_arena_ctx = nullptr;
  struct Restore {
    lmra_context* p;
    ~Restore() { t_arena_ctx = p; }
  } restore{arena_prev};
  const long long launches0 = lmra_dev::g_kernel_launches;
  cudaStream_t st = ctx->stream;
  Engine eng(ctx);
  const auto& cfg = in.cfg;
  const size_t N = in.dims.size();
  for (size_t d : in.dims)
    if (d == 0) throw std::invalid_argument("tensor dimension must be positive");
  Resolved r = resolve(in.dims, cfg);
  res->omega.assign(N, {});
  res->om_rows.assign(N, 0);
  res->om_cols.assign(N, 0);
  res->idx.assign(N, {});
  res->scales.assign(N, {});
  res->norms.assign(N, {});
  res->factors.assign(N, nullptr);
  res->f_rows.assign(N, 0);
  res->f_cols.assign(N, 0);
  std::vector<DevBuf> factors(N);
  std::vector<size_t> width(N, 0);
  auto factor = [&](const double* t, const std::vector<size_t>& d, size_t n) {
    factors[n] = dense_lsv(ctx, t, d, n, r.mu[n], &width[n]);
  };
  // core_from_factors (tucker.cpp:81-92): ascending factor width, stable
  auto core_from = [&](std::vector<size_t>& cur) {
    std::vector<size_t> idx(N);
    std::iota(idx.begin(), idx.end(), size_t{0});
    std::stable_sort(idx.begin(), idx.end(), [&](size_t a, size_t b) { return width[a] < width[b]; });
    DevBuf t;
    const double* src = in.x;
    cur = in.dims;
    for (size_t n : idx) {
      DevBuf y = eng.ttm(src, cur, n, factors[n].get(), width[n], "core_ttm");
      cur[n] = width[n];
      t = std::move(y);
      src = t.get();
    }
    return t;
  };
  std::vector<size_t> cdims;
  DevBuf core;
  auto st_hosvd = [&] {
    DevBuf work;
    const double* src = in.x;
    std::vector<size_t> cur = in.dims;
    for (size_t n : r.order) {
      factor(src, cur, n);
      DevBuf y = eng.ttm(src, cur, n, factors[n].get(), width[n], "shrink_ttm");
      cur[n] = width[n];
      work = std::move(y);
      src = work.get();
    }
    cdims = cur;
    core = std::move(work);
  };
  if (in.alg == LMRA_THOSVD) {  // tucker.cpp:242-248
    for (size_t n = 0; n < N; ++n) factor(in.x, in.dims, n);
    core = core_from(cdims);
  } else if (in.alg == LMRA_STHOSVD) {  // tucker.cpp:250-259
    st_hosvd();
  } else {  // LMRA_HOOI, tucker.cpp:261-316 with init = st_hosvd
    st_hosvd();
    core = core_from(cdims);
    const double norm_a = frobenius_dev(ctx, in.x, prod(in.dims));
    if (norm_a != 0.0) {
      double prev = frobenius_dev(ctx, core.get(), prod(cdims));
      bool converged = false;
      int sweep = 0;
      const size_t last = r.order.back();
      while (sweep < cfg.hooi_max_sweeps) {
        ++sweep;
        for (size_t n : r.order) {
          DevBuf y;
          const double* src = in.x;
          std::vector<size_t> cur = in.dims;
          for (size_t m = 0; m < N; ++m) {
            if (m == n) continue;
            DevBuf z = eng.ttm(src, cur, m, factors[m].get(), width[m], "hooi_ttm");
            cur[m] = width[m];
            y = std::move(z);
            src = y.get();
          }
          factor(src, cur, n);
          if (n == last) {
            DevBuf z = eng.ttm(src, cur, n, factors[n].get(), width[n], "hooi_ttm");
            cur[n] = width[n];
            cdims = cur;
            core = std::move(z);
          }
        }
        const double curn = frobenius_dev(ctx, core.get(), prod(cdims));
        if (std::abs(curn - prev) / norm_a < cfg.hooi_tol) {
          converged = true;
          break;
        }
        prev = curn;
      }
      if (!converged)
        fprintf(stderr, "lmra: hooi stopped after %d sweeps without meeting the tolerance\n", sweep);
      res->hooi_converged = converged ? 1 : 0;
      res->hooi_sweeps = sweep;
    }
  }
  res->core_dims = cdims;
  // result blocks (ResultBlocks) -- detach() needs an active arena context for the block cache
  t_arena_ctx = ctx;
  res->core = core.detach();
  for (size_t n = 0; n < N; ++n) {
    res->f_rows[n] = in.dims[n];
    res->f_cols[n] = width[n];
    res->factors[n] = factors[n].detach();
  }
  ck(cudaStreamSynchronize(st), "sync");
  res->launches = (double)(lmra_dev::g_kernel_launches - launches0);
  res->t_total = now_ms() - t0;
  res->t_device = res->t_total;
}

lmra_host::Config to_config(const lmra_algo_config* c) {
  lmra_host::Config k;
  if (!c) throw std::invalid_argument("null config");
  if (c->n_rank && !c->rank) throw std::invalid_argument("null rank array");
  k.mu.assign(c->rank, c->rank + c->n_rank);
  k.oversampling = c->oversampling;
  k.power = c->power;
  k.alpha = c->alpha;
  k.regime = c->regime;
  k.beta = c->regime_beta;
  if (c->n_t_samples) k.t_samples.assign(c->t_samples, c->t_samples + c->n_t_samples);
  if (c->n_order) k.order.assign(c->order, c->order + c->n_order);
  k.seed = c->seed;
  k.strategy = c->strategy;
  k.hooi_max_sweeps = c->hooi_max_sweeps;
  k.hooi_tol = c->hooi_tol;
  if (k.regime < 0 || k.regime > 2) throw std::invalid_argument("unknown probability regime");
  if (k.strategy != 0 && k.strategy != 1) throw std::invalid_argument("unknown Gram strategy");
  return k;
}

}  // namespace

// ================================================================== C ABI
extern "C" {

const char* lmra_last_error(void) { return g_err.c_str(); }
const char* lmra_version(void) { return "lmra-b200 0.1 (sm_100a, fp64 DMMA)"; }

void lmra_algo_config_init(lmra_algo_config* cfg) {
  std::memset(cfg, 0, sizeof(*cfg));
  cfg->oversampling = 10;
  cfg->power = 1;
  cfg->alpha = 0.2;
  cfg->regime = LMRA_UNIFORM;
  cfg->regime_beta = 0.5;
  cfg->strategy = LMRA_STRATEGY_A;
  cfg->hooi_max_sweeps = 50;
  cfg->hooi_tol = 1e-8;
}

int lmra_context_create(int device, void* stream, lmra_context** out) {
  *out = nullptr;
  return guard([&] {
    auto c = std::make_unique<lmra_context>();
    c->device = device;
    c->results->device = device;
    DeviceGuard dg(device);
    ck(cudaFree(nullptr), "cuda init");
    ck(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device), "attr");
    if (stream) {
      c->stream = static_cast<cudaStream_t>(stream);
    } else {
      ck(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking), "stream");
      c->own_stream = true;
    }
    cudaMemPool_t pool;
    ck(cudaDeviceGetDefaultMemPool(&pool, device), "mempool");
    uint64_t thresh = UINT64_MAX;
    ck(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thresh), "mempool attr");
    *out = c.release();
  });
}

void lmra_context_destroy(lmra_context* ctx) {
  if (!ctx) return;
  {
    // never throws (may run during process teardown, when the CUDA driver is shutting down)
    int prev = -1;
    cudaGetDevice(&prev);
    if (prev != ctx->device) cudaSetDevice(ctx->device);
    cudaGetLastError();
    cudaStreamSynchronize(ctx->stream);
    ctx->comm.reset();
    for (cudaStream_t s : ctx->aux) cudaStreamDestroy(s);
    if (ctx->hi) cudaStreamDestroy(ctx->hi);
    for (cudaEvent_t e : ctx->events) cudaEventDestroy(e);
    if (ctx->pinned) cudaFreeHost(ctx->pinned);
    if (ctx->arena) cudaFree(ctx->arena);
    if (ctx->cusolver) lmra_host::cusolver().Destroy(ctx->cusolver);
    if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
    if (prev >= 0 && prev != ctx->device) cudaSetDevice(prev);
    cudaGetLastError();
  }
  delete ctx;
}

int lmra_context_set_stream(lmra_context* ctx, void* stream) {
  return guard([&] {
    if (!stream) throw std::invalid_argument("null stream");
    ctx->stream = static_cast<cudaStream_t>(stream);
  });
}

int lmra_context_synchronize(lmra_context* ctx) {
  return guard([&] {
    DeviceGuard dg(ctx->device);
    ck(cudaStreamSynchronize(ctx->stream), "sync");
  });
}

int lmra_nccl_unique_id(void* out128) {
  return guard([&] {
    ncclUniqueId id;
    ckn(lmra_host::nccl().GetUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(out128, &id, sizeof(id));
  });
}

int lmra_context_set_comm(lmra_context* ctx, const void* uid, int nranks, int rank) {
  return guard([&] {
    if (nranks < 1 || rank < 0 || rank >= nranks) throw std::invalid_argument("bad rank layout");
    DeviceGuard dg(ctx->device);
    ncclUniqueId id;
    std::memcpy(&id, uid, sizeof(id));
    ctx->comm.reset();
    auto c = std::make_shared<NcclComm>();
    ckn(lmra_host::nccl().CommInitRank(&c->c, nranks, id, rank), "ncclCommInitRank");
    c->nranks = nranks;
    c->rank = rank;
    ctx->comm = c;
    ctx->nranks = nranks;
    ctx->rank = rank;
  });
}

int lmra_thread_group_create(int nranks, void** group) {
  return guard([&] {
    if (nranks < 1) throw std::invalid_argument("bad rank count");
    *group = new std::shared_ptr<ThreadGroup>(std::make_shared<ThreadGroup>(nranks));
  });
}

void lmra_thread_group_destroy(void* group) {
  delete static_cast<std::shared_ptr<ThreadGroup>*>(group);
}

int lmra_context_set_thread_comm(lmra_context* ctx, void* group, int rank) {
  return guard([&] {
    auto g = *static_cast<std::shared_ptr<ThreadGroup>*>(group);
    if (rank < 0 || rank >= g->n) throw std::invalid_argument("bad rank");
    auto c = std::make_shared<ThreadComm>();
    c->g = g;
    c->nranks = g->n;
    c->rank = rank;
    ctx->comm = c;
    ctx->nranks = g->n;
    ctx->rank = rank;
  });
}

int lmra_shard_range(uint64_t extent, int nranks, int rank, uint64_t* start, uint64_t* count) {
  return guard([&] {
    if (nranks < 1 || rank < 0 || rank >= nranks) throw std::invalid_argument("bad rank layout");
    size_t b = 0, c = 0;
    shard_bounds((size_t)extent, (size_t)nranks, (size_t)rank, &b, &c);
    *start = b;
    *count = c;
  });
}

// ------------------------------------------------------------------ algorithm ids, knobs
// tucker.cpp:190-220 (parse_algorithm / algorithm_id / all_algorithm_ids)
static const struct {
  int code;
  const char* id;
} kAlgIds[] = {{LMRA_THOSVD, "thosvd"}, {LMRA_STHOSVD, "sthosvd"}, {LMRA_HOOI, "hooi"}, {LMRA_ALG1, "alg1"},
               {LMRA_ALG2, "alg2"},     {LMRA_ALG4, "alg4"},       {LMRA_ALG5, "alg5"}, {LMRA_ALG6, "alg6"},
               {LMRA_ALG7, "alg7"}};

const char* lmra_algorithm_id(int algorithm) {
  for (const auto& a : kAlgIds)
    if (a.code == algorithm) return a.id;
  return "?";
}

int lmra_parse_algorithm(const char* id, int* algorithm) {
  if (!id) return 0;
  for (const auto& a : kAlgIds)
    if (std::strcmp(a.id, id) == 0) {
      if (algorithm) *algorithm = a.code;
      return 1;
    }
  return 0;
}

int lmra_all_algorithm_ids(const char** ids, int max_ids) {
  const int n = (int)(sizeof(kAlgIds) / sizeof(kAlgIds[0]));
  for (int k = 0; k < n && k < max_ids; ++k) ids[k] = kAlgIds[k].id;
  return n;
}

// tucker.cpp:164-172: LMRA_NUM_THREADS, default 1, clamped to [1, 64]
int lmra_thread_cap(void) {
  static const int cap = [] {
    const char* env = std::getenv("LMRA_NUM_THREADS");
    if (!env) return 1;
    return std::clamp(std::atoi(env), 1, 64);
  }();
  return cap;
}

// the same idiom for devices: LMRA_NUM_GPUS, default 1, clamped to [1, visible devices]
int lmra_device_cap(void) {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count < 1) {
    cudaGetLastError();
    return 1;
  }
  const char* env = std::getenv("LMRA_NUM_GPUS");
  if (!env) return 1;
  return std::clamp(std::atoi(env), 1, count);
}

int lmra_run_algorithm(lmra_context* ctx, int algorithm, const double* x, const uint64_t* dims,
                       int order, int x_location, const lmra_algo_config* cfg,
                       const lmra_overrides* overrides, lmra_result** out) {
  *out = nullptr;
  return guard([&] {
    if (!ctx) throw std::invalid_argument("null context");
    const bool deterministic = algorithm == LMRA_THOSVD || algorithm == LMRA_STHOSVD || algorithm == LMRA_HOOI;
    if (algorithm != LMRA_ALG1 && algorithm != LMRA_ALG2 && algorithm != LMRA_ALG4 &&
        algorithm != LMRA_ALG5 && algorithm != LMRA_ALG6 && algorithm != LMRA_ALG7 && !deterministic)
      throw std::invalid_argument("unknown algorithm");
    if (order < 1) throw std::invalid_argument("cannot decompose an order-0 tensor");
    const bool sharded = ctx->comm && ctx->nranks > 1;
    if (sharded && (algorithm == LMRA_ALG6 || algorithm == LMRA_ALG7))
      throw std::invalid_argument("alg6/alg7 run on one device (no sharded QR-proxy path)");
    if (sharded && deterministic)
      throw std::invalid_argument("the deterministic baselines (thosvd / sthosvd / hooi) run on one device");
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard dg(ctx->device);
    ArenaScope arena(ctx);  // every device buffer of the run (after the device guard)
    RunInputs in;
    in.alg = algorithm;
    in.dims.assign(dims, dims + order);
    in.cfg = to_config(cfg);
    in.ov = overrides;
    auto res = std::make_unique<lmra_result>();
    res->device = ctx->device;
    res->blocks = ctx->results;
    DevBuf staged;
    if (x_location == LMRA_HOST) {
      size_t n = prod(in.dims);
      if (sharded) {  // x is this rank's slab of the last mode
        const size_t L = in.dims.back();
        if (L == 0) throw std::invalid_argument("tensor dimension must be positive");
        size_t b = 0, c = 0;
        shard_bounds(L, (size_t)ctx->nranks, (size_t)ctx->rank, &b, &c);
        n = n / L * c;
      }
      staged = DevBuf(n, ctx->stream);
      ck(cudaMemcpyAsync(staged.get(), x, n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream),
         "H2D tensor");
      in.x = staged.get();
    } else {
      in.x = x;
    }
    if (sharded) {
      try {
        run_sharded_impl(ctx, in, res.get());
      } catch (...) {
        ctx->comm->abort();
        throw;
      }
    } else if (deterministic) {
      run_deterministic_impl(ctx, in, res.get());
    } else {
      run_algorithm_impl(ctx, in, res.get());
    }
    *out = res.release();
  });
}

// ------------------------------------------------------------------ in-process multi-GPU
// One process drives ndev devices (the C++ drop-in's LMRA_NUM_GPUS): one context and one
// host thread per device, the tensor split along its last mode exactly as with one process
// per GPU.  Communicator: NCCL (ncclCommInitAll) when the devices are distinct, else the
// in-process ThreadComm (device copies, peer access enabled).  Groups are cached per device
// list; a group's runs are serialised.
namespace {
struct DeviceGroup {
  std::vector<int> devs;
  std::vector<lmra_context*> ctx;
  std::shared_ptr<ThreadGroup> tg;
  bool nccl = false;
  std::mutex run_mu;
  ~DeviceGroup() {
    for (lmra_context* c : ctx) lmra_context_destroy(c);
  }
};
// never destroyed: tearing contexts down in static destructors would race the CUDA runtime's own
// teardown at process exit
std::mutex& g_groups_mu = *new std::mutex;
std::map<std::vector<int>, std::shared_ptr<DeviceGroup>>& g_groups =
    *new std::map<std::vector<int>, std::shared_ptr<DeviceGroup>>;

std::shared_ptr<DeviceGroup> device_group(const std::vector<int>& devs) {
  std::lock_guard<std::mutex> lk(g_groups_mu);
  auto it = g_groups.find(devs);
  if (it != g_groups.end()) return it->second;
  auto g = std::make_shared<DeviceGroup>();
  g->devs = devs;
  const int n = (int)devs.size();
  for (int d : devs) {
    lmra_context* c = nullptr;
    if (lmra_context_create(d, nullptr, &c) != LMRA_OK) throw CudaError(g_err);
    g->ctx.push_back(c);
  }
  std::vector<int> sorted = devs;
  std::sort(sorted.begin(), sorted.end());
  const bool distinct = std::adjacent_find(sorted.begin(), sorted.end()) == sorted.end();
  if (n > 1 && distinct) {
    try {
      const auto& api = lmra_host::nccl();
      if (api.CommInitAll) {
        std::vector<ncclComm_t> comms(n);
        ckn(api.CommInitAll(comms.data(), n, devs.data()), "ncclCommInitAll");
        for (int r = 0; r < n; ++r) {
          auto c = std::make_shared<NcclComm>();
          c->c = comms[r];
          c->nranks = n;
          c->rank = r;
          g->ctx[r]->comm = c;
          g->ctx[r]->nranks = n;
          g->ctx[r]->rank = r;
        }
        g->nccl = true;
      }
    } catch (const std::exception&) {
      g->nccl = false;  // no NCCL in this process: the in-process communicator below
    }
  }
  if (n > 1 && !g->nccl) {
    for (int a : devs)
      for (int b : devs)
        if (a != b) {
          int ok = 0;
          cudaDeviceCanAccessPeer(&ok, a, b);
          if (ok) {
            DeviceGuard dg(a);
            if (cudaDeviceEnablePeerAccess(b, 0) != cudaSuccess) cudaGetLastError();  // already enabled
          }
        }
    g->tg = std::make_shared<ThreadGroup>(n);
    for (int r = 0; r < n; ++r) {
      auto c = std::make_shared<ThreadComm>();
      c->g = g->tg;
      c->nranks = n;
      c->rank = r;
      g->ctx[r]->comm = c;
      g->ctx[r]->nranks = n;
      g->ctx[r]->rank = r;
    }
  }
  g_groups[devs] = g;
  return g;
}
}  // namespace

int lmra_run_algorithm_multigpu(int ndev, const int* devices, int algorithm, const double* x, const uint64_t* dims,
                                int order, int x_location, const lmra_algo_config* cfg,
                                const lmra_overrides* overrides, lmra_result** out) {
  *out = nullptr;
  return guard([&] {
    if (ndev < 1 || !devices) throw std::invalid_argument("bad device list");
    if (order < 1) throw std::invalid_argument("cannot decompose an order-0 tensor");
    std::vector<int> devs(devices, devices + ndev);
    auto g = device_group(devs);
    std::lock_guard<std::mutex> lk(g->run_mu);
    size_t slice = 1;
    for (int k = 0; k + 1 < order; ++k) slice *= dims[k];
    const uint64_t L = dims[order - 1];
    std::vector<int> rc(ndev, LMRA_OK);
    std::vector<std::string> err(ndev);
    std::vector<lmra_result*> res(ndev, nullptr);
    std::vector<std::thread> th;
    for (int r = 0; r < ndev; ++r)
      th.emplace_back([&, r] {
        uint64_t st = 0, cnt = 0;
        lmra_shard_range(L, ndev, r, &st, &cnt);
        const double* xr = x ? x + st * slice : nullptr;
        void* slab = nullptr;
        if (x_location == LMRA_DEVICE && ndev > 1 && devs[r] != devs[0]) {  // x lives on devices[0]
          DeviceGuard dg(devs[r]);
          const size_t bytes = cnt * slice * sizeof(double);
          if (cudaMalloc(&slab, std::max<size_t>(bytes, 16)) != cudaSuccess ||
              cudaMemcpyPeer(slab, devs[r], xr, devs[0], bytes) != cudaSuccess) {
            rc[r] = LMRA_ECUDA;
            err[r] = "slab copy to device " + std::to_string(devs[r]) + " failed";
            if (g->ctx[r]->comm) g->ctx[r]->comm->abort();
            if (slab) cudaFree(slab);
            return;
          }
          xr = static_cast<const double*>(slab);
        }
        rc[r] = lmra_run_algorithm(g->ctx[r], algorithm, xr, dims, order, x_location, cfg, overrides, &res[r]);
        if (rc[r] != LMRA_OK) err[r] = lmra_last_error();
        if (slab) {
          DeviceGuard dg(devs[r]);
          cudaFree(slab);
        }
      });
    for (auto& t : th) t.join();
    for (int r = 1; r < ndev; ++r)
      if (res[r]) lmra_result_free(res[r]);
    for (int r = 0; r < ndev; ++r)
      if (rc[r] != LMRA_OK) {
        if (res[0]) lmra_result_free(res[0]);
        {  // the communicator was aborted: the next call builds a fresh group
          std::lock_guard<std::mutex> lk2(g_groups_mu);
          g_groups.erase(devs);
        }
        if (rc[r] == LMRA_EINVAL) throw std::invalid_argument(err[r]);
        if (rc[r] == LMRA_ECUDA) throw CudaError(err[r]);
        throw std::runtime_error(err[r]);
      }
    *out = res[0];
  });
}

int lmra_result_order(const lmra_result* r) { return (int)r->factors.size(); }
void lmra_result_hooi_stats(const lmra_result* r, int* converged, int* sweeps) {
  *converged = r->hooi_converged;
  *sweeps = r->hooi_sweeps;
}
void lmra_result_core_dims(const lmra_result* r, uint64_t* dims) {
  for (size_t n = 0; n < r->core_dims.size(); ++n) dims[n] = r->core_dims[n];
}
static int copy_out(int device, double* dst, const double* src, size_t n, int loc) {
  return guard([&] {
    DeviceGuard dg(device);
    ck(cudaMemcpy(dst, src, n * sizeof(double),
                  loc == LMRA_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice),
       "copy out");
  });
}
int lmra_result_copy_core(const lmra_result* r, double* dst, int dst_location) {
  return copy_out(r->device, dst, r->core, prod(r->core_dims), dst_location);
}
void lmra_result_factor_dims(const lmra_result* r, int mode, uint64_t* rows, uint64_t* cols) {
  *rows = r->f_rows[mode];
  *cols = r->f_cols[mode];
}
int lmra_result_copy_factor(const lmra_result* r, int mode, double* dst, int dst_location) {
  return copy_out(r->device, dst, r->factors[mode], r->f_rows[mode] * r->f_cols[mode],
                  dst_location);
}
const double* lmra_result_core_device(const lmra_result* r) {
  r->exposed.store(true);
  return r->core;
}
const double* lmra_result_factor_device(const lmra_result* r, int mode) {
  r->exposed.store(true);
  return r->factors[mode];
}
void lmra_result_omega_dims(const lmra_result* r, int mode, uint64_t* rows, uint64_t* cols) {
  *rows = r->om_rows[mode];
  *cols = r->om_cols[mode];
}
int lmra_result_copy_omega(const lmra_result* r, int mode, double* dst) {
  std::memcpy(dst, r->omega[mode].data(), sizeof(double) * r->omega[mode].size());
  return LMRA_OK;
}
uint64_t lmra_result_num_samples(const lmra_result* r, int mode) { return r->idx[mode].size(); }
int lmra_result_copy_samples(const lmra_result* r, int mode, int64_t* idx, double* scales) {
  std::memcpy(idx, r->idx[mode].data(), sizeof(int64_t) * r->idx[mode].size());
  std::memcpy(scales, r->scales[mode].data(), sizeof(double) * r->scales[mode].size());
  return LMRA_OK;
}
uint64_t lmra_result_num_norms(const lmra_result* r, int mode) { return r->norms[mode].size(); }
int lmra_result_copy_norms(const lmra_result* r, int mode, double* w) {
  std::memcpy(w, r->norms[mode].data(), sizeof(double) * r->norms[mode].size());
  return LMRA_OK;
}
int lmra_result_timings(const lmra_result* r, double* out5) {
  out5[0] = r->t_total;
  out5[1] = r->t_rng;
  out5[2] = r->t_sampling;
  out5[3] = r->t_device;
  out5[4] = r->launches;
  return LMRA_OK;
}
void lmra_result_free(lmra_result* r) { delete r; }

int lmra_result_num_phases(const lmra_result* r) { return (int)r->phases.size(); }
int lmra_result_phase(const lmra_result* r, int i, char* name, size_t name_len, double* ms,
                      int* launches) {
  return guard([&] {
    if (i < 0 || i >= (int)r->phases.size()) throw std::out_of_range("phase index");
    const auto& p = r->phases[i];
    if (name && name_len) {
      std::strncpy(name, p.name.c_str(), name_len - 1);
      name[name_len - 1] = 0;
    }
    *ms = p.ms;
    *launches = p.count;
  });
}

int lmra_context_set_profiling(lmra_context* ctx, int on) {
  return guard([&] { ctx->profile = on < 0 ? 0 : (on > 3 ? 1 : on); });
}

int lmra_context_set_trace(lmra_context* ctx, int on) {
  return guard([&] { ctx->keep_trace = on != 0; });
}

// ------------------------------------------------------------------ primitives
int lmra_mode_n_product(lmra_context* ctx, const double* x, const uint64_t* dims, int order,
                        int mode, const double* b, uint64_t b_rows, double* y) {
  return guard([&] {
    if (mode < 0 || mode >= order) throw std::out_of_range("mode_n_product: mode out of range");
    if (b_rows < 1) throw std::invalid_argument("mode_n_product: empty matrix");
    DeviceGuard dg(ctx->device);
    std::vector<size_t> d(dims, dims + order);
    const size_t I = d[mode];
    Engine eng(ctx);
    DevBuf bt(I * b_rows, ctx->stream);
    eng.launch("transpose", [&] {
      return lmra_dev::launch_transpose(b, (long long)b_rows, (long long)I, bt.get(), ctx->stream);
    });
    eng.launch("ttm", [&] {
      return lmra_dev::launch_ttm(x, view_of(d, (size_t)mode), bt.get(), (int)b_rows, y, ctx->stream);
    });
    ck(cudaStreamSynchronize(ctx->stream), "sync");
  });
}

int lmra_mode0_product_i8(lmra_context* ctx, const double* x, uint64_t K, uint64_t J, const double* q,
                          int mu, const double* w, double* y) {
  return guard([&] {
    if (!lmra_dev::ttm_i8_supported((long long)K, (long long)J, mu, x))
      throw std::invalid_argument("mode0_product_i8: shape not supported (K even <= 4096, mu <= 64)");
    DeviceGuard dg(ctx->device);
    DevBuf work((lmra_dev::ttm_i8_workspace_bytes((long long)K, mu) + 7) / 8, ctx->stream);
    Engine eng(ctx);
    eng.launch("ttm_i8", [&] {
      return lmra_dev::launch_ttm_i8(x, (long long)K, (long long)J, q, mu, w, y, work.get(), ctx->stream);
    });
    ck(cudaStreamSynchronize(ctx->stream), "sync");
  });
}

int lmra_mode1_product_i8(lmra_context* ctx, const double* x, uint64_t R, uint64_t K, uint64_t O,
                          const double* q, int mu, double* y) {
  return guard([&] {
    if (!lmra_dev::ttm_i8_inner_supported((long long)R, (long long)K, (long long)O, mu, x))
      throw std::invalid_argument("mode1_product_i8: shape not supported (R even <= 64, K <= 4096, mu <= 64)");
    DeviceGuard dg(ctx->device);
    DevBuf work((lmra_dev::ttm_i8_workspace_bytes((long long)K, mu) + 7) / 8, ctx->stream);
    DevBuf fexp((R * O + 1) / 2, ctx->stream);
    int* fe = reinterpret_cast<int*>(fexp.get());
    Engine eng(ctx);
    eng.launch("column_exponents", [&] {
      return lmra_dev::launch_column_exponents(x, (long long)R, (long long)K, (long long)O, fe, ctx->stream);
    });
    eng.launch("ttm_i8", [&] {
      return lmra_dev::launch_ttm_i8_inner(x, (long long)R, (long long)K, (long long)O, q, mu, fe, y, work.get(),
                                           ctx->stream);
    });
    ck(cudaStreamSynchronize(ctx->stream), "sync");
  });
}

int lmra_gram_power_apply(lmra_context* ctx, const double* a, uint64_t rows, uint64_t cols,
                          const double* g, uint64_t s, int q, int strategy, double* c) {
  return guard([&] {
    if (q < 1) throw std::invalid_argument("gram_power_apply: q must be >= 1");
    DeviceGuard dg(ctx->device);
    Engine eng(ctx);
    DevBuf cb(rows * s, ctx->stream);
    ck(cudaMemcpyAsync(cb.get(), g, rows * s * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream),
       "copy");
    eng.gram_power(a, ModeView{1, (long long)rows, (long long)cols}, cb, s, q, strategy);
    ck(cudaMemcpyAsync(c, cb.get(), rows * s * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream),
       "copy");
    ck(cudaStreamSynchronize(ctx->stream), "sync");
  });
}

int lmra_leading_left_singular_vectors(lmra_context* ctx, const double* c, uint64_t rows,
                                       uint64_t cols, uint64_t mu, double* u) {
  return guard([&] {
    if (mu < 1 || mu > std::min(rows, cols))
      throw std::invalid_argument("leading_left_singular_vectors: mu out of range");
    if (rows < cols) throw std::invalid_argument("leading_left_singular_vectors: needs rows >= cols");
    DeviceGuard dg(ctx->device);
    Engine eng(ctx);
    DevBuf status(1, ctx->stream);
    ck(cudaMemsetAsync(status.get(), 0, sizeof(double), ctx->stream), "memset");
    DevBuf out = eng.orth(c, rows, cols, mu, reinterpret_cast<int*>(status.get()));
    ck(cudaMemcpyAsync(u, out.get(), rows * mu * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream),
       "copy");
    int st = 0;
    ck(cudaMemcpyAsync(&st, status.get(), sizeof(int), cudaMemcpyDeviceToHost, ctx->stream), "D2H");
    ck(cudaStreamSynchronize(ctx->stream), "sync");
    if (st) throw std::runtime_error("thin_svd: SVD iteration did not converge");
  });
}

int lmra_tnsr_read_header(const char* path, int* order, uint64_t* dims, int max_order) {
  return guard([&] {
    const lmra_host::TnsrHeader h = lmra_host::tnsr_read_header(path);
    *order = (int)h.dims.size();
    for (int k = 0; k < std::min(max_order, *order); ++k) dims[k] = h.dims[k];
  });
}

int lmra_tnsr_load(lmra_context* ctx, const char* path, double* dst, int dst_location) {
  return guard([&] {
    if (dst_location == LMRA_HOST) {
      lmra_host::tnsr_load_host(path, dst);
      return;
    }
    if (!ctx) throw std::invalid_argument("null context");
    DeviceGuard dg(ctx->device);
    lmra_host::tnsr_load_device(path, dst, ctx->stream);
  });
}

int lmra_tnsr_save(lmra_context* ctx, const char* path, const double* src, int src_location,
                   const uint64_t* dims, int order) {
  return guard([&] {
    if (order < 0) throw std::invalid_argument("negative tensor order");
    std::vector<uint64_t> d(dims, dims + order);
    if (src_location == LMRA_HOST) {
      lmra_host::tnsr_save(path, d, src, false, nullptr);
      return;
    }
    if (!ctx) throw std::invalid_argument("null context");
    DeviceGuard dg(ctx->device);
    lmra_host::tnsr_save(path, d, src, true, ctx->stream);
  });
}

int lmra_thin_qr_q(lmra_context* ctx, const double* c, uint64_t rows, uint64_t cols, double* q) {
  return guard([&] {
    if (rows < cols) throw std::invalid_argument("thin_qr: requires rows >= cols");
    if (cols < 1 || cols > (uint64_t)lmra_dev::kMaxWidth)
      throw std::invalid_argument("thin_qr: 1 to 64 columns");
    DeviceGuard dg(ctx->device);
    Engine eng(ctx);
    DevBuf w(lmra_dev::thin_q_workspace_doubles((long long)rows, (int)cols), ctx->stream);
    eng.launch("qr_thin_q", [&] {
      return lmra_dev::launch_thin_q(c, (long long)rows, (int)cols, q, w.get(), ctx->stream);
    });
    ck(cudaStreamSynchronize(ctx->stream), "sync");
  });
}

int lmra_qr_project_extract(lmra_context* ctx, const double* c, uint64_t rows, uint64_t cols,
                            const double* a, uint64_t a_cols, uint64_t mu, double* out) {
  return guard([&] {
    if (mu < 1 || mu > cols) throw std::invalid_argument("qr_project_extract: mu out of range");
    if (rows < cols) throw std::invalid_argument("thin_qr: requires rows >= cols");
    if (cols > (uint64_t)lmra_dev::kMaxWidth) throw std::invalid_argument("qr_project_extract: more than 64 columns");
    if (mu > std::min(cols, a_cols))
      throw std::invalid_argument("leading_left_singular_vectors: mu out of range");
    DeviceGuard dg(ctx->device);
    Engine eng(ctx);
    DevBuf status(1, ctx->stream);
    ck(cudaMemsetAsync(status.get(), 0, sizeof(double), ctx->stream), "memset");
    Engine::QrProxy r = eng.qr_extract(a, {(size_t)rows, (size_t)a_cols}, 0, c, cols, mu,
                                       reinterpret_cast<int*>(status.get()));
    ck(cudaMemcpyAsync(out, r.f.get(), rows * mu * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream),
       "copy");
    int st = 0;
    ck(cudaMemcpyAsync(&st, status.get(), sizeof(int), cudaMemcpyDeviceToHost, ctx->stream), "D2H");
    ck(cudaStreamSynchronize(ctx->stream), "sync");
    if (st) throw std::runtime_error("thin_svd: SVD iteration did not converge");
  });
}

int lmra_column_sqnorms(lmra_context* ctx, const double* x, const uint64_t* dims, int order,
                        int mode, double* w) {
  return guard([&] {
    if (mode < 0 || mode >= order) throw std::out_of_range("mode out of range");
    DeviceGuard dg(ctx->device);
    std::vector<size_t> d(dims, dims + order);
    Engine eng(ctx);
    eng.launch("norms", [&] {
      return lmra_dev::launch_column_sqnorms(x, view_of(d, (size_t)mode), w, ctx->stream);
    });
    ck(cudaStreamSynchronize(ctx->stream), "sync");
  });
}

// diagnostics: [certified chunks, element-exact chunks] of the exact scans since last reset
int lmra_debug_sampler_stats(unsigned long long* out2, int reset) {
  lmra_dev::sampler_walk_stats(out2, reset != 0);
  return LMRA_OK;
}

int lmra_sample_columns_device(lmra_context* ctx, const double* w, uint64_t n, int regime,
                               double beta, uint64_t L, uint64_t seed, uint64_t stream,
                               int64_t* idx, double* scales, double* p) {
  return guard([&] {
    if (n < 1) throw std::invalid_argument("probability distribution must be nonempty");
    if (L < 1) throw std::invalid_argument("randsample: L must be positive");
    if (regime < 0 || regime > 2) throw std::invalid_argument("unknown probability regime");
    DeviceGuard dg(ctx->device);
    Engine eng(ctx);
    DevBuf work(lmra_dev::sampler_workspace_doubles((long long)n), ctx->stream);
    DevBuf status(1, ctx->stream);
    ck(cudaMemsetAsync(status.get(), 0, sizeof(double), ctx->stream), "memset");
    const double* wv = w;
    DevBuf dummy;
    if (regime == 2) {  // uniform never reads w
      dummy = DevBuf(n, ctx->stream);
      wv = dummy.get();
    }
    eng.launch("sampler", [&] {
      return lmra_dev::launch_sampler(wv, (long long)n, regime, beta, (long long)L, seed, stream,
                                      reinterpret_cast<long long*>(idx), scales, p, work.get(),
                                      reinterpret_cast<int*>(status.get()), ctx->stream);
    });
    int f = 0;
    ck(cudaMemcpyAsync(&f, status.get(), sizeof(int), cudaMemcpyDeviceToHost, ctx->stream), "D2H");
    ck(cudaStreamSynchronize(ctx->stream), "sync");
    if (f & 1) throw std::invalid_argument("probability weights must be nonnegative");
    if (f & 32) throw std::invalid_argument("nearly-optimal mixture weight must lie in (0, 1]");
    if (f & 2) throw std::invalid_argument("cannot normalize an all-zero distribution");
    if (f & 4) throw std::invalid_argument("probability weights must sum to one");
    if (f & 8) throw std::invalid_argument("randsample: all-zero distribution");
  });
}

int lmra_gaussian_matrix(uint64_t rows, uint64_t cols, uint64_t seed, uint64_t stream,
                         double* out) {
  return guard([&] {
    if (rows < 1 || cols < 1) throw std::invalid_argument("gaussian_matrix: shape must be positive");
    lmra_host::fill_normals(seed, stream, out, rows * cols, lmra_host::host_threads());
  });
}

int lmra_probabilities(const double* w, uint64_t n, int regime, double beta, double* p) {
  return guard([&] {
    std::vector<double> v(w, w + n);
    auto out = lmra_host::probabilities_from_norms(std::move(v), regime, beta);
    std::memcpy(p, out.data(), sizeof(double) * n);
  });
}

int lmra_randsample(uint64_t L, const double* p, uint64_t n, uint64_t seed, uint64_t stream,
                    int64_t* idx, double* scales) {
  return guard([&] {
    std::vector<double> pv(p, p + n);
    lmra_host::check_distribution(pv);
    auto s = lmra_host::randsample(L, pv, seed, stream);
    std::memcpy(idx, s.idx.data(), sizeof(int64_t) * L);
    std::memcpy(scales, s.scales.data(), sizeof(double) * L);
  });
}

int lmra_amm_sample_counts(const uint64_t* dims, int order, const lmra_algo_config* cfg,
                           int sequential, uint64_t* out) {
  return guard([&] {
    std::vector<size_t> d(dims, dims + order);
    auto c = lmra_host::amm_sample_counts(d, to_config(cfg), sequential != 0);
    for (int n = 0; n < order; ++n) out[n] = c[n];
  });
}

// ------------------------------------------------------------------ generators
// Definitions: gen/portable_gen.hpp (bit-identical to the host generators of the oracle).
// Every generator writes the slab [start, start + count) of the last mode (the whole tensor
// for start = 0, count = dims[N-1]); a multi-GPU rank generates only its own slab.
namespace {
struct GenShape {
  std::vector<size_t> d;
  size_t L = 0, slice = 1, start = 0, count = 0;
};
GenShape gen_shape(const uint64_t* dims, int order, uint64_t start, uint64_t count) {
  if (order < 1 || order > 8) throw std::invalid_argument("generator: order must be 1..8");
  GenShape g;
  g.d.assign(dims, dims + order);
  for (size_t v : g.d)
    if (v == 0) throw std::invalid_argument("tensor dimension must be positive");
  g.L = g.d.back();
  for (int k = 0; k + 1 < order; ++k) g.slice *= g.d[k];
  if (start > g.L || count > g.L - start) throw std::invalid_argument("generator: slab out of range");
  g.start = start;
  g.count = count;
  return g;
}
}  // namespace

int lmra_gen_hilbert_slab(lmra_context* ctx, const uint64_t* dims, int order, uint64_t start, uint64_t count,
                          double* x) {
  return guard([&] {
    const GenShape g = gen_shape(dims, order, start, count);
    DeviceGuard dg(ctx->device);
    std::vector<long long> d(g.d.begin(), g.d.end());
    ck(lmra_dev::launch_gen_hilbert(x, d.data(), order, (long long)start, (long long)count, ctx->stream),
       "gen_hilbert");
    ck(cudaStreamSynchronize(ctx->stream), "sync");
  });
}

int lmra_gen_hilbert(lmra_context* ctx, const uint64_t* dims, int order, double* x) {
  if (order < 1) return lmra_gen_hilbert_slab(ctx, dims, order, 0, 0, x);
  return lmra_gen_hilbert_slab(ctx, dims, order, 0, dims[order - 1], x);
}

int lmra_gen_tucker_signal_slab(lmra_context* ctx, const uint64_t* dims, const uint64_t* core_dims, int order,
                                uint64_t seed, uint64_t start, uint64_t count, double* x, double* slice_b,
                                double* slice_e) {
  return guard([&] {
    using namespace lmra_gen;
    const GenShape g = gen_shape(dims, order, start, count);
    if (order == 1 && (start != 0 || count != g.L)) throw std::invalid_argument("generator: an order-1 slab is the whole tensor");
    std::vector<size_t> cd(core_dims, core_dims + order);
    for (int n = 0; n < order; ++n)
      if (cd[n] < 1 || cd[n] > g.d[n]) throw std::invalid_argument("core dimensions must lie in [1, I_n]");
    DeviceGuard dg(ctx->device);
    cudaStream_t st = ctx->stream;
    // host halves: G (stream 100) and the orthonormal factors U_n (stream 101 + n)
    std::vector<double> hg(prod(cd));
    gp_normals_range(seed, kStreamCore, hg.data(), 0, hg.size());
    std::vector<std::vector<double>> hu(order);
    for (int n = 0; n < order; ++n) {
      hu[n].resize(g.d[n] * cd[n]);
      gp_orthonormal_factor(g.d[n], cd[n], seed, (uint64_t)n, hu[n].data());
    }
    // B = G x_0 U_0 x_1 U_1 ... (mode order), the last product only for the slab's rows
    Engine eng(ctx);
    DevBuf cur = eng.upload(hg.data(), hg.size());
    std::vector<size_t> cdim = cd;
    for (int n = 0; n < order; ++n) {
      DevBuf u = eng.upload(hu[n].data(), hu[n].size());
      const bool last = n == order - 1;
      const size_t rows = last ? g.count : g.d[n];
      long long inner = 1, outer = 1;
      for (int k = 0; k < n; ++k) inner *= (long long)cdim[k];
      for (int k = n + 1; k < order; ++k) outer *= (long long)cdim[k];
      double* dst = nullptr;
      DevBuf y;
      if (last) {
        dst = x;
      } else {
        y = DevBuf((size_t)inner * rows * (size_t)outer, st);
        dst = y.get();
      }
      ck(lmra_dev::launch_gen_ttm(cur.get(), inner, (long long)cd[n], (long long)rows, outer,
                                  u.get() + (last ? g.start : 0), (long long)g.d[n], dst, st),
         "gen_ttm");
      cdim[n] = g.d[n];
      if (!last) cur = std::move(y);
      ck(cudaStreamSynchronize(st), "sync");  // u / cur are released at the end of the iteration
    }
    // per-slice sums of squares of B and of the noise E (stream 200, regenerated)
    const size_t d0 = g.d[0];
    const size_t local = g.slice * g.count;
    const size_t nfib = local / d0, per = g.slice / d0;
    const size_t sl = order == 1 ? 1 : g.count;  // an order-1 tensor is one slice
    const size_t perf = order == 1 ? nfib : per;
    DevBuf fb(nfib, st), fe(nfib, st), sb(sl, st), se(sl, st);
    ck(lmra_dev::launch_gen_fiber_sumsq(x, (long long)d0, (long long)nfib, fb.get(), st), "fiber sumsq");
    ck(lmra_dev::launch_gen_noise_fiber_sumsq(seed, kStreamNoise, (long long)(g.start * g.slice), (long long)d0,
                                              (long long)nfib, fe.get(), st),
       "noise sumsq");
    ck(lmra_dev::launch_gen_slice_sum(fb.get(), (long long)perf, (long long)sl, sb.get(), st), "slice sum");
    ck(lmra_dev::launch_gen_slice_sum(fe.get(), (long long)perf, (long long)sl, se.get(), st), "slice sum");
    ck(cudaMemcpyAsync(slice_b, sb.get(), sl * sizeof(double), cudaMemcpyDeviceToHost, st), "D2H");
    ck(cudaMemcpyAsync(slice_e, se.get(), sl * sizeof(double), cudaMemcpyDeviceToHost, st), "D2H");
    ck(cudaStreamSynchronize(st), "sync");
  });
}

int lmra_gen_noise_coef(const double* slice_b, const double* slice_e, uint64_t nslices, double gamma,
                        double* coef) {
  return guard([&] { *coef = lmra_gen::gp_noise_coef(slice_b, slice_e, nslices, gamma); });
}

int lmra_gen_add_noise_slab(lmra_context* ctx, const uint64_t* dims, int order, uint64_t seed, uint64_t start,
                            uint64_t count, double coef, double* x) {
  return guard([&] {
    const GenShape g = gen_shape(dims, order, start, count);
    DeviceGuard dg(ctx->device);
    ck(lmra_dev::launch_gen_add_noise(x, (long long)(g.slice * g.count), (long long)(g.start * g.slice), coef,
                                      seed, lmra_gen::kStreamNoise, ctx->stream),
       "add noise");
    ck(cudaStreamSynchronize(ctx->stream), "sync");
  });
}

int lmra_gen_tucker_noise(lmra_context* ctx, const uint64_t* dims, const uint64_t* core_dims, int order,
                          double gamma, uint64_t seed, double* x) {
  return guard([&] {
    if (order < 1) throw std::invalid_argument("generator: order must be 1..8");
    const uint64_t L = dims[order - 1];
    const size_t sl = order == 1 ? 1 : L;
    std::vector<double> sb(sl), se(sl);
    auto rethrow = [](int rc) {  // keep the error class of the step that failed
      if (rc == LMRA_EINVAL) throw std::invalid_argument(g_err);
      if (rc == LMRA_ECUDA) throw CudaError(g_err);
      if (rc != LMRA_OK) throw std::runtime_error(g_err);
    };
    rethrow(lmra_gen_tucker_signal_slab(ctx, dims, core_dims, order, seed, 0, L, x, sb.data(), se.data()));
    const double coef = lmra_gen::gp_noise_coef(sb.data(), se.data(), sl, gamma);
    rethrow(lmra_gen_add_noise_slab(ctx, dims, order, seed, 0, L, coef, x));
  });
}

int lmra_gen_video_slab(lmra_context* ctx, const uint64_t* dims, int order, uint64_t n_terms, double noise,
                        uint64_t seed, uint64_t start, uint64_t count, double* x) {
  return guard([&] {
    const GenShape g = gen_shape(dims, order, start, count);
    if (n_terms < 1) throw std::invalid_argument("video generator: n_terms must be positive");
    DeviceGuard dg(ctx->device);
    cudaStream_t st = ctx->stream;
    size_t tot = 0;
    for (size_t v : g.d) tot += v * n_terms;
    std::vector<double> prof(tot), w(n_terms);
    lmra_gen::gp_video_profiles(dims, order, n_terms, seed, prof.data(), w.data());
    Engine eng(ctx);
    DevBuf dp = eng.upload(prof.data(), tot), dw = eng.upload(w.data(), n_terms);
    std::vector<long long> dl(g.d.begin(), g.d.end());
    ck(lmra_dev::launch_gen_video(x, dl.data(), order, (long long)start, (long long)count, dp.get(), dw.get(),
                                  (int)n_terms, noise, seed, lmra_gen::kStreamVideoNoise, st),
       "gen_video");
    ck(cudaStreamSynchronize(st), "sync");
  });
}

int lmra_gen_video(lmra_context* ctx, const uint64_t* dims, int order, uint64_t n_terms, double noise,
                   uint64_t seed, double* x) {
  if (order < 1) return lmra_gen_video_slab(ctx, dims, order, n_terms, noise, seed, 0, 0, x);
  return lmra_gen_video_slab(ctx, dims, order, n_terms, noise, seed, 0, dims[order - 1], x);
}

// ------------------------------------------------------------------ verification
// reconstruct (tucker.cpp:222-227): core x_0 Q_0 x_1 Q_1 ... (mode order), into out
static void reconstruct_into(lmra_context* ctx, const double* core, const std::vector<size_t>& cdims,
                             const std::vector<const double*>& factors, const std::vector<size_t>& rows,
                             double* out) {
  cudaStream_t st = ctx->stream;
  Engine eng(ctx);
  const size_t N = cdims.size();
  std::vector<size_t> cur = cdims;
  DevBuf t;
  const double* src = core;
  if (N == 0) {
    ck(cudaMemcpyAsync(out, core, sizeof(double), cudaMemcpyDeviceToDevice, st), "copy");
    return;
  }
  for (size_t n = 0; n < N; ++n) {
    const size_t mu = cur[n], I = rows[n];
    DevBuf qt(I * mu, st);
    eng.launch("transpose", [&] {
      return lmra_dev::launch_transpose(factors[n], (long long)I, (long long)mu, qt.get(), st);
    });
    std::vector<size_t> od = cur;
    od[n] = I;
    const bool last = n + 1 == N;
    DevBuf y;
    double* dst = last ? out : nullptr;
    if (!last) {
      y = DevBuf(prod(od), st);
      dst = y.get();
    }
    eng.launch("reconstruct", [&] { return lmra_dev::launch_ttm(src, view_of(cur, n), qt.get(), (int)I, dst, st); });
    ck(cudaStreamSynchronize(st), "sync");
    cur = od;
    if (!last) {
      t = std::move(y);
      src = t.get();
    }
  }
}

static double relative_error_dev(lmra_context* ctx, const double* a, const double* r, size_t n) {
  cudaStream_t st = ctx->stream;
  DevBuf work(lmra_dev::diff_sumsq_workspace_doubles(), st), out(2, st);
  ck(lmra_dev::launch_diff_sumsq(a, r, (long long)n, work.get(), out.get(), st), "diff_sumsq");
  double h[2];
  ck(cudaMemcpyAsync(h, out.get(), sizeof(h), cudaMemcpyDeviceToHost, st), "D2H");
  ck(cudaStreamSynchronize(st), "sync");
  if (h[1] == 0.0) throw std::invalid_argument("relative_error: zero reference tensor");
  return std::sqrt(h[0] / h[1]);
}

// stages a host buffer on the device (or returns the device pointer as is)
static const double* staged(lmra_context* ctx, const double* p, size_t n, int loc, DevBuf& keep) {
  if (loc == LMRA_DEVICE) return p;
  keep = DevBuf(n, ctx->stream);
  ck(cudaMemcpyAsync(keep.get(), p, n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream), "H2D");
  return keep.get();
}

int lmra_reconstruct(lmra_context* ctx, const double* core, const uint64_t* core_dims, int order,
                     const double* const* factors, const uint64_t* factor_rows, int location, double* out,
                     int out_location) {
  return guard([&] {
    if (!ctx) throw std::invalid_argument("null context");
    if (order < 0) throw std::invalid_argument("negative tensor order");
    DeviceGuard dg(ctx->device);
    std::vector<size_t> cd(core_dims, core_dims + order), rows(factor_rows, factor_rows + order);
    std::vector<DevBuf> keep(order + 1);
    const double* c = staged(ctx, core, prod(cd), location, keep[order]);
    std::vector<const double*> f(order);
    for (int n = 0; n < order; ++n) f[n] = staged(ctx, factors[n], rows[n] * cd[n], location, keep[n]);
    const size_t total = prod(rows);
    DevBuf tmp;
    double* dst = out;
    if (out_location == LMRA_HOST) {
      tmp = DevBuf(total, ctx->stream);
      dst = tmp.get();
    }
    reconstruct_into(ctx, c, cd, f, rows, dst);
    if (out_location == LMRA_HOST)
      ck(cudaMemcpyAsync(out, dst, total * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream), "D2H");
    ck(cudaStreamSynchronize(ctx->stream), "sync");
  });
}

int lmra_relative_error(lmra_context* ctx, const double* a, const double* approx, const uint64_t* dims, int order,
                        int location, double* re) {
  return guard([&] {
    if (!ctx) throw std::invalid_argument("null context");
    DeviceGuard dg(ctx->device);
    std::vector<size_t> d(dims, dims + order);
    const size_t n = prod(d);
    DevBuf ka, kr;
    const double* da = staged(ctx, a, n, location, ka);
    const double* dr = staged(ctx, approx, n, location, kr);
    *re = relative_error_dev(ctx, da, dr, n);
  });
}

int lmra_result_relative_error(lmra_context* ctx, const lmra_result* r, const double* a, const uint64_t* dims,
                               int order, int location, double* re) {
  return guard([&] {
    if (!ctx || !r) throw std::invalid_argument("null context or result");
    if ((size_t)order != r->factors.size()) throw std::invalid_argument("relative_error: shape mismatch");
    std::vector<size_t> d(dims, dims + order);
    for (int n = 0; n < order; ++n)
      if (r->f_rows[n] != d[n]) throw std::invalid_argument("relative_error: shape mismatch");
    DeviceGuard dg(ctx->device);
    const size_t n = prod(d);
    DevBuf ka;
    const double* da = staged(ctx, a, n, location, ka);
    DevBuf rec(n, ctx->stream);
    std::vector<const double*> f(r->factors.begin(), r->factors.end());
    reconstruct_into(ctx, r->core, r->core_dims, f, r->f_rows, rec.get());
    *re = relative_error_dev(ctx, da, rec.get(), n);
  });
}

int lmra_device_alloc(lmra_context* ctx, size_t bytes, void** out) {
  return guard([&] {
    DeviceGuard dg(ctx->device);
    ck(cudaMalloc(out, std::max<size_t>(bytes, 16)), "cudaMalloc");
  });
}

int lmra_device_free(lmra_context* ctx, void* p) {
  return guard([&] {
    DeviceGuard dg(ctx->device);
    ck(cudaFree(p), "cudaFree");
  });
}

int lmra_memcpy(lmra_context* ctx, void* dst, const void* src, size_t bytes, int dst_location,
                int src_location) {
  return guard([&] {
    DeviceGuard dg(ctx->device);
    cudaMemcpyKind k = src_location == LMRA_HOST
                           ? (dst_location == LMRA_HOST ? cudaMemcpyHostToHost : cudaMemcpyHostToDevice)
                           : (dst_location == LMRA_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice);
    ck(cudaMemcpyAsync(dst, src, bytes, k, ctx->stream), "memcpy");
    ck(cudaStreamSynchronize(ctx->stream), "sync");
  });
}

}  // extern "C"

extern "C" int lmra_debug_jacobi_sweeps(void) { return lmra_dev::last_jacobi_sweeps(); }
extern "C" void lmra_debug_orth_clocks(long long* out7) { lmra_dev::last_orth_clocks(out7); }

namespace lmra_dev {  // scratch of the launchers (kernels.hpp)
cudaError_t scratch_alloc(void** p, size_t bytes, cudaStream_t st) {
  if ((*p = arena_take(bytes))) return cudaSuccess;
  return cudaMallocAsync(p, bytes, st);
}
void scratch_free(void* p, cudaStream_t st) {
  if (p && !in_arena(p)) cudaFreeAsync(p, st);
}
}  // namespace lmra_dev

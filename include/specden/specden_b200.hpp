// specden_b200.hpp — C++ drop-in for the reference's specden API
// (proj/include/specden/{errors,precision,rng,layout,reduction,pool,sharded,
// operators}.hpp and the SPEC-only lanczos_run / ritz_decompose / hvp),
// header-only over the C-ABI of include/specden_b200.h. The reference's
// module headers (specden/pool.hpp, specden/sharded.hpp, ...) in this
// directory forward here, so reference callers -- and the reference's own
// doctest suites (proj/tests/*.cpp), built unchanged against this header by
// oracle/build_dropin_tests.sh -- compile as they are.
//
// B200 mapping:
//  * WorkerPool (pool.hpp:47-94): n worker threads with FIFO mailboxes, one
//    exactly-once reply per message, per-kind counters, the jitter test hook.
//    Worker w owns CUDA device worker_device(w) = w mod (visible devices) and
//    one stream on it; its shard of every ShardedVector lives on that device.
//  * Every vector operation is one message per worker (the reference's
//    message pattern: DotPartial, Axpy, Scale, Gather, Scatter, ApplyShard)
//    whose work is an sm_100a kernel on the worker's stream; dot partials are
//    the fixed 1024-block folds, folded by the coordinator in worker order
//    (combine_blocked, reduction.hpp:76-107) -- bitwise the reference.
//  * lanczos_run on an engine-native operator runs the device Lanczos engine
//    on the workers' own threads and devices, one rank per worker, exchanging
//    f64 partials through an in-process communicator; an operator given only
//    by apply_fn runs the SPEC recurrence composed from the vector ops.
// Streams are created blocking (cudaStreamCreate), so the legacy default
// stream orders with them; every op synchronises its stream before replying.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <atomic>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <deque>
#include <fstream>
#include <functional>
#include <future>
#include <map>
#include <memory>
#include <mutex>
#include <numbers>
#include <random>
#include <span>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "specden_b200.h"

namespace specden {

// ---------------------------------------------------------------- errors
// errors.hpp:13-41 (same six classes; device_error for CUDA/NCCL failures)
#define SPECDEN_ERROR_CLASS(name) \
  struct name : std::runtime_error { \
    explicit name(const std::string& w) : std::runtime_error(w) {} \
  }
SPECDEN_ERROR_CLASS(config_error);
SPECDEN_ERROR_CLASS(layout_error);
SPECDEN_ERROR_CLASS(argument_error);
SPECDEN_ERROR_CLASS(numerical_error);
SPECDEN_ERROR_CLASS(state_error);
SPECDEN_ERROR_CLASS(protocol_error);
SPECDEN_ERROR_CLASS(device_error);
#undef SPECDEN_ERROR_CLASS

[[noreturn]] inline void throw_status(sd_status s, const std::string& m) {
  switch (s) {
    case SD_CONFIG_ERROR: throw config_error(m);
    case SD_LAYOUT_ERROR: throw layout_error(m);
    case SD_ARGUMENT_ERROR: throw argument_error(m);
    case SD_NUMERICAL_ERROR: throw numerical_error(m);
    case SD_STATE_ERROR: throw state_error(m);
    case SD_PROTOCOL_ERROR: throw protocol_error(m);
    default: throw device_error(m);
  }
}
inline void check(sd_status s) {
  if (s != SD_OK) throw_status(s, sd_last_error());
}
inline void cuda_ok(cudaError_t e) {
  if (e != cudaSuccess) throw device_error(cudaGetErrorString(e));
}

// ------------------------------------------------------------- precision
// precision.hpp:15-34
enum class Precision { f32, f64 };
inline int prec_code(Precision p) { return p == Precision::f32 ? SD_F32 : SD_F64; }
inline double round_elem(double x, Precision p) { return p == Precision::f32 ? double(float(x)) : x; }
inline double unit_roundoff(Precision p) { return p == Precision::f32 ? 0x1p-24 : 0x1p-53; }
inline const char* precision_name(Precision p) { return p == Precision::f32 ? "f32" : "f64"; }
inline Precision parse_precision(const std::string& s) {
  if (s == "f32") return Precision::f32;
  if (s == "f64") return Precision::f64;
  throw config_error("unknown precision '" + s + "' (expected f32 or f64)");
}

// ------------------------------------------------------------------- rng
// rng.hpp:17-52: counter-based draws, a pure function of (seed, counter).
// Host copies (tests, setup); the device kernels use the same integer path.
inline std::uint64_t mix64(std::uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
inline std::uint64_t keyed_counter(std::uint64_t seed, std::uint64_t counter) { return sd_keyed_counter(seed, counter); }
inline double uniform01(std::uint64_t seed, std::uint64_t counter) {
  return double(keyed_counter(seed, counter) >> 11) * 0x1p-53 + 0x1p-54;
}
inline double gaussian(std::uint64_t seed, std::uint64_t i) {
  constexpr double two_pi = 2.0 * std::numbers::pi;  // exact doubling
  const double r = std::sqrt(-2.0 * std::log(uniform01(seed, 2 * i)));
  return r * std::cos(two_pi * uniform01(seed, 2 * i + 1));
}
inline double rademacher(std::uint64_t seed, std::uint64_t i) { return sd_rademacher(seed, i); }
inline std::uint64_t uniform_index(std::uint64_t seed, std::uint64_t i, std::uint64_t n) {
  return sd_uniform_index(seed, i, n);
}

// ---------------------------------------------------------------- layout
// layout.hpp:12-72
struct ShardRange {
  std::size_t begin = 0, end = 0;
  std::size_t size() const { return end - begin; }
};
struct ShardLayout {
  std::size_t total_dim = 0;
  std::vector<ShardRange> shard_bounds;
  std::size_t worker_count() const { return shard_bounds.size(); }
  std::vector<uint64_t> begins() const {
    std::vector<uint64_t> b;
    for (auto& r : shard_bounds) b.push_back(r.begin);
    return b;
  }
  std::vector<uint64_t> ends() const {
    std::vector<uint64_t> e;
    for (auto& r : shard_bounds) e.push_back(r.end);
    return e;
  }
  std::size_t owner(std::size_t i) const {
    uint64_t o = 0;
    const auto e = ends();
    check(sd_layout_owner(e.size(), e.data(), i, &o));
    return std::size_t(o);
  }
  bool operator==(const ShardLayout& o) const {
    if (total_dim != o.total_dim || shard_bounds.size() != o.shard_bounds.size()) return false;
    for (std::size_t w = 0; w < shard_bounds.size(); ++w)
      if (shard_bounds[w].begin != o.shard_bounds[w].begin || shard_bounds[w].end != o.shard_bounds[w].end)
        return false;
    return true;
  }
};
inline void validate_layout(const ShardLayout& l) {
  const auto b = l.begins(), e = l.ends();
  check(sd_validate_layout(l.total_dim, b.size(), b.data(), e.data()));
}
inline ShardLayout split_evenly(std::size_t dim, std::size_t n) {
  if (dim == 0 || n == 0) throw layout_error("split_evenly needs dim > 0 and n > 0");
  std::vector<uint64_t> b(n), e(n);
  uint64_t cnt = 0;
  check(sd_split_evenly(dim, n, b.data(), e.data(), &cnt));
  ShardLayout l;
  l.total_dim = dim;
  for (uint64_t i = 0; i < cnt; ++i) l.shard_bounds.push_back({std::size_t(b[i]), std::size_t(e[i])});
  return l;
}

// ------------------------------------------------------------- reduction
// reduction.hpp:30-115: the fixed global block grid. Host forms for callers
// that build partials themselves; the library's device partials follow the
// same DAG (sd_k_dot_partial + sd_combine_partials_host).
inline constexpr std::size_t kReduceBlock = 1024;
inline double fold_left(std::span<const double> xs) {
  double acc = 0.0;
  for (double x : xs) acc += x;
  return acc;
}
struct BlockedPartial {
  std::size_t begin = 0, end = 0;
  std::vector<double> head, sums, tail;
};
template <class TermFn>
BlockedPartial make_blocked_partial(std::size_t begin, std::size_t end, std::size_t total, TermFn&& term,
                                    std::size_t block = kReduceBlock) {
  BlockedPartial p;
  p.begin = begin;
  p.end = end;
  std::size_t i = begin;
  const std::size_t head_end = std::min(end, (begin + block - 1) / block * block);
  while (i < head_end) p.head.push_back(term(i++));
  // whole blocks [i, min(i + block, total)) that end inside [begin, end)
  for (std::size_t blk = std::min(i + block, total); i < end && blk <= end; blk = std::min(i + block, total)) {
    double acc = 0.0;
    while (i < blk) acc += term(i++);
    p.sums.push_back(acc);
  }
  while (i < end) p.tail.push_back(term(i++));
  return p;
}
inline double combine_blocked(const std::vector<BlockedPartial>& parts, std::size_t total,
                              std::size_t block = kReduceBlock) {
  double closed = 0.0, open = 0.0;
  std::size_t at = 0;
  const auto next_edge = [&](std::size_t i) { return std::min((i / block + 1) * block, total); };
  const auto feed = [&](double t) {
    const std::size_t edge = next_edge(at);
    open += t;
    if (++at == edge) {
      closed += open;
      open = 0.0;
    }
  };
  for (const BlockedPartial& p : parts) {
    if (p.begin != at) throw protocol_error("blocked partials are not contiguous in worker order");
    for (double t : p.head) feed(t);
    for (double s : p.sums) {
      if (at % block) throw protocol_error("blocked partial misaligned with the reduction grid");
      closed += s;
      at = next_edge(at);
    }
    for (double t : p.tail) feed(t);
    if (at != p.end) throw protocol_error("blocked partial does not cover its range");
  }
  if (at != total) throw protocol_error("blocked partials do not cover the vector");
  return closed;
}
inline double reduce_ordered(std::span<const double> partials) { return fold_left(partials); }

// --------------------------------------------------------------- devices
inline int device_count() {
  static const int n = [] {
    int c = 0;
    if (cudaGetDeviceCount(&c) != cudaSuccess || c < 1) throw device_error("no CUDA device visible");
    return c;
  }();
  return n;
}
// the device that owns worker / shard w (round robin over the visible devices)
inline int worker_device(std::size_t w) { return int(w % std::size_t(device_count())); }

struct DeviceGuard {
  int prev = 0;
  explicit DeviceGuard(int dev) {
    cuda_ok(cudaGetDevice(&prev));
    if (prev != dev) cuda_ok(cudaSetDevice(dev));
  }
  ~DeviceGuard() { cudaSetDevice(prev); }
};

// RAII device allocation on a given device
class DeviceBuffer {
 public:
  DeviceBuffer() = default;
  explicit DeviceBuffer(std::size_t bytes, int device = -1) : bytes_(bytes) {
    if (device < 0) cuda_ok(cudaGetDevice(&device));
    dev_ = device;
    if (bytes) {
      DeviceGuard g(dev_);
      cuda_ok(cudaMalloc(&p_, bytes));
    }
  }
  DeviceBuffer(const DeviceBuffer& o) : DeviceBuffer(o.bytes_, o.dev_) {
    if (bytes_) cuda_ok(cudaMemcpy(p_, o.p_, bytes_, cudaMemcpyDefault));
  }
  DeviceBuffer(DeviceBuffer&& o) noexcept { swap(o); }
  DeviceBuffer& operator=(DeviceBuffer o) noexcept {
    swap(o);
    return *this;
  }
  ~DeviceBuffer() {
    if (p_) {
      DeviceGuard g(dev_);
      cudaFree(p_);
    }
  }
  void* get() const { return p_; }
  std::size_t bytes() const { return bytes_; }
  int device() const { return dev_; }

 private:
  void swap(DeviceBuffer& o) noexcept {
    std::swap(p_, o.p_);
    std::swap(bytes_, o.bytes_);
    std::swap(dev_, o.dev_);
  }
  void* p_ = nullptr;
  std::size_t bytes_ = 0;
  int dev_ = 0;
};

// One shard of a ShardedVector: device storage in the vector's precision
// (f32 shards hold floats -- exactly the reference's f32-representable
// doubles) with element access through the host, as the reference's
// std::vector<double> shards offer (sharded.hpp:17-22).
class DeviceShard {
 public:
  class Ref {
   public:
    Ref(const DeviceShard* s, std::size_t j) : s_(s), j_(j) {}
    operator double() const { return s_->read(j_); }
    Ref& operator=(double v) {
      s_->write(j_, v);
      return *this;
    }
    Ref& operator=(const Ref& o) { return *this = double(o); }

   private:
    const DeviceShard* s_;
    std::size_t j_;
  };
  DeviceShard() = default;
  DeviceShard(std::size_t n, Precision prec, int device) : n_(n), prec_(prec), buf_(n * esize(prec), device) {
    if (n) {
      DeviceGuard g(device);  // legacy-stream zero fill: the workers' blocking streams order after it
      cuda_ok(cudaMemset(buf_.get(), 0, n * esize(prec)));
    }
  }
  static std::size_t esize(Precision p) { return p == Precision::f32 ? 4 : 8; }
  std::size_t size() const { return n_; }
  bool empty() const { return n_ == 0; }
  void* data() const { return buf_.get(); }
  int device() const { return buf_.device(); }
  Precision precision() const { return prec_; }
  Ref operator[](std::size_t j) const { return Ref(this, j); }
  double read(std::size_t j) const {
    if (j >= n_) throw argument_error("shard element index out of range");
    if (prec_ == Precision::f32) {
      float f;
      cuda_ok(cudaMemcpy(&f, static_cast<char*>(data()) + j * 4, 4, cudaMemcpyDefault));
      return f;
    }
    double d;
    cuda_ok(cudaMemcpy(&d, static_cast<char*>(data()) + j * 8, 8, cudaMemcpyDefault));
    return d;
  }
  void write(std::size_t j, double v) const {
    if (j >= n_) throw argument_error("shard element index out of range");
    if (prec_ == Precision::f32) {
      const float f = float(v);
      cuda_ok(cudaMemcpy(static_cast<char*>(data()) + j * 4, &f, 4, cudaMemcpyDefault));
    } else {
      cuda_ok(cudaMemcpy(static_cast<char*>(data()) + j * 8, &v, 8, cudaMemcpyDefault));
    }
  }

 private:
  std::size_t n_ = 0;
  Precision prec_ = Precision::f64;
  DeviceBuffer buf_;
};

// ------------------------------------------------------------------ pool
// pool.hpp:21-94
enum class MsgKind : int { ApplyShard, DotPartial, Axpy, Scale, Gather, Scatter, Shutdown };
inline constexpr std::size_t kMsgKindCount = 7;
struct PoolOptions {
  unsigned delay_jitter_us = 0;  // sleep U[0, jitter] before each reply (test hook)
  std::uint64_t delay_seed = 0;
};

class WorkerPool {
 public:
  WorkerPool(std::size_t n, ShardLayout layout, PoolOptions opt = {}) : layout_(std::move(layout)), opt_(opt) {
    validate_layout(layout_);
    if (n != layout_.worker_count()) throw layout_error("worker count does not match layout shard count");
    workers_.reserve(n);
    for (std::size_t w = 0; w < n; ++w) workers_.push_back(std::make_unique<Worker>());
    std::vector<std::promise<void>> ready(n);
    for (std::size_t w = 0; w < n; ++w)
      workers_[w]->thread = std::thread([this, w, p = &ready[w]] { worker_main(w, *p); });
    std::exception_ptr failed;
    for (auto& p : ready) {  // streams exist before the first message
      try {
        p.get_future().get();
      } catch (...) {
        if (!failed) failed = std::current_exception();
      }
    }
    if (failed) {  // release the workers that did start, then report the first failure
      shut_down_ = true;
      for (std::size_t w = 0; w < n; ++w) enqueue(w, MsgKind::Shutdown, nullptr);
      for (auto& wk : workers_) wk->thread.join();
      std::rethrow_exception(failed);
    }
  }
  ~WorkerPool() {
    shut_down_ = true;
    for (std::size_t w = 0; w < workers_.size(); ++w) enqueue(w, MsgKind::Shutdown, nullptr);
    for (auto& wk : workers_)
      if (wk->thread.joinable()) wk->thread.join();
  }
  WorkerPool(const WorkerPool&) = delete;
  WorkerPool& operator=(const WorkerPool&) = delete;

  const ShardLayout& layout() const { return layout_; }
  std::size_t worker_count() const { return layout_.worker_count(); }

  // one message to worker w; the future resolves when the worker has replied
  std::future<void> post(std::size_t w, MsgKind kind, std::function<void(std::size_t)> work) {
    if (w >= workers_.size()) throw protocol_error("message posted to an unknown worker");
    if (shut_down_) throw protocol_error("message posted after shutdown");
    return enqueue(w, kind, std::move(work));
  }
  // broadcast, wait for every reply, rethrow the lowest worker's exception
  void run_all(MsgKind kind, const std::function<void(std::size_t)>& work) {
    std::vector<std::future<void>> f;
    f.reserve(workers_.size());
    for (std::size_t w = 0; w < workers_.size(); ++w) f.push_back(post(w, kind, work));
    std::exception_ptr first;
    for (auto& x : f) {
      try {
        x.get();
      } catch (...) {
        if (!first) first = std::current_exception();
      }
    }
    if (first) std::rethrow_exception(first);
  }
  void run_on(std::size_t w, MsgKind kind, std::function<void(std::size_t)> work) {
    post(w, kind, std::move(work)).get();
  }
  std::uint64_t message_count(MsgKind kind) const { return counters_[static_cast<int>(kind)].load(); }
  std::uint64_t total_messages() const {
    std::uint64_t t = 0;
    for (const auto& c : counters_) t += c.load();
    return t;
  }

  // B200 extensions: worker w's device and stream (valid on any thread)
  int device(std::size_t w) const { return workers_.at(w)->device; }
  cudaStream_t stream(std::size_t w) const { return workers_.at(w)->stream; }
  sd_stream sd_stream_of(std::size_t w) const { return reinterpret_cast<sd_stream>(stream(w)); }
  void sync(std::size_t w) const { cuda_ok(cudaStreamSynchronize(stream(w))); }
  // 8-byte device scratch per worker for scalar operands of the kernels
  double* scalar_slot(std::size_t w, int i) const { return static_cast<double*>(workers_.at(w)->scratch.get()) + i; }

 private:
  struct Envelope {
    MsgKind kind;
    std::function<void(std::size_t)> work;
    std::promise<void> reply;
  };
  struct Worker {
    std::thread thread;
    std::mutex m;
    std::condition_variable cv;
    std::deque<Envelope> q;
    int device = 0;
    cudaStream_t stream = nullptr;
    DeviceBuffer scratch;
  };
  std::future<void> enqueue(std::size_t w, MsgKind kind, std::function<void(std::size_t)> work) {
    Worker& wk = *workers_[w];
    Envelope e{kind, std::move(work), {}};
    std::future<void> f = e.reply.get_future();
    counters_[static_cast<int>(kind)].fetch_add(1);
    {
      std::lock_guard<std::mutex> lk(wk.m);
      wk.q.push_back(std::move(e));
    }
    wk.cv.notify_one();
    return f;
  }
  void worker_main(std::size_t w, std::promise<void>& ready) {
    Worker& wk = *workers_[w];
    try {
      wk.device = worker_device(w);
      cuda_ok(cudaSetDevice(wk.device));
      cuda_ok(cudaStreamCreate(&wk.stream));  // blocking: ordered with the legacy default stream
      wk.scratch = DeviceBuffer(8 * sizeof(double), wk.device);
      ready.set_value();
    } catch (...) {
      ready.set_exception(std::current_exception());
      return;
    }
    std::mt19937_64 jitter(opt_.delay_seed ^ (0x9e3779b97f4a7c15ull * (w + 1)));
    while (true) {
      Envelope e;
      {
        std::unique_lock<std::mutex> lk(wk.m);
        wk.cv.wait(lk, [&] { return !wk.q.empty(); });
        e = std::move(wk.q.front());
        wk.q.pop_front();
      }
      if (e.kind == MsgKind::Shutdown) {
        e.reply.set_value();
        break;
      }
      try {
        if (e.work) e.work(w);
        if (opt_.delay_jitter_us)
          std::this_thread::sleep_for(std::chrono::microseconds(jitter() % (opt_.delay_jitter_us + 1ull)));
        e.reply.set_value();
      } catch (...) {
        e.reply.set_exception(std::current_exception());
      }
    }
    cudaStreamSynchronize(wk.stream);
    cudaStreamDestroy(wk.stream);
  }

  ShardLayout layout_;
  PoolOptions opt_;
  std::vector<std::unique_ptr<Worker>> workers_;
  std::array<std::atomic<std::uint64_t>, kMsgKindCount> counters_{};
  std::atomic<bool> shut_down_{false};
};

// --------------------------------------------------------------- sharded
// sharded.hpp:17-69
struct ShardedVector {
  ShardLayout layout;
  Precision prec = Precision::f64;
  std::vector<DeviceShard> shards;
  std::size_t dim() const { return layout.total_dim; }
  std::size_t esize() const { return DeviceShard::esize(prec); }
  double get(std::size_t i) const {
    const std::size_t w = layout.owner(i);
    return shards[w].read(i - layout.shard_bounds[w].begin);
  }
  void set(std::size_t i, double v) {
    const std::size_t w = layout.owner(i);
    shards[w].write(i - layout.shard_bounds[w].begin, round_elem(v, prec));
  }
};

// zero vector; shard w on worker_device(w)
inline ShardedVector make_sharded(const ShardLayout& layout, Precision prec) {
  ShardedVector v;
  v.layout = layout;
  v.prec = prec;
  v.shards.reserve(layout.worker_count());
  for (std::size_t w = 0; w < layout.worker_count(); ++w)
    v.shards.emplace_back(layout.shard_bounds[w].size(), prec, worker_device(w));
  return v;
}

enum class ProbeDist { gaussian, rademacher, one_hot };
struct ProbeSpec {
  std::uint64_t seed = 42;
  ProbeDist distribution = ProbeDist::gaussian;
  std::size_t one_hot_index = 0;
  bool normalize = true;
};
inline int dist_code(ProbeDist d) {
  return d == ProbeDist::gaussian ? SD_GAUSSIAN : (d == ProbeDist::rademacher ? SD_RADEMACHER : SD_ONE_HOT);
}
inline ProbeDist parse_probe_dist(const std::string& s) {
  if (s == "gaussian") return ProbeDist::gaussian;
  if (s == "rademacher") return ProbeDist::rademacher;
  if (s == "one_hot") return ProbeDist::one_hot;
  throw config_error("unknown probe distribution '" + s + "'");
}
inline const char* probe_dist_name(ProbeDist d) {
  return d == ProbeDist::gaussian ? "gaussian" : (d == ProbeDist::rademacher ? "rademacher" : "one_hot");
}

namespace detail {
inline void check_pool(const WorkerPool& pool, const ShardedVector& a) {
  if (!(a.layout == pool.layout())) throw layout_error("sharded vector does not belong to this pool's layout");
}
inline void check_same(const WorkerPool& pool, const ShardedVector& a, const ShardedVector& b) {
  check_pool(pool, a);
  if (!(a.layout == b.layout)) throw layout_error("sharded vectors have different layouts");
  if (a.prec != b.prec) throw layout_error("sharded vectors have different precision");
}
// upload a scalar operand into worker w's slot i (pageable copy: synchronous)
inline const double* put_scalar(WorkerPool& pool, std::size_t w, int i, double v) {
  double* d = pool.scalar_slot(w, i);
  cuda_ok(cudaMemcpyAsync(d, &v, 8, cudaMemcpyHostToDevice, pool.stream(w)));
  return d;
}
}  // namespace detail

// dot (sharded.cpp:85-100): each worker its blocked partial (one DotPartial
// message), the coordinator folds them in worker order.
inline double dot(WorkerPool& pool, const ShardedVector& a, const ShardedVector& b) {
  detail::check_same(pool, a, b);
  const ShardLayout& L = a.layout;
  const std::size_t n = L.worker_count();
  std::vector<std::vector<double>> parts(n);
  pool.run_all(MsgKind::DotPartial, [&](std::size_t w) {
    const auto r = L.shard_bounds[w];
    const uint64_t len = sd_partial_len(r.begin, r.end, L.total_dim);
    DeviceBuffer dp(len * sizeof(double), pool.device(w));
    check(sd_k_dot_partial(a.shards[w].data(), b.shards[w].data(), r.begin, r.end, L.total_dim, prec_code(a.prec),
                           static_cast<double*>(dp.get()), pool.sd_stream_of(w)));
    parts[w].resize(len);
    cuda_ok(cudaMemcpyAsync(parts[w].data(), dp.get(), len * sizeof(double), cudaMemcpyDeviceToHost, pool.stream(w)));
    pool.sync(w);
  });
  std::vector<const double*> ptr(n);
  for (std::size_t w = 0; w < n; ++w) ptr[w] = parts[w].data();
  const auto bg = L.begins(), en = L.ends();
  double out = 0;
  check(sd_combine_partials_host(n, bg.data(), en.data(), L.total_dim, ptr.data(), &out));
  return out;
}

inline double norm2(WorkerPool& pool, const ShardedVector& x) { return std::sqrt(dot(pool, x, x)); }

// axpy (sharded.cpp:106-118): round(y + alpha*x) into a fresh vector
inline ShardedVector axpy(WorkerPool& pool, double alpha, const ShardedVector& x, const ShardedVector& y) {
  detail::check_same(pool, x, y);
  ShardedVector out = make_sharded(x.layout, x.prec);
  pool.run_all(MsgKind::Axpy, [&](std::size_t w) {
    const std::size_t n = x.layout.shard_bounds[w].size();
    cuda_ok(cudaMemcpyAsync(out.shards[w].data(), y.shards[w].data(), n * x.esize(), cudaMemcpyDeviceToDevice,
                            pool.stream(w)));
    check(sd_k_axpy(x.shards[w].data(), out.shards[w].data(), n, detail::put_scalar(pool, w, 0, alpha), 1.0,
                    prec_code(x.prec), pool.sd_stream_of(w)));
    pool.sync(w);
  });
  return out;
}

// scale (sharded.cpp:120-130)
inline ShardedVector scale(WorkerPool& pool, const ShardedVector& x, double c) {
  if (!std::isfinite(c)) throw argument_error("scale factor is not finite");
  detail::check_pool(pool, x);
  ShardedVector out = make_sharded(x.layout, x.prec);
  pool.run_all(MsgKind::Scale, [&](std::size_t w) {
    check(sd_k_scale(x.shards[w].data(), out.shards[w].data(), x.layout.shard_bounds[w].size(),
                     detail::put_scalar(pool, w, 0, c), 0, prec_code(x.prec), pool.sd_stream_of(w)));
    pool.sync(w);
  });
  return out;
}

// draw_probe (sharded.cpp:59-83): fill per worker, then norm2 + scale(1/n)
inline ShardedVector draw_probe(WorkerPool& pool, const ProbeSpec& spec, Precision prec) {
  const ShardLayout& L = pool.layout();
  if (spec.distribution == ProbeDist::one_hot && spec.one_hot_index >= L.total_dim)
    throw argument_error("one_hot index out of range");
  ShardedVector v = make_sharded(L, prec);
  pool.run_all(MsgKind::ApplyShard, [&](std::size_t w) {
    check(sd_k_probe_fill(v.shards[w].data(), L.shard_bounds[w].begin, L.shard_bounds[w].end, spec.seed,
                          dist_code(spec.distribution), spec.one_hot_index, prec_code(prec), pool.sd_stream_of(w)));
    pool.sync(w);
  });
  if (spec.normalize) {
    const double n = norm2(pool, v);
    if (!(n > 0.0)) throw numerical_error("probe has zero norm");
    v = scale(pool, v, 1.0 / n);
  }
  return v;
}

// gather / scatter (sharded.cpp:132-154)
inline std::vector<double> gather(WorkerPool& pool, const ShardedVector& x) {
  detail::check_pool(pool, x);
  std::vector<double> full(x.dim());
  pool.run_all(MsgKind::Gather, [&](std::size_t w) {
    const auto r = x.layout.shard_bounds[w];
    if (x.prec == Precision::f64) {
      cuda_ok(cudaMemcpyAsync(full.data() + r.begin, x.shards[w].data(), r.size() * 8, cudaMemcpyDeviceToHost,
                              pool.stream(w)));
      pool.sync(w);
    } else {
      std::vector<float> tmp(r.size());
      cuda_ok(cudaMemcpyAsync(tmp.data(), x.shards[w].data(), r.size() * 4, cudaMemcpyDeviceToHost, pool.stream(w)));
      pool.sync(w);
      for (std::size_t j = 0; j < r.size(); ++j) full[r.begin + j] = tmp[j];
    }
  });
  return full;
}

inline ShardedVector scatter(WorkerPool& pool, const std::vector<double>& full, Precision prec) {
  const ShardLayout& L = pool.layout();
  if (full.size() != L.total_dim) throw layout_error("scatter source length does not match layout");
  ShardedVector v = make_sharded(L, prec);
  pool.run_all(MsgKind::Scatter, [&](std::size_t w) {
    const auto r = L.shard_bounds[w];
    if (prec == Precision::f64) {
      cuda_ok(cudaMemcpyAsync(v.shards[w].data(), full.data() + r.begin, r.size() * 8, cudaMemcpyHostToDevice,
                              pool.stream(w)));
      pool.sync(w);
    } else {
      std::vector<float> tmp(r.size());
      for (std::size_t j = 0; j < r.size(); ++j) tmp[j] = float(full[r.begin + j]);
      cuda_ok(cudaMemcpyAsync(v.shards[w].data(), tmp.data(), r.size() * 4, cudaMemcpyHostToDevice, pool.stream(w)));
      pool.sync(w);
    }
  });
  return v;
}

// ------------------------------------------------------------- operators
// operators.hpp:15-54
inline constexpr std::size_t kDenseCap = 2048;
struct DenseSymmetric {
  std::size_t n = 0;
  std::vector<double> a;  // row-major n*n
  double at(std::size_t i, std::size_t j) const { return a[i * n + j]; }
  double& at(std::size_t i, std::size_t j) { return a[i * n + j]; }
};

// Engine-native form of an operator: builds the sd_operator the device
// Lanczos engine drives, on the calling thread's current device (one per
// worker device when the engine runs sharded).
using NativeFactory = std::function<sd_operator()>;

struct OperatorHandle {
  std::size_t dim = 0;
  std::string label;
  std::function<void(WorkerPool&, const ShardedVector&, ShardedVector&)> apply_fn;
  NativeFactory native;         // extension: empty for operators given only by apply_fn
  bool native_sharded = false;  // the native form applies a sharded layout (rank rows of the gathered x)

  // operators.cpp:12-17: dimension check, fresh output in x's layout, apply_fn
  ShardedVector apply(WorkerPool& pool, const ShardedVector& x) const {
    if (x.dim() != dim) throw layout_error("operator/vector dimension mismatch");
    ShardedVector y = make_sharded(x.layout, x.prec);
    apply_fn(pool, x, y);
    return y;
  }
};

namespace detail {
inline void check_dense_size(std::size_t n) {
  if (n < 2) throw argument_error("dense operators need n >= 2");
  if (n > kDenseCap) throw argument_error("dense operator size exceeds the desk-scale cap (2048)");
}
// the matrix uploaded once per device
struct DenseOnDevices {
  std::shared_ptr<const DenseSymmetric> m;
  std::mutex mu;
  std::map<int, std::shared_ptr<DeviceBuffer>> per_dev;
  const double* on(int dev) {
    std::lock_guard<std::mutex> lk(mu);
    auto& b = per_dev[dev];
    if (!b) {
      b = std::make_shared<DeviceBuffer>(m->a.size() * sizeof(double), dev);
      cuda_ok(cudaMemcpy(b->get(), m->a.data(), m->a.size() * sizeof(double), cudaMemcpyHostToDevice));
    }
    return static_cast<const double*>(b->get());
  }
};
}  // namespace detail

// dense_operator (operators.cpp:26-48): gather x (Gather messages), then each
// worker computes its own rows from the full x (ApplyShard) -- serial f64
// fold per row on the device, bitwise the reference for any layout
inline OperatorHandle dense_operator(std::shared_ptr<const DenseSymmetric> m, std::string label) {
  detail::check_dense_size(m->n);
  auto dev = std::make_shared<detail::DenseOnDevices>();
  dev->m = m;
  OperatorHandle op;
  op.dim = m->n;
  op.label = std::move(label);
  op.apply_fn = [dev](WorkerPool& pool, const ShardedVector& x, ShardedVector& y) {
    const std::vector<double> xf = gather(pool, x);
    const std::size_t n = xf.size();
    pool.run_all(MsgKind::ApplyShard, [&](std::size_t w) {
      const auto r = y.layout.shard_bounds[w];
      const double* a = dev->on(pool.device(w));
      DeviceBuffer xd(n * y.esize(), pool.device(w));
      if (y.prec == Precision::f64) {
        cuda_ok(cudaMemcpyAsync(xd.get(), xf.data(), n * 8, cudaMemcpyHostToDevice, pool.stream(w)));
        check(sd_k_dense_apply(a, n, xd.get(), y.shards[w].data(), r.begin, r.end, SD_F64, pool.sd_stream_of(w)));
        pool.sync(w);
      } else {
        std::vector<float> xs(xf.begin(), xf.end());
        cuda_ok(cudaMemcpyAsync(xd.get(), xs.data(), n * 4, cudaMemcpyHostToDevice, pool.stream(w)));
        check(sd_k_dense_apply(a, n, xd.get(), y.shards[w].data(), r.begin, r.end, SD_F32, pool.sd_stream_of(w)));
        pool.sync(w);
      }
    });
  };
  op.native = [m]() {
    sd_operator o = nullptr;
    check(sd_operator_dense(m->n, m->a.data(), &o));
    return o;
  };
  op.native_sharded = true;
  return op;
}
inline DenseSymmetric wigner_dense(std::size_t n, double sigma, std::uint64_t seed) {
  DenseSymmetric m;
  m.n = n;
  if (n >= 2 && n <= kDenseCap) m.a.resize(n * n);
  check(sd_wigner_dense(n, sigma, seed, m.a.data()));
  return m;
}
inline OperatorHandle wigner_operator(std::size_t n, double sigma, std::uint64_t seed) {
  return dense_operator(std::make_shared<DenseSymmetric>(wigner_dense(n, sigma, seed)),
                        "wigner(n=" + std::to_string(n) + ",sigma=" + std::to_string(sigma) +
                            ",seed=" + std::to_string(seed) + ")");
}
inline DenseSymmetric spiked_dense(std::size_t n, double sigma, const std::vector<double>& spikes,
                                   std::uint64_t seed) {
  DenseSymmetric m;
  m.n = n;
  if (n >= 2 && n <= kDenseCap) m.a.resize(n * n);
  check(sd_spiked_dense(n, sigma, spikes.data(), spikes.size(), seed, m.a.data()));
  return m;
}
inline OperatorHandle spiked_operator(std::size_t n, double sigma, const std::vector<double>& spikes,
                                      std::uint64_t seed) {
  return dense_operator(std::make_shared<DenseSymmetric>(spiked_dense(n, sigma, spikes, seed)),
                        "spiked(n=" + std::to_string(n) + ")");
}
// load_dense (operators.cpp:114-135): "dim N" then N rows of N reals; every
// malformed file is a config_error, an out-of-range N an argument_error
inline DenseSymmetric load_dense(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw config_error("cannot open dense operator file '" + path + "'");
  std::string tag;
  std::size_t n = 0;
  if (!(in >> tag >> n) || tag != "dim") throw config_error("dense operator file must start with a 'dim N' header");
  detail::check_dense_size(n);
  DenseSymmetric m;
  m.n = n;
  m.a.resize(n * n);
  for (double& x : m.a)
    if (!(in >> x)) throw config_error("dense operator file ended early (expected " + std::to_string(n * n) + " entries)");
  for (std::size_t i = 0; i < n; ++i)
    for (std::size_t j = 0; j < i; ++j)
      if (m.at(i, j) != m.at(j, i))
        throw config_error("dense operator file is not symmetric at (" + std::to_string(j) + "," + std::to_string(i) +
                           ")");
  return m;
}

// ------------------------------------------- lanczos
enum class Reorthogonalize { none, full, selective };
enum class Reduction { ordered, tree };
struct LanczosConfig {
  std::size_t k_max = 10;
  double breakdown_tol = -1.0;  // <= 0: 1e-12 (f64) / 1e-7 (f32)
  Reorthogonalize reorthogonalize = Reorthogonalize::none;
  ProbeSpec probe;
  Precision prec = Precision::f64;
  std::size_t window = 0;                 // selective: the W >= 2 most recent basis vectors (extension)
  Reduction reduction = Reduction::ordered;  // tree: fused GEMV passes (extension; HVP operators)
};
struct TridiagonalMatrix {
  std::vector<double> alphas, betas;
  std::size_t k() const { return alphas.size(); }
};
struct LanczosRun {
  TridiagonalMatrix t;
  bool breakdown = false;
  double ms_apply = 0, ms_recurrence = 0, ms_reorth = 0;
};

namespace detail {
inline sd_lanczos_config native_config(const LanczosConfig& cfg) {
  sd_lanczos_config c{};
  c.k_max = cfg.k_max;
  c.eps = cfg.breakdown_tol;
  c.reorth = cfg.reorthogonalize == Reorthogonalize::full        ? SD_REORTH_FULL
             : cfg.reorthogonalize == Reorthogonalize::selective ? SD_REORTH_SELECTIVE
                                                                 : SD_REORTH_NONE;
  c.prec = prec_code(cfg.prec);
  c.probe_seed = cfg.probe.seed;
  c.probe_dist = dist_code(cfg.probe.distribution);
  c.selective_window = cfg.window;
  c.reduction = cfg.reduction == Reduction::tree ? SD_REDUCE_TREE : SD_REDUCE_ORDERED;
  return c;
}

// The SPEC recurrence composed from the vector operations (operators given
// only by apply_fn): each op is a kernel per worker, bitwise the reference.
inline LanczosRun lanczos_composed(const OperatorHandle& op, const LanczosConfig& cfg, WorkerPool& pool) {
  if (cfg.k_max < 1) throw config_error("k_max must be >= 1");
  if (cfg.reorthogonalize == Reorthogonalize::selective && cfg.window < 2)
    throw config_error("selective reorthogonalisation needs a window >= 2");
  const double eps = cfg.breakdown_tol > 0 ? cfg.breakdown_tol : (cfg.prec == Precision::f64 ? 1e-12 : 1e-7);
  LanczosRun run;
  ShardedVector q = draw_probe(pool, cfg.probe, cfg.prec), qp;
  std::vector<ShardedVector> Q;
  if (cfg.reorthogonalize != Reorthogonalize::none) Q.push_back(q);
  for (std::size_t k = 0; k < cfg.k_max; ++k) {
    ShardedVector r = op.apply(pool, q);
    if (k > 0) r = axpy(pool, -run.t.betas[k - 1], qp, r);
    const double alpha = dot(pool, q, r);
    if (!std::isfinite(alpha)) throw numerical_error("non-finite alpha (partial tridiagonal discarded)");
    r = axpy(pool, -alpha, q, r);
    for (int pass = 0; pass < 2 && !Q.empty(); ++pass) {
      std::vector<double> c(Q.size());
      for (std::size_t i = 0; i < Q.size(); ++i) c[i] = dot(pool, Q[i], r);
      for (std::size_t i = 0; i < Q.size(); ++i) r = axpy(pool, -c[i], Q[i], r);
    }
    const double beta = norm2(pool, r);
    run.t.alphas.push_back(alpha);
    if (!std::isfinite(beta)) throw numerical_error("non-finite beta");
    if (beta < eps) {
      run.breakdown = true;
      break;
    }
    if (k + 1 == cfg.k_max) break;
    run.t.betas.push_back(beta);
    qp = q;
    q = scale(pool, r, 1.0 / beta);
    if (cfg.reorthogonalize == Reorthogonalize::full) Q.push_back(q);
    if (cfg.reorthogonalize == Reorthogonalize::selective) {
      if (Q.size() == cfg.window) Q[(k + 1) % cfg.window] = q;  // ring of the W most recent, slot order
      else Q.push_back(q);
    }
  }
  return run;
}
}  // namespace detail

// lanczos_run: the device engine, one rank per worker on the worker's own
// thread, device and stream (in-process communicator for the f64 partials and
// the gathered operator input); operators without a native form run the
// composed recurrence.
inline LanczosRun lanczos_run(const OperatorHandle& op, const LanczosConfig& cfg, WorkerPool& pool) {
  if (op.dim != pool.layout().total_dim) throw layout_error("operator/vector dimension mismatch");
  const std::size_t n = pool.worker_count();
  if (!op.native || (n > 1 && !op.native_sharded)) return detail::lanczos_composed(op, cfg, pool);
  const sd_lanczos_config c = detail::native_config(cfg);
  const auto b = pool.layout().begins(), e = pool.layout().ends();
  std::vector<sd_comm> comms(n, nullptr);
  if (n > 1) check(sd_comm_local_create(int(n), comms.data()));
  std::vector<std::vector<double>> al(n, std::vector<double>(cfg.k_max)), be(n, std::vector<double>(cfg.k_max));
  std::vector<sd_lanczos_info> info(n);
  std::vector<sd_status> st(n, SD_OK);
  std::vector<std::string> msg(n);
  std::vector<std::future<void>> f;
  for (std::size_t w = 0; w < n; ++w)
    f.push_back(pool.post(w, MsgKind::ApplyShard, [&, w](std::size_t) {
      std::shared_ptr<sd_operator_s> o(op.native(), sd_operator_destroy);
      const uint64_t bytes = sd_lanczos_workspace_bytes(b.data(), e.data(), op.dim, &c, int(n), int(w));
      if (!bytes) {
        st[w] = SD_CONFIG_ERROR;
        msg[w] = sd_last_error();
        if (n > 1) sd_comm_abort(comms[w]);
        return;
      }
      DeviceBuffer ws(bytes, pool.device(w));
      st[w] = sd_lanczos_run(o.get(), comms[w], b.data(), e.data(), op.dim, &c, ws.get(), bytes, al[w].data(),
                             be[w].data(), &info[w], pool.sd_stream_of(w));
      if (st[w] != SD_OK) {
        msg[w] = sd_last_error();
        if (n > 1) sd_comm_abort(comms[w]);
      }
    }));
  for (auto& x : f) x.get();
  for (sd_comm cm : comms)
    if (cm) sd_comm_destroy(cm);
  for (std::size_t w = 0; w < n; ++w)  // the lowest failing worker's error (pool.cpp:54-64)
    if (st[w] != SD_OK && st[w] != SD_PROTOCOL_ERROR) throw_status(st[w], msg[w]);
  for (std::size_t w = 0; w < n; ++w)
    if (st[w] != SD_OK) throw_status(st[w], msg[w]);
  LanczosRun r;
  r.t.alphas.assign(al[0].begin(), al[0].begin() + info[0].n_alpha);
  r.t.betas.assign(be[0].begin(), be[0].begin() + info[0].n_beta);
  r.breakdown = info[0].breakdown != 0;
  r.ms_apply = info[0].ms_apply;
  r.ms_recurrence = info[0].ms_recurrence;
  r.ms_reorth = info[0].ms_reorth;
  return r;
}

// ------------------------------------------- quadrature
struct RitzSpectrum {
  std::vector<double> values, weights;
  double residual = 0;
};
inline RitzSpectrum ritz_decompose(const TridiagonalMatrix& t) {
  RitzSpectrum s;
  s.values.resize(t.k());
  s.weights.resize(t.k());
  check(sd_ritz_decompose(t.k(), t.alphas.data(), t.betas.empty() ? nullptr : t.betas.data(), s.values.data(),
                          s.weights.data(), &s.residual));
  return s;
}
struct SmoothedDensity {
  std::vector<double> grid, density;
  double kernel_sigma = 0;
};
inline SmoothedDensity smooth_density(const RitzSpectrum& s, double sigma = -1.0, std::size_t grid_points = 512) {
  SmoothedDensity d;
  d.grid.resize(grid_points);
  d.density.resize(grid_points);
  check(sd_smooth_density(s.values.size(), s.values.data(), s.weights.data(), sigma, grid_points, d.grid.data(),
                          d.density.data(), &d.kernel_sigma));
  return d;
}
// average_spectra: union of (theta, w / n_runs), renormalised
inline RitzSpectrum average_spectra(const std::vector<RitzSpectrum>& runs) {
  if (runs.empty()) throw argument_error("average_spectra needs at least one run");
  std::vector<std::pair<double, double>> all;
  for (const auto& r : runs)
    for (std::size_t i = 0; i < r.values.size(); ++i) all.push_back({r.values[i], r.weights[i] / double(runs.size())});
  std::stable_sort(all.begin(), all.end(), [](auto& a, auto& b) { return a.first < b.first; });
  double tot = 0;
  for (auto& p : all) tot += p.second;
  RitzSpectrum out;
  for (auto& p : all) {
    out.values.push_back(p.first);
    out.weights.push_back(p.second / tot);
  }
  return out;
}

// ---- autodiff: hvp / batched_hvp (Alg. 1)
// ModelSpec architectures: mlp(layer_widths) with mse and the
// decoder family the SPEC's attention_block grows into (GPT-2 style, or
// Llama style: sd_gpt_config.arch). The device engine computes in fp32
// (3xTF32 tensor-core GEMMs), so vectors must be Precision::f32. The model
// lives on worker 0's device.
struct ModelSpec {
  enum class Arch { mlp, transformer } arch = Arch::mlp;
  std::vector<std::uint64_t> layer_widths;  // mlp
  sd_gpt_config transformer{};              // transformer
  static ModelSpec mlp(std::vector<std::uint64_t> widths) {
    ModelSpec m;
    m.arch = Arch::mlp;
    m.layer_widths = std::move(widths);
    return m;
  }
  static ModelSpec decoder(const sd_gpt_config& c) {
    ModelSpec m;
    m.arch = Arch::transformer;
    m.transformer = c;
    return m;
  }
  std::size_t parameter_count() const {
    return arch == Arch::mlp ? sd_mlp_param_count(layer_widths.data(), int(layer_widths.size()))
                             : sd_gpt_param_count(&transformer);
  }
};

// One batch: token rows (transformer: rows x seq tokens and next-token
// targets) or feature rows (mlp: rows x w0 features, rows x w_last targets).
struct Batch {
  int rows = 0, seq = 0;
  std::vector<int> tokens, token_targets;
  std::vector<float> x, y;
  // the samples Alg. 1 weights by: tokens (cross-entropy) or rows (mse)
  std::size_t samples() const { return tokens.empty() ? std::size_t(rows) : tokens.size(); }
};

// Parameters (device, f32) plus the HVP engines of one model; transformer
// engines are built per batch shape on first use and share the parameters.
// Every engine call runs on worker 0 (its device and stream).
class Model {
 public:
  // transformer with the synthetic counter-keyed init (sd_gpt_init_params)
  Model(WorkerPool& pool, const ModelSpec& spec, std::uint64_t init_seed, double gain_scale = 0.0,
        double bias_scale = 0.0)
      : spec_(spec), P_(spec.parameter_count()), dev_(pool.device(0)), theta_(P_ * 4, dev_) {
    if (spec.arch != ModelSpec::Arch::transformer) throw config_error("this constructor builds transformer models");
    if (P_ == 0) check(SD_CONFIG_ERROR);
    pool.run_on(0, MsgKind::ApplyShard, [&](std::size_t) {
      check(sd_gpt_init_params(&spec_.transformer, init_seed, gain_scale, bias_scale,
                               static_cast<float*>(theta_.get()), pool.sd_stream_of(0)));
      pool.sync(0);
    });
  }
  // mlp with caller parameters (flat declaration order, f32-representable), n_max rows per batch
  Model(WorkerPool& pool, const ModelSpec& spec, const std::vector<double>& params, int n_max)
      : spec_(spec), P_(spec.parameter_count()), dev_(pool.device(0)), theta_(P_ * 4, dev_) {
    if (spec.arch != ModelSpec::Arch::mlp) throw config_error("this constructor builds mlp models");
    if (params.size() != P_) throw layout_error("parameter count does not match the model");
    std::vector<float> f(params.begin(), params.end());
    pool.run_on(0, MsgKind::ApplyShard, [&](std::size_t) {
      cuda_ok(cudaMemcpyAsync(theta_.get(), f.data(), P_ * 4, cudaMemcpyHostToDevice, pool.stream(0)));
      sd_mlp m = nullptr;
      check(sd_mlp_create(spec_.layer_widths.data(), int(spec_.layer_widths.size()), n_max,
                          static_cast<const float*>(theta_.get()), pool.sd_stream_of(0), &m));
      mlp_.reset(m, sd_mlp_destroy);
      pool.sync(0);
    });
    n_max_ = n_max;
  }
  std::size_t parameter_count() const { return P_; }
  const ModelSpec& spec() const { return spec_; }
  int device() const { return dev_; }

  // Hv (full logical vectors on the model's device) of one batch with loss
  // weight `scale`, on stream s of the model's device
  void hvp_device(const Batch& b, float scale, const float* v, float* hv, sd_stream s) {
    if (spec_.arch == ModelSpec::Arch::mlp) {
      const int w0 = int(spec_.layer_widths.front()), wl = int(spec_.layer_widths.back());
      if (b.rows < 1) throw argument_error("empty batch");
      if (b.rows > n_max_) throw argument_error("batch exceeds the engine's row capacity");
      if (b.x.size() != std::size_t(b.rows) * w0 || b.y.size() != std::size_t(b.rows) * wl)
        throw argument_error("inconsistent sample dimensions");
      check(sd_mlp_set_batch(mlp_.get(), b.x.data(), b.y.data(), b.rows, scale, s));
      check(sd_mlp_hvp(mlp_.get(), v, hv, s));
      return;
    }
    if (b.rows < 1 || b.seq < 1) throw argument_error("empty batch");
    if (b.tokens.size() != std::size_t(b.rows) * b.seq || b.token_targets.size() != b.tokens.size())
      throw argument_error("inconsistent sample dimensions");
    Engine& e = engine(b.rows, b.seq, s);
    check(sd_gpt_set_batch(e.g.get(), b.tokens.data(), b.token_targets.data(), scale, s));
    check(sd_gpt_hvp(e.g.get(), v, hv, s));
  }

 private:
  struct Engine {
    DeviceBuffer ws;
    std::shared_ptr<sd_gpt_s> g;
  };
  Engine& engine(int rows, int seq, sd_stream s) {
    std::lock_guard<std::mutex> lk(mu_);
    const auto key = std::make_pair(rows, seq);
    auto it = engines_.find(key);
    if (it != engines_.end()) return it->second;
    const uint64_t bytes = sd_gpt_workspace_bytes(&spec_.transformer, rows, seq);
    if (!bytes) {  // invalid shape: the create call reports the precise error class
      sd_gpt g = nullptr;
      check(sd_gpt_create(&spec_.transformer, rows, seq, static_cast<const float*>(theta_.get()), nullptr, 0, s, &g));
    }
    // built in place: the engine keeps pointers into its workspace
    Engine& e = engines_[key];
    try {
      e.ws = DeviceBuffer(bytes, dev_);
      sd_gpt g = nullptr;
      check(sd_gpt_create(&spec_.transformer, rows, seq, static_cast<const float*>(theta_.get()), e.ws.get(), bytes, s,
                          &g));
      e.g.reset(g, sd_gpt_destroy);
    } catch (...) {
      engines_.erase(key);
      throw;
    }
    return e;
  }
  ModelSpec spec_;
  std::size_t P_ = 0;
  int dev_ = 0;
  DeviceBuffer theta_;
  std::shared_ptr<sd_mlp_s> mlp_;
  int n_max_ = 0;
  std::mutex mu_;
  std::map<std::pair<int, int>, Engine> engines_;
};

namespace detail {
// full logical vector on device `dev` from the shards (peer copies across devices)
inline DeviceBuffer gather_device(WorkerPool& pool, const ShardedVector& x, int dev) {
  const std::size_t es = x.esize();
  DeviceBuffer full(x.dim() * es, dev);
  pool.run_all(MsgKind::Gather, [&](std::size_t w) {
    const auto r = x.layout.shard_bounds[w];
    cuda_ok(cudaMemcpyAsync(static_cast<char*>(full.get()) + r.begin * es, x.shards[w].data(), r.size() * es,
                            cudaMemcpyDefault, pool.stream(w)));
    pool.sync(w);
  });
  return full;
}
inline void scatter_device(WorkerPool& pool, const DeviceBuffer& full, ShardedVector& y) {
  const std::size_t es = y.esize();
  pool.run_all(MsgKind::Scatter, [&](std::size_t w) {
    const auto r = y.layout.shard_bounds[w];
    cuda_ok(cudaMemcpyAsync(y.shards[w].data(), static_cast<const char*>(full.get()) + r.begin * es, r.size() * es,
                            cudaMemcpyDefault, pool.stream(w)));
    pool.sync(w);
  });
}
inline void check_model_vector(WorkerPool& pool, const Model& m, const ShardedVector& v) {
  check_pool(pool, v);
  if (v.dim() != m.parameter_count()) throw layout_error("vector dimension does not match the model");
  if (v.prec != Precision::f32) throw config_error("the HVP engine computes in f32: use Precision::f32 vectors");
}
inline double batch_norm(const Model& m, const Batch& b) {
  return double(b.samples()) * (m.spec().arch == ModelSpec::Arch::mlp ? double(m.spec().layer_widths.back()) : 1.0);
}
}  // namespace detail

// Hv of the batch-mean loss (Pearlmutter, forward-over-reverse on device)
inline ShardedVector hvp(WorkerPool& pool, Model& m, const Batch& batch, const ShardedVector& v) {
  detail::check_model_vector(pool, m, v);
  DeviceBuffer xf = detail::gather_device(pool, v, m.device()), yf(v.dim() * 4, m.device());
  pool.run_on(0, MsgKind::ApplyShard, [&](std::size_t) {
    m.hvp_device(batch, float(1.0 / detail::batch_norm(m, batch)), static_cast<const float*>(xf.get()),
                 static_cast<float*>(yf.get()), pool.sd_stream_of(0));
    pool.sync(0);
  });
  ShardedVector y = make_sharded(v.layout, v.prec);
  detail::scatter_device(pool, yf, y);
  return y;
}

// SPEC.md:202-210 / Alg. 1 lines 5-16: sum_b |B_b| u_b / N -- every batch's
// loss is weighted 1/N_total so its Hv already carries |B_b|/N; the per-batch
// results are summed in loader order with the f32 axpy kernel.
inline ShardedVector batched_hvp(WorkerPool& pool, Model& m, const std::vector<Batch>& loader,
                                 const ShardedVector& v) {
  detail::check_model_vector(pool, m, v);
  if (loader.empty()) throw argument_error("batched_hvp needs at least one batch");
  double N = 0;
  for (const Batch& b : loader) N += detail::batch_norm(m, b);
  DeviceBuffer xf = detail::gather_device(pool, v, m.device()), tmp(v.dim() * 4, m.device()),
      acc(v.dim() * 4, m.device());
  pool.run_on(0, MsgKind::ApplyShard, [&](std::size_t) {
    cuda_ok(cudaMemsetAsync(acc.get(), 0, v.dim() * 4, pool.stream(0)));
    const double* one = detail::put_scalar(pool, 0, 0, 1.0);
    for (const Batch& b : loader) {
      m.hvp_device(b, float(1.0 / N), static_cast<const float*>(xf.get()), static_cast<float*>(tmp.get()),
                   pool.sd_stream_of(0));
      check(sd_k_axpy(tmp.get(), acc.get(), v.dim(), one, 1.0, SD_F32, pool.sd_stream_of(0)));
    }
    pool.sync(0);
  });
  ShardedVector y = make_sharded(v.layout, v.prec);
  detail::scatter_device(pool, acc, y);
  return y;
}

// The model's Hessian on one batch as an OperatorHandle (what lanczos_run
// drives): apply_fn for pool callers; the native form is an sd_operator_custom
// over the engine (the device Lanczos engine then runs it on the model's
// device, single rank).
inline OperatorHandle hvp_operator(WorkerPool& pool, Model& m, const Batch& batch) {
  (void)pool;
  const float scale = float(1.0 / detail::batch_norm(m, batch));
  struct Ctx {
    Model* m;
    Batch b;
    float scale;
  };
  auto ctx = std::make_shared<Ctx>(Ctx{&m, batch, scale});
  OperatorHandle op;
  op.dim = m.parameter_count();
  op.label = "hvp";
  op.apply_fn = [ctx](WorkerPool& p, const ShardedVector& x, ShardedVector& y) {
    y = hvp(p, *ctx->m, ctx->b, x);
  };
  op.native = [ctx]() {
    static const sd_apply_fn fn = [](void* c, const void* x, void* y, sd_stream s) -> sd_status {
      auto* k = static_cast<Ctx*>(c);
      try {
        k->m->hvp_device(k->b, k->scale, static_cast<const float*>(x), static_cast<float*>(y), s);
      } catch (const std::exception&) {
        return SD_ARGUMENT_ERROR;
      }
      return SD_OK;
    };
    sd_operator o = nullptr;
    check(sd_operator_custom(ctx->m->parameter_count(), fn, ctx.get(), &o));
    return o;
  };
  return op;
}

}  // namespace specden

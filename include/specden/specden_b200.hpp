// specden_b200.hpp — C++ drop-in for the reference's specden API
// (proj/include/specden/{errors,precision,layout,pool,sharded,operators}.hpp
// and the SPEC-only lanczos_run / ritz_decompose), header-only over the C-ABI
// of include/specden_b200.h. Vectors live on the current CUDA device; every
// floating-point operation runs in libspecden_b200.so (sm_100a kernels).
//
// Differences a reference caller sees: none in names, argument meaning or
// exception types; ShardedVector shards are device buffers (get/set/gather
// copy through the host), and WorkerPool workers are shards of one device
// driven on one CUDA stream (multi-GPU = one process per GPU + sd_comm).
#pragma once

#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "specden_b200.h"

namespace specden {

// ---- errors.hpp:13-41
struct config_error : std::runtime_error {
  explicit config_error(const std::string& w) : std::runtime_error(w) {}
};
struct layout_error : std::runtime_error {
  explicit layout_error(const std::string& w) : std::runtime_error(w) {}
};
struct argument_error : std::runtime_error {
  explicit argument_error(const std::string& w) : std::runtime_error(w) {}
};
struct numerical_error : std::runtime_error {
  explicit numerical_error(const std::string& w) : std::runtime_error(w) {}
};
struct state_error : std::runtime_error {
  explicit state_error(const std::string& w) : std::runtime_error(w) {}
};
struct protocol_error : std::runtime_error {
  explicit protocol_error(const std::string& w) : std::runtime_error(w) {}
};
struct device_error : std::runtime_error {
  explicit device_error(const std::string& w) : std::runtime_error(w) {}
};

inline void check(sd_status s) {
  if (s == SD_OK) return;
  const std::string m = sd_last_error();
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
inline void cuda_ok(cudaError_t e) {
  if (e != cudaSuccess) throw device_error(cudaGetErrorString(e));
}

// ---- precision.hpp:15-34
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

// ---- layout.hpp:12-72
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

// ---- device buffer (RAII)
class DeviceBuffer {
 public:
  DeviceBuffer() = default;
  explicit DeviceBuffer(std::size_t bytes) : bytes_(bytes) {
    if (bytes) cuda_ok(cudaMalloc(&p_, bytes));
  }
  DeviceBuffer(const DeviceBuffer& o) : DeviceBuffer(o.bytes_) {
    if (bytes_) cuda_ok(cudaMemcpy(p_, o.p_, bytes_, cudaMemcpyDeviceToDevice));
  }
  DeviceBuffer& operator=(DeviceBuffer o) {
    std::swap(p_, o.p_);
    std::swap(bytes_, o.bytes_);
    return *this;
  }
  ~DeviceBuffer() {
    if (p_) cudaFree(p_);
  }
  void* get() const { return p_; }
  std::size_t bytes() const { return bytes_; }

 private:
  void* p_ = nullptr;
  std::size_t bytes_ = 0;
};

// ---- pool.hpp:47-94: n shard "workers" of one device, one stream
class WorkerPool {
 public:
  WorkerPool(std::size_t n, ShardLayout layout) : layout_(std::move(layout)) {
    validate_layout(layout_);
    if (n != layout_.worker_count()) throw layout_error("worker count does not match layout shard count");
    cuda_ok(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
  }
  ~WorkerPool() {
    if (stream_) {
      cudaStreamSynchronize(stream_);
      cudaStreamDestroy(stream_);
    }
  }
  WorkerPool(const WorkerPool&) = delete;
  WorkerPool& operator=(const WorkerPool&) = delete;
  const ShardLayout& layout() const { return layout_; }
  std::size_t worker_count() const { return layout_.worker_count(); }
  sd_stream stream() const { return reinterpret_cast<sd_stream>(stream_); }
  void sync() const { cuda_ok(cudaStreamSynchronize(stream_)); }

 private:
  ShardLayout layout_;
  cudaStream_t stream_ = nullptr;
};

// ---- sharded.hpp:17-69
struct ShardedVector {
  ShardLayout layout;
  Precision prec = Precision::f64;
  std::vector<DeviceBuffer> shards;
  std::size_t dim() const { return layout.total_dim; }
  std::size_t esize() const { return prec == Precision::f32 ? 4 : 8; }
  double get(std::size_t i) const {
    const std::size_t w = layout.owner(i);
    const std::size_t off = (i - layout.shard_bounds[w].begin) * esize();
    if (prec == Precision::f32) {
      float v;
      cuda_ok(cudaMemcpy(&v, static_cast<char*>(shards[w].get()) + off, 4, cudaMemcpyDeviceToHost));
      return v;
    }
    double v;
    cuda_ok(cudaMemcpy(&v, static_cast<char*>(shards[w].get()) + off, 8, cudaMemcpyDeviceToHost));
    return v;
  }
  void set(std::size_t i, double v) {
    const std::size_t w = layout.owner(i);
    const std::size_t off = (i - layout.shard_bounds[w].begin) * esize();
    if (prec == Precision::f32) {
      const float f = float(v);
      cuda_ok(cudaMemcpy(static_cast<char*>(shards[w].get()) + off, &f, 4, cudaMemcpyHostToDevice));
    } else {
      cuda_ok(cudaMemcpy(static_cast<char*>(shards[w].get()) + off, &v, 8, cudaMemcpyHostToDevice));
    }
  }
};

inline ShardedVector make_sharded(const ShardLayout& layout, Precision prec) {
  ShardedVector v;
  v.layout = layout;
  v.prec = prec;
  for (const auto& r : layout.shard_bounds) {
    v.shards.emplace_back(r.size() * v.esize());
    cuda_ok(cudaMemset(v.shards.back().get(), 0, r.size() * v.esize()));
  }
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

namespace detail {
inline void check_pool(const WorkerPool& pool, const ShardedVector& a) {
  if (!(a.layout == pool.layout())) throw layout_error("sharded vector does not belong to this pool's layout");
}
inline void check_same(const WorkerPool& pool, const ShardedVector& a, const ShardedVector& b) {
  check_pool(pool, a);
  if (!(a.layout == b.layout)) throw layout_error("sharded vectors have different layouts");
  if (a.prec != b.prec) throw layout_error("sharded vectors have different precision");
}
struct DevScalar {
  DeviceBuffer b{sizeof(double)};
  explicit DevScalar(double v) { cuda_ok(cudaMemcpy(b.get(), &v, 8, cudaMemcpyHostToDevice)); }
  const double* p() const { return static_cast<const double*>(b.get()); }
};
}  // namespace detail

// dot (sharded.cpp:85-100): per-shard blocked partials, folded in shard order.
inline double dot(WorkerPool& pool, const ShardedVector& a, const ShardedVector& b) {
  detail::check_same(pool, a, b);
  const ShardLayout& L = a.layout;
  const auto bg = L.begins(), en = L.ends();
  uint64_t pmax = 0;
  for (std::size_t w = 0; w < L.worker_count(); ++w) pmax = std::max(pmax, sd_partial_len(bg[w], en[w], L.total_dim));
  DeviceBuffer parts(L.worker_count() * pmax * sizeof(double)), out(sizeof(double));
  for (std::size_t w = 0; w < L.worker_count(); ++w)
    check(sd_k_dot_partial(a.shards[w].get(), b.shards[w].get(), bg[w], en[w], L.total_dim, prec_code(a.prec),
                           static_cast<double*>(parts.get()) + w * pmax, pool.stream()));
  check(sd_k_combine(L.worker_count(), bg.data(), en.data(), L.total_dim, 1, static_cast<double*>(parts.get()),
                     static_cast<double*>(out.get()), pool.stream()));
  double r = 0;
  cuda_ok(cudaMemcpyAsync(&r, out.get(), 8, cudaMemcpyDeviceToHost, reinterpret_cast<cudaStream_t>(pool.stream())));
  pool.sync();
  return r;
}

inline double norm2(WorkerPool& pool, const ShardedVector& x) { return std::sqrt(dot(pool, x, x)); }

// axpy (sharded.cpp:106-118): round(y + alpha*x) into a fresh vector
inline ShardedVector axpy(WorkerPool& pool, double alpha, const ShardedVector& x, const ShardedVector& y) {
  detail::check_same(pool, x, y);
  ShardedVector out = y;
  detail::DevScalar a(alpha);
  for (std::size_t w = 0; w < x.layout.worker_count(); ++w)
    check(sd_k_axpy(x.shards[w].get(), out.shards[w].get(), x.layout.shard_bounds[w].size(), a.p(), 1.0,
                    prec_code(x.prec), pool.stream()));
  pool.sync();
  return out;
}

// scale (sharded.cpp:120-130)
inline ShardedVector scale(WorkerPool& pool, const ShardedVector& x, double c) {
  if (!std::isfinite(c)) throw argument_error("scale factor is not finite");
  detail::check_pool(pool, x);
  ShardedVector out = make_sharded(x.layout, x.prec);
  detail::DevScalar cc(c);
  for (std::size_t w = 0; w < x.layout.worker_count(); ++w)
    check(sd_k_scale(x.shards[w].get(), out.shards[w].get(), x.layout.shard_bounds[w].size(), cc.p(), 0,
                     prec_code(x.prec), pool.stream()));
  pool.sync();
  return out;
}

// draw_probe (sharded.cpp:59-83)
inline ShardedVector draw_probe(WorkerPool& pool, const ProbeSpec& spec, Precision prec) {
  const ShardLayout& L = pool.layout();
  if (spec.distribution == ProbeDist::one_hot && spec.one_hot_index >= L.total_dim)
    throw argument_error("one_hot index out of range");
  ShardedVector v = make_sharded(L, prec);
  for (std::size_t w = 0; w < L.worker_count(); ++w)
    check(sd_k_probe_fill(v.shards[w].get(), L.shard_bounds[w].begin, L.shard_bounds[w].end, spec.seed,
                          dist_code(spec.distribution), spec.one_hot_index, prec_code(prec), pool.stream()));
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
  pool.sync();
  std::vector<double> full(x.dim());
  for (std::size_t w = 0; w < x.layout.worker_count(); ++w) {
    const auto r = x.layout.shard_bounds[w];
    if (x.prec == Precision::f64) {
      cuda_ok(cudaMemcpy(full.data() + r.begin, x.shards[w].get(), r.size() * 8, cudaMemcpyDeviceToHost));
    } else {
      std::vector<float> tmp(r.size());
      cuda_ok(cudaMemcpy(tmp.data(), x.shards[w].get(), r.size() * 4, cudaMemcpyDeviceToHost));
      for (std::size_t j = 0; j < r.size(); ++j) full[r.begin + j] = tmp[j];
    }
  }
  return full;
}

inline ShardedVector scatter(WorkerPool& pool, const std::vector<double>& full, Precision prec) {
  const ShardLayout& L = pool.layout();
  if (full.size() != L.total_dim) throw layout_error("scatter source length does not match layout");
  ShardedVector v = make_sharded(L, prec);
  for (std::size_t w = 0; w < L.worker_count(); ++w) {
    const auto r = L.shard_bounds[w];
    if (prec == Precision::f64) {
      cuda_ok(cudaMemcpy(v.shards[w].get(), full.data() + r.begin, r.size() * 8, cudaMemcpyHostToDevice));
    } else {
      std::vector<float> tmp(r.size());
      for (std::size_t j = 0; j < r.size(); ++j) tmp[j] = float(full[r.begin + j]);
      cuda_ok(cudaMemcpy(v.shards[w].get(), tmp.data(), r.size() * 4, cudaMemcpyHostToDevice));
    }
  }
  return v;
}

// ---- operators.hpp:15-54
struct DenseSymmetric {
  std::size_t n = 0;
  std::vector<double> a;
  double at(std::size_t i, std::size_t j) const { return a[i * n + j]; }
  double& at(std::size_t i, std::size_t j) { return a[i * n + j]; }
};
inline constexpr std::size_t kDenseCap = 2048;

struct OperatorHandle {
  std::size_t dim = 0;
  std::string label;
  std::shared_ptr<sd_operator_s> native;

  // operators.cpp:12-17: dimension check, fresh output in x's layout
  ShardedVector apply(WorkerPool& pool, const ShardedVector& x) const {
    if (x.dim() != dim) throw layout_error("operator/vector dimension mismatch");
    ShardedVector y = make_sharded(x.layout, x.prec);
    const std::size_t es = x.esize();
    DeviceBuffer xf(dim * es), yf(dim * es);
    for (std::size_t w = 0; w < x.layout.worker_count(); ++w)
      cuda_ok(cudaMemcpy(static_cast<char*>(xf.get()) + x.layout.shard_bounds[w].begin * es, x.shards[w].get(),
                         x.layout.shard_bounds[w].size() * es, cudaMemcpyDeviceToDevice));
    check(sd_operator_apply(native.get(), xf.get(), yf.get(), prec_code(x.prec), pool.stream()));
    pool.sync();
    for (std::size_t w = 0; w < x.layout.worker_count(); ++w)
      cuda_ok(cudaMemcpy(y.shards[w].get(), static_cast<char*>(yf.get()) + x.layout.shard_bounds[w].begin * es,
                         x.layout.shard_bounds[w].size() * es, cudaMemcpyDeviceToDevice));
    return y;
  }
};

inline OperatorHandle dense_operator(std::shared_ptr<const DenseSymmetric> m, std::string label) {
  sd_operator op = nullptr;
  check(sd_operator_dense(m->n, m->a.data(), &op));
  return OperatorHandle{m->n, std::move(label), std::shared_ptr<sd_operator_s>(op, sd_operator_destroy)};
}
inline DenseSymmetric wigner_dense(std::size_t n, double sigma, std::uint64_t seed) {
  DenseSymmetric m;
  m.n = n;
  m.a.resize(n * n);
  check(sd_wigner_dense(n, sigma, seed, m.a.data()));
  return m;
}
inline OperatorHandle wigner_operator(std::size_t n, double sigma, std::uint64_t seed) {
  return dense_operator(std::make_shared<DenseSymmetric>(wigner_dense(n, sigma, seed)),
                        "wigner(n=" + std::to_string(n) + ")");
}
inline DenseSymmetric spiked_dense(std::size_t n, double sigma, const std::vector<double>& spikes,
                                   std::uint64_t seed) {
  DenseSymmetric m;
  m.n = n;
  m.a.resize(n * n);
  check(sd_spiked_dense(n, sigma, spikes.data(), spikes.size(), seed, m.a.data()));
  return m;
}
inline OperatorHandle spiked_operator(std::size_t n, double sigma, const std::vector<double>& spikes,
                                      std::uint64_t seed) {
  return dense_operator(std::make_shared<DenseSymmetric>(spiked_dense(n, sigma, spikes, seed)),
                        "spiked(n=" + std::to_string(n) + ")");
}

// ---- lanczos and quadrature
enum class Reorthogonalize { none, full, selective };
struct LanczosConfig {
  std::size_t k_max = 10;
  double breakdown_tol = -1.0;  // <= 0: 1e-12 (f64) / 1e-7 (f32)
  Reorthogonalize reorthogonalize = Reorthogonalize::none;
  ProbeSpec probe;
  Precision prec = Precision::f64;
  std::size_t window = 0;  // selective: keep the W >= 2 most recent basis vectors (extension)
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

inline LanczosRun lanczos_run(const OperatorHandle& op, const LanczosConfig& cfg, WorkerPool& pool) {
  const int ro = cfg.reorthogonalize == Reorthogonalize::full        ? SD_REORTH_FULL
                 : cfg.reorthogonalize == Reorthogonalize::selective ? SD_REORTH_SELECTIVE
                                                                     : SD_REORTH_NONE;
  sd_lanczos_config c{cfg.k_max, cfg.breakdown_tol, ro, prec_code(cfg.prec), cfg.probe.seed,
                      dist_code(cfg.probe.distribution), 0};
  c.selective_window = cfg.window;
  const uint64_t b = 0, e = op.dim;
  const uint64_t bytes = sd_lanczos_workspace_bytes(&b, &e, op.dim, &c, 1, 0);
  if (!bytes) check(SD_CONFIG_ERROR);
  DeviceBuffer ws(bytes);
  std::vector<double> al(cfg.k_max), be(cfg.k_max);
  sd_lanczos_info info{};
  const sd_status st = sd_lanczos_run(op.native.get(), nullptr, &b, &e, op.dim, &c, ws.get(), bytes, al.data(),
                                      be.data(), &info, pool.stream());
  check(st);
  LanczosRun r;
  r.t.alphas.assign(al.begin(), al.begin() + info.n_alpha);
  r.t.betas.assign(be.begin(), be.begin() + info.n_beta);
  r.breakdown = info.breakdown != 0;
  r.ms_apply = info.ms_apply;
  r.ms_recurrence = info.ms_recurrence;
  r.ms_reorth = info.ms_reorth;
  return r;
}

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


// ---- autodiff: hvp / batched_hvp (Alg. 1)
// ModelSpec architectures: mlp(layer_widths) with mse and the
// decoder family the SPEC's attention_block grows into (GPT-2 style, or
// Llama style: sd_gpt_config.arch). The device engine computes in fp32
// (3xTF32 tensor-core GEMMs), so vectors must be Precision::f32.
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
class Model {
 public:
  // transformer with the synthetic counter-keyed init (sd_gpt_init_params)
  Model(WorkerPool& pool, const ModelSpec& spec, std::uint64_t init_seed, double gain_scale = 0.0,
        double bias_scale = 0.0)
      : spec_(spec), P_(spec.parameter_count()), theta_(P_ * 4) {
    if (spec.arch != ModelSpec::Arch::transformer) throw config_error("this constructor builds transformer models");
    if (P_ == 0) check(SD_CONFIG_ERROR);
    check(sd_gpt_init_params(&spec_.transformer, init_seed, gain_scale, bias_scale,
                             static_cast<float*>(theta_.get()), pool.stream()));
    pool.sync();
  }
  // mlp with caller parameters (flat declaration order, f32-representable), n_max rows per batch
  Model(WorkerPool& pool, const ModelSpec& spec, const std::vector<double>& params, int n_max)
      : spec_(spec), P_(spec.parameter_count()), theta_(P_ * 4) {
    (void)pool;
    if (spec.arch != ModelSpec::Arch::mlp) throw config_error("this constructor builds mlp models");
    if (params.size() != P_) throw layout_error("parameter count does not match the model");
    std::vector<float> f(params.begin(), params.end());
    cuda_ok(cudaMemcpy(theta_.get(), f.data(), P_ * 4, cudaMemcpyHostToDevice));
    sd_mlp m = nullptr;
    check(sd_mlp_create(spec_.layer_widths.data(), int(spec_.layer_widths.size()), n_max,
                        static_cast<const float*>(theta_.get()), pool.stream(), &m));
    mlp_.reset(m, sd_mlp_destroy);
    n_max_ = n_max;
  }
  std::size_t parameter_count() const { return P_; }
  const ModelSpec& spec() const { return spec_; }

  // Hv (full logical vectors on device) of one batch with loss weight `scale`
  void hvp_device(WorkerPool& pool, const Batch& b, float scale, const float* v, float* hv) {
    if (spec_.arch == ModelSpec::Arch::mlp) {
      const int w0 = int(spec_.layer_widths.front()), wl = int(spec_.layer_widths.back());
      if (b.rows < 1) throw argument_error("empty batch");
      if (b.rows > n_max_) throw argument_error("batch exceeds the engine's row capacity");
      if (b.x.size() != std::size_t(b.rows) * w0 || b.y.size() != std::size_t(b.rows) * wl)
        throw argument_error("inconsistent sample dimensions");
      check(sd_mlp_set_batch(mlp_.get(), b.x.data(), b.y.data(), b.rows, scale, pool.stream()));
      check(sd_mlp_hvp(mlp_.get(), v, hv, pool.stream()));
      return;
    }
    if (b.rows < 1 || b.seq < 1) throw argument_error("empty batch");
    if (b.tokens.size() != std::size_t(b.rows) * b.seq || b.token_targets.size() != b.tokens.size())
      throw argument_error("inconsistent sample dimensions");
    Engine& e = engine(pool, b.rows, b.seq);
    check(sd_gpt_set_batch(e.g.get(), b.tokens.data(), b.token_targets.data(), scale, pool.stream()));
    check(sd_gpt_hvp(e.g.get(), v, hv, pool.stream()));
  }

 private:
  struct Engine {
    DeviceBuffer ws;
    std::shared_ptr<sd_gpt_s> g;
  };
  Engine& engine(WorkerPool& pool, int rows, int seq) {
    const auto key = std::make_pair(rows, seq);
    auto it = engines_.find(key);
    if (it != engines_.end()) return it->second;
    const uint64_t bytes = sd_gpt_workspace_bytes(&spec_.transformer, rows, seq);
    if (!bytes) {  // invalid shape: the create call reports the precise error class
      sd_gpt g = nullptr;
      check(sd_gpt_create(&spec_.transformer, rows, seq, static_cast<const float*>(theta_.get()), nullptr, 0,
                          pool.stream(), &g));
    }
    // built in place: the engine keeps pointers into its workspace (DeviceBuffer copies, it does not move)
    Engine& e = engines_[key];
    try {
      e.ws = DeviceBuffer(bytes);
      sd_gpt g = nullptr;
      check(sd_gpt_create(&spec_.transformer, rows, seq, static_cast<const float*>(theta_.get()), e.ws.get(), bytes,
                          pool.stream(), &g));
      e.g.reset(g, sd_gpt_destroy);
    } catch (...) {
      engines_.erase(key);
      throw;
    }
    return e;
  }
  ModelSpec spec_;
  std::size_t P_ = 0;
  DeviceBuffer theta_;
  std::shared_ptr<sd_mlp_s> mlp_;
  int n_max_ = 0;
  std::map<std::pair<int, int>, Engine> engines_;
};

namespace detail {
inline DeviceBuffer gather_device(const ShardedVector& x) {
  const std::size_t es = x.esize();
  DeviceBuffer full(x.dim() * es);
  for (std::size_t w = 0; w < x.layout.worker_count(); ++w)
    cuda_ok(cudaMemcpy(static_cast<char*>(full.get()) + x.layout.shard_bounds[w].begin * es, x.shards[w].get(),
                       x.layout.shard_bounds[w].size() * es, cudaMemcpyDeviceToDevice));
  return full;
}
inline void scatter_device(const DeviceBuffer& full, ShardedVector& y) {
  const std::size_t es = y.esize();
  for (std::size_t w = 0; w < y.layout.worker_count(); ++w)
    cuda_ok(cudaMemcpy(y.shards[w].get(), static_cast<const char*>(full.get()) + y.layout.shard_bounds[w].begin * es,
                       y.layout.shard_bounds[w].size() * es, cudaMemcpyDeviceToDevice));
}
inline void check_model_vector(WorkerPool& pool, const Model& m, const ShardedVector& v) {
  check_pool(pool, v);
  if (v.dim() != m.parameter_count()) throw layout_error("vector dimension does not match the model");
  if (v.prec != Precision::f32) throw config_error("the HVP engine computes in f32: use Precision::f32 vectors");
}
}  // namespace detail

// Hv of the batch-mean loss (Pearlmutter, forward-over-reverse on device)
inline ShardedVector hvp(WorkerPool& pool, Model& m, const Batch& batch, const ShardedVector& v) {
  detail::check_model_vector(pool, m, v);
  DeviceBuffer xf = detail::gather_device(v), yf(v.dim() * 4);
  const double n = double(batch.samples()) *
                   (m.spec().arch == ModelSpec::Arch::mlp ? double(m.spec().layer_widths.back()) : 1.0);
  m.hvp_device(pool, batch, float(1.0 / n), static_cast<const float*>(xf.get()), static_cast<float*>(yf.get()));
  pool.sync();
  ShardedVector y = make_sharded(v.layout, v.prec);
  detail::scatter_device(yf, y);
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
  for (const Batch& b : loader) N += double(b.samples());
  if (m.spec().arch == ModelSpec::Arch::mlp) N *= double(m.spec().layer_widths.back());
  DeviceBuffer xf = detail::gather_device(v), tmp(v.dim() * 4), acc(v.dim() * 4);
  cuda_ok(cudaMemset(acc.get(), 0, v.dim() * 4));
  detail::DevScalar one(1.0);
  for (const Batch& b : loader) {
    m.hvp_device(pool, b, float(1.0 / N), static_cast<const float*>(xf.get()), static_cast<float*>(tmp.get()));
    check(sd_k_axpy(tmp.get(), acc.get(), v.dim(), one.p(), 1.0, SD_F32, pool.stream()));
  }
  pool.sync();
  ShardedVector y = make_sharded(v.layout, v.prec);
  detail::scatter_device(acc, y);
  return y;
}

// The model's Hessian on one batch as an OperatorHandle (what lanczos_run drives).
inline OperatorHandle hvp_operator(WorkerPool& pool, Model& m, const Batch& batch) {
  struct Ctx {
    Model* m;
    Batch b;
    WorkerPool* pool;
    float scale;
  };
  const double n = double(batch.samples()) *
                   (m.spec().arch == ModelSpec::Arch::mlp ? double(m.spec().layer_widths.back()) : 1.0);
  auto* ctx = new Ctx{&m, batch, &pool, float(1.0 / n)};
  static const sd_apply_fn fn = [](void* c, const void* x, void* y, sd_stream) -> sd_status {
    auto* k = static_cast<Ctx*>(c);
    try {
      k->m->hvp_device(*k->pool, k->b, k->scale, static_cast<const float*>(x), static_cast<float*>(y));
    } catch (const std::exception&) {
      return SD_ARGUMENT_ERROR;
    }
    return SD_OK;
  };
  sd_operator op = nullptr;
  check(sd_operator_custom(m.parameter_count(), fn, ctx, &op));
  std::shared_ptr<sd_operator_s> h(op, [ctx](sd_operator o) {
    sd_operator_destroy(o);
    delete ctx;
  });
  return OperatorHandle{m.parameter_count(), "hvp", std::move(h)};
}

}  // namespace specden

// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// CPU restatement of the HessFormer SLQ path (arxiv 2505.11564) as specified by
// the C++ reference under /root/reference/proj and SPEC.md. Only tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
// may load it; the product path (paper_2505_11564_b200/) never does.
//
// Parity status: the RNG, layout, blocked reduction, vector ops and dense
// operators are PINNED bitwise against the compiled reference (oracle/_ref,
// built from /root/reference/proj/src by oracle/build_ref.sh) and against the
// Appendix-A golden values in SURVEY.md. Lanczos, Ritz, density, the autodiff
// Graph and the HVP have no reference implementation (SPEC only); they are
// pinned by SPEC known answers (tests/test_oracle_*.py) and finite differences.
#pragma once

#include <cmath>
#include <cstddef>
#include <cstdint>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

namespace sdo {

// ---- errors: the six classes of proj/include/specden/errors.hpp:13-41 -----
enum class Err { ok = 0, config = 1, layout = 2, argument = 3, numerical = 4, state = 5, protocol = 6 };
struct error : std::runtime_error {
  Err kind;
  error(Err k, const std::string& w) : std::runtime_error(w), kind(k) {}
};
[[noreturn]] inline void fail(Err k, const std::string& w) { throw error(k, w); }

// ---- precision: proj/include/specden/precision.hpp:15-24 -------------------
enum class Precision { f32 = 0, f64 = 1 };
inline double round_elem(double x, Precision p) {
  return p == Precision::f32 ? double(float(x)) : x;
}
inline double unit_roundoff(Precision p) { return p == Precision::f32 ? 0x1p-24 : 0x1p-53; }

// ---- counter RNG: proj/include/specden/rng.hpp:17-52 -----------------------
inline uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z ^= z >> 30;
  z *= 0xbf58476d1ce4e5b9ull;
  z ^= z >> 27;
  z *= 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
inline uint64_t keyed_counter(uint64_t seed, uint64_t ctr) {
  const uint64_t key = mix64(seed);
  return mix64(key ^ (ctr * 0x9e3779b97f4a7c15ull));
}
inline double uniform01(uint64_t seed, uint64_t ctr) {
  return double(keyed_counter(seed, ctr) >> 11) * 0x1p-53 + 0x1p-54;
}
inline double gaussian(uint64_t seed, uint64_t i) {
  const double a = uniform01(seed, 2 * i), b = uniform01(seed, 2 * i + 1);
  const double two_pi = 2.0 * 3.141592653589793;  // std::numbers::pi, (2*pi) rounded first
  return std::sqrt(-2.0 * std::log(a)) * std::cos(two_pi * b);
}
inline double rademacher(uint64_t seed, uint64_t i) {
  return (keyed_counter(seed, i) & 1ull) != 0 ? 1.0 : -1.0;
}
inline uint64_t uniform_index(uint64_t seed, uint64_t i, uint64_t n) { return keyed_counter(seed, i) % n; }

// ---- layout: proj/include/specden/layout.hpp:12-72 -------------------------
struct Range {
  size_t begin = 0, end = 0;
  size_t size() const { return end - begin; }
};
struct Layout {
  size_t total = 0;
  std::vector<Range> shards;
  size_t workers() const { return shards.size(); }
};
void validate_layout(const Layout& l);
Layout split_evenly(size_t dim, size_t n);
size_t layout_owner(const Layout& l, size_t i);

// ---- blocked reduction: proj/include/specden/reduction.hpp:30-115 ----------
constexpr size_t kBlock = 1024;
size_t oracle_threads();  // matmul worker threads (ORACLE_THREADS, default all cores)
// One worker's share of the fixed-grid fold over [begin, end).
struct Partial {
  size_t begin = 0, end = 0;
  std::vector<double> head, sums, tail;
};
Partial make_partial(size_t begin, size_t end, size_t total, const std::function<double(size_t)>& term,
                     size_t block = kBlock);
double combine_partials(const std::vector<Partial>& parts, size_t total, size_t block = kBlock);
// Whole-vector evaluation of the same DAG (block folds, then fold of block sums).
double blocked_sum(const double* terms, size_t n, size_t block = kBlock);

// ---- vectors: proj/src/sharded.cpp:59-154 ----------------------------------
// A logical vector; sharding never changes a value (all ops are layout
// invariant by construction), so the oracle keeps it flat.
struct Vec {
  Precision prec = Precision::f64;
  std::vector<double> x;
  size_t dim() const { return x.size(); }
};
enum class ProbeDist { gaussian = 0, rademacher = 1, one_hot = 2 };
struct ProbeSpec {
  uint64_t seed = 42;
  ProbeDist dist = ProbeDist::gaussian;
  size_t one_hot_index = 0;
  bool normalize = true;
};
Vec draw_probe(size_t dim, const ProbeSpec& spec, Precision prec);
double dot(const Vec& a, const Vec& b);
double norm2(const Vec& a);
Vec axpy(double alpha, const Vec& x, const Vec& y);
Vec scale(const Vec& x, double c);

// ---- dense operators: proj/src/operators.cpp:19-112 ------------------------
constexpr size_t kDenseCap = 2048;
struct Dense {
  size_t n = 0;
  std::vector<double> a;
};
Dense wigner_dense(size_t n, double sigma, uint64_t seed);
Dense spiked_dense(size_t n, double sigma, const std::vector<double>& spikes, uint64_t seed);
Vec dense_apply(const Dense& m, const Vec& x);

// ---- Lanczos: Alg. 2 ------------------------------
enum class Reorth { none = 0, full = 1, selective = 2 };
struct LanczosConfig {
  size_t k_max = 10;
  double eps = -1.0;  // <0: default 1e-12 (f64) / 1e-7 (f32)
  Reorth reorth = Reorth::none;
  ProbeSpec probe;
  Precision prec = Precision::f64;
  bool store_basis = false;  // forced on by full reorth
  size_t window = 0;         // selective: the most recent `window` columns (>= 2)
};
struct LanczosResult {
  std::vector<double> alphas, betas;
  std::vector<double> step_beta;  // every computed beta, including the breaking one
  std::vector<Vec> basis;
  bool breakdown = false;  // beta < eps (benign)
  bool numerical_failure = false;
  std::string message;
};
using ApplyFn = std::function<void(const Vec& x, Vec& y)>;
LanczosResult lanczos_run(size_t dim, const ApplyFn& apply, const LanczosConfig& cfg);
double loss_of_orthogonality(const std::vector<Vec>& basis);

// ---- quadrature: SPEC.md:302-368 -------------------------------------------
struct Ritz {
  std::vector<double> values, weights;
};
Ritz ritz_decompose(const std::vector<double>& alphas, const std::vector<double>& betas);
struct Density {
  std::vector<double> grid, density;
  double sigma = 0.0;
};
Density smooth_density(const Ritz& s, double sigma, size_t grid_points);
Ritz average_spectra(const std::vector<Ritz>& runs);

// ---- autodiff Graph: proj/include/specden/autodiff.hpp:14-101 --------------
struct Tensor {
  size_t rows = 0, cols = 0;
  std::vector<double> v;
  Tensor() = default;
  Tensor(size_t r, size_t c, double fill = 0.0) : rows(r), cols(c), v(r * c, fill) {}
  size_t numel() const { return rows * cols; }
  double& at(size_t i, size_t j) { return v[i * cols + j]; }
  double at(size_t i, size_t j) const { return v[i * cols + j]; }
};

class Graph {
 public:
  explicit Graph(Precision p = Precision::f64) : prec_(p) {}
  int constant(Tensor t);
  int param(Tensor t);
  int add(int a, int b);
  int sub(int a, int b);
  int mul(int a, int b);
  int smul(int a, double c);
  int addrow(int a, int row);
  int mulcol(int a, int col);
  int matmul(int a, int b, bool ta = false, bool tb = false);
  int tanh_(int a);
  int exp_(int a);
  int log_(int a);
  int recip(int a);
  int softmax_rows(int a);
  int sum_rows(int a);
  int sum_cols(int a);
  int sum_all(int a);
  int mean_all(int a);
  int mse(int pred, int target);
  int cross_entropy(int logits, int onehot);
  std::vector<int> grad(int loss, const std::vector<int>& wrt, bool create_graph = true);
  const Tensor& val(int id) const { return nodes_.at(size_t(id)).val; }
  size_t node_count() const { return nodes_.size(); }
  Precision precision() const { return prec_; }
  int ones(size_t r, size_t c);

 private:
  enum class Op { Const, Param, Add, Sub, Mul, Smul, AddRow, MulCol, Matmul, Tanh, Exp, Log, Recip, Softmax, SumRows, SumCols, SumAll };
  struct Node {
    Op op;
    int a = -1, b = -1;
    bool ta = false, tb = false;
    double c = 0.0;
    bool rg = false;
    Tensor val;
  };
  int push(Node n);
  bool rg(int id) const { return nodes_[size_t(id)].rg; }
  void accumulate(std::vector<int>& adj, int node, int term);
  std::vector<Node> nodes_;
  Precision prec_;
  bool detached_ = false;
};

// ---- models and HVP: Alg. 1 ----------------------
// GPT-style decoder (GPT-2 block structure, tied embeddings, pre-LN, GELU-tanh,
// causal softmax attention composed from primitives). Flat parameter order is
// declaration order, row-major:
//   wte[V,d], wpe[S,d], per layer {ln1.g[d], ln1.b[d], attn.W[d,3d], attn.b[3d],
//   proj.W[d,d], proj.b[d], ln2.g[d], ln2.b[d], fc.W[d,ff], fc.b[ff],
//   fcp.W[ff,d], fcp.b[d]}, lnf.g[d], lnf.b[d].
struct GptConfig {
  size_t n_layer = 1, d = 64, n_head = 4, ff = 256, vocab = 64, ctx = 32;
  double ln_eps = 1e-5;
  int arch = 0;              // 0: GPT-2 block; 1: Llama-style (RMSNorm, RoPE, SwiGLU, untied head, no biases)
  double rope_base = 10000.0;
  size_t n_kv_head = 0;      // Llama: key/value heads (grouped-query attention); 0 = n_head
};
struct ParamSlot {
  std::string name;
  size_t offset, rows, cols;
  int kind;  // 0 matrix, 1 ln gain, 2 ln bias / linear bias
};
std::vector<ParamSlot> gpt_layout(const GptConfig& c);
size_t gpt_param_count(const GptConfig& c);
// theta[i] = base(kind) + scale(kind) * gaussian(seed, i); scales {0.02, gain_s, bias_s}.
std::vector<double> gpt_init(const GptConfig& c, uint64_t seed, double gain_scale, double bias_scale, Precision p);
struct Batch {
  size_t B = 1, S = 1;
  std::vector<uint32_t> tokens, targets;  // B*S each
};
Batch synthetic_batch(const GptConfig& c, size_t B, size_t S, uint64_t seed_tok, uint64_t first_seq);
double gpt_loss(const GptConfig& c, const std::vector<double>& theta, const Batch& b, Precision p);
std::vector<double> gpt_grad(const GptConfig& c, const std::vector<double>& theta, const Batch& b, Precision p);
std::vector<double> gpt_hvp(const GptConfig& c, const std::vector<double>& theta, const Batch& b,
                            const std::vector<double>& v, Precision p);
// Alg. 1: sum_b |B| * u_b / N.
std::vector<double> gpt_batched_hvp(const GptConfig& c, const std::vector<double>& theta,
                                    const std::vector<Batch>& loader, const std::vector<double>& v, Precision p);

// MLP with tanh hidden layers and mse loss (mlp(layer_widths)).
struct MlpData {
  size_t n = 0;
  std::vector<double> x, y;  // n x widths.front(), n x widths.back()
};
size_t mlp_param_count(const std::vector<size_t>& widths);
std::vector<double> mlp_grad(const std::vector<size_t>& widths, const std::vector<double>& theta, const MlpData& d,
                             Precision p);
std::vector<double> mlp_hvp(const std::vector<size_t>& widths, const std::vector<double>& theta, const MlpData& d,
                            const std::vector<double>& v, Precision p);

}  // namespace sdo

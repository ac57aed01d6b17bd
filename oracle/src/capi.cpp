// ORACLE — TEST INFRASTRUCTURE ONLY (see sdo.hpp header).
// extern "C" surface of the oracle for tests/ (ctypes) and bench.py's
// cpu_baseline / --impl reference legs. Status codes follow sdo::Err.
#include <cstring>
#include <string>

#include "sdo.hpp"

using namespace sdo;

static thread_local std::string g_err;

#define ORACLE_TRY(...)                    \
  try {                                    \
    __VA_ARGS__;                           \
    return 0;                              \
  } catch (const sdo::error& e) {          \
    g_err = e.what();                      \
    return int(e.kind);                    \
  } catch (const std::exception& e) {      \
    g_err = e.what();                      \
    return 99;                             \
  }

static GptConfig gcfg(const long long* c) {
  GptConfig g;
  g.n_layer = size_t(c[0]);
  g.d = size_t(c[1]);
  g.n_head = size_t(c[2]);
  g.ff = size_t(c[3]);
  g.vocab = size_t(c[4]);
  g.ctx = size_t(c[5]);
  g.arch = int(c[6]);
  g.rope_base = double(c[7]);
  g.n_kv_head = size_t(c[8]);
  return g;
}

static Batch gbatch(long long B, long long S, const unsigned* tok, const unsigned* tgt) {
  Batch b;
  b.B = size_t(B);
  b.S = size_t(S);
  b.tokens.assign(tok, tok + B * S);
  b.targets.assign(tgt, tgt + B * S);
  return b;
}

extern "C" {

const char* oracle_last_error() { return g_err.c_str(); }

unsigned long long oracle_mix64(unsigned long long x) { return mix64(x); }
unsigned long long oracle_keyed_counter(unsigned long long s, unsigned long long c) { return keyed_counter(s, c); }
double oracle_uniform01(unsigned long long s, unsigned long long c) { return uniform01(s, c); }
double oracle_gaussian(unsigned long long s, unsigned long long i) { return gaussian(s, i); }
double oracle_rademacher(unsigned long long s, unsigned long long i) { return rademacher(s, i); }
unsigned long long oracle_uniform_index(unsigned long long s, unsigned long long i, unsigned long long n) {
  return uniform_index(s, i, n);
}

void oracle_gaussian_fill(unsigned long long seed, unsigned long long first, long long n, double* out) {
  for (long long i = 0; i < n; ++i) out[i] = gaussian(seed, first + (unsigned long long)i);
}

int oracle_split_evenly(long long dim, long long n, long long* begins, long long* ends, long long* count) {
  ORACLE_TRY({
    const Layout l = split_evenly(size_t(dim < 0 ? 0 : dim), size_t(n < 0 ? 0 : n));
    for (size_t w = 0; w < l.workers(); ++w) {
      begins[w] = (long long)l.shards[w].begin;
      ends[w] = (long long)l.shards[w].end;
    }
    *count = (long long)l.workers();
  })
}

int oracle_validate_layout(long long total, long long n, const long long* begins, const long long* ends) {
  ORACLE_TRY({
    Layout l;
    l.total = size_t(total);
    for (long long w = 0; w < n; ++w) l.shards.push_back({size_t(begins[w]), size_t(ends[w])});
    validate_layout(l);
  })
}

int oracle_draw_probe(long long dim, unsigned long long seed, int dist, long long one_hot, int normalize, int prec,
                      double* out) {
  ORACLE_TRY({
    ProbeSpec s;
    s.seed = seed;
    s.dist = ProbeDist(dist);
    s.one_hot_index = size_t(one_hot);
    s.normalize = normalize != 0;
    const Vec v = draw_probe(size_t(dim), s, Precision(prec));
    std::memcpy(out, v.x.data(), v.x.size() * sizeof(double));
  })
}

double oracle_dot(long long n, const double* a, const double* b) {
  Vec x, y;
  x.x.assign(a, a + n);
  y.x.assign(b, b + n);
  return dot(x, y);
}

double oracle_blocked_sum(long long n, const double* terms) { return blocked_sum(terms, size_t(n)); }

int oracle_axpy(long long n, double alpha, const double* x, const double* y, int prec, double* out) {
  ORACLE_TRY({
    Vec a, b;
    a.prec = b.prec = Precision(prec);
    a.x.assign(x, x + n);
    b.x.assign(y, y + n);
    const Vec o = axpy(alpha, a, b);
    std::memcpy(out, o.x.data(), size_t(n) * sizeof(double));
  })
}

int oracle_scale(long long n, const double* x, double c, int prec, double* out) {
  ORACLE_TRY({
    Vec a;
    a.prec = Precision(prec);
    a.x.assign(x, x + n);
    const Vec o = scale(a, c);
    std::memcpy(out, o.x.data(), size_t(n) * sizeof(double));
  })
}

// Blocked partial of sum_i a[i]*b[i] over [begin,end) of a length-`total`
// vector (a, b are the shard slices). Writes head/sums/tail into `buf` in that
// order and their counts into counts[3].
int oracle_dot_partial(long long begin, long long end, long long total, const double* a, const double* b, double* buf,
                       long long* counts) {
  ORACLE_TRY({
    const Partial p = make_partial(size_t(begin), size_t(end), size_t(total),
                                   [&](size_t i) { return a[i - size_t(begin)] * b[i - size_t(begin)]; });
    size_t k = 0;
    for (double t : p.head) buf[k++] = t;
    for (double t : p.sums) buf[k++] = t;
    for (double t : p.tail) buf[k++] = t;
    counts[0] = (long long)p.head.size();
    counts[1] = (long long)p.sums.size();
    counts[2] = (long long)p.tail.size();
  })
}

// parts: n workers; for worker w, range [begins[w], ends[w]), counts[3w..3w+2],
// and its head/sums/tail values concatenated in `buf` (worker order).
int oracle_combine_partials(long long n, long long total, const long long* begins, const long long* ends,
                            const long long* counts, const double* buf, double* out) {
  ORACLE_TRY({
    std::vector<Partial> parts((size_t)n);
    size_t k = 0;
    for (long long w = 0; w < n; ++w) {
      Partial& p = parts[size_t(w)];
      p.begin = size_t(begins[w]);
      p.end = size_t(ends[w]);
      for (long long i = 0; i < counts[3 * w]; ++i) p.head.push_back(buf[k++]);
      for (long long i = 0; i < counts[3 * w + 1]; ++i) p.sums.push_back(buf[k++]);
      for (long long i = 0; i < counts[3 * w + 2]; ++i) p.tail.push_back(buf[k++]);
    }
    *out = combine_partials(parts, size_t(total));
  })
}

int oracle_wigner(long long n, double sigma, unsigned long long seed, double* out) {
  ORACLE_TRY({
    const Dense m = wigner_dense(size_t(n), sigma, seed);
    std::memcpy(out, m.a.data(), m.a.size() * sizeof(double));
  })
}

int oracle_spiked(long long n, double sigma, const double* spikes, long long ns, unsigned long long seed, double* out) {
  ORACLE_TRY({
    const Dense m = spiked_dense(size_t(n), sigma, std::vector<double>(spikes, spikes + ns), seed);
    std::memcpy(out, m.a.data(), m.a.size() * sizeof(double));
  })
}

int oracle_dense_apply(long long n, const double* a, const double* x, int prec, double* y) {
  ORACLE_TRY({
    Dense m;
    m.n = size_t(n);
    m.a.assign(a, a + n * n);
    Vec v;
    v.prec = Precision(prec);
    v.x.assign(x, x + n);
    const Vec o = dense_apply(m, v);
    std::memcpy(y, o.x.data(), size_t(n) * sizeof(double));
  })
}

// Lanczos over a dense operator. out_alpha/out_beta sized k_max; out_basis
// (optional) sized (k_max+1)*n. info[0]=#alphas, info[1]=#betas,
// info[2]=breakdown, info[3]=numerical failure, info[4]=#basis columns.
int oracle_lanczos_dense(long long n, const double* a, long long k_max, double eps, int reorth, long long window,
                         unsigned long long seed,
                         int dist, int prec, double* out_alpha, double* out_beta, double* out_step_beta,
                         double* out_basis, long long* info) {
  ORACLE_TRY({
    Dense m;
    m.n = size_t(n);
    m.a.assign(a, a + n * n);
    LanczosConfig cfg;
    cfg.k_max = size_t(k_max);
    cfg.eps = eps;
    cfg.reorth = Reorth(reorth);
    cfg.window = size_t(window);
    cfg.probe.seed = seed;
    cfg.probe.dist = ProbeDist(dist);
    cfg.prec = Precision(prec);
    cfg.store_basis = out_basis != nullptr;
    const LanczosResult r = lanczos_run(size_t(n), [&](const Vec& x, Vec& y) { y = dense_apply(m, x); }, cfg);
    for (size_t i = 0; i < r.alphas.size(); ++i) out_alpha[i] = r.alphas[i];
    for (size_t i = 0; i < r.betas.size(); ++i) out_beta[i] = r.betas[i];
    for (size_t i = 0; i < r.step_beta.size(); ++i) out_step_beta[i] = r.step_beta[i];
    if (out_basis)
      for (size_t j = 0; j < r.basis.size(); ++j)
        std::memcpy(out_basis + j * size_t(n), r.basis[j].x.data(), size_t(n) * sizeof(double));
    info[0] = (long long)r.alphas.size();
    info[1] = (long long)r.betas.size();
    info[2] = r.breakdown;
    info[3] = r.numerical_failure;
    info[4] = (long long)r.basis.size();
  })
}

// Lanczos over the diagonal operator y_i = round(d_i * x_i) (exact product, one rounding).
int oracle_lanczos_diag(long long n, const double* d, long long k_max, double eps, int reorth, long long window,
                        unsigned long long seed,
                        int dist, int prec, double* out_alpha, double* out_beta, long long* info) {
  ORACLE_TRY({
    LanczosConfig cfg;
    cfg.k_max = size_t(k_max);
    cfg.eps = eps;
    cfg.reorth = Reorth(reorth);
    cfg.window = size_t(window);
    cfg.probe.seed = seed;
    cfg.probe.dist = ProbeDist(dist);
    cfg.prec = Precision(prec);
    const LanczosResult r = lanczos_run(
        size_t(n),
        [&](const Vec& x, Vec& y) {
          for (size_t i = 0; i < x.dim(); ++i) y.x[i] = round_elem(d[i] * x.x[i], x.prec);
        },
        cfg);
    for (size_t i = 0; i < r.alphas.size(); ++i) out_alpha[i] = r.alphas[i];
    for (size_t i = 0; i < r.betas.size(); ++i) out_beta[i] = r.betas[i];
    info[0] = (long long)r.alphas.size();
    info[1] = (long long)r.betas.size();
    info[2] = r.breakdown;
    info[3] = r.numerical_failure;
  })
}

int oracle_ritz(long long k, const double* alphas, const double* betas, double* values, double* weights) {
  ORACLE_TRY({
    const Ritz r = ritz_decompose(std::vector<double>(alphas, alphas + k), std::vector<double>(betas, betas + (k - 1)));
    std::memcpy(values, r.values.data(), size_t(k) * sizeof(double));
    std::memcpy(weights, r.weights.data(), size_t(k) * sizeof(double));
  })
}

int oracle_smooth_density(long long k, const double* values, const double* weights, double sigma, long long npts,
                          double* grid, double* dens, double* sigma_used) {
  ORACLE_TRY({
    Ritz r;
    r.values.assign(values, values + k);
    r.weights.assign(weights, weights + k);
    const Density d = smooth_density(r, sigma, size_t(npts));
    std::memcpy(grid, d.grid.data(), size_t(npts) * sizeof(double));
    std::memcpy(dens, d.density.data(), size_t(npts) * sizeof(double));
    *sigma_used = d.sigma;
  })
}

// ---- GPT. cfg = {n_layer, d, n_head, ff, vocab, ctx}
long long oracle_gpt_param_count(const long long* cfg) { return (long long)gpt_param_count(gcfg(cfg)); }

int oracle_gpt_layout(const long long* cfg, long long* offsets, long long* rows, long long* cols, int* kinds,
                      long long* count) {
  ORACLE_TRY({
    const auto s = gpt_layout(gcfg(cfg));
    for (size_t i = 0; i < s.size(); ++i) {
      offsets[i] = (long long)s[i].offset;
      rows[i] = (long long)s[i].rows;
      cols[i] = (long long)s[i].cols;
      kinds[i] = s[i].kind;
    }
    *count = (long long)s.size();
  })
}

int oracle_gpt_init(const long long* cfg, unsigned long long seed, double gain_scale, double bias_scale, int prec,
                    double* out) {
  ORACLE_TRY({
    const auto th = gpt_init(gcfg(cfg), seed, gain_scale, bias_scale, Precision(prec));
    std::memcpy(out, th.data(), th.size() * sizeof(double));
  })
}

int oracle_gpt_batch(const long long* cfg, long long B, long long S, unsigned long long seed_tok, long long first_seq,
                     unsigned* tokens, unsigned* targets) {
  ORACLE_TRY({
    const Batch b = synthetic_batch(gcfg(cfg), size_t(B), size_t(S), seed_tok, (uint64_t)first_seq);
    std::memcpy(tokens, b.tokens.data(), b.tokens.size() * sizeof(unsigned));
    std::memcpy(targets, b.targets.data(), b.targets.size() * sizeof(unsigned));
  })
}

int oracle_gpt_loss(const long long* cfg, const double* theta, long long B, long long S, const unsigned* tok,
                    const unsigned* tgt, int prec, double* out) {
  ORACLE_TRY({
    const GptConfig c = gcfg(cfg);
    *out = gpt_loss(c, std::vector<double>(theta, theta + gpt_param_count(c)), gbatch(B, S, tok, tgt), Precision(prec));
  })
}

int oracle_gpt_grad(const long long* cfg, const double* theta, long long B, long long S, const unsigned* tok,
                    const unsigned* tgt, int prec, double* out) {
  ORACLE_TRY({
    const GptConfig c = gcfg(cfg);
    const size_t P = gpt_param_count(c);
    const auto g = gpt_grad(c, std::vector<double>(theta, theta + P), gbatch(B, S, tok, tgt), Precision(prec));
    std::memcpy(out, g.data(), P * sizeof(double));
  })
}

int oracle_gpt_hvp(const long long* cfg, const double* theta, long long B, long long S, const unsigned* tok,
                   const unsigned* tgt, const double* v, int prec, double* out) {
  ORACLE_TRY({
    const GptConfig c = gcfg(cfg);
    const size_t P = gpt_param_count(c);
    const auto h = gpt_hvp(c, std::vector<double>(theta, theta + P), gbatch(B, S, tok, tgt),
                           std::vector<double>(v, v + P), Precision(prec));
    std::memcpy(out, h.data(), P * sizeof(double));
  })
}

// Lanczos (the same restatement as oracle_lanczos_dense)
// driven by the oracle's own GPT Hessian-vector product (SPEC.md:193-210,
// PAPER.md Alg. 1): the CPU side of the end-to-end SLQ parity check of
// BASELINE configs[0]. Vectors in `prec`; the HVP tape runs in `hvp_prec` and
// its output is rounded to `prec` (round_elem). info as oracle_lanczos_dense.
int oracle_lanczos_gpt(const long long* cfg, const double* theta, long long B, long long S, const unsigned* tok,
                       const unsigned* tgt, long long k_max, double eps, int reorth, long long window,
                       unsigned long long seed, int dist, int prec, int hvp_prec, double* out_alpha, double* out_beta,
                       long long* info) {
  ORACLE_TRY({
    const GptConfig c = gcfg(cfg);
    const size_t P = gpt_param_count(c);
    const std::vector<double> th(theta, theta + P);
    const Batch bt = gbatch(B, S, tok, tgt);
    LanczosConfig lc;
    lc.k_max = size_t(k_max);
    lc.eps = eps;
    lc.reorth = Reorth(reorth);
    lc.window = size_t(window);
    lc.probe.seed = seed;
    lc.probe.dist = ProbeDist(dist);
    lc.prec = Precision(prec);
    const LanczosResult r = lanczos_run(
        P,
        [&](const Vec& x, Vec& y) {
          const auto h = gpt_hvp(c, th, bt, x.x, Precision(hvp_prec));
          for (size_t i = 0; i < P; ++i) y.x[i] = round_elem(h[i], y.prec);
        },
        lc);
    for (size_t i = 0; i < r.alphas.size(); ++i) out_alpha[i] = r.alphas[i];
    for (size_t i = 0; i < r.betas.size(); ++i) out_beta[i] = r.betas[i];
    info[0] = (long long)r.alphas.size();
    info[1] = (long long)r.betas.size();
    info[2] = r.breakdown;
    info[3] = r.numerical_failure;
  })
}

// loader: nb batches with sizes Bs[i] (all of length S), tokens concatenated.
int oracle_gpt_batched_hvp(const long long* cfg, const double* theta, long long nb, const long long* Bs, long long S,
                           const unsigned* tok, const unsigned* tgt, const double* v, int prec, double* out) {
  ORACLE_TRY({
    const GptConfig c = gcfg(cfg);
    const size_t P = gpt_param_count(c);
    std::vector<Batch> loader;
    long long off = 0;
    for (long long i = 0; i < nb; ++i) {
      loader.push_back(gbatch(Bs[i], S, tok + off, tgt + off));
      off += Bs[i] * S;
    }
    const auto h = gpt_batched_hvp(c, std::vector<double>(theta, theta + P), loader, std::vector<double>(v, v + P),
                                   Precision(prec));
    std::memcpy(out, h.data(), P * sizeof(double));
  })
}

long long oracle_mlp_param_count(const long long* widths, long long nw) {
  return (long long)mlp_param_count(std::vector<size_t>(widths, widths + nw));
}

int oracle_mlp_grad(const long long* widths, long long nw, const double* theta, long long n, const double* x,
                    const double* y, int prec, double* out) {
  ORACLE_TRY({
    const std::vector<size_t> w(widths, widths + nw);
    MlpData d;
    d.n = size_t(n);
    d.x.assign(x, x + n * widths[0]);
    d.y.assign(y, y + n * widths[nw - 1]);
    const size_t P = mlp_param_count(w);
    const auto g = mlp_grad(w, std::vector<double>(theta, theta + P), d, Precision(prec));
    std::memcpy(out, g.data(), P * sizeof(double));
  })
}

int oracle_mlp_hvp(const long long* widths, long long nw, const double* theta, long long n, const double* x,
                   const double* y, const double* v, int prec, double* out) {
  ORACLE_TRY({
    const std::vector<size_t> w(widths, widths + nw);
    MlpData d;
    d.n = size_t(n);
    d.x.assign(x, x + n * widths[0]);
    d.y.assign(y, y + n * widths[nw - 1]);
    const size_t P = mlp_param_count(w);
    const auto h = mlp_hvp(w, std::vector<double>(theta, theta + P), d, std::vector<double>(v, v + P), Precision(prec));
    std::memcpy(out, h.data(), P * sizeof(double));
  })
}

}  // extern "C"

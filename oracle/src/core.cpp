// ORACLE — TEST INFRASTRUCTURE ONLY (see sdo.hpp header).
// Layout, blocked reduction, vector algebra, dense operators, Lanczos and
// quadrature restated from the reference and SPEC.md.
#include <algorithm>
#include <cmath>

#include "sdo.hpp"

namespace sdo {

// proj/include/specden/layout.hpp:45-55
void validate_layout(const Layout& l) {
  if (l.total == 0) fail(Err::layout, "layout covers zero dimensions");
  if (l.shards.empty()) fail(Err::layout, "layout has no shards");
  size_t at = 0;
  for (const Range& r : l.shards) {
    if (r.begin != at) fail(Err::layout, "shard bounds leave a gap or overlap");
    if (!(r.end > r.begin)) fail(Err::layout, "empty shard range");
    at = r.end;
  }
  if (at != l.total) fail(Err::layout, "shard bounds do not cover total_dim");
}

// proj/include/specden/layout.hpp:59-72: first dim%n shards get one extra; n clamped to dim.
Layout split_evenly(size_t dim, size_t n) {
  if (dim == 0 || n == 0) fail(Err::layout, "split_evenly needs dim > 0 and n > 0");
  const size_t w = std::min(dim, n);
  Layout l;
  l.total = dim;
  const size_t q = dim / w, rem = dim % w;
  size_t at = 0;
  for (size_t i = 0; i < w; ++i) {
    const size_t len = q + (i < rem);
    l.shards.push_back({at, at + len});
    at += len;
  }
  validate_layout(l);
  return l;
}

// proj/include/specden/layout.hpp:28-32 (linear scan; first shard whose end exceeds i)
size_t layout_owner(const Layout& l, size_t i) {
  for (size_t w = 0; w < l.shards.size(); ++w)
    if (l.shards[w].end > i) return w;
  fail(Err::argument, "index out of range in ShardLayout::owner");
}

// proj/include/specden/reduction.hpp:50-71
Partial make_partial(size_t begin, size_t end, size_t total, const std::function<double(size_t)>& term,
                     size_t block) {
  Partial p;
  p.begin = begin;
  p.end = end;
  size_t blk = (begin + block - 1) / block;  // first grid block starting at or after begin
  size_t i = begin;
  const size_t head_end = std::min(end, blk * block);
  while (i < head_end) p.head.push_back(term(i++));
  for (;;) {
    const size_t stop = std::min(total, (blk + 1) * block);
    if (i >= end || stop > end) break;
    double s = 0.0;
    while (i < stop) s += term(i++);
    p.sums.push_back(s);
    ++blk;
  }
  while (i < end) p.tail.push_back(term(i++));
  return p;
}

// proj/include/specden/reduction.hpp:76-107: resumes straddled blocks term by term.
double combine_partials(const std::vector<Partial>& parts, size_t total, size_t block) {
  double closed = 0.0, open = 0.0;
  size_t at = 0;
  auto grid_end = [&](size_t i) { return std::min(total, (i / block + 1) * block); };
  auto feed = [&](double t) {
    open += t;
    ++at;
    if (at == grid_end(at - 1)) {
      closed += open;
      open = 0.0;
    }
  };
  for (const Partial& p : parts) {
    if (p.begin != at) fail(Err::protocol, "blocked partials are not contiguous in worker order");
    for (double t : p.head) feed(t);
    for (double s : p.sums) {
      if (at % block != 0) fail(Err::protocol, "blocked partial misaligned with the reduction grid");
      closed += s;
      at = grid_end(at);
    }
    for (double t : p.tail) feed(t);
    if (at != p.end) fail(Err::protocol, "blocked partial does not cover its range");
  }
  if (at != total) fail(Err::protocol, "blocked partials do not cover the vector");
  return closed;
}

double blocked_sum(const double* terms, size_t n, size_t block) {
  double total = 0.0;
  for (size_t b0 = 0; b0 < n; b0 += block) {
    double s = 0.0;
    const size_t e = std::min(n, b0 + block);
    for (size_t i = b0; i < e; ++i) s += terms[i];
    total += s;
  }
  return total;
}

// ---------------------------------------------------------------- vectors
static void same_shape(const Vec& a, const Vec& b) {
  if (a.dim() != b.dim()) fail(Err::layout, "sharded vectors have different layouts");
  if (a.prec != b.prec) fail(Err::layout, "sharded vectors have different precision");
}

// proj/src/sharded.cpp:59-83
Vec draw_probe(size_t dim, const ProbeSpec& spec, Precision prec) {
  if (spec.dist == ProbeDist::one_hot && spec.one_hot_index >= dim) fail(Err::argument, "one_hot index out of range");
  Vec v;
  v.prec = prec;
  v.x.resize(dim);
  for (size_t i = 0; i < dim; ++i) {
    double e;
    if (spec.dist == ProbeDist::gaussian)
      e = gaussian(spec.seed, i);
    else if (spec.dist == ProbeDist::rademacher)
      e = rademacher(spec.seed, i);
    else
      e = (i == spec.one_hot_index) ? 1.0 : 0.0;
    v.x[i] = round_elem(e, prec);
  }
  if (spec.normalize) {
    const double n = norm2(v);
    if (!(n > 0.0)) fail(Err::numerical, "probe has zero norm");
    v = scale(v, 1.0 / n);
  }
  return v;
}

// proj/src/sharded.cpp:85-100: terms a[i]*b[i] in f64 on the 1024-block grid.
double dot(const Vec& a, const Vec& b) {
  same_shape(a, b);
  const size_t n = a.dim();
  double total = 0.0;
  for (size_t b0 = 0; b0 < n; b0 += kBlock) {
    double s = 0.0;
    const size_t e = std::min(n, b0 + kBlock);
    for (size_t i = b0; i < e; ++i) s += a.x[i] * b.x[i];
    total += s;
  }
  return total;
}

double norm2(const Vec& a) { return std::sqrt(dot(a, a)); }

// proj/src/sharded.cpp:106-118: round(y + alpha*x), product first, no FMA.
Vec axpy(double alpha, const Vec& x, const Vec& y) {
  same_shape(x, y);
  Vec o;
  o.prec = x.prec;
  o.x.resize(x.dim());
  for (size_t i = 0; i < x.dim(); ++i) {
    const double t = alpha * x.x[i];
    o.x[i] = round_elem(y.x[i] + t, o.prec);
  }
  return o;
}

// proj/src/sharded.cpp:120-130
Vec scale(const Vec& x, double c) {
  if (!std::isfinite(c)) fail(Err::argument, "scale factor is not finite");
  Vec o;
  o.prec = x.prec;
  o.x.resize(x.dim());
  for (size_t i = 0; i < x.dim(); ++i) o.x[i] = round_elem(c * x.x[i], o.prec);
  return o;
}

// ---------------------------------------------------------------- dense
static void dense_size_ok(size_t n) {
  if (n < 2) fail(Err::argument, "dense operators need n >= 2");
  if (n > kDenseCap) fail(Err::argument, "dense operator size exceeds the desk-scale cap");
}

// proj/src/operators.cpp:50-63: upper triangle (i<=j) drawn at counter i*n+j, mirrored.
Dense wigner_dense(size_t n, double sigma, uint64_t seed) {
  dense_size_ok(n);
  if (!(sigma > 0.0)) fail(Err::argument, "wigner sigma must be positive");
  Dense m;
  m.n = n;
  m.a.assign(n * n, 0.0);
  for (size_t i = 0; i < n; ++i)
    for (size_t j = i; j < n; ++j) m.a[j * n + i] = m.a[i * n + j] = sigma * gaussian(seed, i * n + j);
  return m;
}

// proj/src/operators.cpp:72-102
Dense spiked_dense(size_t n, double sigma, const std::vector<double>& spikes, uint64_t seed) {
  if (!(n > spikes.size())) fail(Err::argument, "spiked operator needs n > number of spikes");
  Dense m = wigner_dense(n, sigma, seed);
  const uint64_t dseed = mix64(seed ^ 0x5eedd1ce5ull);
  std::vector<std::vector<double>> prev;
  for (size_t s = 0; s < spikes.size(); ++s) {
    std::vector<double> u(n);
    for (size_t i = 0; i < n; ++i) u[i] = gaussian(dseed, s * n + i);
    for (const auto& w : prev) {
      double c = 0.0;
      for (size_t i = 0; i < n; ++i) c += w[i] * u[i];
      for (size_t i = 0; i < n; ++i) u[i] -= c * w[i];
    }
    double nn = 0.0;
    for (size_t i = 0; i < n; ++i) nn += u[i] * u[i];
    nn = std::sqrt(nn);
    if (!(nn > 0.0)) fail(Err::numerical, "degenerate spike direction");
    for (size_t i = 0; i < n; ++i) u[i] /= nn;
    for (size_t i = 0; i < n; ++i)
      for (size_t j = 0; j < n; ++j) m.a[i * n + j] += spikes[s] * (u[i] * u[j]);
    prev.push_back(std::move(u));
  }
  return m;
}

// proj/src/operators.cpp:30-46: per row serial f64 fold over the gathered x, then round.
Vec dense_apply(const Dense& m, const Vec& x) {
  if (x.dim() != m.n) fail(Err::layout, "operator/vector dimension mismatch");
  Vec y;
  y.prec = x.prec;
  y.x.resize(m.n);
  for (size_t i = 0; i < m.n; ++i) {
    const double* row = &m.a[i * m.n];
    double acc = 0.0;
    for (size_t j = 0; j < m.n; ++j) acc += row[j] * x.x[j];
    y.x[i] = round_elem(acc, y.prec);
  }
  return y;
}

// ---------------------------------------------------------------- Lanczos
// SPEC.md:257-265 and PAPER.md Alg. 2 (lines 3-14); full reorth = two classical
// Gram-Schmidt passes over every stored column q_0..q_k:
// c_i = dot(q_i, r) for all i against the same r, then r = axpy(-c_i, q_i, r)
// for i ascending. q_{k+1} = scale(r, 1/beta) (reciprocal multiply, as
// draw_probe normalises, proj/src/sharded.cpp:80).
LanczosResult lanczos_run(size_t dim, const ApplyFn& apply, const LanczosConfig& cfg) {
  if (dim < 2) fail(Err::argument, "operator dimension must be >= 2");
  if (cfg.k_max < 1) fail(Err::config, "k_max must be >= 1");
  const double eps = cfg.eps > 0 ? cfg.eps : (cfg.prec == Precision::f64 ? 1e-12 : 1e-7);
  const bool keep = cfg.store_basis || cfg.reorth == Reorth::full;
  // selective (this project's definition, SURVEY 8(a) row 20 -- the SPEC
  // leaves it to the builder): two classical Gram-Schmidt passes over the
  // most recent W columns, kept in a ring (column i in slot i % W) and swept
  // in slot order 0..min(k+1, W)-1; memory is W vectors instead of k+1.
  const bool sel = cfg.reorth == Reorth::selective;
  const size_t W = cfg.window;
  if (sel && W < 2) fail(Err::config, "selective reorthogonalisation needs a window >= 2");
  LanczosResult res;
  Vec q = draw_probe(dim, cfg.probe, cfg.prec), q_prev;
  std::vector<Vec> Q, ring(sel ? W : 0);
  size_t stored = 1;
  Q.push_back(q);
  if (sel) ring[0] = q;
  for (size_t k = 0; k < cfg.k_max; ++k) {
    Vec r;
    r.prec = cfg.prec;
    r.x.assign(dim, 0.0);
    apply(q, r);
    if (k > 0) r = axpy(-res.betas[k - 1], q_prev, r);
    const double alpha = dot(q, r);
    if (!std::isfinite(alpha)) {
      res.numerical_failure = true;
      res.message = "non-finite alpha";
      break;
    }
    r = axpy(-alpha, q, r);
    if (cfg.reorth == Reorth::full) {
      for (int pass = 0; pass < 2; ++pass) {
        std::vector<double> c(Q.size());
        for (size_t i = 0; i < Q.size(); ++i) c[i] = dot(Q[i], r);
        for (size_t i = 0; i < Q.size(); ++i) r = axpy(-c[i], Q[i], r);
      }
    } else if (sel) {
      for (int pass = 0; pass < 2; ++pass) {
        std::vector<double> c(stored);
        for (size_t i = 0; i < stored; ++i) c[i] = dot(ring[i], r);
        for (size_t i = 0; i < stored; ++i) r = axpy(-c[i], ring[i], r);
      }
    }
    const double beta = norm2(r);
    res.alphas.push_back(alpha);
    res.step_beta.push_back(beta);
    if (!std::isfinite(beta)) {
      res.numerical_failure = true;
      res.message = "non-finite beta";
      break;
    }
    if (beta < eps) {
      res.breakdown = true;
      break;
    }
    if (k + 1 == cfg.k_max) break;
    res.betas.push_back(beta);
    q_prev = q;
    q = scale(r, 1.0 / beta);
    if (keep) Q.push_back(q);
    if (sel) {
      ring[(k + 1) % W] = q;
      stored = std::min(stored + 1, W);
    }
  }
  if (keep) res.basis = std::move(Q);
  return res;
}

double loss_of_orthogonality(const std::vector<Vec>& basis) {
  double m = 0.0;
  for (size_t i = 0; i < basis.size(); ++i)
    for (size_t j = i + 1; j < basis.size(); ++j) m = std::max(m, std::abs(dot(basis[i], basis[j])));
  return m;
}

// ---------------------------------------------------------------- quadrature
// Independent of the product's implicit-QL solver: cyclic Jacobi on the dense
// k x k tridiagonal (k <= a few hundred), eigenvectors accumulated in full.
Ritz ritz_decompose(const std::vector<double>& alphas, const std::vector<double>& betas) {
  const size_t k = alphas.size();
  if (k == 0 || betas.size() + 1 != k) fail(Err::argument, "tridiagonal needs k alphas and k-1 betas");
  for (double a : alphas)
    if (!std::isfinite(a)) fail(Err::numerical, "non-finite tridiagonal entry");
  for (double b : betas)
    if (!std::isfinite(b)) fail(Err::numerical, "non-finite tridiagonal entry");
  std::vector<double> A(k * k, 0.0), V(k * k, 0.0);
  for (size_t i = 0; i < k; ++i) {
    A[i * k + i] = alphas[i];
    V[i * k + i] = 1.0;
    if (i + 1 < k) A[i * k + i + 1] = A[(i + 1) * k + i] = betas[i];
  }
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0;
    for (size_t p = 0; p < k; ++p)
      for (size_t q = p + 1; q < k; ++q) off += A[p * k + q] * A[p * k + q];
    if (off == 0.0) break;
    for (size_t p = 0; p < k; ++p)
      for (size_t q = p + 1; q < k; ++q) {
        const double apq = A[p * k + q];
        if (apq == 0.0) continue;
        const double app = A[p * k + p], aqq = A[q * k + q];
        const double theta = (aqq - app) / (2.0 * apq);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (std::abs(theta) + std::sqrt(theta * theta + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (size_t r = 0; r < k; ++r) {
          const double arp = A[r * k + p], arq = A[r * k + q];
          A[r * k + p] = c * arp - s * arq;
          A[r * k + q] = s * arp + c * arq;
        }
        for (size_t r = 0; r < k; ++r) {
          const double apr = A[p * k + r], aqr = A[q * k + r];
          A[p * k + r] = c * apr - s * aqr;
          A[q * k + r] = s * apr + c * aqr;
        }
        for (size_t r = 0; r < k; ++r) {
          const double vrp = V[r * k + p], vrq = V[r * k + q];
          V[r * k + p] = c * vrp - s * vrq;
          V[r * k + q] = s * vrp + c * vrq;
        }
      }
  }
  std::vector<size_t> idx(k);
  for (size_t i = 0; i < k; ++i) idx[i] = i;
  std::sort(idx.begin(), idx.end(), [&](size_t x, size_t y) { return A[x * k + x] < A[y * k + y]; });
  Ritz r;
  for (size_t i : idx) {
    r.values.push_back(A[i * k + i]);
    double n2 = 0.0;
    for (size_t j = 0; j < k; ++j) n2 += V[j * k + i] * V[j * k + i];
    r.weights.push_back(V[i] * V[i] / n2);  // first component of column i, squared
  }
  return r;
}

// sum_i w_i N(x; theta_i, sigma^2) on a uniform grid over
// [min - 5 sigma, max + 5 sigma]; sigma <= 0 selects (max - min)/100.
Density smooth_density(const Ritz& s, double sigma, size_t grid_points) {
  if (s.values.empty()) fail(Err::argument, "degenerate spectrum (k = 0)");
  if (grid_points < 2) fail(Err::argument, "grid_points must be >= 2");
  const double lo = *std::min_element(s.values.begin(), s.values.end());
  const double hi = *std::max_element(s.values.begin(), s.values.end());
  if (!(sigma > 0)) sigma = (hi - lo) / 100.0;
  if (!(sigma > 0)) sigma = 1.0;
  Density d;
  d.sigma = sigma;
  const double a = lo - 5 * sigma, b = hi + 5 * sigma;
  const double norm = 1.0 / (sigma * std::sqrt(2.0 * 3.141592653589793));
  for (size_t g = 0; g < grid_points; ++g) {
    const double x = a + (b - a) * double(g) / double(grid_points - 1);
    double acc = 0.0;
    for (size_t i = 0; i < s.values.size(); ++i) {
      const double z = (x - s.values[i]) / sigma;
      acc += s.weights[i] * norm * std::exp(-0.5 * z * z);
    }
    d.grid.push_back(x);
    d.density.push_back(acc);
  }
  return d;
}

// union of (theta, w / n_runs), renormalised to sum 1.
Ritz average_spectra(const std::vector<Ritz>& runs) {
  if (runs.empty()) fail(Err::argument, "average_spectra needs at least one run");
  Ritz out;
  const double inv = 1.0 / double(runs.size());
  double tot = 0.0;
  for (const Ritz& r : runs)
    for (size_t i = 0; i < r.values.size(); ++i) {
      out.values.push_back(r.values[i]);
      out.weights.push_back(r.weights[i] * inv);
      tot += r.weights[i] * inv;
    }
  std::vector<size_t> idx(out.values.size());
  for (size_t i = 0; i < idx.size(); ++i) idx[i] = i;
  std::stable_sort(idx.begin(), idx.end(), [&](size_t x, size_t y) { return out.values[x] < out.values[y]; });
  Ritz s;
  for (size_t i : idx) {
    s.values.push_back(out.values[i]);
    s.weights.push_back(out.weights[i] / tot);
  }
  return s;
}

}  // namespace sdo

// ORACLE — TEST INFRASTRUCTURE ONLY.
// extern "C" wrapper around the COMPILED REFERENCE (proj/src/{pool,sharded,
// operators}.cpp, built in place from /root/reference by oracle/build_ref.sh
// into oracle/_ref/libspecden_ref.so). Used (1) to pin the restatement in
// oracle/src bitwise against the reference and (2) as the "reference" CPU arm
// of bench.py: the Lanczos recurrence below composes the reference's own
// draw_probe/dot/axpy/scale/OperatorHandle::apply (SPEC.md:257-265 defines the
// recurrence; the reference has no lanczos_run of its own).
#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>

#include "specden/errors.hpp"
#include "specden/operators.hpp"
#include "specden/pool.hpp"
#include "specden/sharded.hpp"

using namespace specden;

static thread_local std::string g_err;

#define REF_TRY(...)                                                      \
  try {                                                                   \
    __VA_ARGS__;                                                          \
    return 0;                                                             \
  } catch (const config_error& e) { g_err = e.what(); return 1; }         \
  catch (const layout_error& e) { g_err = e.what(); return 2; }           \
  catch (const argument_error& e) { g_err = e.what(); return 3; }         \
  catch (const numerical_error& e) { g_err = e.what(); return 4; }        \
  catch (const state_error& e) { g_err = e.what(); return 5; }            \
  catch (const protocol_error& e) { g_err = e.what(); return 6; }         \
  catch (const std::exception& e) { g_err = e.what(); return 99; }

static Precision P(int p) { return p == 0 ? Precision::f32 : Precision::f64; }

static WorkerPool* pool_for(long long dim, long long workers) {
  const std::size_t n = std::size_t(workers < 1 ? 1 : workers);
  const std::size_t w = std::min<std::size_t>(n, std::size_t(dim));
  return new WorkerPool(w, split_evenly(std::size_t(dim), n));
}

static ShardedVector from_full(WorkerPool& pool, const double* x, long long n, int prec) {
  return scatter(pool, std::vector<double>(x, x + n), P(prec));
}

static void to_full(WorkerPool& pool, const ShardedVector& v, double* out) {
  const auto f = gather(pool, v);
  std::memcpy(out, f.data(), f.size() * sizeof(double));
}

extern "C" {

const char* refc_last_error() { return g_err.c_str(); }

int refc_draw_probe(long long dim, long long workers, unsigned long long seed, int dist, long long one_hot,
                    int normalize, int prec, double* out) {
  REF_TRY({
    std::unique_ptr<WorkerPool> pool(pool_for(dim, workers));
    ProbeSpec s;
    s.seed = seed;
    s.distribution = dist == 0 ? ProbeDist::gaussian : (dist == 1 ? ProbeDist::rademacher : ProbeDist::one_hot);
    s.one_hot_index = std::size_t(one_hot);
    s.normalize = normalize != 0;
    to_full(*pool, draw_probe(*pool, s, P(prec)), out);
  })
}

int refc_dot(long long dim, long long workers, const double* a, const double* b, int prec, double* out) {
  REF_TRY({
    std::unique_ptr<WorkerPool> pool(pool_for(dim, workers));
    *out = dot(*pool, from_full(*pool, a, dim, prec), from_full(*pool, b, dim, prec));
  })
}

int refc_axpy(long long dim, long long workers, double alpha, const double* x, const double* y, int prec, double* out) {
  REF_TRY({
    std::unique_ptr<WorkerPool> pool(pool_for(dim, workers));
    to_full(*pool, axpy(*pool, alpha, from_full(*pool, x, dim, prec), from_full(*pool, y, dim, prec)), out);
  })
}

int refc_scale(long long dim, long long workers, const double* x, double c, int prec, double* out) {
  REF_TRY({
    std::unique_ptr<WorkerPool> pool(pool_for(dim, workers));
    to_full(*pool, scale(*pool, from_full(*pool, x, dim, prec), c), out);
  })
}

int refc_wigner(long long n, double sigma, unsigned long long seed, double* out) {
  REF_TRY({
    const DenseSymmetric m = wigner_dense(std::size_t(n), sigma, seed);
    std::memcpy(out, m.a.data(), m.a.size() * sizeof(double));
  })
}

int refc_spiked(long long n, double sigma, const double* spikes, long long ns, unsigned long long seed, double* out) {
  REF_TRY({
    const DenseSymmetric m = spiked_dense(std::size_t(n), sigma, std::vector<double>(spikes, spikes + ns), seed);
    std::memcpy(out, m.a.data(), m.a.size() * sizeof(double));
  })
}

int refc_dense_apply(long long n, const double* a, long long workers, const double* x, int prec, double* out) {
  REF_TRY({
    auto m = std::make_shared<DenseSymmetric>();
    m->n = std::size_t(n);
    m->a.assign(a, a + n * n);
    const OperatorHandle op = dense_operator(m, "dense");
    std::unique_ptr<WorkerPool> pool(pool_for(n, workers));
    to_full(*pool, op.apply(*pool, from_full(*pool, x, n, prec)), out);
  })
}

// Lanczos (full reorth = two classical Gram-Schmidt passes
// against every stored column) composed from the reference's own primitives.
int refc_lanczos_dense(long long n, const double* a, long long workers, long long k_max, double eps, int reorth,
                       unsigned long long seed, int dist, int prec, double* out_alpha, double* out_beta,
                       long long* info) {
  REF_TRY({
    auto m = std::make_shared<DenseSymmetric>();
    m->n = std::size_t(n);
    m->a.assign(a, a + n * n);
    const OperatorHandle op = dense_operator(m, "dense");
    std::unique_ptr<WorkerPool> pool(pool_for(n, workers));
    ProbeSpec s;
    s.seed = seed;
    s.distribution = dist == 0 ? ProbeDist::gaussian : ProbeDist::rademacher;
    const Precision pr = P(prec);
    if (!(eps > 0)) eps = pr == Precision::f64 ? 1e-12 : 1e-7;
    ShardedVector q = draw_probe(*pool, s, pr), qp;
    std::vector<ShardedVector> Q{q};
    long long na = 0, nb = 0, brk = 0;
    std::vector<double> betas;
    for (long long k = 0; k < k_max; ++k) {
      ShardedVector r = op.apply(*pool, q);
      if (k > 0) r = axpy(*pool, -betas[std::size_t(k - 1)], qp, r);
      const double al = dot(*pool, q, r);
      if (!std::isfinite(al)) throw numerical_error("non-finite alpha");
      r = axpy(*pool, -al, q, r);
      if (reorth) {
        for (int pass = 0; pass < 2; ++pass) {
          std::vector<double> c(Q.size());
          for (std::size_t i = 0; i < Q.size(); ++i) c[i] = dot(*pool, Q[i], r);
          for (std::size_t i = 0; i < Q.size(); ++i) r = axpy(*pool, -c[i], Q[i], r);
        }
      }
      const double be = norm2(*pool, r);
      out_alpha[na++] = al;
      if (!std::isfinite(be)) throw numerical_error("non-finite beta");
      if (be < eps) {
        brk = 1;
        break;
      }
      if (k + 1 == k_max) break;
      betas.push_back(be);
      out_beta[nb++] = be;
      qp = q;
      q = scale(*pool, r, 1.0 / be);
      if (reorth) Q.push_back(q);
    }
    info[0] = na;
    info[1] = nb;
    info[2] = brk;
  })
}

// Times the reference primitives' share of one Lanczos step at full P
// (2 axpy + 1 dot + 1 norm2 + 1 scale, plus 2x CGS over j stored columns:
// 2j dot + 2j axpy) on `workers` host threads. Returns seconds per step.
int refc_time_recurrence(long long dim, long long workers, long long j, long long reps, int prec, double* seconds) {
  REF_TRY({
    std::unique_ptr<WorkerPool> pool(pool_for(dim, workers));
    ProbeSpec s;
    s.seed = 1;
    s.distribution = ProbeDist::rademacher;
    const Precision pr = P(prec);
    ShardedVector q = draw_probe(*pool, s, pr);
    s.seed = 2;
    ShardedVector qp = draw_probe(*pool, s, pr);
    s.seed = 3;
    ShardedVector hv = draw_probe(*pool, s, pr);
    std::vector<ShardedVector> Q;
    for (long long i = 0; i < j; ++i) {
      s.seed = 100 + std::uint64_t(i);
      Q.push_back(draw_probe(*pool, s, pr));
    }
    const auto t0 = std::chrono::steady_clock::now();
    for (long long rep = 0; rep < reps; ++rep) {
      ShardedVector r = axpy(*pool, -0.5, qp, hv);
      const double al = dot(*pool, q, r);
      r = axpy(*pool, -al, q, r);
      for (int pass = 0; pass < 2 && j > 0; ++pass) {
        std::vector<double> c(Q.size());
        for (std::size_t i = 0; i < Q.size(); ++i) c[i] = dot(*pool, Q[i], r);
        for (std::size_t i = 0; i < Q.size(); ++i) r = axpy(*pool, -c[i], Q[i], r);
      }
      const double be = norm2(*pool, r);
      ShardedVector qn = scale(*pool, r, 1.0 / (be > 0 ? be : 1.0));
      (void)qn;
    }
    const auto t1 = std::chrono::steady_clock::now();
    *seconds = std::chrono::duration<double>(t1 - t0).count() / double(reps);
  })
}

}  // extern "C"

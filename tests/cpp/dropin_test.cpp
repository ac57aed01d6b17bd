// The reference's own test idioms (proj/tests/test_sharded_core.cpp,
// test_runtime.cpp, test_operators.cpp), recompiled against the drop-in
// header include/specden/specden_b200.hpp: a reference caller switches by
// changing the include. Built and run by tests/test_dropin_gpu.py.
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include "doctest.h"

#include <cstring>

#include "specden/specden_b200.hpp"

using namespace specden;

static WorkerPool* pool_ptr(std::size_t dim, std::size_t n) {
  return new WorkerPool(std::min(n, dim), split_evenly(dim, n));
}
static ShardedVector random_vector(WorkerPool& pool, std::uint64_t seed, Precision prec = Precision::f64) {
  ProbeSpec s;
  s.seed = seed;
  s.normalize = false;
  return draw_probe(pool, s, prec);  // counter Gaussians, like test_util.hpp random_vector
}

TEST_CASE("split_evenly covers the index space with contiguous shards") {
  for (std::size_t dim : {1u, 2u, 7u, 10u, 1000u})
    for (std::size_t n : {1u, 2u, 3u, 4u, 8u, 16u}) {
      ShardLayout l = split_evenly(dim, n);
      CHECK(l.worker_count() == std::min(dim, n));
      std::size_t covered = 0;
      for (const auto& r : l.shard_bounds) covered += r.size();
      CHECK(covered == dim);
    }
  ShardLayout l;
  l.total_dim = 10;
  l.shard_bounds = {{0, 4}, {5, 10}};
  CHECK_THROWS_AS(validate_layout(l), layout_error);
}

TEST_CASE("probe layout invariance holds for many dims, layouts, precisions") {
  for (std::size_t dim : {5u, 129u, 1025u, 5000u})
    for (Precision prec : {Precision::f64, Precision::f32}) {
      ProbeSpec spec;
      spec.seed = 99;
      spec.distribution = ProbeDist::rademacher;
      std::unique_ptr<WorkerPool> ref(pool_ptr(dim, 1));
      auto expect = gather(*ref, draw_probe(*ref, spec, prec));
      for (std::size_t n : {2u, 3u, 7u}) {
        std::unique_ptr<WorkerPool> pool(pool_ptr(dim, n));
        CHECK(gather(*pool, draw_probe(*pool, spec, prec)) == expect);
      }
    }
}

TEST_CASE("dot is bitwise identical across shard counts; symmetric") {
  for (std::size_t dim : {1000u, 5000u, 70001u})
    for (Precision prec : {Precision::f64, Precision::f32}) {
      std::unique_ptr<WorkerPool> ref(pool_ptr(dim, 1));
      double expect = dot(*ref, random_vector(*ref, 21, prec), random_vector(*ref, 22, prec));
      for (std::size_t n : {2u, 4u, 7u}) {
        std::unique_ptr<WorkerPool> pool(pool_ptr(dim, n));
        auto a = random_vector(*pool, 21, prec), b = random_vector(*pool, 22, prec);
        double got = dot(*pool, a, b), sym = dot(*pool, b, a);
        CHECK(std::memcmp(&got, &expect, sizeof got) == 0);
        CHECK(std::memcmp(&got, &sym, sizeof got) == 0);
      }
    }
}

TEST_CASE("axpy and scale results are bitwise layout invariant; f32 storage") {
  const std::size_t dim = 2050;
  for (Precision prec : {Precision::f64, Precision::f32}) {
    std::unique_ptr<WorkerPool> ref(pool_ptr(dim, 1));
    auto x1 = random_vector(*ref, 51, prec), y1 = random_vector(*ref, 52, prec);
    auto ax = gather(*ref, axpy(*ref, 0.7, x1, y1));
    auto sc = gather(*ref, scale(*ref, x1, -1.25));
    for (std::size_t n : {3u, 8u}) {
      std::unique_ptr<WorkerPool> pool(pool_ptr(dim, n));
      auto x = random_vector(*pool, 51, prec), y = random_vector(*pool, 52, prec);
      CHECK(gather(*pool, axpy(*pool, 0.7, x, y)) == ax);
      CHECK(gather(*pool, scale(*pool, x, -1.25)) == sc);
    }
    if (prec == Precision::f32)
      for (double v : ax) CHECK(double(float(v)) == v);
  }
}

TEST_CASE("normalized probe has unit norm; errors") {
  std::unique_ptr<WorkerPool> pool(pool_ptr(300, 3));
  ProbeSpec spec;
  spec.seed = 4;
  for (Precision prec : {Precision::f64, Precision::f32}) {
    auto v = draw_probe(*pool, spec, prec);
    CHECK(std::abs(norm2(*pool, v) - 1.0) < (prec == Precision::f64 ? 4e-16 : 4e-7));
  }
  std::unique_ptr<WorkerPool> p3(pool_ptr(3, 1)), p4(pool_ptr(4, 1));
  auto a = scatter(*p3, {1, 2, 3}, Precision::f64);
  auto b = scatter(*p4, {1, 2, 3, 4}, Precision::f64);
  CHECK_THROWS_AS(dot(*p3, a, b), layout_error);
  CHECK_THROWS_AS(scale(*p3, a, INFINITY), argument_error);
  CHECK(dot(*p3, a, scatter(*p3, {4, 5, 6}, Precision::f64)) == 32.0);
  ProbeSpec oh;
  oh.distribution = ProbeDist::one_hot;
  oh.one_hot_index = 5;
  std::unique_ptr<WorkerPool> p5(pool_ptr(5, 2));
  CHECK_THROWS_AS(draw_probe(*p5, oh, Precision::f64), argument_error);
}

TEST_CASE("dense apply is bitwise layout invariant in both precisions") {
  const std::size_t n = 512;
  auto op = wigner_operator(n, 1.0, 15);
  for (Precision prec : {Precision::f64, Precision::f32}) {
    std::unique_ptr<WorkerPool> ref(pool_ptr(n, 1));
    auto expect = gather(*ref, op.apply(*ref, random_vector(*ref, 16, prec)));
    for (std::size_t workers : {2u, 5u, 8u}) {
      std::unique_ptr<WorkerPool> pool(pool_ptr(n, workers));
      CHECK(gather(*pool, op.apply(*pool, random_vector(*pool, 16, prec))) == expect);
    }
  }
  std::unique_ptr<WorkerPool> p5(pool_ptr(5, 1));
  CHECK_THROWS_AS(op.apply(*p5, random_vector(*p5, 1)), layout_error);
}

TEST_CASE("lanczos on diag(1,2,3) with full reorth recovers its eigenvalues") {
  DenseSymmetric d;
  d.n = 3;
  d.a = {1, 0, 0, 0, 2, 0, 0, 0, 3};
  auto op = dense_operator(std::make_shared<DenseSymmetric>(d), "diag");
  std::unique_ptr<WorkerPool> pool(pool_ptr(3, 1));
  LanczosConfig cfg;
  cfg.k_max = 3;
  cfg.reorthogonalize = Reorthogonalize::full;
  auto run = lanczos_run(op, cfg, *pool);
  auto s = ritz_decompose(run.t);
  CHECK(std::abs(s.values[0] - 1) < 1e-10);
  CHECK(std::abs(s.values[1] - 2) < 1e-10);
  CHECK(std::abs(s.values[2] - 3) < 1e-10);
  double w = 0;
  for (double x : s.weights) w += x;
  CHECK(std::abs(w - 1) < 1e-12);
}

// ---- autodiff surface: hvp / batched_hvp on the device engines
static sd_gpt_config tiny_decoder() {
  sd_gpt_config c{};
  c.n_layer = 1, c.d = 32, c.n_head = 2, c.ff = 64, c.vocab = 48, c.ctx = 16, c.arch = SD_ARCH_GPT2;
  c.rope_base = 10000.f, c.n_kv_head = 0;
  return c;
}
static Batch token_batch(int rows, int seq, int vocab, std::uint64_t seed) {
  Batch b;
  b.rows = rows, b.seq = seq;
  for (int i = 0; i < rows * seq; ++i) {
    b.tokens.push_back(int(sd_uniform_index(seed, 2 * i, vocab)));
    b.token_targets.push_back(int(sd_uniform_index(seed, 2 * i + 1, vocab)));
  }
  return b;
}
static Batch concat(const Batch& a, const Batch& b) {
  Batch c = a;
  c.rows += b.rows;
  c.tokens.insert(c.tokens.end(), b.tokens.begin(), b.tokens.end());
  c.token_targets.insert(c.token_targets.end(), b.token_targets.begin(), b.token_targets.end());
  c.x.insert(c.x.end(), b.x.begin(), b.x.end());
  c.y.insert(c.y.end(), b.y.begin(), b.y.end());
  return c;
}
static double host_dot(const std::vector<double>& a, const std::vector<double>& b) {
  double s = 0;
  for (std::size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
  return s;
}
static double rel_l2(const std::vector<double>& a, const std::vector<double>& b) {
  double n = 0, d = 0;
  for (std::size_t i = 0; i < a.size(); ++i) n += (a[i] - b[i]) * (a[i] - b[i]), d += b[i] * b[i];
  return std::sqrt(n / d);
}

TEST_CASE("hvp on a decoder is symmetric and linear; batched_hvp weights batches by size") {
  const ModelSpec spec = ModelSpec::decoder(tiny_decoder());
  const std::size_t P = spec.parameter_count();
  std::unique_ptr<WorkerPool> pool(pool_ptr(P, 3));
  Model m(*pool, spec, 0, 0.1, 0.1);
  const Batch b = token_batch(2, 16, 48, 7);
  auto u = random_vector(*pool, 31, Precision::f32), w = random_vector(*pool, 32, Precision::f32);
  auto hu = gather(*pool, hvp(*pool, m, b, u)), hw = gather(*pool, hvp(*pool, m, b, w));
  const double a = host_dot(hu, gather(*pool, w)), c = host_dot(gather(*pool, u), hw);
  CHECK(std::abs(a - c) <= 1e-5 * std::max(std::abs(a), std::abs(c)));
  // linearity: H(u + w) = Hu + Hw
  auto uw = hvp(*pool, m, b, axpy(*pool, 1.0, u, w));
  std::vector<double> sum(hu.size());
  for (std::size_t i = 0; i < sum.size(); ++i) sum[i] = hu[i] + hw[i];
  CHECK(rel_l2(gather(*pool, uw), sum) < 1e-5);
  // batches of 1 and 3 sequences == hvp over the concatenated 4
  const Batch b1 = token_batch(1, 16, 48, 11), b3 = token_batch(3, 16, 48, 12);
  auto split = gather(*pool, batched_hvp(*pool, m, {b1, b3}, u));
  auto whole = gather(*pool, hvp(*pool, m, concat(b1, b3), u));
  CHECK(rel_l2(split, whole) < 1e-5);
  // a single batch is identical to hvp
  CHECK(gather(*pool, batched_hvp(*pool, m, {b}, u)) == hu);
  // errors
  CHECK_THROWS_AS(hvp(*pool, m, b, random_vector(*pool, 1, Precision::f64)), config_error);
  std::unique_ptr<WorkerPool> small(pool_ptr(P - 1, 1));
  CHECK_THROWS_AS(hvp(*small, m, b, random_vector(*small, 1, Precision::f32)), layout_error);
  CHECK_THROWS_AS(batched_hvp(*pool, m, {}, u), argument_error);
  Batch bad = b;
  bad.token_targets.pop_back();
  CHECK_THROWS_AS(hvp(*pool, m, bad, u), argument_error);
}

TEST_CASE("mlp [4,8,1] with mse: batched_hvp over rows {1, 3} equals the 4-row batch") {
  const ModelSpec spec = ModelSpec::mlp({4, 8, 1});
  const std::size_t P = spec.parameter_count();
  CHECK(P == 4 * 8 + 8 + 8 * 1 + 1);
  std::unique_ptr<WorkerPool> pool(pool_ptr(P, 2));
  std::vector<double> theta(P);
  for (std::size_t i = 0; i < P; ++i) theta[i] = double(float(0.5 * sd_rademacher(3, i) * (1.0 + (i % 7) / 7.0)));
  Model m(*pool, spec, theta, 8);
  auto rows = [](int n, std::uint64_t seed) {
    Batch b;
    b.rows = n;
    for (int i = 0; i < 4 * n; ++i) b.x.push_back(float(sd_rademacher(seed, i) * 0.25 * (1 + i % 3)));
    for (int i = 0; i < n; ++i) b.y.push_back(float(0.1 * (i + 1)));
    return b;
  };
  const Batch r1 = rows(1, 5), r3 = rows(3, 6);
  auto v = random_vector(*pool, 41, Precision::f32);
  auto split = gather(*pool, batched_hvp(*pool, m, {r1, r3}, v));
  auto whole = gather(*pool, hvp(*pool, m, concat(r1, r3), v));
  CHECK(rel_l2(split, whole) < 1e-6);
  Batch too_big = rows(9, 1);
  CHECK_THROWS_AS(hvp(*pool, m, too_big, v), argument_error);
}

TEST_CASE("lanczos_run drives the model's Hessian (full and selective reorth)") {
  const ModelSpec spec = ModelSpec::decoder(tiny_decoder());
  std::unique_ptr<WorkerPool> pool(pool_ptr(spec.parameter_count(), 1));
  Model m(*pool, spec, 1, 0.1, 0.1);
  auto op = hvp_operator(*pool, m, token_batch(2, 16, 48, 9));
  LanczosConfig cfg;
  cfg.k_max = 8;
  cfg.prec = Precision::f32;
  cfg.probe.distribution = ProbeDist::rademacher;
  cfg.reorthogonalize = Reorthogonalize::full;
  auto full = lanczos_run(op, cfg, *pool);
  CHECK(full.t.k() == 8);
  for (double a : full.t.alphas) CHECK(std::isfinite(a));
  cfg.reorthogonalize = Reorthogonalize::selective;
  cfg.window = 9;  // window >= k_max + 1 keeps every column: identical to full
  auto sel = lanczos_run(op, cfg, *pool);
  CHECK(sel.t.alphas == full.t.alphas);
  CHECK(sel.t.betas == full.t.betas);
}

TEST_CASE("lanczos_run: device engine sharded over pool workers == one worker == the apply_fn-composed recurrence") {
  // operators.hpp:15-21 plug-in point: an operator given ONLY by apply_fn runs
  // the SPEC recurrence composed from the pool's vector ops; the dense
  // operator's native form runs the device engine, one rank per worker thread
  // (its own device and stream), partials exchanged in-process. Both are the
  // reference's arithmetic, so all three agree bit for bit.
  auto S = std::make_shared<DenseSymmetric>(spiked_dense(300, 1.0, {40.0, -40.0}, 3));
  auto op = dense_operator(S, "spiked");
  OperatorHandle plain;
  plain.dim = op.dim;
  plain.label = "apply_fn only";
  plain.apply_fn = op.apply_fn;
  for (Precision prec : {Precision::f64, Precision::f32}) {
    LanczosConfig cfg;
    cfg.k_max = 14;
    cfg.prec = prec;
    cfg.reorthogonalize = Reorthogonalize::full;
    cfg.probe.distribution = ProbeDist::rademacher;
    std::unique_ptr<WorkerPool> one(pool_ptr(300, 1)), five(pool_ptr(300, 5));
    const auto a = lanczos_run(op, cfg, *one);
    const auto b = lanczos_run(op, cfg, *five);
    const auto c = lanczos_run(plain, cfg, *five);
    CHECK(a.t.alphas.size() == 14);
    CHECK(a.t.alphas == b.t.alphas);
    CHECK(a.t.betas == b.t.betas);
    CHECK(a.t.alphas == c.t.alphas);
    CHECK(a.t.betas == c.t.betas);
    // tree reductions (extension): the same recurrence within rounding
    cfg.reduction = Reduction::tree;
    const auto t = lanczos_run(op, cfg, *one);
    const double tol = prec == Precision::f64 ? 1e-12 : 2e-6;
    for (std::size_t i = 0; i < t.t.alphas.size(); ++i) CHECK(std::abs(t.t.alphas[i] - a.t.alphas[i]) <= tol * 50);
  }
  // a custom apply_fn: y = 3 x -> alpha_0 = 3, benign breakdown at k = 1
  OperatorHandle three;
  three.dim = 64;
  three.label = "3I";
  three.apply_fn = [](WorkerPool& p, const ShardedVector& x, ShardedVector& y) { y = scale(p, x, 3.0); };
  std::unique_ptr<WorkerPool> p4(pool_ptr(64, 4));
  LanczosConfig c3;
  c3.k_max = 5;
  const auto r3 = lanczos_run(three, c3, *p4);
  CHECK(r3.t.alphas.size() == 1);
  CHECK(r3.t.alphas[0] == doctest::Approx(3.0).epsilon(1e-15));
  CHECK(r3.breakdown);
}

TEST_CASE("WorkerPool: one device and stream per worker, message counts, exactly-once replies") {
  std::unique_ptr<WorkerPool> pool(pool_ptr(100, 4));
  for (std::size_t w = 0; w < 4; ++w) {
    CHECK(pool->device(w) == worker_device(w));
    CHECK(pool->stream(w) != nullptr);
  }
  auto a = random_vector(*pool, 91), b = random_vector(*pool, 92);
  const auto d0 = pool->message_count(MsgKind::DotPartial), g0 = pool->message_count(MsgKind::Gather);
  (void)dot(*pool, a, b);
  (void)gather(*pool, a);
  CHECK(pool->message_count(MsgKind::DotPartial) == d0 + 4);
  CHECK(pool->message_count(MsgKind::Gather) == g0 + 4);
  std::atomic<int> hits{0};
  pool->run_all(MsgKind::ApplyShard, [&](std::size_t) { hits.fetch_add(1); });
  CHECK(hits.load() == 4);
  CHECK_THROWS_AS(pool->post(4, MsgKind::ApplyShard, [](std::size_t) {}), protocol_error);
}

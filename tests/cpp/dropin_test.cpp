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

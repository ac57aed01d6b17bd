// ORACLE — TEST INFRASTRUCTURE ONLY (see sdo.hpp header).
// Eager double-backward tape restating proj/include/specden/autodiff.hpp:26-101:
// grad() emits VJP nodes built from the same primitive set, so the gradient is
// itself differentiable (create_graph), and f32 mode rounds every node value.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <thread>

#include "sdo.hpp"

namespace sdo {

static void need_same(const Tensor& a, const Tensor& b, const char* op) {
  if (a.rows != b.rows || a.cols != b.cols) fail(Err::argument, std::string("shape mismatch in ") + op);
}

int Graph::push(Node n) {
  if (prec_ == Precision::f32)
    for (double& x : n.val.v) x = double(float(x));
  nodes_.push_back(std::move(n));
  return int(nodes_.size() - 1);
}

int Graph::constant(Tensor t) {
  Node n{Op::Const};
  n.val = std::move(t);
  return push(std::move(n));
}

int Graph::param(Tensor t) {
  Node n{Op::Param};
  n.rg = true;
  n.val = std::move(t);
  return push(std::move(n));
}

int Graph::ones(size_t r, size_t c) { return constant(Tensor(r, c, 1.0)); }

#define SDO_NODE(OPC, A, B)                         \
  Node n{Op::OPC};                                  \
  n.a = (A);                                        \
  n.b = (B);                                        \
  n.rg = !detached_ && (rg(A) || ((B) >= 0 && rg(B)));

int Graph::add(int a, int b) {
  const Tensor &x = val(a), &y = val(b);
  need_same(x, y, "add");
  SDO_NODE(Add, a, b)
  n.val = Tensor(x.rows, x.cols);
  for (size_t i = 0; i < x.numel(); ++i) n.val.v[i] = x.v[i] + y.v[i];
  return push(std::move(n));
}

int Graph::sub(int a, int b) {
  const Tensor &x = val(a), &y = val(b);
  need_same(x, y, "sub");
  SDO_NODE(Sub, a, b)
  n.val = Tensor(x.rows, x.cols);
  for (size_t i = 0; i < x.numel(); ++i) n.val.v[i] = x.v[i] - y.v[i];
  return push(std::move(n));
}

int Graph::mul(int a, int b) {
  const Tensor &x = val(a), &y = val(b);
  need_same(x, y, "mul");
  SDO_NODE(Mul, a, b)
  n.val = Tensor(x.rows, x.cols);
  for (size_t i = 0; i < x.numel(); ++i) n.val.v[i] = x.v[i] * y.v[i];
  return push(std::move(n));
}

int Graph::smul(int a, double c) {
  const Tensor& x = val(a);
  SDO_NODE(Smul, a, -1)
  n.c = c;
  n.val = Tensor(x.rows, x.cols);
  for (size_t i = 0; i < x.numel(); ++i) n.val.v[i] = c * x.v[i];
  return push(std::move(n));
}

int Graph::addrow(int a, int row) {
  const Tensor &x = val(a), &r = val(row);
  if (r.rows != 1 || r.cols != x.cols) fail(Err::argument, "shape mismatch in addrow");
  SDO_NODE(AddRow, a, row)
  n.val = Tensor(x.rows, x.cols);
  for (size_t i = 0; i < x.rows; ++i)
    for (size_t j = 0; j < x.cols; ++j) n.val.at(i, j) = x.at(i, j) + r.v[j];
  return push(std::move(n));
}

int Graph::mulcol(int a, int col) {
  const Tensor &x = val(a), &c = val(col);
  if (c.cols != 1 || c.rows != x.rows) fail(Err::argument, "shape mismatch in mulcol");
  SDO_NODE(MulCol, a, col)
  n.val = Tensor(x.rows, x.cols);
  for (size_t i = 0; i < x.rows; ++i)
    for (size_t j = 0; j < x.cols; ++j) n.val.at(i, j) = x.at(i, j) * c.v[i];
  return push(std::move(n));
}

size_t oracle_threads() {
  static const size_t n = [] {
    const char* e = std::getenv("ORACLE_THREADS");
    const long v = e ? std::atol(e) : 0;
    return v > 0 ? size_t(v) : std::max<size_t>(1, std::thread::hardware_concurrency());
  }();
  return n;
}

// C[i][j] = sum_k A'[i][k] B'[k][j], k ascending, f64. Row-parallel; the
// per-element summation order does not depend on the thread count.
static Tensor matmul_eval(const Tensor& a, const Tensor& b, bool ta, bool tb) {
  const size_t m = ta ? a.cols : a.rows, ka = ta ? a.rows : a.cols;
  const size_t kb = tb ? b.cols : b.rows, nn = tb ? b.rows : b.cols;
  if (ka != kb) fail(Err::argument, "shape mismatch in matmul");
  Tensor A(m, ka), B(kb, nn);
  if (ta) {
    for (size_t i = 0; i < a.rows; ++i)
      for (size_t j = 0; j < a.cols; ++j) A.at(j, i) = a.at(i, j);
  } else {
    A.v = a.v;
  }
  if (tb) {
    for (size_t i = 0; i < b.rows; ++i)
      for (size_t j = 0; j < b.cols; ++j) B.at(j, i) = b.at(i, j);
  } else {
    B.v = b.v;
  }
  Tensor C(m, nn);
  auto rows = [&](size_t i0, size_t i1) {
    for (size_t i = i0; i < i1; ++i) {
      double* c = &C.v[i * nn];
      const double* ar = &A.v[i * ka];
      for (size_t k = 0; k < ka; ++k) {
        const double av = ar[k];
        const double* br = &B.v[k * nn];
        for (size_t j = 0; j < nn; ++j) c[j] += av * br[j];
      }
    }
  };
  const size_t work = m * ka * nn;
  const size_t nt = work < (size_t(1) << 22) ? 1 : std::min<size_t>(oracle_threads(), m);
  if (nt <= 1) {
    rows(0, m);
  } else {
    std::vector<std::thread> th;
    for (size_t t = 0; t < nt; ++t) th.emplace_back(rows, m * t / nt, m * (t + 1) / nt);
    for (auto& t : th) t.join();
  }
  return C;
}

int Graph::matmul(int a, int b, bool ta, bool tb) {
  Tensor C = matmul_eval(val(a), val(b), ta, tb);
  SDO_NODE(Matmul, a, b)
  n.ta = ta;
  n.tb = tb;
  n.val = std::move(C);
  return push(std::move(n));
}

#define SDO_UNARY(NAME, OPC, EXPR)                                      \
  int Graph::NAME(int a) {                                              \
    const Tensor& x = val(a);                                           \
    SDO_NODE(OPC, a, -1)                                                \
    n.val = Tensor(x.rows, x.cols);                                     \
    for (size_t i = 0; i < x.numel(); ++i) {                            \
      const double t = x.v[i];                                          \
      n.val.v[i] = (EXPR);                                              \
    }                                                                   \
    return push(std::move(n));                                          \
  }
SDO_UNARY(tanh_, Tanh, std::tanh(t))
SDO_UNARY(exp_, Exp, std::exp(t))
SDO_UNARY(log_, Log, std::log(t))
SDO_UNARY(recip, Recip, 1.0 / t)

int Graph::softmax_rows(int a) {
  const Tensor& x = val(a);
  SDO_NODE(Softmax, a, -1)
  n.val = Tensor(x.rows, x.cols);
  for (size_t i = 0; i < x.rows; ++i) {
    double mx = -INFINITY;
    for (size_t j = 0; j < x.cols; ++j) mx = std::max(mx, x.at(i, j));
    double s = 0.0;
    for (size_t j = 0; j < x.cols; ++j) s += (n.val.at(i, j) = std::exp(x.at(i, j) - mx));
    for (size_t j = 0; j < x.cols; ++j) n.val.at(i, j) /= s;
  }
  return push(std::move(n));
}

int Graph::sum_rows(int a) {
  const Tensor& x = val(a);
  SDO_NODE(SumRows, a, -1)
  n.val = Tensor(1, x.cols);
  for (size_t i = 0; i < x.rows; ++i)
    for (size_t j = 0; j < x.cols; ++j) n.val.v[j] += x.at(i, j);
  return push(std::move(n));
}

int Graph::sum_cols(int a) {
  const Tensor& x = val(a);
  SDO_NODE(SumCols, a, -1)
  n.val = Tensor(x.rows, 1);
  for (size_t i = 0; i < x.rows; ++i) {
    double s = 0.0;
    for (size_t j = 0; j < x.cols; ++j) s += x.at(i, j);
    n.val.v[i] = s;
  }
  return push(std::move(n));
}

int Graph::sum_all(int a) {
  const Tensor& x = val(a);
  SDO_NODE(SumAll, a, -1)
  n.val = Tensor(1, 1);
  double s = 0.0;
  for (double t : x.v) s += t;
  n.val.v[0] = s;
  return push(std::move(n));
}

int Graph::mean_all(int a) { return smul(sum_all(a), 1.0 / double(val(a).numel())); }

int Graph::mse(int pred, int target) {
  const int d = sub(pred, target);
  return mean_all(mul(d, d));
}

// mean over rows of -<onehot_row, log softmax(logits_row)>
int Graph::cross_entropy(int logits, int onehot) {
  const int lp = log_(softmax_rows(logits));
  return smul(sum_all(mul(onehot, lp)), -1.0 / double(val(logits).rows));
}

void Graph::accumulate(std::vector<int>& adj, int node, int term) {
  if (!rg(node)) return;
  int& slot = adj[size_t(node)];
  slot = slot < 0 ? term : add(slot, term);
}

std::vector<int> Graph::grad(int loss, const std::vector<int>& wrt, bool create_graph) {
  if (val(loss).numel() != 1) fail(Err::argument, "grad needs a scalar loss");
  const bool saved = detached_;
  detached_ = !create_graph;
  std::vector<int> adj(size_t(loss) + 1, -1);
  adj[size_t(loss)] = ones(1, 1);
  for (int id = loss; id >= 0; --id) {
    const int g = adj[size_t(id)];
    if (g < 0 || !rg(id)) continue;
    const Node nd = Node{nodes_[size_t(id)].op, nodes_[size_t(id)].a, nodes_[size_t(id)].b,
                         nodes_[size_t(id)].ta, nodes_[size_t(id)].tb, nodes_[size_t(id)].c};
    const int a = nd.a, b = nd.b;
    const size_t r = val(id).rows, c = val(id).cols;
    switch (nd.op) {
      case Op::Const:
      case Op::Param:
        break;
      case Op::Add:
        accumulate(adj, a, g);
        accumulate(adj, b, g);
        break;
      case Op::Sub:
        accumulate(adj, a, g);
        if (rg(b)) accumulate(adj, b, smul(g, -1.0));
        break;
      case Op::Mul:
        if (rg(a)) accumulate(adj, a, mul(g, b));
        if (rg(b)) accumulate(adj, b, mul(g, a));
        break;
      case Op::Smul:
        accumulate(adj, a, smul(g, nd.c));
        break;
      case Op::AddRow:
        accumulate(adj, a, g);
        if (rg(b)) accumulate(adj, b, sum_rows(g));
        break;
      case Op::MulCol:
        if (rg(a)) accumulate(adj, a, mulcol(g, b));
        if (rg(b)) accumulate(adj, b, sum_cols(mul(g, a)));
        break;
      case Op::Matmul:
        // C = A'B' with A' = op(a), B' = op(b); dA' = g B'^T, dB' = A'^T g.
        if (rg(a)) accumulate(adj, a, nd.ta ? matmul(b, g, nd.tb, true) : matmul(g, b, false, !nd.tb));
        if (rg(b)) accumulate(adj, b, nd.tb ? matmul(g, a, true, nd.ta) : matmul(a, g, !nd.ta, false));
        break;
      case Op::Tanh:
        accumulate(adj, a, mul(g, sub(ones(r, c), mul(id, id))));
        break;
      case Op::Exp:
        accumulate(adj, a, mul(g, id));
        break;
      case Op::Log:
        accumulate(adj, a, mul(g, recip(a)));
        break;
      case Op::Recip:
        accumulate(adj, a, mul(g, smul(mul(id, id), -1.0)));
        break;
      case Op::Softmax: {
        const int rs = matmul(sum_cols(mul(g, id)), ones(1, c));
        accumulate(adj, a, mul(id, sub(g, rs)));
        break;
      }
      case Op::SumRows: {
        const size_t ar = val(a).rows;
        accumulate(adj, a, matmul(ones(ar, 1), g));
        break;
      }
      case Op::SumCols: {
        const size_t ac = val(a).cols;
        accumulate(adj, a, matmul(g, ones(1, ac)));
        break;
      }
      case Op::SumAll: {
        const size_t ar = val(a).rows, ac = val(a).cols;
        accumulate(adj, a, matmul(matmul(ones(ar, 1), g), ones(1, ac)));
        break;
      }
    }
  }
  std::vector<int> out;
  for (int w : wrt) {
    int g = w <= loss ? adj[size_t(w)] : -1;
    if (g < 0) g = constant(Tensor(val(w).rows, val(w).cols));
    out.push_back(g);
  }
  detached_ = saved;
  return out;
}

}  // namespace sdo

// ORACLE — TEST INFRASTRUCTURE ONLY (see sdo.hpp header).
// Models expressed purely in Graph primitives (attention is
// composed from matmul + softmax + scaling, never fused) and the Pearlmutter
// HVP of SPEC.md:193-210 / PAPER.md Alg. 1.
#include <cmath>

#include "sdo.hpp"

namespace sdo {

std::vector<ParamSlot> gpt_layout(const GptConfig& c) {
  std::vector<ParamSlot> s;
  size_t off = 0;
  auto add = [&](const std::string& name, size_t r, size_t cc, int kind) {
    s.push_back({name, off, r, cc, kind});
    off += r * cc;
  };
  if (c.arch == 1) {
    // Llama-style (this project's declaration order; [in][out] matrices, the
    // q|k|v and gate|up projections fused column-wise, untied head [V][d])
    add("tok_embeddings", c.vocab, c.d, 0);
    for (size_t l = 0; l < c.n_layer; ++l) {
      const std::string p = "layers." + std::to_string(l) + ".";
      add(p + "attention_norm.weight", 1, c.d, 1);
      const size_t kvd = (c.n_kv_head ? c.n_kv_head : c.n_head) * (c.d / c.n_head);
      add(p + "attention.wqkv", c.d, c.d + 2 * kvd, 0);
      add(p + "attention.wo", c.d, c.d, 0);
      add(p + "ffn_norm.weight", 1, c.d, 1);
      add(p + "feed_forward.w_gate_up", c.d, 2 * c.ff, 0);
      add(p + "feed_forward.w_down", c.ff, c.d, 0);
    }
    add("norm.weight", 1, c.d, 1);
    add("output", c.vocab, c.d, 0);
    return s;
  }
  add("wte", c.vocab, c.d, 0);
  add("wpe", c.ctx, c.d, 0);
  for (size_t l = 0; l < c.n_layer; ++l) {
    const std::string p = "h" + std::to_string(l) + ".";
    add(p + "ln_1.weight", 1, c.d, 1);
    add(p + "ln_1.bias", 1, c.d, 2);
    add(p + "attn.c_attn.weight", c.d, 3 * c.d, 0);
    add(p + "attn.c_attn.bias", 1, 3 * c.d, 2);
    add(p + "attn.c_proj.weight", c.d, c.d, 0);
    add(p + "attn.c_proj.bias", 1, c.d, 2);
    add(p + "ln_2.weight", 1, c.d, 1);
    add(p + "ln_2.bias", 1, c.d, 2);
    add(p + "mlp.c_fc.weight", c.d, c.ff, 0);
    add(p + "mlp.c_fc.bias", 1, c.ff, 2);
    add(p + "mlp.c_proj.weight", c.ff, c.d, 0);
    add(p + "mlp.c_proj.bias", 1, c.d, 2);
  }
  add("ln_f.weight", 1, c.d, 1);
  add("ln_f.bias", 1, c.d, 2);
  return s;
}

size_t gpt_param_count(const GptConfig& c) {
  const auto s = gpt_layout(c);
  return s.back().offset + s.back().rows * s.back().cols;
}

std::vector<double> gpt_init(const GptConfig& c, uint64_t seed, double gain_scale, double bias_scale, Precision p) {
  std::vector<double> th(gpt_param_count(c));
  for (const ParamSlot& s : gpt_layout(c)) {
    const double base = s.kind == 1 ? 1.0 : 0.0;
    const double sc = s.kind == 0 ? 0.02 : (s.kind == 1 ? gain_scale : bias_scale);
    for (size_t e = 0; e < s.rows * s.cols; ++e) {
      const size_t i = s.offset + e;
      th[i] = round_elem(sc == 0.0 ? base : base + sc * gaussian(seed, i), p);
    }
  }
  return th;
}

// Sequence q of length S+1 is the token stream uniform_index(seed, q*(S+1)+s, V);
// inputs are its first S tokens, targets the next-token shift.
Batch synthetic_batch(const GptConfig& c, size_t B, size_t S, uint64_t seed_tok, uint64_t first_seq) {
  if (S > c.ctx) fail(Err::argument, "sequence longer than context");
  Batch b;
  b.B = B;
  b.S = S;
  for (size_t q = 0; q < B; ++q)
    for (size_t s = 0; s < S; ++s) {
      const uint64_t base = (first_seq + q) * (S + 1) + s;
      b.tokens.push_back(uint32_t(uniform_index(seed_tok, base, c.vocab)));
      b.targets.push_back(uint32_t(uniform_index(seed_tok, base + 1, c.vocab)));
    }
  return b;
}

namespace {

struct GptNodes {
  std::vector<int> params;
  int loss = -1;
};

Tensor slice(const std::vector<double>& flat, const ParamSlot& s) {
  Tensor t(s.rows, s.cols);
  for (size_t i = 0; i < t.numel(); ++i) t.v[i] = flat[s.offset + i];
  return t;
}

int layernorm(Graph& g, int x, int gamma, int beta, size_t T, size_t d, double eps) {
  const int mu = g.smul(g.sum_cols(x), 1.0 / double(d));
  const int xc = g.sub(x, g.matmul(mu, g.ones(1, d)));
  const int var = g.smul(g.sum_cols(g.mul(xc, xc)), 1.0 / double(d));
  const int r = g.exp_(g.smul(g.log_(g.add(var, g.constant(Tensor(T, 1, eps)))), -0.5));
  const int xh = g.mulcol(xc, r);
  return g.addrow(g.mul(xh, g.matmul(g.ones(T, 1), gamma)), beta);
}

// RMSNorm: h = gamma * x * (mean(x^2) + eps)^-1/2 (exp(-1/2 log) as in layernorm)
int rmsnorm(Graph& g, int x, int gamma, size_t T, size_t d, double eps) {
  const int ms = g.smul(g.sum_cols(g.mul(x, x)), 1.0 / double(d));
  const int r = g.exp_(g.smul(g.log_(g.add(ms, g.constant(Tensor(T, 1, eps)))), -0.5));
  return g.mul(g.mulcol(x, r), g.matmul(g.ones(T, 1), gamma));
}

// SiLU: x * 1 / (1 + exp(-x))
int silu(Graph& g, int x) {
  const Tensor& xv = g.val(x);
  return g.mul(x, g.recip(g.add(g.ones(xv.rows, xv.cols), g.exp_(g.smul(x, -1.0)))));
}

int gelu_tanh(Graph& g, int x) {
  const Tensor& xv = g.val(x);
  const double k = std::sqrt(2.0 / 3.141592653589793);
  const int x3 = g.mul(g.mul(x, x), x);
  const int inner = g.smul(g.add(x, g.smul(x3, 0.044715)), k);
  const int t = g.tanh_(inner);
  return g.mul(g.smul(x, 0.5), g.add(g.ones(xv.rows, xv.cols), t));
}

GptNodes build_llama(Graph& g, const GptConfig& c, const std::vector<double>& theta, const Batch& bt);

GptNodes build_gpt(Graph& g, const GptConfig& c, const std::vector<double>& theta, const Batch& bt) {
  if (c.arch == 1) return build_llama(g, c, theta, bt);
  const auto slots = gpt_layout(c);
  GptNodes out;
  for (const auto& s : slots) out.params.push_back(g.param(slice(theta, s)));
  const size_t B = bt.B, S = bt.S, T = B * S, d = c.d, H = c.n_head, dh = d / H;
  if (d % H) fail(Err::argument, "d must be divisible by n_head");
  Tensor tok(T, c.vocab), pos(T, c.ctx), tgt(T, c.vocab);
  for (size_t t = 0; t < T; ++t) {
    tok.at(t, bt.tokens[t]) = 1.0;
    pos.at(t, t % S) = 1.0;
    tgt.at(t, bt.targets[t]) = 1.0;
  }
  size_t pi = 0;
  const int wte = out.params[pi++], wpe = out.params[pi++];
  int x = g.add(g.matmul(g.constant(tok), wte), g.matmul(g.constant(pos), wpe));
  Tensor mask(S, S);
  for (size_t i = 0; i < S; ++i)
    for (size_t j = i + 1; j < S; ++j) mask.at(i, j) = -1e30;
  const int maskn = g.constant(mask);
  std::vector<int> rsel(B);
  for (size_t b = 0; b < B; ++b) {
    Tensor r(S, T);
    for (size_t s = 0; s < S; ++s) r.at(s, b * S + s) = 1.0;
    rsel[b] = g.constant(r);
  }
  std::vector<int> qsel(H), ksel(H), vsel(H), place(H);
  for (size_t h = 0; h < H; ++h) {
    Tensor q(3 * d, dh), k(3 * d, dh), v(3 * d, dh), p(dh, d);
    for (size_t e = 0; e < dh; ++e) {
      q.at(h * dh + e, e) = 1.0;
      k.at(d + h * dh + e, e) = 1.0;
      v.at(2 * d + h * dh + e, e) = 1.0;
      p.at(e, h * dh + e) = 1.0;
    }
    qsel[h] = g.constant(q);
    ksel[h] = g.constant(k);
    vsel[h] = g.constant(v);
    place[h] = g.constant(p);
  }
  const double sc = 1.0 / std::sqrt(double(dh));
  for (size_t l = 0; l < c.n_layer; ++l) {
    const int g1 = out.params[pi++], b1 = out.params[pi++], wa = out.params[pi++], ba = out.params[pi++];
    const int wp = out.params[pi++], bp = out.params[pi++], g2 = out.params[pi++], b2 = out.params[pi++];
    const int wf = out.params[pi++], bf = out.params[pi++], wq = out.params[pi++], bq = out.params[pi++];
    const int h1 = layernorm(g, x, g1, b1, T, d, c.ln_eps);
    const int qkv = g.addrow(g.matmul(h1, wa), ba);
    int att = -1;
    for (size_t b = 0; b < B; ++b) {
      const int xb = g.matmul(rsel[b], qkv);
      int ob = -1;
      for (size_t h = 0; h < H; ++h) {
        const int q = g.matmul(xb, qsel[h]), k = g.matmul(xb, ksel[h]), v = g.matmul(xb, vsel[h]);
        const int s = g.add(g.smul(g.matmul(q, k, false, true), sc), maskn);
        const int o = g.matmul(g.softmax_rows(s), v);
        const int oh = g.matmul(o, place[h]);
        ob = ob < 0 ? oh : g.add(ob, oh);
      }
      const int back = g.matmul(rsel[b], ob, true, false);
      att = att < 0 ? back : g.add(att, back);
    }
    x = g.add(x, g.addrow(g.matmul(att, wp), bp));
    const int h2 = layernorm(g, x, g2, b2, T, d, c.ln_eps);
    const int f = gelu_tanh(g, g.addrow(g.matmul(h2, wf), bf));
    x = g.add(x, g.addrow(g.matmul(f, wq), bq));
  }
  const int gf = out.params[pi++], bfn = out.params[pi++];
  const int hf = layernorm(g, x, gf, bfn, T, d, c.ln_eps);
  const int logits = g.matmul(hf, wte, false, true);
  out.loss = g.cross_entropy(logits, g.constant(tgt));
  return out;
}

// Llama-style decoder in the same primitives: RMSNorm (pre-norm), RoPE on q/k
// (rotate-half convention: t*cos + (t R)*sin with the constant R), causal
// softmax attention, SwiGLU MLP (silu(gate) * up), untied output head.
GptNodes build_llama(Graph& g, const GptConfig& c, const std::vector<double>& theta, const Batch& bt) {
  const auto slots = gpt_layout(c);
  GptNodes out;
  for (const auto& s : slots) out.params.push_back(g.param(slice(theta, s)));
  const size_t B = bt.B, S = bt.S, T = B * S, d = c.d, H = c.n_head, dh = d / H, ff = c.ff;
  if (d % H || dh % 2) fail(Err::argument, "d must be divisible by n_head (even head dim)");
  Tensor tok(T, c.vocab), tgt(T, c.vocab);
  for (size_t t = 0; t < T; ++t) {
    tok.at(t, bt.tokens[t]) = 1.0;
    tgt.at(t, bt.targets[t]) = 1.0;
  }
  size_t pi = 0;
  const int emb = out.params[pi++];
  int x = g.matmul(g.constant(tok), emb);
  Tensor mask(S, S), cosT(S, dh), sinT(S, dh), rot(dh, dh);
  for (size_t i = 0; i < S; ++i)
    for (size_t j = i + 1; j < S; ++j) mask.at(i, j) = -1e30;
  const size_t half = dh / 2;
  for (size_t p = 0; p < S; ++p)
    for (size_t i = 0; i < half; ++i) {
      const double theta_i = std::pow(c.rope_base, -2.0 * double(i) / double(dh));
      const double ang = double(p) * theta_i;
      cosT.at(p, i) = cosT.at(p, i + half) = std::cos(ang);
      sinT.at(p, i) = sinT.at(p, i + half) = std::sin(ang);
    }
  for (size_t i = 0; i < half; ++i) {
    rot.at(i + half, i) = -1.0;  // (t R)[i] = -t[i + half]
    rot.at(i, i + half) = 1.0;   // (t R)[i + half] = t[i]
  }
  const int maskn = g.constant(mask), cosn = g.constant(cosT), sinn = g.constant(sinT), rotn = g.constant(rot);
  auto rope = [&](int t) { return g.add(g.mul(t, cosn), g.mul(g.matmul(t, rotn), sinn)); };
  std::vector<int> rsel(B);
  for (size_t b = 0; b < B; ++b) {
    Tensor r(S, T);
    for (size_t s2 = 0; s2 < S; ++s2) r.at(s2, b * S + s2) = 1.0;
    rsel[b] = g.constant(r);
  }
  // grouped-query attention: query head h reads key/value head h / (H / KV)
  const size_t KV = c.n_kv_head ? c.n_kv_head : H;
  if (H % KV) fail(Err::argument, "n_head must be a multiple of n_kv_head");
  const size_t kvd = KV * dh, W = d + 2 * kvd, G = H / KV;
  std::vector<int> qsel(H), ksel(H), vsel(H), place(H);
  for (size_t h = 0; h < H; ++h) {
    Tensor q(W, dh), k(W, dh), v(W, dh), p(dh, d);
    const size_t kv = h / G;
    for (size_t e = 0; e < dh; ++e) {
      q.at(h * dh + e, e) = 1.0;
      k.at(d + kv * dh + e, e) = 1.0;
      v.at(d + kvd + kv * dh + e, e) = 1.0;
      p.at(e, h * dh + e) = 1.0;
    }
    qsel[h] = g.constant(q);
    ksel[h] = g.constant(k);
    vsel[h] = g.constant(v);
    place[h] = g.constant(p);
  }
  Tensor gsel(2 * ff, ff), usel(2 * ff, ff);
  for (size_t e = 0; e < ff; ++e) {
    gsel.at(e, e) = 1.0;
    usel.at(ff + e, e) = 1.0;
  }
  const int gseln = g.constant(gsel), useln = g.constant(usel);
  const double sc = 1.0 / std::sqrt(double(dh));
  for (size_t l = 0; l < c.n_layer; ++l) {
    const int g1 = out.params[pi++], wqkv = out.params[pi++], wo = out.params[pi++];
    const int g2 = out.params[pi++], wgu = out.params[pi++], wd = out.params[pi++];
    const int h1 = rmsnorm(g, x, g1, T, d, c.ln_eps);
    const int qkv = g.matmul(h1, wqkv);
    int att = -1;
    for (size_t b = 0; b < B; ++b) {
      const int xb = g.matmul(rsel[b], qkv);
      int ob = -1;
      for (size_t h = 0; h < H; ++h) {
        const int q = rope(g.matmul(xb, qsel[h])), k = rope(g.matmul(xb, ksel[h])), v = g.matmul(xb, vsel[h]);
        const int s2 = g.add(g.smul(g.matmul(q, k, false, true), sc), maskn);
        const int o = g.matmul(g.softmax_rows(s2), v);
        const int oh = g.matmul(o, place[h]);
        ob = ob < 0 ? oh : g.add(ob, oh);
      }
      const int back = g.matmul(rsel[b], ob, true, false);
      att = att < 0 ? back : g.add(att, back);
    }
    x = g.add(x, g.matmul(att, wo));
    const int h2 = rmsnorm(g, x, g2, T, d, c.ln_eps);
    const int fu = g.matmul(h2, wgu);
    const int a = g.mul(silu(g, g.matmul(fu, gseln)), g.matmul(fu, useln));
    x = g.add(x, g.matmul(a, wd));
  }
  const int gf = out.params[pi++], head = out.params[pi++];
  const int hf = rmsnorm(g, x, gf, T, d, c.ln_eps);
  const int logits = g.matmul(hf, head, false, true);
  out.loss = g.cross_entropy(logits, g.constant(tgt));
  return out;
}

std::vector<double> flatten(const Graph& g, const std::vector<int>& ids, size_t P) {
  std::vector<double> out;
  out.reserve(P);
  for (int id : ids) {
    const Tensor& t = g.val(id);
    out.insert(out.end(), t.v.begin(), t.v.end());
  }
  return out;
}

// Pearlmutter: u = grad(<grad(L), v>) with the first gradient kept differentiable.
std::vector<double> hvp_of(Graph& g, const std::vector<int>& params, int loss, const std::vector<double>& v, size_t P) {
  if (v.size() != P) fail(Err::layout, "hvp vector dimension mismatch");
  const std::vector<int> gr = g.grad(loss, params, true);
  int d = -1;
  size_t off = 0;
  for (size_t i = 0; i < params.size(); ++i) {
    const Tensor& pv = g.val(params[i]);
    Tensor vt(pv.rows, pv.cols);
    for (size_t e = 0; e < vt.numel(); ++e) vt.v[e] = v[off + e];
    off += vt.numel();
    const int term = g.sum_all(g.mul(gr[i], g.constant(std::move(vt))));
    d = d < 0 ? term : g.add(d, term);
  }
  const std::vector<int> u = g.grad(d, params, false);
  return flatten(g, u, P);
}

}  // namespace

double gpt_loss(const GptConfig& c, const std::vector<double>& theta, const Batch& b, Precision p) {
  Graph g(p);
  const GptNodes n = build_gpt(g, c, theta, b);
  return g.val(n.loss).v[0];
}

std::vector<double> gpt_grad(const GptConfig& c, const std::vector<double>& theta, const Batch& b, Precision p) {
  Graph g(p);
  const GptNodes n = build_gpt(g, c, theta, b);
  return flatten(g, g.grad(n.loss, n.params, false), theta.size());
}

std::vector<double> gpt_hvp(const GptConfig& c, const std::vector<double>& theta, const Batch& b,
                            const std::vector<double>& v, Precision p) {
  if (b.tokens.empty()) fail(Err::argument, "empty batch");
  Graph g(p);
  const GptNodes n = build_gpt(g, c, theta, b);
  return hvp_of(g, n.params, n.loss, v, theta.size());
}

std::vector<double> gpt_batched_hvp(const GptConfig& c, const std::vector<double>& theta,
                                    const std::vector<Batch>& loader, const std::vector<double>& v, Precision p) {
  if (loader.empty()) fail(Err::argument, "batched_hvp needs at least one batch");
  std::vector<double> h(theta.size(), 0.0);
  double N = 0.0;
  for (const Batch& b : loader) {
    const std::vector<double> u = gpt_hvp(c, theta, b, v, p);
    const double bs = double(b.B);
    for (size_t i = 0; i < h.size(); ++i) h[i] += u[i] * bs;
    N += bs;
  }
  for (double& x : h) x /= N;
  return h;
}

// ---------------------------------------------------------------- MLP
size_t mlp_param_count(const std::vector<size_t>& w) {
  size_t n = 0;
  for (size_t l = 0; l + 1 < w.size(); ++l) n += w[l] * w[l + 1] + w[l + 1];
  return n;
}

namespace {
GptNodes build_mlp(Graph& g, const std::vector<size_t>& w, const std::vector<double>& th, const MlpData& d) {
  if (w.size() < 2) fail(Err::config, "mlp needs at least two widths");
  if (th.size() != mlp_param_count(w)) fail(Err::layout, "mlp parameter count mismatch");
  GptNodes out;
  Tensor xt(d.n, w.front()), yt(d.n, w.back());
  xt.v = d.x;
  yt.v = d.y;
  int h = g.constant(xt);
  size_t off = 0;
  for (size_t l = 0; l + 1 < w.size(); ++l) {
    Tensor W(w[l], w[l + 1]), bb(1, w[l + 1]);
    for (size_t i = 0; i < W.numel(); ++i) W.v[i] = th[off + i];
    off += W.numel();
    for (size_t i = 0; i < bb.numel(); ++i) bb.v[i] = th[off + i];
    off += bb.numel();
    const int wn = g.param(W), bn = g.param(bb);
    out.params.push_back(wn);
    out.params.push_back(bn);
    h = g.addrow(g.matmul(h, wn), bn);
    if (l + 2 < w.size()) h = g.tanh_(h);
  }
  out.loss = g.mse(h, g.constant(yt));
  return out;
}
}  // namespace

std::vector<double> mlp_grad(const std::vector<size_t>& w, const std::vector<double>& th, const MlpData& d,
                             Precision p) {
  Graph g(p);
  const GptNodes n = build_mlp(g, w, th, d);
  return flatten(g, g.grad(n.loss, n.params, false), th.size());
}

std::vector<double> mlp_hvp(const std::vector<size_t>& w, const std::vector<double>& th, const MlpData& d,
                            const std::vector<double>& v, Precision p) {
  Graph g(p);
  const GptNodes n = build_mlp(g, w, th, d);
  return hvp_of(g, n.params, n.loss, v, th.size());
}

}  // namespace sdo

// GPT-decoder Hessian-vector product engine (Alg. 1)
// as forward-over-reverse on B200:
//   1. forward pass carrying primal AND tangent (R-op along v) activations;
//   2. backward pass carrying adjoints AND adjoint tangents; the parameter
//      "gradients" of the tangent backward ARE Hv (first-order weight
//      gradients are never formed).
// Every matrix product runs on the tcgen05 3xTF32 GEMM (sd_gemm.cu); every
// nonlinearity (LayerNorm, GELU, causal softmax, cross-entropy) is one fused
// kernel computing value, tangent, adjoint and adjoint tangent terms
// (sd_gpt_kernels.cu). Hv is written straight into the flat parameter-order
// output vector (declaration order, row-major: SPEC.md:180), so the Lanczos
// engine consumes it without any gather.
//
// Architecture: GPT-2 block (pre-LN, fused QKV with bias, causal softmax
// attention, GELU-tanh MLP, tied wte/LM head), loss = mean next-token
// cross-entropy over the batch's B*S tokens (scaled by `loss_scale` so that a
// data-sharded sum of per-rank Hv equals the global mean, Alg. 1 line 14-17).
#include <cuda_runtime.h>

#include <cstdlib>

#include <algorithm>
#include <cmath>
#include <memory>
#include <cstring>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "sd_common.cuh"
#include "sd_engine.h"
#include "sd_gemm.h"
#include "sd_gpt.h"

namespace {

using sd::fail;

struct Slot {
  uint64_t off, rows, cols;
  int kind;  // 0 matrix, 1 LN gain, 2 bias
};

// Declaration order of oracle/src/models.cpp gpt_layout (GPT-2 parameter names).
std::vector<Slot> layout(const sd_gpt_config& c) {
  std::vector<Slot> s;
  uint64_t off = 0;
  auto add = [&](uint64_t r, uint64_t cc, int k) {
    s.push_back({off, r, cc, k});
    off += r * cc;
  };
  if (c.arch == SD_ARCH_LLAMA) {
    // oracle/src/models.cpp gpt_layout (arch 1): tok_embeddings, per layer
    // [attention_norm, wqkv [d][3d], wo, ffn_norm, w_gate_up [d][2ff], w_down],
    // norm, output [V][d]
    const uint64_t kvd = uint64_t(c.n_kv_head > 0 ? c.n_kv_head : c.n_head) * (c.d / c.n_head);
    add(c.vocab, c.d, 0);
    for (int l = 0; l < c.n_layer; ++l) {
      add(1, c.d, 1);
      add(c.d, c.d + 2 * kvd, 0);
      add(c.d, c.d, 0);
      add(1, c.d, 1);
      add(c.d, 2 * c.ff, 0);
      add(c.ff, c.d, 0);
    }
    add(1, c.d, 1);
    add(c.vocab, c.d, 0);
    return s;
  }
  add(c.vocab, c.d, 0);
  add(c.ctx, c.d, 0);
  for (int l = 0; l < c.n_layer; ++l) {
    add(1, c.d, 1);
    add(1, c.d, 2);
    add(c.d, 3 * c.d, 0);
    add(1, 3 * c.d, 2);
    add(c.d, c.d, 0);
    add(1, c.d, 2);
    add(1, c.d, 1);
    add(1, c.d, 2);
    add(c.d, c.ff, 0);
    add(1, c.ff, 2);
    add(c.ff, c.d, 0);
    add(1, c.d, 2);
  }
  add(1, c.d, 1);
  add(1, c.d, 2);
  return s;
}

uint64_t param_count(const sd_gpt_config& c) {
  const auto s = layout(c);
  return s.back().off + s.back().rows * s.back().cols;
}

void check_cfg(const sd_gpt_config& c, int B, int S) {
  if (c.n_layer < 1 || c.d < 4 || c.n_head < 1 || c.ff < 4 || c.vocab < 2 || c.ctx < 1)
    fail(SD_CONFIG_ERROR, "gpt config out of range");
  if (c.d % c.n_head) fail(SD_CONFIG_ERROR, "d must be divisible by n_head");
  if (c.d % 4 || c.ff % 4 || (c.d / c.n_head) % 4) fail(SD_CONFIG_ERROR, "d, ff and head dim must be multiples of 4");
  if (B < 1 || S < 1) fail(SD_ARGUMENT_ERROR, "empty batch");
  if (S > c.ctx) fail(SD_ARGUMENT_ERROR, "sequence longer than context");
  if (S % 4) fail(SD_CONFIG_ERROR, "sequence length must be a multiple of 4");
  if (c.arch != SD_ARCH_GPT2 && c.arch != SD_ARCH_LLAMA) fail(SD_CONFIG_ERROR, "unknown architecture");
  if (c.arch == SD_ARCH_LLAMA && !(c.rope_base > 1.0f)) fail(SD_CONFIG_ERROR, "rope_base must exceed 1");
  if (c.n_kv_head < 0 || (c.n_kv_head > 0 && (c.arch != SD_ARCH_LLAMA || c.n_head % c.n_kv_head)))
    fail(SD_CONFIG_ERROR, "n_kv_head must divide n_head (Llama-style only)");
  if (c.arch == SD_ARCH_LLAMA && (c.d / c.n_head) % 2) fail(SD_CONFIG_ERROR, "RoPE needs an even head dim");
}

struct Layer {
  float *xh1, *dxh1, *r1, *dr1, *h1, *h1s, *dh1, *dh1s;
  float *a, *as, *da, *das;
  float *P, *Ps, *dP, *dPs;
  float *o, *os, *dO, *dOs;
  float *xh2, *dxh2, *r2, *dr2, *h2, *h2s, *dh2, *dh2s;
  float *f, *df, *u, *us, *du, *dus;
  float *qkv = nullptr, *qkvs = nullptr, *dqkv = nullptr, *dqkvs = nullptr;  // GQA raw q|k|v (+tangent)
};

struct Plan {
  uint64_t bytes = 0;
  char* base = nullptr;
  template <class T>
  T* take(uint64_t n) {
    const uint64_t off = bytes;
    bytes += (n * sizeof(T) + 255) / 256 * 256;
    return base ? reinterpret_cast<T*>(base + off) : nullptr;
  }
};

}  // namespace

struct sd_gpt_s {
  sd_gpt_config c{};
  int B = 0, S = 0, T = 0, H = 0, dh = 0;
  long long Vp = 0, BHSS = 0, P = 0;
  std::vector<Slot> slots;
  const float* theta = nullptr;
  float *theta_s = nullptr, *v_s = nullptr;
  // Pipeline stage (Llama-style family; the whole model is the one-stage
  // case): layers [l0, l1), the token embedding on the first stage, the final
  // norm + head + loss on the last. The stage's parameters are the contiguous
  // slice [pbase, pbase + Pst) of the flat declaration-order layout, so theta,
  // v and Hv are stage-local. Micro-batches (nmb of B x S tokens) run through
  // `nsets` activation sets (set = micro-batch % nsets: a 1F1B schedule keeps
  // at most n_stages - stage micro-batches in flight on a stage).
  int l0 = 0, l1 = 0, nmb = 1, nsets = 1;
  bool first = true, last = true;
  long long pbase = 0, Pst = 0;
  Layer* L = nullptr;  // layers of the current set, indexed l - l0
  std::vector<std::vector<Layer>> LS;
  std::vector<float*> XS;  // per set: [x | dx] (2 T d, contiguous: one message)
  float *x, *dx;
  float *xhf, *dxhf, *rf, *drf, *hf, *hfs, *dhf, *dhfs;
  float *z, *zs, *dz, *dzs;
  float *gx, *gdx, *gxs, *gdxs, *gh, *ghs, *gdh, *gdhs;  // gx | gdx contiguous (2 T d)
  float *go, *gos, *gdo, *gdos, *ga, *gas, *gda, *gdas;
  float *gP, *gPs, *gdP, *gdPs, *gu, *gus, *gdu, *gdus;
  float *ga_mlp = nullptr, *gda_mlp = nullptr;
  // grouped-query attention: adjoints of the raw [T, d + 2 kvd] q|k|v product
  float *gqkv = nullptr, *gqkvs = nullptr, *gdqkv = nullptr, *gdqkvs = nullptr;
  int KV = 0, W = 0;  // key/value heads, raw q|k|v width
  bool gqa() const { return KV != H; }
  double* loss_rows = nullptr;  // nmb * T (last stage)
  float* red = nullptr;  // column-reduction scratch
  // per micro-batch m: tok/tgt/upos at m T, uniq/ustart at m (T + 1)
  int *tok = nullptr, *tgt = nullptr, *uniq = nullptr, *ustart = nullptr, *upos = nullptr;
  int* nuniq = nullptr;  // [nmb] distinct tokens per micro-batch (device)
  // pinned staging of the host tokens | targets (set_batch returns before the
  // upload runs; the next call waits for the previous upload's event)
  int* h_stage = nullptr;
  cudaEvent_t ev_stage = nullptr;
  void* csr_scratch = nullptr;  // device scratch of gpt_token_csr (allocated at the first set_batch)
  size_t csr_bytes = 0;
  ~sd_gpt_s() {
    if (gexec) cudaGraphExecDestroy(gexec);
    if (cap_stream) cudaStreamDestroy(cap_stream);
    if (vfix) cudaFree(vfix);
    if (csr_scratch) cudaFree(csr_scratch);
    if (ev_stage) {
      cudaEventSynchronize(ev_stage);
      cudaEventDestroy(ev_stage);
    }
    if (h_stage) cudaFreeHost(h_stage);
  }
  float loss_scale = 1.0f;
  bool have_batch = false;
  std::vector<double> h_loss;
  // current stage pass: v, Hv (stage-local), micro-batch accumulation flag
  const float* vcur = nullptr;
  float* hvcur = nullptr;
  bool acc = false;
  // SD_GPT_RECOMPUTE: a set keeps only each layer's input [x | dx] (XIN) and
  // the backward re-runs the layer into the one scratch layer (Lscratch, xr);
  // SD_GPT_NO_PROBE_RESIDUAL: no v residual array (v_s), the tangent products
  // form all residuals on chip
  bool recompute = false, probe_res = true;
  Layer Lscratch{};
  std::vector<std::vector<float*>> XIN;
  float* xr = nullptr;
  int set_of(int m) const { return m % nsets; }

  void carve(Plan& p) {
    const long long T_ = T, d = c.d, ff = c.ff, ffw = c.arch == SD_ARCH_LLAMA ? 2 * ff : ff;
    auto td = [&] { return p.take<float>(T_ * d); };
    LS.assign(nsets, std::vector<Layer>(recompute ? 0 : l1 - l0));
    XS.assign(nsets, nullptr);
    XIN.assign(nsets, std::vector<float*>(recompute ? l1 - l0 : 0, nullptr));
    auto layer_arrays = [&](Layer& l) {
        l.xh1 = td(), l.dxh1 = td(), l.h1 = td(), l.h1s = td(), l.dh1 = td(), l.dh1s = td();
        l.r1 = p.take<float>(T_), l.dr1 = p.take<float>(T_);
        l.a = p.take<float>(T_ * 3 * d), l.as = p.take<float>(T_ * 3 * d);
        l.da = p.take<float>(T_ * 3 * d), l.das = p.take<float>(T_ * 3 * d);
        // P, dP residuals are formed on chip by their (64-wide attention) consumers
        l.P = p.take<float>(BHSS), l.Ps = nullptr, l.dP = p.take<float>(BHSS), l.dPs = nullptr;
        l.o = td(), l.os = td(), l.dO = td(), l.dOs = td();
        l.xh2 = td(), l.dxh2 = td(), l.h2 = td(), l.h2s = td(), l.dh2 = td(), l.dh2s = td();
        l.r2 = p.take<float>(T_), l.dr2 = p.take<float>(T_);
        // GPT-2: MLP pre-activation [T, ff]; Llama: [gate | up] pre-activations [T, 2ff]
        l.f = p.take<float>(T_ * ffw), l.df = p.take<float>(T_ * ffw);
        l.u = p.take<float>(T_ * ff), l.us = p.take<float>(T_ * ff);
        l.du = p.take<float>(T_ * ff), l.dus = p.take<float>(T_ * ff);
        if (gqa())
          l.qkv = p.take<float>(T_ * W), l.qkvs = p.take<float>(T_ * W), l.dqkv = p.take<float>(T_ * W),
          l.dqkvs = p.take<float>(T_ * W);
    };
    for (int si = 0; si < nsets; ++si) {
      for (auto& l : LS[si]) layer_arrays(l);
      for (auto& xi : XIN[si]) xi = p.take<float>(2 * T_ * d);
      XS[si] = p.take<float>(2 * T_ * d);
    }
    if (recompute) {
      layer_arrays(Lscratch);
      xr = p.take<float>(2 * T_ * d);
    }
    if (last) {
      xhf = td(), dxhf = td(), hf = td(), hfs = td(), dhf = td(), dhfs = td();
      rf = p.take<float>(T_), drf = p.take<float>(T_);
      z = p.take<float>(T_ * Vp), zs = p.take<float>(T_ * Vp), dz = p.take<float>(T_ * Vp),
      dzs = p.take<float>(T_ * Vp);
      loss_rows = p.take<double>(T_ * nmb);
    }
    gx = p.take<float>(2 * T_ * d), gdx = gx ? gx + T_ * d : nullptr;
    gxs = td(), gdxs = td(), gh = td(), ghs = td(), gdh = td(), gdhs = td();
    go = td(), gos = td(), gdo = td(), gdos = td();
    ga = p.take<float>(T_ * 3 * d), gas = p.take<float>(T_ * 3 * d);
    gda = p.take<float>(T_ * 3 * d), gdas = p.take<float>(T_ * 3 * d);
    gP = p.take<float>(BHSS), gPs = nullptr, gdP = p.take<float>(BHSS), gdPs = nullptr;
    gu = p.take<float>(T_ * ffw), gus = p.take<float>(T_ * ffw), gdu = p.take<float>(T_ * ffw),
    gdus = p.take<float>(T_ * ffw);
    if (c.arch == SD_ARCH_LLAMA) {  // adjoint (+ tangent) of the SwiGLU output [T, ff]
      ga_mlp = p.take<float>(T_ * ff), gda_mlp = p.take<float>(T_ * ff);
    }
    if (gqa())
      gqkv = p.take<float>(T_ * W), gqkvs = p.take<float>(T_ * W), gdqkv = p.take<float>(T_ * W),
      gdqkvs = p.take<float>(T_ * W);
    theta_s = c.bf16_weights ? nullptr : p.take<float>(Pst);  // bf16 weights: exact in tf32, no residual
    v_s = probe_res ? p.take<float>(Pst) : nullptr;
    red = p.take<float>(sd::kColredReserve + 2LL * 64 * std::max(3 * d, ff));
    if (first) {
      tok = p.take<int>(T_ * nmb), uniq = p.take<int>((T_ + 1) * nmb), ustart = p.take<int>((T_ + 1) * nmb);
      upos = p.take<int>(T_ * nmb), nuniq = p.take<int>(nmb);
    }
    if (last) tgt = p.take<int>(T_ * nmb);
    use_set(0);
  }
  void use_set(int m) {
    const int si = m % nsets;
    L = recompute ? nullptr : LS[si].data();
    x = XS[si];
    dx = x ? x + (long long)T * c.d : nullptr;
  }

  // ---- GEMM helper: C = alpha op(A) op(B) + beta C (+bias), 3xTF32
  struct Op {
    const float *p, *s;
    long long ld;
    bool mn;
    long long s1 = 0, s2 = 0;
    bool exact = false;  // tf32-exact values (bf16 weights): no residual
  };
  // weight operand of parameter slot i
  Op Wt(int i, long long ld, bool mn) const { return Op{th(i), ths(i), ld, mn, 0, 0, c.bf16_weights != 0}; }
  void mm(int M, int N, int K, Op A, Op Bo, float* C, long long ldc, float alpha, float beta, cudaStream_t st,
          const float* bias = nullptr, float* Cs = nullptr, int Z1 = 1, int Z2 = 1, long long c1 = 0,
          long long c2 = 0) {
    sd::GemmArgs g;
    g.M = M, g.N = N, g.K = K;
    g.A = A.p, g.As = A.s, g.lda = A.ld, g.a_mn = A.mn;
    g.B = Bo.p, g.Bs = Bo.s, g.ldb = Bo.ld, g.b_mn = Bo.mn, g.b_exact = Bo.exact;
    g.C = C, g.ldc = ldc, g.alpha = alpha, g.beta = beta, g.bias = bias, g.Cs = Cs;
    g.Z1 = Z1, g.Z2 = Z2, g.sa1 = A.s1, g.sa2 = A.s2, g.sb1 = Bo.s1, g.sb2 = Bo.s2, g.sc1 = c1, g.sc2 = c2;
    g.causal = cmode;
    onchip_residuals(g);
    sd::gemm(g, st);
  }
  // dual source: C = alpha (op(A) op(B) + op(A2) op(B2)) + beta C (+bias), one
  // launch and one accumulation (the tangent products of Pearlmutter's R-op)
  void mm2(int M, int N, int K, Op A, Op Bo, Op A2, Op B2, float* C, long long ldc, float alpha, float beta,
           cudaStream_t st, const float* bias = nullptr, float* Cs = nullptr, int Z1 = 1, int Z2 = 1,
           long long c1 = 0, long long c2 = 0) {
    sd::GemmArgs g;
    g.M = M, g.N = N, g.K = K;
    g.A = A.p, g.As = A.s, g.lda = A.ld, g.a_mn = A.mn;
    g.B = Bo.p, g.Bs = Bo.s, g.ldb = Bo.ld, g.b_mn = Bo.mn, g.b_exact = Bo.exact;
    if (A2.mn != A.mn || B2.mn != Bo.mn) fail(SD_ARGUMENT_ERROR, "gpt: dual product majors differ");
    g.A2 = A2.p, g.A2s = A2.s, g.lda2 = A2.ld, g.B2 = B2.p, g.B2s = B2.s, g.ldb2 = B2.ld, g.b2_exact = B2.exact;
    g.sa1_2 = A2.s1, g.sa2_2 = A2.s2, g.sb1_2 = B2.s1, g.sb2_2 = B2.s2;
    g.C = C, g.ldc = ldc, g.alpha = alpha, g.beta = beta, g.bias = bias, g.Cs = Cs;
    g.Z1 = Z1, g.Z2 = Z2, g.sa1 = A.s1, g.sa2 = A.s2, g.sb1 = Bo.s1, g.sb2 = Bo.s2, g.sc1 = c1, g.sc2 = c2;
    g.causal = cmode;
    onchip_residuals(g);
    sd::gemm(g, st);
  }
  // twin products of one weight (GemmArgs::twin): C = alpha A B + beta C (+bias,
  // Cs) and its tangent C2 = alpha (A2 B + A B2) + beta C2 (+bias2, Cs2) -- the
  // primal and tangent products of the R-op forward and adjoint -- as one
  // launch over both outputs' tiles (SD_GEMM_TWIN=0: the two launches)
  void mm_tw(int M, int N, int K, Op A, Op Bo, Op A2, Op B2, float* C, float* C2, long long ldc, float alpha,
             float beta, cudaStream_t st, const float* bias, float* Cs, const float* bias2, float* Cs2, int Z1 = 1,
             int Z2 = 1, long long c1 = 0, long long c2 = 0) {
    sd::GemmArgs g;
    g.M = M, g.N = N, g.K = K;
    g.A = A.p, g.As = A.s, g.lda = A.ld, g.a_mn = A.mn;
    g.B = Bo.p, g.Bs = Bo.s, g.ldb = Bo.ld, g.b_mn = Bo.mn, g.b_exact = Bo.exact;
    if (A2.mn != A.mn || B2.mn != Bo.mn) fail(SD_ARGUMENT_ERROR, "gpt: twin product majors differ");
    g.A2 = A2.p, g.A2s = A2.s, g.lda2 = A2.ld, g.B2 = B2.p, g.B2s = B2.s, g.ldb2 = B2.ld, g.b2_exact = B2.exact;
    g.C = C, g.ldc = ldc, g.alpha = alpha, g.beta = beta, g.bias = bias, g.Cs = Cs;
    g.twin = true, g.C2 = C2, g.Cs2 = Cs2, g.alpha2 = alpha, g.beta2 = beta, g.bias2 = bias2;
    g.Z1 = Z1, g.Z2 = Z2, g.sa1 = A.s1, g.sa2 = A.s2, g.sb1 = Bo.s1, g.sb2 = Bo.s2, g.sc1 = c1, g.sc2 = c2;
    g.sa1_2 = A2.s1, g.sa2_2 = A2.s2, g.sb1_2 = B2.s1, g.sb2_2 = B2.s2;
    g.causal = cmode;
    onchip_residuals(g);
    sd::gemm(g, st);
  }
  // merged pair of 64-wide per-head products sharing A (sd_gemm.cu launch_split):
  // C = alpha A B, C2 = alpha (A B2 + A2 B) -- the [o | dO], [gv | gdv],
  // [gq | gdq], [gk | gdk] pairs of the attention R-op in one launch each
  void mm_pair(int M, int K, Op A, Op Bo, Op B2, Op A2, float* C, float* Cs, float* C2, float* Cs2, long long ldc,
               float alpha, cudaStream_t st, int Z1, int Z2, long long c1, long long c2) {
    sd::GemmArgs g;
    g.M = M, g.N = 64, g.K = K;
    g.A = A.p, g.lda = A.ld, g.a_mn = A.mn, g.sa1 = A.s1, g.sa2 = A.s2;
    g.B = Bo.p, g.ldb = Bo.ld, g.b_mn = Bo.mn, g.sb1 = Bo.s1, g.sb2 = Bo.s2;
    g.B2 = B2.p, g.ldb2 = B2.ld;
    g.A2 = A2.p, g.lda2 = A2.ld, g.sa1_2 = A2.s1, g.sa2_2 = A2.s2;
    if (A2.mn != A.mn || !Bo.mn || !B2.mn || B2.ld != Bo.ld || B2.s1 != Bo.s1 || B2.s2 != Bo.s2)
      fail(SD_ARGUMENT_ERROR, "gpt: split pair operands differ in layout");
    g.C = C, g.Cs = Cs, g.C2 = C2, g.Cs2 = Cs2, g.ldc = ldc, g.alpha = alpha, g.beta = 0.0f;
    g.Z1 = Z1, g.Z2 = Z2, g.sc1 = c1, g.sc2 = c2;
    g.causal = cmode;
    g.onchip = true;
    g.split = true;
    sd::gemm(g, st);
  }
  static bool split_pairs() {
    static const bool on = [] {  // SD_ATTN_SPLIT=0: the two products as separate launches
      const char* e = std::getenv("SD_ATTN_SPLIT");
      return !(e && e[0] == '0') && dh_ok;
    }();
    return on;
  }
  static constexpr bool dh_ok = true;
  int cmode = 0;  // causal tile/K skipping for the per-head S x S products (sd_gemm.cu)
  // Products with residual arrays use them (on-chip residuals for the MN-major-A
  // weight products measured neutral on the whole HVP: SD_GEMM_ONCHIP=1).
  static void onchip_residuals(sd::GemmArgs& g) {
    // an operand without a residual array (P, dP, gS, gdS) -> on-chip residuals
    if (!g.As || (!g.Bs && !g.b_exact) || (g.A2 && (!g.A2s || (!g.B2s && !g.b2_exact)))) {
      g.onchip = true;
      return;
    }
    static const bool onchip = [] {  // SD_GEMM_ONCHIP=1: let the GEMM choose (measured neutral)
      const char* e = std::getenv("SD_GEMM_ONCHIP");
      return e && e[0] == '1';
    }();
    if (!onchip) return;
    g.onchip = true;
  }

  const float* th(int i) const { return theta + (slots[i].off - pbase); }
  const float* ths(int i) const { return theta_s ? theta_s + (slots[i].off - pbase) : nullptr; }

  // Hv of the batch: the whole model as a one-stage pipeline -- begin, then
  // forward + backward of each micro-batch (Hv of micro-batches after the
  // first accumulates: GEMM beta = 1, accumulate flags of the column and
  // embedding reductions; Alg. 1's h += u b over the loader)
  // ---- CUDA graph of the whole-model HVP. The launch sequence of one HVP is
  // fixed once the batch shape is, so it is captured once and replayed: v is
  // first copied into the engine-owned vfix (the graph's fixed input) and the
  // graph is keyed by everything else it captured by value -- the Hv pointer,
  // loss_scale, the issuing thread (whose split-K workspace the GEMMs bound)
  // and the workspace generation. A key seen for the first time runs eagerly
  // (allocations happen there); its second occurrence is captured. Any
  // capture failure falls back to eager launches for good. SD_GPT_GRAPH=0:
  // always eager.
  struct GraphKey {
    const float* hv = nullptr;
    float loss_scale = 0.0f;
    std::thread::id tid;
    uint64_t gen = 0;
    bool operator==(const GraphKey& o) const {
      return hv == o.hv && loss_scale == o.loss_scale && tid == o.tid && gen == o.gen;
    }
  };
  float* vfix = nullptr;
  cudaStream_t cap_stream = nullptr;
  cudaGraphExec_t gexec = nullptr;
  GraphKey gkey, gpending;
  bool have_pending = false, graph_off = false;
  uint64_t glaunches = 0;
  static bool graphs_enabled() {
    static const bool on = [] {
      const char* e = std::getenv("SD_GPT_GRAPH");
      return !(e && e[0] == '0');
    }();
    return on;
  }
  void drop_graph() {
    if (gexec) cudaGraphExecDestroy(gexec);
    gexec = nullptr;
  }

  void hvp(const float* v, float* hv, cudaStream_t st) {
    if (graph_off || !graphs_enabled() || !first || !last || sd::gemm_profiling()) {
      hvp_eager(v, hv, st);
      return;
    }
    if (!vfix) SD_CUDA(cudaMalloc(&vfix, size_t(Pst) * sizeof(float)));
    SD_CUDA(cudaMemcpyAsync(vfix, v, size_t(Pst) * sizeof(float), cudaMemcpyDeviceToDevice, st));
    const GraphKey k{hv, loss_scale, std::this_thread::get_id(), sd::gemm_scratch_generation()};
    if (gexec && k == gkey) {
      SD_CUDA(cudaGraphLaunch(gexec, st));
      sd::add_launches(glaunches);
      return;
    }
    if (!(have_pending && k == gpending)) {
      hvp_eager(vfix, hv, st);  // first sighting: warm-up (workspaces grow here, outside any capture)
      gpending = k, have_pending = true;
      return;
    }
    drop_graph();
    // captured on the engine's own stream (capture only records; the legacy
    // default stream cannot capture), launched on st
    if (!cap_stream) SD_CUDA(cudaStreamCreateWithFlags(&cap_stream, cudaStreamNonBlocking));
    cudaGraph_t graph = nullptr;
    const uint64_t n0 = sd_launch_count();
    SD_CUDA(cudaStreamBeginCapture(cap_stream, cudaStreamCaptureModeThreadLocal));
    bool ok = true;
    try {
      hvp_eager(vfix, hv, cap_stream);
    } catch (...) {
      ok = false;
    }
    const cudaError_t ce = cudaStreamEndCapture(cap_stream, &graph);
    ok = ok && ce == cudaSuccess && graph && sd::gemm_scratch_generation() == k.gen;
    if (ok) ok = cudaGraphInstantiateWithFlags(&gexec, graph, 0) == cudaSuccess;
    if (graph) cudaGraphDestroy(graph);
    if (!ok) {  // not capturable here: eager from now on
      (void)cudaGetLastError();
      gexec = nullptr;
      graph_off = true;
      hvp_eager(vfix, hv, st);
      return;
    }
    glaunches = sd_launch_count() - n0;  // counted while capturing; they run now
    gkey = k, have_pending = false;
    SD_CUDA(cudaGraphLaunch(gexec, st));
  }

  void hvp_eager(const float* v, float* hv, cudaStream_t st) {
    stage_begin(v, hv, st);
    for (int m = 0; m < nmb; ++m) {
      if (c.arch == SD_ARCH_LLAMA) {
        stage_fwd(m, st);
        stage_bwd(m, st);
      } else {
        gpt2_fwd(m, st);
        gpt2_bwd(m, st);
      }
    }
  }

  // ---- GPT-2 block (pre-LN, biases, GELU, learned positions, tied head).
  // Whole-model stage only (the tied embedding is read by the first and the
  // last layer); micro-batches and SD_GPT_RECOMPUTE as for the Llama family.
  void gpt2_fwd(int m, cudaStream_t st) {
    use_set(m);
    sd::gpt_embed(tok + (long long)m * T, T, S, c.d, th(0), th(1), V_(0), V_(1), x, dx, st);
    const size_t xb = 2ull * size_t(T) * c.d * sizeof(float);
    for (int l = 0; l < c.n_layer; ++l) {
      if (recompute) {
        SD_CUDA(cudaMemcpyAsync(XIN[set_of(m)][l], x, xb, cudaMemcpyDeviceToDevice, st));
        gpt2_layer_fwd(Lscratch, l, x, dx, st);
      } else {
        gpt2_layer_fwd(L[l], l, x, dx, st);
      }
    }
  }

  void gpt2_layer_fwd(Layer& Ly, int l, float* x, float* dx, cudaStream_t st) {
    const int d = c.d, ff = c.ff;
    const float sc = 1.0f / std::sqrt(float(dh));
    const int b = 2 + 12 * l;  // slot index of h{l}.ln_1.weight
    sd::LnArgs la{x, dx, th(b), th(b + 1), V_(b), V_(b + 1), T, d, 1e-5f,
                  Ly.h1, Ly.h1s, Ly.dh1, Ly.dh1s, Ly.xh1, Ly.dxh1, Ly.r1, Ly.dr1};
    sd::gpt_ln_fwd(la, st);
    // qkv = h Wa + ba ; dqkv = dh Wa + h VWa + Vba
    mm_tw(T, 3 * d, d, {Ly.h1, Ly.h1s, d, false}, Wt(b + 2, 3 * d, true), {Ly.dh1, Ly.dh1s, d, false}, {V_(b + 2), Vs(b + 2), 3 * d, true}, Ly.a, Ly.da, 3 * d, 1, 0, st, th(b + 3), Ly.as, V_(b + 3), Ly.das);
    attention_fwd(Ly, sc, st);
    // x += o Wp + bp ; dx += do Wp + o VWp + Vbp
    mm_tw(T, d, d, {Ly.o, Ly.os, d, false}, Wt(b + 4, d, true), {Ly.dO, Ly.dOs, d, false}, {V_(b + 4), Vs(b + 4), d, true}, x, dx, d, 1, 1, st, th(b + 5), nullptr, V_(b + 5), nullptr);
    sd::LnArgs lb{x, dx, th(b + 6), th(b + 7), V_(b + 6), V_(b + 7), T, d, 1e-5f,
                  Ly.h2, Ly.h2s, Ly.dh2, Ly.dh2s, Ly.xh2, Ly.dxh2, Ly.r2, Ly.dr2};
    sd::gpt_ln_fwd(lb, st);
    mm_tw(T, ff, d, {Ly.h2, Ly.h2s, d, false}, Wt(b + 8, ff, true), {Ly.dh2, Ly.dh2s, d, false}, {V_(b + 8), Vs(b + 8), ff, true}, Ly.f, Ly.df, ff, 1, 0, st, th(b + 9), nullptr, V_(b + 9), nullptr);
    sd::gpt_gelu_fwd(Ly.f, Ly.df, Ly.u, Ly.us, Ly.du, Ly.dus, (long long)T * ff, st);
    mm_tw(T, d, ff, {Ly.u, Ly.us, ff, false}, Wt(b + 10, d, true), {Ly.du, Ly.dus, ff, false}, {V_(b + 10), Vs(b + 10), d, true}, x, dx, d, 1, 1, st, th(b + 11), nullptr, V_(b + 11), nullptr);
  }

  void gpt2_bwd(int m, cudaStream_t st) {
    const int d = c.d, V = c.vocab;
    const long long Td = (long long)T * d;
    const float hb = m > 0 ? 1.0f : 0.0f;  // beta of the Hv products
    use_set(m);
    acc = m > 0;
    const int fL = 2 + 12 * c.n_layer;
    sd::LnArgs lf{x, dx, th(fL), th(fL + 1), V_(fL), V_(fL + 1), T, d, 1e-5f, hf, hfs, dhf, dhfs, xhf, dxhf, rf, drf};
    sd::gpt_ln_fwd(lf, st);
    // logits z = hf wte^T ; dz = dhf wte^T + hf Vwte^T
    mm_tw(T, V, d, {hf, hfs, d, false}, Wt(0, d, false), {dhf, dhfs, d, false}, {V_(0), Vs(0), d, false}, z, dz, Vp, 1, 0, st, nullptr, nullptr, nullptr, nullptr);
    sd::gpt_ce(z, dz, zs, dzs, tgt + (long long)m * T, T, V, Vp, loss_scale, loss_rows + (long long)m * T, st);
    // ghf = gz wte ; gdhf = gdz wte + gz Vwte ; Hv_wte(head) (+)= gdz^T hf + gz^T dhf
    mm_tw(T, d, V, {z, zs, Vp, false}, Wt(0, d, true), {dz, dzs, Vp, false}, {V_(0), Vs(0), d, true}, gh, gdh, d, 1, 0, st, nullptr, nullptr, nullptr, nullptr);
    mm2(V, d, T, {dz, dzs, Vp, true}, {hf, hfs, d, true}, {z, zs, Vp, true}, {dhf, dhfs, d, true}, HV(0), d, 1, hb,
        st);
    SD_CUDA(cudaMemsetAsync(gx, 0, 2 * Td * sizeof(float), st));
    sd::LnBwdArgs bf{gh, gdh, th(fL), V_(fL), xhf, dxhf, rf, drf, T, d, gx, gdx, gxs, gdxs, HV(fL), HV(fL + 1), red, 0,
                     int(acc)};
    sd::gpt_ln_bwd(bf, st);
    for (int l = c.n_layer - 1; l >= 0; --l) {
      if (recompute) {  // re-run the layer from its saved input (bit-identical activations)
        SD_CUDA(cudaMemcpyAsync(xr, XIN[set_of(m)][l], 2ull * size_t(T) * c.d * sizeof(float),
                                cudaMemcpyDeviceToDevice, st));
        gpt2_layer_fwd(Lscratch, l, xr, xr + Td, st);
        gpt2_layer_bwd(Lscratch, l, hb, st);
      } else {
        gpt2_layer_bwd(L[l], l, hb, st);
      }
    }
    // embeddings (wte also carries the head contribution written above)
    if (!acc) SD_CUDA(cudaMemsetAsync(HV(1), 0, slots[1].rows * slots[1].cols * sizeof(float), st));
    sd::gpt_embed_bwd(uniq + (long long)m * (T + 1), ustart + (long long)m * (T + 1), upos + (long long)m * T,
                      nuniq + m, B, S, d, gdx, HV(0), HV(1), st, int(acc));
  }

  void gpt2_layer_bwd(Layer& Ly, int l, float hb, cudaStream_t st) {
    const int d = c.d, ff = c.ff;
    const float sc = 1.0f / std::sqrt(float(dh));
    const int b = 2 + 12 * l;
    // MLP out: gu = gx Wq^T ; gdu = gdx Wq^T + gx VWq^T ; Hv_Wq = du^T gx + u^T gdx
    mm_tw(T, ff, d, {gx, gxs, d, false}, Wt(b + 10, d, false), {gdx, gdxs, d, false}, {V_(b + 10), Vs(b + 10), d, false}, gu, gdu, ff, 1, 0, st, nullptr, nullptr, nullptr, nullptr);
    mm2(ff, d, T, {Ly.du, Ly.dus, ff, true}, {gx, gxs, d, true}, {Ly.u, Ly.us, ff, true}, {gdx, gdxs, d, true},
        HV(b + 10), d, 1, hb, st);
    sd::gpt_colsum(gdx, T, d, d, HV(b + 11), red, st, int(acc));
    sd::gpt_gelu_bwd(Ly.f, Ly.df, gu, gdu, gus, gdus, (long long)T * ff, st);
    // MLP in: gh = gf Wf^T ; gdh = gdf Wf^T + gf VWf^T ; Hv_Wf = dh2^T gf + h2^T gdf
    mm_tw(T, d, ff, {gu, gus, ff, false}, Wt(b + 8, ff, false), {gdu, gdus, ff, false}, {V_(b + 8), Vs(b + 8), ff, false}, gh, gdh, d, 1, 0, st, nullptr, nullptr, nullptr, nullptr);
    mm2(d, ff, T, {Ly.dh2, Ly.dh2s, d, true}, {gu, gus, ff, true}, {Ly.h2, Ly.h2s, d, true}, {gdu, gdus, ff, true},
        HV(b + 8), ff, 1, hb, st);
    sd::gpt_colsum(gdu, T, ff, ff, HV(b + 9), red, st, int(acc));
    sd::LnBwdArgs b2{gh, gdh, th(b + 6), V_(b + 6), Ly.xh2, Ly.dxh2, Ly.r2, Ly.dr2, T, d,
                     gx, gdx, gxs, gdxs, HV(b + 6), HV(b + 7), red, 0, int(acc)};
    sd::gpt_ln_bwd(b2, st);
    // attention out-projection
    mm_tw(T, d, d, {gx, gxs, d, false}, Wt(b + 4, d, false), {gdx, gdxs, d, false}, {V_(b + 4), Vs(b + 4), d, false}, go, gdo, d, 1, 0, st, nullptr, gos, nullptr, gdos);
    mm2(d, d, T, {Ly.dO, Ly.dOs, d, true}, {gx, gxs, d, true}, {Ly.o, Ly.os, d, true}, {gdx, gdxs, d, true},
        HV(b + 4), d, 1, hb, st);
    sd::gpt_colsum(gdx, T, d, d, HV(b + 5), red, st, int(acc));
    attention_bwd(Ly, sc, st);
    // QKV: gh = ga Wa^T ; gdh = gda Wa^T + ga VWa^T ; Hv_Wa = dh1^T ga + h1^T gda
    mm_tw(T, d, 3 * d, {ga, gas, 3 * d, false}, Wt(b + 2, 3 * d, false), {gda, gdas, 3 * d, false}, {V_(b + 2), Vs(b + 2), 3 * d, false}, gh, gdh, d, 1, 0, st, nullptr, nullptr, nullptr, nullptr);
    mm2(d, 3 * d, T, {Ly.dh1, Ly.dh1s, d, true}, {ga, gas, 3 * d, true}, {Ly.h1, Ly.h1s, d, true},
        {gda, gdas, 3 * d, true}, HV(b + 2), 3 * d, 1, hb, st);
    sd::gpt_colsum(gda, T, 3 * d, 3 * d, HV(b + 3), red, st, int(acc));
    sd::LnBwdArgs b1{gh, gdh, th(b), V_(b), Ly.xh1, Ly.dxh1, Ly.r1, Ly.dr1, T, d,
                     gx, gdx, gxs, gdxs, HV(b), HV(b + 1), red, 0, int(acc)};
    sd::gpt_ln_bwd(b1, st);
  }

  // Llama-style decoder (oracle/src/models.cpp build_llama): the same
  // forward-over-reverse scheme, stage_fwd / stage_bwd below (RMSNorm via the
  // LN kernels' rms mode, RoPE on q/k after the fused QKV product with the
  // inverse rotation on their adjoints, SwiGLU on the fused [gate | up]
  // product, untied head, no biases).

  // stage-local views of v, its tf32 residual and Hv for parameter slot i
  const float* V_(int i) const { return vcur + (slots[i].off - pbase); }
  const float* Vs(int i) const { return v_s ? v_s + (slots[i].off - pbase) : nullptr; }
  float* HV(int i) const { return hvcur + (slots[i].off - pbase); }

  void stage_begin(const float* v, float* hv, cudaStream_t st) {
    if (!have_batch) fail(SD_STATE_ERROR, "gpt: set_batch was not called");
    vcur = v, hvcur = hv;
    if (v_s) sd::gpt_residual(v, v_s, Pst, st);
  }

  // Forward (primal + tangent) of micro-batch m through layers [l0, l1). The
  // set's [x | dx] holds the stage input (the first stage embeds the tokens)
  // and, on return, the stage output.
  void stage_fwd(int m, cudaStream_t st) {
    use_set(m);
    if (first) sd::gpt_embed(tok + (long long)m * T, T, S, c.d, th(0), nullptr, V_(0), nullptr, x, dx, st);
    const size_t xb = 2ull * size_t(T) * c.d * sizeof(float);
    for (int l = l0; l < l1; ++l) {
      if (recompute) {  // keep only the layer input; the backward re-runs the layer
        SD_CUDA(cudaMemcpyAsync(XIN[set_of(m)][l - l0], x, xb, cudaMemcpyDeviceToDevice, st));
        layer_fwd(Lscratch, l, x, dx, st);
      } else {
        layer_fwd(L[l - l0], l, x, dx, st);
      }
    }
  }

  // one Llama layer, primal + tangent: [x | dx] += attention and MLP blocks;
  // the layer's activations (those the double backward reads) land in Ly
  void layer_fwd(Layer& Ly, int l, float* x, float* dx, cudaStream_t st) {
    const int d = c.d, ff = c.ff;
    const float sc = 1.0f / std::sqrt(float(dh)), eps = 1e-5f;
    {
      const int b = 1 + 6 * l;  // attention_norm
      sd::LnArgs la{x, dx, th(b), nullptr, V_(b), nullptr, T, d, eps,
                    Ly.h1, Ly.h1s, Ly.dh1, Ly.dh1s, Ly.xh1, Ly.dxh1, Ly.r1, Ly.dr1, 1};
      sd::gpt_ln_fwd(la, st);
      // q|k|v = h1 Wqkv (width W = d + 2 kvd); grouped-query attention expands
      // the KV heads to the MHA [T, 3d] layout the attention products use
      float *qa = gqa() ? Ly.qkv : Ly.a, *qas = gqa() ? Ly.qkvs : Ly.as;
      float *qd = gqa() ? Ly.dqkv : Ly.da, *qds = gqa() ? Ly.dqkvs : Ly.das;
      mm_tw(T, W, d, {Ly.h1, Ly.h1s, d, false}, Wt(b + 1, W, true), {Ly.dh1, Ly.dh1s, d, false}, {V_(b + 1), Vs(b + 1), W, true}, qa, qd, W, 1, 0, st, nullptr, qas, nullptr, qds);
      if (gqa()) sd::llama_gqa_expand(Ly.qkv, Ly.qkvs, Ly.dqkv, Ly.dqkvs, Ly.a, Ly.as, Ly.da, Ly.das, T, d, dh, KV, H, st);
      sd::llama_rope(Ly.a, Ly.as, Ly.da, Ly.das, T, S, d, dh, c.rope_base, 0, st);
      attention_fwd(Ly, sc, st);
      mm_tw(T, d, d, {Ly.o, Ly.os, d, false}, Wt(b + 2, d, true), {Ly.dO, Ly.dOs, d, false}, {V_(b + 2), Vs(b + 2), d, true}, x, dx, d, 1, 1, st, nullptr, nullptr, nullptr, nullptr);
      sd::LnArgs lb{x, dx, th(b + 3), nullptr, V_(b + 3), nullptr, T, d, eps,
                    Ly.h2, Ly.h2s, Ly.dh2, Ly.dh2s, Ly.xh2, Ly.dxh2, Ly.r2, Ly.dr2, 1};
      sd::gpt_ln_fwd(lb, st);
      mm_tw(T, 2 * ff, d, {Ly.h2, Ly.h2s, d, false}, Wt(b + 4, 2 * ff, true), {Ly.dh2, Ly.dh2s, d, false}, {V_(b + 4), Vs(b + 4), 2 * ff, true}, Ly.f, Ly.df, 2 * ff, 1, 0, st, nullptr, nullptr, nullptr, nullptr);
      sd::llama_swiglu_fwd(Ly.f, Ly.df, Ly.u, Ly.us, Ly.du, Ly.dus, T, ff, st);
      mm_tw(T, d, ff, {Ly.u, Ly.us, ff, false}, Wt(b + 5, d, true), {Ly.du, Ly.dus, ff, false}, {V_(b + 5), Vs(b + 5), d, true}, x, dx, d, 1, 1, st, nullptr, nullptr, nullptr, nullptr);
    }
  }

  // Backward (adjoint + adjoint tangent) of micro-batch m. The last stage
  // forms the adjoint from the head and the loss; other stages find the
  // adjoint of their output in [gx | gdx]. On return [gx | gdx] holds the
  // adjoint of the stage input (the first stage scatters it into the
  // embedding's Hv instead). Hv of micro-batch m > 0 accumulates.
  void stage_bwd(int m, cudaStream_t st) {
    const int d = c.d, V = c.vocab;
    const long long Td = (long long)T * d;
    const float sc = 1.0f / std::sqrt(float(dh)), eps = 1e-5f;
    const float hb = m > 0 ? 1.0f : 0.0f;  // beta of the Hv products
    const int fL = 1 + 6 * c.n_layer, head = fL + 1;  // final norm, output head
    use_set(m);
    acc = m > 0;
    if (last) {
      sd::LnArgs lf{x, dx, th(fL), nullptr, V_(fL), nullptr, T, d, eps, hf, hfs, dhf, dhfs, xhf, dxhf, rf, drf, 1};
      sd::gpt_ln_fwd(lf, st);
      // logits z = hf W_out^T ; dz = dhf W_out^T + hf VW_out^T
      mm_tw(T, V, d, {hf, hfs, d, false}, Wt(head, d, false), {dhf, dhfs, d, false}, {V_(head), Vs(head), d, false}, z, dz, Vp, 1, 0, st, nullptr, nullptr, nullptr, nullptr);
      sd::gpt_ce(z, dz, zs, dzs, tgt + (long long)m * T, T, V, Vp, loss_scale, loss_rows + (long long)m * T, st);
      mm_tw(T, d, V, {z, zs, Vp, false}, Wt(head, d, true), {dz, dzs, Vp, false}, {V_(head), Vs(head), d, true}, gh, gdh, d, 1, 0, st, nullptr, nullptr, nullptr, nullptr);
      mm2(V, d, T, {dz, dzs, Vp, true}, {hf, hfs, d, true}, {z, zs, Vp, true}, {dhf, dhfs, d, true}, HV(head), d, 1,
          hb, st);
      SD_CUDA(cudaMemsetAsync(gx, 0, 2 * Td * sizeof(float), st));
      sd::LnBwdArgs bf{gh, gdh, th(fL), V_(fL), xhf, dxhf, rf, drf, T, d, gx, gdx, gxs, gdxs, HV(fL), nullptr, red, 1,
                       int(acc)};
      sd::gpt_ln_bwd(bf, st);
    } else {  // received adjoint: its tf32 residuals (what the producing ln_bwd wrote)
      sd::gpt_residual(gx, gxs, Td, st);
      sd::gpt_residual(gdx, gdxs, Td, st);
    }
    for (int l = l1 - 1; l >= l0; --l) {
      if (recompute) {  // re-run the layer from its saved input (bit-identical activations)
        SD_CUDA(cudaMemcpyAsync(xr, XIN[set_of(m)][l - l0], 2ull * size_t(T) * c.d * sizeof(float),
                                cudaMemcpyDeviceToDevice, st));
        layer_fwd(Lscratch, l, xr, xr + (long long)T * c.d, st);
        layer_bwd(Lscratch, l, hb, st);
      } else {
        layer_bwd(L[l - l0], l, hb, st);
      }
    }
    if (first) {
      if (!acc) SD_CUDA(cudaMemsetAsync(HV(0), 0, slots[0].rows * slots[0].cols * sizeof(float), st));
      sd::gpt_embed_bwd(uniq + (long long)m * (T + 1), ustart + (long long)m * (T + 1), upos + (long long)m * T,
                        nuniq + m, B, S, d, gdx, HV(0), nullptr, st);
    }
  }

  // one Llama layer backward: [gx | gdx] hold the adjoint of the layer output
  // and, on return, of its input; Hv of the layer's parameters (beta hb)
  void layer_bwd(Layer& Ly, int l, float hb, cudaStream_t st) {
    const int d = c.d, ff = c.ff;
    const float sc = 1.0f / std::sqrt(float(dh));
    {
      const int b = 1 + 6 * l;
      // down projection: ga = gx Wd^T ; gda = gdx Wd^T + gx VWd^T ; Hv_Wd = da^T gx + a^T gdx
      mm_tw(T, ff, d, {gx, gxs, d, false}, Wt(b + 5, d, false), {gdx, gdxs, d, false}, {V_(b + 5), Vs(b + 5), d, false}, ga_mlp, gda_mlp, ff, 1, 0, st, nullptr, nullptr, nullptr, nullptr);
      mm2(ff, d, T, {Ly.du, Ly.dus, ff, true}, {gx, gxs, d, true}, {Ly.u, Ly.us, ff, true}, {gdx, gdxs, d, true},
          HV(b + 5), d, 1, hb, st);
      sd::llama_swiglu_bwd(Ly.f, Ly.df, ga_mlp, gda_mlp, gu, gus, gdu, gdus, T, ff, st);
      // gate|up: gh = gfu Wgu^T ; gdh = gdfu Wgu^T + gfu VWgu^T ; Hv_Wgu = dh2^T gfu + h2^T gdfu
      mm_tw(T, d, 2 * ff, {gu, gus, 2 * ff, false}, Wt(b + 4, 2 * ff, false), {gdu, gdus, 2 * ff, false}, {V_(b + 4), Vs(b + 4), 2 * ff, false}, gh, gdh, d, 1, 0, st, nullptr, nullptr, nullptr, nullptr);
      mm2(d, 2 * ff, T, {Ly.dh2, Ly.dh2s, d, true}, {gu, gus, 2 * ff, true}, {Ly.h2, Ly.h2s, d, true},
          {gdu, gdus, 2 * ff, true}, HV(b + 4), 2 * ff, 1, hb, st);
      sd::LnBwdArgs b2{gh, gdh, th(b + 3), V_(b + 3), Ly.xh2, Ly.dxh2, Ly.r2, Ly.dr2, T, d,
                       gx, gdx, gxs, gdxs, HV(b + 3), nullptr, red, 1, int(acc)};
      sd::gpt_ln_bwd(b2, st);
      // attention output projection
      mm_tw(T, d, d, {gx, gxs, d, false}, Wt(b + 2, d, false), {gdx, gdxs, d, false}, {V_(b + 2), Vs(b + 2), d, false}, go, gdo, d, 1, 0, st, nullptr, gos, nullptr, gdos);
      mm2(d, d, T, {Ly.dO, Ly.dOs, d, true}, {gx, gxs, d, true}, {Ly.o, Ly.os, d, true}, {gdx, gdxs, d, true},
          HV(b + 2), d, 1, hb, st);
      attention_bwd(Ly, sc, st);
      // adjoints of the pre-rotation q, k: the inverse rotation; GQA: sum the
      // expanded heads' k/v adjoints back into their KV heads
      sd::llama_rope(ga, gas, gda, gdas, T, S, d, dh, c.rope_base, 1, st);
      const float *qg = ga, *qgs = gas, *qgd = gda, *qgds = gdas;
      if (gqa()) {
        sd::llama_gqa_reduce(ga, gda, gqkv, gqkvs, gdqkv, gdqkvs, T, d, dh, KV, H, st);
        qg = gqkv, qgs = gqkvs, qgd = gdqkv, qgds = gdqkvs;
      }
      mm_tw(T, d, W, {qg, qgs, W, false}, Wt(b + 1, W, false), {qgd, qgds, W, false}, {V_(b + 1), Vs(b + 1), W, false}, gh, gdh, d, 1, 0, st, nullptr, nullptr, nullptr, nullptr);
      mm2(d, W, T, {Ly.dh1, Ly.dh1s, d, true}, {qg, qgs, W, true}, {Ly.h1, Ly.h1s, d, true}, {qgd, qgds, W, true},
          HV(b + 1), W, 1, hb, st);
      sd::LnBwdArgs b1{gh, gdh, th(b), V_(b), Ly.xh1, Ly.dxh1, Ly.r1, Ly.dr1, T, d,
                       gx, gdx, gxs, gdxs, HV(b), nullptr, red, 1, int(acc)};
      sd::gpt_ln_bwd(b1, st);
    }
  }

  // per (batch b, head h): S = sc q k^T ; dS = sc (dq k^T + q dk^T) ; P, dP = softmax R-op ;
  // o = P v ; do = dP v + P dv   (o written into the merged [T, d] layout)
  void attention_fwd(Layer& Ly, float sc, cudaStream_t st) {
    const int d = c.d, Sq = S;
    const long long ha = dh, ba = (long long)Sq * 3 * d;      // head / batch strides in a [T, 3d]
    const long long hs = (long long)Sq * Sq, bs = (long long)H * Sq * Sq;  // in P [B, H, S, S]
    const long long ho = dh, bo = (long long)Sq * d;          // in o [T, d]
    auto q = [&](float* base, float* res) { return Op{base, res, 3 * d, false, ha, ba}; };
    cmode = 1;  // scores: only j <= i tiles
    // S = sc q k^T and dS = sc (dq k^T + q dk^T): one twin launch
    mm_tw(Sq, Sq, dh, q(Ly.a, Ly.as), {Ly.a + d, Ly.as + d, 3 * d, false, ha, ba}, q(Ly.da, Ly.das),
          {Ly.da + d, Ly.das + d, 3 * d, false, ha, ba}, Ly.P, Ly.dP, Sq, sc, 0, st, nullptr, nullptr, nullptr, nullptr,
          H, B, hs, bs);
    sd::gpt_attn_softmax_fwd(Ly.P, Ly.dP, Ly.Ps, Ly.dPs, Sq, (long long)B * H * Sq, st);
    const Op Pm{Ly.P, Ly.Ps, Sq, false, hs, bs}, dPm{Ly.dP, Ly.dPs, Sq, false, hs, bs};
    const Op vv{Ly.a + 2 * d, Ly.as + 2 * d, 3 * d, true, ha, ba}, dvv{Ly.da + 2 * d, Ly.das + 2 * d, 3 * d, true, ha, ba};
    cmode = 2;  // P, dP lower-triangular: keys k <= query i
    if (dh == 64 && split_pairs()) {
      mm_pair(Sq, Sq, Pm, vv, dvv, dPm, Ly.o, Ly.os, Ly.dO, Ly.dOs, d, 1.0f, st, H, B, ho, bo);
    } else {
      mm(Sq, dh, Sq, Pm, vv, Ly.o, d, 1, 0, st, nullptr, Ly.os, H, B, ho, bo);
      mm2(Sq, dh, Sq, dPm, vv, Pm, dvv, Ly.dO, d, 1, 0, st, nullptr, Ly.dOs, H, B, ho, bo);
    }
    cmode = 0;
  }

  // gP = go v^T ; gdP = gdo v^T + go dv^T ; (gS, gdS) = softmax double-backward ;
  // gv = P^T go ; gdv = dP^T go + P^T gdo ; gq = sc gS k ; gdq = sc (gdS k + gS dk) ;
  // gk = sc gS^T q ; gdk = sc (gdS^T q + gS^T dq)      -> ga / gda [T, 3d]
  void attention_bwd(Layer& Ly, float sc, cudaStream_t st) {
    const int d = c.d, Sq = S;
    const long long ha = dh, ba = (long long)Sq * 3 * d;
    const long long hs = (long long)Sq * Sq, bs = (long long)H * Sq * Sq;
    const long long ho = dh, bo = (long long)Sq * d;
    const Op goK{go, gos, d, false, ho, bo}, gdoK{gdo, gdos, d, false, ho, bo};
    const Op vK{Ly.a + 2 * d, Ly.as + 2 * d, 3 * d, false, ha, ba}, dvK{Ly.da + 2 * d, Ly.das + 2 * d, 3 * d, false, ha, ba};
    cmode = 1;
    mm_tw(Sq, Sq, dh, goK, vK, gdoK, dvK, gP, gdP, Sq, 1, 0, st, nullptr, nullptr, nullptr, nullptr, H, B, hs, bs);
    sd::gpt_attn_softmax_bwd(Ly.P, Ly.dP, gP, gdP, gPs, gdPs, Sq, (long long)B * H * Sq, st);
    // value adjoints
    const Op PT{Ly.P, Ly.Ps, Sq, true, hs, bs}, dPT{Ly.dP, Ly.dPs, Sq, true, hs, bs};
    const Op goM{go, gos, d, true, ho, bo}, gdoM{gdo, gdos, d, true, ho, bo};
    cmode = 3;  // P^T upper-triangular: queries i >= key j
    const bool pairs = dh == 64 && split_pairs();
    if (pairs) {
      mm_pair(Sq, Sq, PT, goM, gdoM, dPT, ga + 2 * d, gas + 2 * d, gda + 2 * d, gdas + 2 * d, 3 * d, 1.0f, st, H, B, ha,
              ba);
    } else {
      mm(Sq, dh, Sq, PT, goM, ga + 2 * d, 3 * d, 1, 0, st, nullptr, gas + 2 * d, H, B, ha, ba);
      mm2(Sq, dh, Sq, dPT, goM, PT, gdoM, gda + 2 * d, 3 * d, 1, 0, st, nullptr, gdas + 2 * d, H, B, ha, ba);
    }
    // query adjoints
    const Op gS{gP, gPs, Sq, false, hs, bs}, gdS{gdP, gdPs, Sq, false, hs, bs};
    const Op kM{Ly.a + d, Ly.as + d, 3 * d, true, ha, ba}, dkM{Ly.da + d, Ly.das + d, 3 * d, true, ha, ba};
    cmode = 2;
    if (pairs) {
      mm_pair(Sq, Sq, gS, kM, dkM, gdS, ga, gas, gda, gdas, 3 * d, sc, st, H, B, ha, ba);
    } else {
      mm(Sq, dh, Sq, gS, kM, ga, 3 * d, sc, 0, st, nullptr, gas, H, B, ha, ba);
      mm2(Sq, dh, Sq, gdS, kM, gS, dkM, gda, 3 * d, sc, 0, st, nullptr, gdas, H, B, ha, ba);
    }
    // key adjoints
    const Op gST{gP, gPs, Sq, true, hs, bs}, gdST{gdP, gdPs, Sq, true, hs, bs};
    const Op qM{Ly.a, Ly.as, 3 * d, true, ha, ba}, dqM{Ly.da, Ly.das, 3 * d, true, ha, ba};
    cmode = 3;
    if (pairs) {
      mm_pair(Sq, Sq, gST, qM, dqM, gdST, ga + d, gas + d, gda + d, gdas + d, 3 * d, sc, st, H, B, ha, ba);
    } else {
      mm(Sq, dh, Sq, gST, qM, ga + d, 3 * d, sc, 0, st, nullptr, gas + d, H, B, ha, ba);
      mm2(Sq, dh, Sq, gdST, qM, gST, dqM, gda + d, 3 * d, sc, 0, st, nullptr, gdas + d, H, B, ha, ba);
    }
    cmode = 0;
  }
};

namespace {

// First parameter slot of layer l (l = n_layer: the final norm) in the Llama layout.
int llama_slot(const sd_gpt_config& c, int l) { return l == 0 ? 0 : 1 + 6 * l; }

// Stage parameter slice [begin, end) of the flat layout: the embedding goes
// with layer 0, the final norm and head with the last layer.
void stage_range(const sd_gpt_config& c, int l0, int l1, const std::vector<Slot>& s, uint64_t* b, uint64_t* e) {
  *b = s[llama_slot(c, l0)].off;
  *e = l1 == c.n_layer ? s.back().off + s.back().rows * s.back().cols : s[1 + 6 * l1].off;
}

struct StageSpec {
  int l0 = 0, l1 = -1, nmb = 1, nsets = 1, flags = 0;
};

Plan plan_for(const sd_gpt_config& c, int B, int S, char* base, sd_gpt_s* g, StageSpec sp = {}) {
  sd_gpt_s tmp;
  sd_gpt_s* e = g ? g : &tmp;
  e->c = c;
  e->B = B, e->S = S, e->T = B * S, e->H = c.n_head, e->dh = c.d / c.n_head;
  e->Vp = (c.vocab + 31) / 32 * 32;  // logits rows padded to 32: whole 5-D TMA boxes for the head products
  e->BHSS = (long long)B * c.n_head * S * S;
  e->P = (long long)param_count(c);
  e->KV = c.n_kv_head > 0 ? c.n_kv_head : c.n_head;
  e->W = c.d + 2 * e->KV * e->dh;
  e->l0 = sp.l0, e->l1 = sp.l1 < 0 ? c.n_layer : sp.l1;
  e->nmb = sp.nmb, e->nsets = sp.nsets;
  e->recompute = (sp.flags & SD_GPT_RECOMPUTE) != 0;
  e->probe_res = (sp.flags & SD_GPT_NO_PROBE_RESIDUAL) == 0;
  e->first = e->l0 == 0, e->last = e->l1 == c.n_layer;
  if (e->first && e->last) {
    e->pbase = 0, e->Pst = e->P;
  } else {
    uint64_t b0, b1;
    stage_range(c, e->l0, e->l1, layout(c), &b0, &b1);
    e->pbase = (long long)b0, e->Pst = (long long)(b1 - b0);
  }
  Plan p;
  p.base = base;
  e->carve(p);
  return p;
}

void check_stage(const sd_gpt_config& c, const StageSpec& sp) {
  const bool whole = sp.l0 == 0 && sp.l1 == c.n_layer;
  if (sp.l0 < 0 || sp.l1 > c.n_layer || sp.l0 >= sp.l1) fail(SD_LAYOUT_ERROR, "stage layer range out of bounds");
  if (sp.nmb < 1 || sp.nsets < 1 || sp.nsets > sp.nmb) fail(SD_ARGUMENT_ERROR, "need 1 <= n_sets <= n_micro");
  // the GPT-2 block ties the head to the token embedding (first and last
  // layer): it runs micro-batches and the engine flags as one whole-model stage
  if (!whole && c.arch != SD_ARCH_LLAMA)
    fail(SD_CONFIG_ERROR, "pipeline stages need the untied Llama-style layout");
  if (sp.flags & ~(SD_GPT_RECOMPUTE | SD_GPT_NO_PROBE_RESIDUAL)) fail(SD_ARGUMENT_ERROR, "unknown engine flags");
}

struct GptOpCtx {
  sd_gpt g;
  sd_comm comm;
};

// Parameter-sharded Lanczos over a data-sharded HVP: each rank
// owns [begin_r, end_r) of the Lanczos vectors; per apply the slices of x are
// all-gathered straight into the full vector, the local batch's Hv runs on it,
// and Hv's slices are reduce-scattered (rank-ordered sums) into the owners'
// shards -- the replicated recurrence and reorthogonalisation shrink by the
// rank count, and no padded slots or compaction copies sit on the data path.
struct GptShardCtx {
  sd_gpt g;
  sd_comm comm;
  int nranks = 1, rank = 0;
  std::vector<uint64_t> rb, re;
  float *full = nullptr, *hv = nullptr;
};

sd_status gpt_shard_apply(void* ctx, const void* x, void* y, sd_stream st) {
  auto* c = static_cast<GptShardCtx*>(ctx);
  return sd::guard([&] {
    const cudaStream_t s = (cudaStream_t)st;
    sd::comm_allgatherv_f32(c->comm, static_cast<const float*>(x), c->full, c->rb.data(), c->re.data(), s);
    c->g->hvp(c->full, c->hv, s);
    sd::comm_reducescatterv_f32(c->comm, c->hv, static_cast<float*>(y), c->rb.data(), c->re.data(), s);
  });
}

// Pipeline-parallel apply (sd_operator_gpt_pipeline): stage = comm rank; x, y
// are this stage's parameter slice of the Lanczos vectors. The 1F1B schedule
// (sd_pipeline_schedule) drives the engine's per-micro-batch forward and
// backward; [x | dx] of a set and [gx | gdx] are the boundary messages.
struct GptPipeCtx {
  sd_gpt g;
  sd_comm comm;
  int nst = 1, st = 0;
  std::vector<int> ops;
};

sd_status gpt_pipe_apply(void* ctx, const void* x, void* y, sd_stream sp) {
  auto* c = static_cast<GptPipeCtx*>(ctx);
  return sd::guard([&] {
    const cudaStream_t s = (cudaStream_t)sp;
    sd_gpt g = c->g;
    const uint64_t n2 = 2ull * uint64_t(g->T) * uint64_t(g->c.d);
    g->stage_begin(static_cast<const float*>(x), static_cast<float*>(y), s);
    for (size_t i = 0; i < c->ops.size(); i += 2) {
      const int m = c->ops[i + 1];
      switch (c->ops[i]) {
        case SD_PIPE_F: g->stage_fwd(m, s); break;
        case SD_PIPE_B: g->stage_bwd(m, s); break;
        case SD_PIPE_SEND_F: g->use_set(m), sd::comm_send_f32(c->comm, g->x, n2, c->st + 1, s); break;
        case SD_PIPE_RECV_F: g->use_set(m), sd::comm_recv_f32(c->comm, g->x, n2, c->st - 1, s); break;
        case SD_PIPE_SEND_B: sd::comm_send_f32(c->comm, g->gx, n2, c->st - 1, s); break;
        case SD_PIPE_RECV_B: sd::comm_recv_f32(c->comm, g->gx, n2, c->st + 1, s); break;
        case SD_PIPE_GROUP_BEGIN: sd::comm_group_begin(c->comm); break;
        case SD_PIPE_GROUP_END: sd::comm_group_end(c->comm, s); break;
        default: fail(SD_PROTOCOL_ERROR, "pipeline: unknown schedule op");
      }
    }
  });
}

sd_status gpt_apply(void* ctx, const void* x, void* y, sd_stream s) {
  auto* c = static_cast<GptOpCtx*>(ctx);
  return sd::guard([&] {
    c->g->hvp(static_cast<const float*>(x), static_cast<float*>(y), (cudaStream_t)s);
    sd::comm_allreduce_f32(c->comm, static_cast<float*>(y), uint64_t(c->g->P), (cudaStream_t)s);
  });
}

}  // namespace

extern "C" {

uint64_t sd_gpt_param_count(const sd_gpt_config* c) { return c ? param_count(*c) : 0; }

sd_status sd_gpt_param_layout(const sd_gpt_config* c, uint64_t* offsets, uint64_t* rows, uint64_t* cols, int* kinds,
                              uint64_t* count) {
  return sd::guard([&] {
    const auto s = layout(*c);
    for (size_t i = 0; i < s.size(); ++i) {
      offsets[i] = s[i].off;
      rows[i] = s[i].rows;
      cols[i] = s[i].cols;
      kinds[i] = s[i].kind;
    }
    *count = s.size();
  });
}

// theta[i] = base(kind) + scale(kind) * gaussian(seed, i): matrices 0.02,
// LN gains 1 + gain_scale*N, biases bias_scale*N (oracle gpt_init).
sd_status sd_gpt_init_params(const sd_gpt_config* c, uint64_t seed, double gain_scale, double bias_scale,
                             float* theta, sd_stream s) {
  return sd::guard([&] {
    for (const Slot& sl : layout(*c)) {
      const double base = sl.kind == 1 ? 1.0 : 0.0;
      const double sc = sl.kind == 0 ? 0.02 : (sl.kind == 1 ? gain_scale : bias_scale);
      sd::gpt_init_slot(theta, (long long)sl.off, (long long)(sl.rows * sl.cols), seed, base, sc, (cudaStream_t)s,
                        c->bf16_weights != 0);
    }
  });
}

// The same values for the flat-index range [begin, end) only (a pipeline
// stage's slice: theta_slice[i - begin]); bit-identical to the full init.
sd_status sd_gpt_init_params_range(const sd_gpt_config* c, uint64_t seed, double gain_scale, double bias_scale,
                                   uint64_t begin, uint64_t end, float* theta_slice, sd_stream s) {
  return sd::guard([&] {
    if (!c || !theta_slice) fail(SD_ARGUMENT_ERROR, "null argument");
    const auto lay = layout(*c);
    const uint64_t P = lay.back().off + lay.back().rows * lay.back().cols;
    if (begin >= end || end > P) fail(SD_LAYOUT_ERROR, "init range out of bounds");
    for (const Slot& sl : lay) {
      const uint64_t a = std::max<uint64_t>(sl.off, begin), b = std::min<uint64_t>(sl.off + sl.rows * sl.cols, end);
      if (a >= b) continue;
      const double base = sl.kind == 1 ? 1.0 : 0.0;
      const double sc = sl.kind == 0 ? 0.02 : (sl.kind == 1 ? gain_scale : bias_scale);
      sd::gpt_init_slot(theta_slice, (long long)a, (long long)(b - a), seed, base, sc, (cudaStream_t)s,
                        c->bf16_weights != 0, (long long)begin);
    }
  });
}

uint64_t sd_gpt_workspace_bytes(const sd_gpt_config* c, int batch, int seq) {
  return sd_gpt_stage_workspace_bytes(c, batch, seq, 1, 0, c ? c->n_layer : 0, 1, 0);
}

uint64_t sd_gpt_stage_workspace_bytes(const sd_gpt_config* c, int micro_batch, int seq, int n_micro, int layer_begin,
                                      int layer_end, int n_sets, int flags) {
  try {
    if (!c) fail(SD_ARGUMENT_ERROR, "null config");
    check_cfg(*c, micro_batch, seq);
    const StageSpec sp{layer_begin, layer_end, n_micro, n_sets, flags};
    check_stage(*c, sp);
    return plan_for(*c, micro_batch, seq, nullptr, nullptr, sp).bytes;
  } catch (const std::exception& e) {
    sd::set_last_error(e.what());
    return 0;
  }
}

sd_status sd_gpt_stage_params(const sd_gpt_config* c, int layer_begin, int layer_end, uint64_t* begin,
                              uint64_t* end) {
  return sd::guard([&] {
    if (!c || !begin || !end) fail(SD_ARGUMENT_ERROR, "null argument");
    check_cfg(*c, 1, 4);
    check_stage(*c, StageSpec{layer_begin, layer_end, 1, 1, 0});
    if (layer_begin == 0 && layer_end == c->n_layer) {
      *begin = 0, *end = param_count(*c);
      return;
    }
    stage_range(*c, layer_begin, layer_end, layout(*c), begin, end);
  });
}

sd_status sd_gpt_stage_create(const sd_gpt_config* c, int micro_batch, int seq, int n_micro, int layer_begin,
                              int layer_end, int n_sets, int flags, const float* theta_stage, void* ws,
                              uint64_t bytes, sd_stream s, sd_gpt* out) {
  return sd::guard([&] {
    if (!c || !out) fail(SD_ARGUMENT_ERROR, "null argument");
    check_cfg(*c, micro_batch, seq);
    const StageSpec sp{layer_begin, layer_end, n_micro, n_sets, flags};
    check_stage(*c, sp);
    auto g = std::make_unique<sd_gpt_s>();
    const Plan p = plan_for(*c, micro_batch, seq, static_cast<char*>(ws), g.get(), sp);
    if (bytes < p.bytes) fail(SD_ARGUMENT_ERROR, "gpt workspace too small");
    g->slots = layout(*c);
    g->theta = theta_stage;
    if (c->bf16_weights) {
      if (sd::gpt_count_not_bf16(theta_stage, g->Pst, reinterpret_cast<unsigned long long*>(g->red),
                                 (cudaStream_t)s) != 0)
        fail(SD_CONFIG_ERROR, "bf16_weights: the parameters are not bf16-valued");
    } else {
      sd::gpt_residual(theta_stage, g->theta_s, g->Pst, (cudaStream_t)s);
    }
    SD_CUDA(cudaMemsetAsync(g->red, 0, sd::kColredReserve * sizeof(float), (cudaStream_t)s));  // colred counters
    if (g->last) {  // padded logits columns are never read as values but feed TMA boxes: zero them once
      for (float* z : {g->z, g->zs, g->dz, g->dzs})
        SD_CUDA(cudaMemsetAsync(z, 0, size_t(g->T) * g->Vp * 4, (cudaStream_t)s));
    }
    *out = g.release();
  });
}

sd_status sd_gpt_create(const sd_gpt_config* c, int batch, int seq, const float* theta, void* ws, uint64_t bytes,
                        sd_stream s, sd_gpt* out) {
  return sd_gpt_stage_create(c, batch, seq, 1, 0, c ? c->n_layer : 0, 1, 0, theta, ws, bytes, s, out);
}

// Uploads a batch (host int32 tokens/targets, n_micro * batch * seq each) and
// builds per micro-batch the token -> positions CSR of the deterministic
// embedding backward. Tokens are used by the first stage, targets by the last.
sd_status sd_gpt_set_batch(sd_gpt g, const int* tokens, const int* targets, float loss_scale, sd_stream s) {
  return sd::guard([&] {
    const int T = g->T, M = g->nmb;
    for (long long t = 0; t < (long long)T * M; ++t)
      if (tokens[t] < 0 || tokens[t] >= g->c.vocab || targets[t] < 0 || targets[t] >= g->c.vocab)
        fail(SD_ARGUMENT_ERROR, "token id out of range");
    cudaStream_t st = (cudaStream_t)s;
    // tokens | targets through the engine's pinned staging buffer (the caller's
    // buffers are free on return); the embedding backward's CSR is built on
    // the device (gpt_token_csr), so the call never waits for the GPU's work
    const size_t n = size_t(T) * M;
    if (!g->h_stage) {
      SD_CUDA(cudaMallocHost(&g->h_stage, 2 * n * sizeof(int)));
      SD_CUDA(cudaEventCreateWithFlags(&g->ev_stage, cudaEventDisableTiming));
    } else {
      SD_CUDA(cudaEventSynchronize(g->ev_stage));  // the previous upload has read the staging buffer
    }
    std::memcpy(g->h_stage, tokens, n * sizeof(int));
    std::memcpy(g->h_stage + n, targets, n * sizeof(int));
    if (g->first) {
      SD_CUDA(cudaMemcpyAsync(g->tok, g->h_stage, n * sizeof(int), cudaMemcpyHostToDevice, st));
      if (!g->csr_scratch) {
        g->csr_bytes = sd::gpt_token_csr_scratch(T, M, g->c.vocab);
        SD_CUDA(cudaMalloc(&g->csr_scratch, g->csr_bytes));
      }
      sd::gpt_token_csr(g->tok, T, M, g->c.vocab, g->uniq, g->ustart, g->upos, g->nuniq, g->csr_scratch, g->csr_bytes,
                        st);
    }
    if (g->last) SD_CUDA(cudaMemcpyAsync(g->tgt, g->h_stage + n, n * sizeof(int), cudaMemcpyHostToDevice, st));
    SD_CUDA(cudaEventRecord(g->ev_stage, st));
    g->loss_scale = loss_scale;
    g->have_batch = true;
  });
}

sd_status sd_gpt_hvp(sd_gpt g, const float* v, float* hv, sd_stream s) {
  return sd::guard([&] {
    if (!g->first || !g->last) fail(SD_STATE_ERROR, "gpt: a pipeline stage runs through the stage calls");
    g->hvp(v, hv, (cudaStream_t)s);
  });
}

sd_status sd_gpt_stage_begin(sd_gpt g, const float* v_stage, float* hv_stage, sd_stream s) {
  return sd::guard([&] {
    if (g->c.arch != SD_ARCH_LLAMA) fail(SD_CONFIG_ERROR, "pipeline stages need the Llama-style layout");
    g->stage_begin(v_stage, hv_stage, (cudaStream_t)s);
  });
}

// x_in/dx_in: stage input (ignored on the first stage); x_out/dx_out: stage
// output (may be null; the last stage keeps it for its backward).
sd_status sd_gpt_stage_forward(sd_gpt g, int m, const float* x_in, const float* dx_in, float* x_out, float* dx_out,
                               sd_stream s) {
  return sd::guard([&] {
    if (!g->vcur) fail(SD_STATE_ERROR, "gpt: stage_begin was not called");
    if (m < 0 || m >= g->nmb) fail(SD_ARGUMENT_ERROR, "micro-batch index out of range");
    const cudaStream_t st = (cudaStream_t)s;
    const size_t n = size_t(g->T) * g->c.d * sizeof(float);
    g->use_set(m);
    if (!g->first) {
      if (!x_in || !dx_in) fail(SD_ARGUMENT_ERROR, "stage input missing");
      SD_CUDA(cudaMemcpyAsync(g->x, x_in, n, cudaMemcpyDeviceToDevice, st));
      SD_CUDA(cudaMemcpyAsync(g->dx, dx_in, n, cudaMemcpyDeviceToDevice, st));
    }
    g->stage_fwd(m, st);
    if (x_out) SD_CUDA(cudaMemcpyAsync(x_out, g->x, n, cudaMemcpyDeviceToDevice, st));
    if (dx_out) SD_CUDA(cudaMemcpyAsync(dx_out, g->dx, n, cudaMemcpyDeviceToDevice, st));
  });
}

// gx_in/gdx_in: adjoint of the stage output (ignored on the last stage);
// gx_out/gdx_out: adjoint of the stage input (may be null).
sd_status sd_gpt_stage_backward(sd_gpt g, int m, const float* gx_in, const float* gdx_in, float* gx_out,
                                float* gdx_out, sd_stream s) {
  return sd::guard([&] {
    if (!g->vcur) fail(SD_STATE_ERROR, "gpt: stage_begin was not called");
    if (m < 0 || m >= g->nmb) fail(SD_ARGUMENT_ERROR, "micro-batch index out of range");
    const cudaStream_t st = (cudaStream_t)s;
    const size_t n = size_t(g->T) * g->c.d * sizeof(float);
    if (!g->last) {
      if (!gx_in || !gdx_in) fail(SD_ARGUMENT_ERROR, "stage adjoint input missing");
      SD_CUDA(cudaMemcpyAsync(g->gx, gx_in, n, cudaMemcpyDeviceToDevice, st));
      SD_CUDA(cudaMemcpyAsync(g->gdx, gdx_in, n, cudaMemcpyDeviceToDevice, st));
    }
    g->stage_bwd(m, st);
    if (gx_out) SD_CUDA(cudaMemcpyAsync(gx_out, g->gx, n, cudaMemcpyDeviceToDevice, st));
    if (gdx_out) SD_CUDA(cudaMemcpyAsync(gdx_out, g->gdx, n, cudaMemcpyDeviceToDevice, st));
  });
}

// mean per-token loss of the most recent hvp (synchronises the stream)
sd_status sd_gpt_last_loss(sd_gpt g, double* loss, sd_stream s) {
  return sd::guard([&] {
    if (!g->last) fail(SD_STATE_ERROR, "gpt: the loss lives on the last pipeline stage");
    const size_t n = size_t(g->T) * g->nmb;
    g->h_loss.resize(n);
    SD_CUDA(cudaMemcpyAsync(g->h_loss.data(), g->loss_rows, n * sizeof(double), cudaMemcpyDeviceToHost,
                            (cudaStream_t)s));
    SD_CUDA(cudaStreamSynchronize((cudaStream_t)s));
    double acc = 0.0;
    for (double x : g->h_loss) acc += x;
    *loss = acc / double(n);
  });
}

sd_status sd_gpt_destroy(sd_gpt g) {
  return sd::guard([&] { delete g; });
}

// Lanczos operator: y = H x on this rank's batch shard, summed over `comm`
// (data-sharded HVP; the loss_scale of every rank is 1/global_tokens).
sd_status sd_operator_gpt(sd_gpt g, sd_comm comm, sd_operator* out) {
  return sd::guard([&] {
    if (!g || !g->first || !g->last) fail(SD_ARGUMENT_ERROR, "gpt operator needs a whole-model engine");
    auto* ctx = new GptOpCtx{g, comm};
    const sd_status st = sd_operator_custom(uint64_t(g->P), gpt_apply, ctx, out);
    if (st != SD_OK) {
      delete ctx;
      fail(st, "operator_custom failed");
    }
    sd::operator_set_dtor(*out, [](void* p) { delete static_cast<GptOpCtx*>(p); });
  });
}

sd_status sd_operator_gpt_pipeline(sd_gpt g, sd_comm comm, sd_operator* out) {
  return sd::guard([&] {
    if (!g || !out) fail(SD_ARGUMENT_ERROR, "null argument");
    auto c = std::make_unique<GptPipeCtx>();
    c->g = g, c->comm = comm;
    c->nst = sd::comm_size(comm), c->st = sd::comm_rank(comm);
    if (g->first != (c->st == 0) || g->last != (c->st == c->nst - 1))
      fail(SD_LAYOUT_ERROR, "pipeline: the engine's layers do not match this rank's stage");
    const int need = std::min(g->nmb, c->nst - c->st);
    if (g->nsets < need) fail(SD_CONFIG_ERROR, "pipeline: stage needs min(n_micro, n_stages - stage) activation sets");
    uint64_t n = 0;
    if (sd_pipeline_schedule(c->nst, c->st, g->nmb, nullptr, 0, &n) != SD_OK) fail(SD_ARGUMENT_ERROR, sd_last_error());
    c->ops.resize(2 * n);
    if (sd_pipeline_schedule(c->nst, c->st, g->nmb, c->ops.data(), n, &n) != SD_OK)
      fail(SD_ARGUMENT_ERROR, sd_last_error());
    const sd_status st = sd_operator_custom(uint64_t(g->P), gpt_pipe_apply, c.get(), out);
    if (st != SD_OK) fail(st, "operator_custom failed");
    c.release();  // owned by the operator from here on
    sd::operator_set_dtor(*out, [](void* p) { delete static_cast<GptPipeCtx*>(p); });
  });
}

// Sharded operator: Lanczos vectors split by (begins, ends) over the comm's
// ranks (f32 only); see GptShardCtx. Scratch (2 full vectors) is owned here.
sd_status sd_operator_gpt_sharded(sd_gpt g, sd_comm comm, const uint64_t* begins, const uint64_t* ends,
                                  sd_operator* out) {
  return sd::guard([&] {
    if (!g || !begins || !ends) sd::fail(SD_ARGUMENT_ERROR, "null argument");
    if (!g->first || !g->last) fail(SD_ARGUMENT_ERROR, "sharded gpt operator needs a whole-model engine");
    auto* c = new GptShardCtx();  // owned by the operator (released by sd_operator_destroy)
    c->g = g;
    c->comm = comm;
    c->nranks = sd::comm_size(comm);
    c->rank = sd::comm_rank(comm);
    uint64_t at = 0;
    for (int r = 0; r < c->nranks; ++r) {
      if (begins[r] != at || ends[r] <= begins[r]) sd::fail(SD_LAYOUT_ERROR, "shard bounds leave a gap or overlap");
      c->rb.push_back(begins[r]);
      c->re.push_back(ends[r]);
      at = ends[r];
    }
    if (at != uint64_t(g->P)) sd::fail(SD_LAYOUT_ERROR, "shard bounds do not cover the parameter vector");
    SD_CUDA(cudaMalloc(&c->full, uint64_t(g->P) * sizeof(float)));
    SD_CUDA(cudaMalloc(&c->hv, uint64_t(g->P) * sizeof(float)));
    const sd_status st = sd_operator_custom(uint64_t(g->P), gpt_shard_apply, c, out);
    if (st != SD_OK) sd::fail(st, "operator_custom failed");
    sd::operator_set_dtor(*out, [](void* p) {
      auto* k = static_cast<GptShardCtx*>(p);
      for (float* b : {k->full, k->hv})
        if (b) cudaFree(b);
      delete k;
    });
  });
}

}  // extern "C"

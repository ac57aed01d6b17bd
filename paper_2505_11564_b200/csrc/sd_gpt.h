// Internal interfaces of the GPT HVP engine (kernels in sd_gpt_kernels.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace sd {

struct LnArgs {
  const float *x, *dx, *g, *b, *vg, *vb;
  int T, d;
  float eps;
  float *h, *hs, *dh, *dhs, *xh, *dxh, *r, *dr;
  int rms = 0;  // RMSNorm: no centring, no bias (b, vb null)
};
struct LnBwdArgs {
  const float *gy, *gdy, *g, *vg, *xh, *dxh, *r, *dr;
  int T, d;
  float *gx, *gdx, *gxs, *gdxs;
  float *hv_g, *hv_b;
  float* scratch;  // >= kColredReserve + 2 * 64 * d floats, the first kColredReserve zeroed once
  int rms = 0;
  int acc = 0;  // hv_g/hv_b += (micro-batch accumulation) instead of =
};

void gpt_embed(const int* tok, int T, int S, int d, const float* wte, const float* wpe, const float* vwte,
               const float* vwpe, float* x, float* dx, cudaStream_t s);
// RoPE (rotate-half) on the q and k parts of a [T, 3d] q|k|v buffer and its
// tangent, in place (inverse = backward adjoint); residuals rewritten.
void llama_rope(float* a, float* as, float* da, float* das, int T, int S, int d, int dh, float base, int inverse,
                cudaStream_t s);
// grouped-query attention: raw [T, d + 2 KV dh] q|k|v (+tangent, residuals) ->
// the MHA [T, 3d] layout (query head h reads KV head h / (H / KV)); and the
// adjoint reduction back (sums over each KV head's query group; residuals)
void llama_gqa_expand(const float* raw, const float* raws, const float* draw, const float* draws, float* a, float* as,
                      float* da, float* das, int T, int d, int dh, int KV, int H, cudaStream_t s);
void llama_gqa_reduce(const float* ga, const float* gda, float* graw, float* graws, float* gdraw, float* gdraws, int T,
                      int d, int dh, int KV, int H, cudaStream_t s);
// SwiGLU: fu = [gate | up] [T, 2ff] -> a = silu(gate) * up (and tangent, residuals)
void llama_swiglu_fwd(const float* fu, const float* dfu, float* a, float* as, float* da, float* das, int T, int ff,
                      cudaStream_t s);
// adjoints of [gate | up] from ga (and tangents), residuals
void llama_swiglu_bwd(const float* fu, const float* dfu, const float* ga, const float* gda, float* gfu, float* gfus,
                      float* gdfu, float* gdfus, int T, int ff, cudaStream_t s);
void gpt_ln_fwd(const LnArgs& a, cudaStream_t s);
void gpt_ln_bwd(const LnBwdArgs& a, cudaStream_t s);
// column-reduction scratch: kColredReserve floats of arrival counters (zeroed
// once at creation; each reduction leaves them zero) + 2 * 64 * n partials
constexpr int kColredReserve = 4096;
void gpt_colsum(const float* a, int T, int n, long long lda, float* out, float* scratch, cudaStream_t s,
                int acc = 0);
void gpt_gelu_fwd(const float* f, const float* df, float* u, float* us, float* du, float* dus, long long n,
                  cudaStream_t s);
void gpt_gelu_bwd(const float* f, const float* df, float* gu, float* gdu, float* gus, float* gdus, long long n,
                  cudaStream_t s);
void gpt_attn_softmax_fwd(float* Sm, float* dS, float* Ps, float* dPs, int S, long long rows, cudaStream_t s);
void gpt_attn_softmax_bwd(const float* P, const float* dP, float* gP, float* gdP, float* gPs, float* gdPs, int S,
                          long long rows, cudaStream_t s);
void gpt_ce(float* z, float* dz, float* zs, float* dzs, const int* tgt, int T, int V, long long ld, float scale,
            double* loss_rows, cudaStream_t s);
// Hv of the embeddings: hv_wte rows += scattered adjoint tangents; hv_wpe
// = (acc: +=) the per-position sums
void gpt_embed_bwd(const int* uniq, const int* start, const int* pos, const int* n_uniq_dev, int B, int S, int d,
                   const float* gdx, float* hv_wte, float* hv_wpe, cudaStream_t s, int acc = 0);
// device-side token -> positions CSR of M micro-batches of T tokens (see sd_gpt_kernels.cu)
size_t gpt_token_csr_scratch(int T, int M, int V);
void gpt_token_csr(const int* tok, int T, int M, int V, int* uniq, int* ustart, int* upos, int* nuniq,
                   void* scratch, size_t scratch_bytes, cudaStream_t s);
void gpt_residual(const float* x, float* xs, long long n, cudaStream_t s);
void gpt_fill(float* x, float v, long long n, cudaStream_t s);
// theta[i - th_base] for global flat indices i in [off, off + n)
void gpt_init_slot(float* th, long long off, long long n, uint64_t seed, double base, double scale, cudaStream_t s,
                   bool bf16 = false, long long th_base = 0);
// elements of x that are not bf16-valued (synchronises the stream; scratch: one u64 on device)
unsigned long long gpt_count_not_bf16(const float* x, long long n, unsigned long long* scratch, cudaStream_t s);

}  // namespace sd

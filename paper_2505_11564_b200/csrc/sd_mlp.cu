// MLP Hessian-vector products on sm_100a: the SPEC's mlp(layer_widths)
// model family (tanh hidden layers, mse loss), restated by the
// oracle in oracle/src/models.cpp (build_mlp). Same forward-over-reverse
// scheme as the GPT engine (Alg. 1): the forward carries the tangent
// (primal z = a W + b, dz = da W + a V_W + V_b), the backward carries the
// adjoint and its tangent, and the parameter tangent-adjoint is Hv.
//
// Products run on the 3xTF32 tcgen05 GEMM (sd_gemm.cu), tangent pairs as one
// dual-source launch. Widths are padded to multiples of 4 (16-byte TMA
// strides); padded columns carry exact zeros through every layer.
#include <cuda_runtime.h>

#include <memory>
#include <vector>

#include "sd_common.cuh"
#include "sd_engine.h"
#include "sd_gemm.h"
#include "sd_gpt.h"

namespace sd {
namespace {

// flat [rows x cols] block at `off` <-> padded [rows x ldp] device buffer
__global__ void k_pack(const float* __restrict__ flat, long long off, int rows, int cols, int ldp,
                       float* __restrict__ out) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long n = (long long)rows * ldp;
  if (i >= n) return;
  const int r = int(i / ldp), c = int(i % ldp);
  out[i] = c < cols ? flat[off + (long long)r * cols + c] : 0.0f;
}
__global__ void k_unpack(const float* __restrict__ padded, int rows, int cols, int ldp, float* __restrict__ flat,
                         long long off) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= (long long)rows * cols) return;
  const int r = int(i / cols), c = int(i % cols);
  flat[off + i] = padded[(long long)r * ldp + c];
}
// hidden layer: a = tanh(z), da = (1 - a^2) dz
__global__ void k_tanh_fwd(const float* __restrict__ z, const float* __restrict__ dz, float* __restrict__ a,
                           float* __restrict__ da, long long n) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  // f64 internals, one rounding per stored value
  const double t = tanh(double(z[i]));
  const float tf = float(t);
  a[i] = tf;
  const double tr = double(tf);
  da[i] = float((1.0 - tr * tr) * double(dz[i]));
}
// output: loss += s sum (p - y)^2 ; g = 2 s (p - y) ; gd = 2 s dp  (mse, graph.cpp mse)
__global__ void k_mse(const float* __restrict__ p, const float* __restrict__ dp, const float* __restrict__ y,
                      float s, long long n, float* __restrict__ g, float* __restrict__ gd, double* __restrict__ loss) {
  __shared__ double red[256];
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  double l = 0.0;
  if (i < n) {
    const double e = double(p[i]) - double(y[i]);
    g[i] = float(2.0 * double(s) * e);
    gd[i] = float(2.0 * double(s) * double(dp[i]));
    l = e * e;
  }
  red[threadIdx.x] = l;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) loss[blockIdx.x] = red[0];
}
// hidden adjoint through tanh: gz = ga (1 - a^2); gdz = gda (1 - a^2) - 2 ga a da
__global__ void k_tanh_bwd(const float* __restrict__ a, const float* __restrict__ da, const float* __restrict__ ga,
                           const float* __restrict__ gda, float* __restrict__ gz, float* __restrict__ gdz,
                           long long n) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double t = double(a[i]), d1 = 1.0 - t * t, g = double(ga[i]);
  gz[i] = float(g * d1);
  gdz[i] = float(double(gda[i]) * d1 - 2.0 * g * t * double(da[i]));
}

unsigned blocks(long long n, int t = 256) { return unsigned((n + t - 1) / t); }

}  // namespace
}  // namespace sd

struct sd_mlp_s {
  std::vector<int> w, wp;            // widths, padded widths
  std::vector<long long> offW, offb;  // flat offsets of W_l, b_l
  long long P = 0;
  int n_max = 0, n = 0;
  float loss_scale = 0.0f;
  const float* theta = nullptr;
  // device buffers (padded)
  std::vector<float*> W, Ws, b, VW, VWs, Vb, HW, Hb;
  std::vector<float*> a, as, da, das;  // activations a_0..a_{L} (a_L = output z)
  std::vector<float*> z, dz;
  float *x = nullptr, *y = nullptr, *g = nullptr, *gs = nullptr, *gd = nullptr, *gds = nullptr;
  float *ga = nullptr, *gda = nullptr, *red = nullptr;
  double* loss_part = nullptr;
  std::vector<void*> owned;
  double last_loss = 0.0;
  bool have_batch = false;

  float* alloc(long long nfl) {
    void* p = nullptr;
    SD_CUDA(cudaMalloc(&p, size_t(std::max<long long>(nfl, 4)) * sizeof(float)));
    SD_CUDA(cudaMemset(p, 0, size_t(std::max<long long>(nfl, 4)) * sizeof(float)));
    owned.push_back(p);
    return static_cast<float*>(p);
  }
  ~sd_mlp_s() {
    for (void* p : owned) cudaFree(p);
  }
  int L() const { return int(w.size()) - 1; }

  void mm(int M, int N, int K, const float* A, const float* As, long long lda, bool amn, const float* B,
          const float* Bs, long long ldb, bool bmn, float* C, long long ldc, float beta, cudaStream_t st,
          const float* bias = nullptr, const float* A2 = nullptr, const float* A2s = nullptr,
          const float* B2 = nullptr, const float* B2s = nullptr) {
    sd::GemmArgs q;
    q.M = M, q.N = N, q.K = K;
    q.A = A, q.As = As, q.lda = lda, q.a_mn = amn;
    q.B = B, q.Bs = Bs, q.ldb = ldb, q.b_mn = bmn;
    q.C = C, q.ldc = ldc, q.beta = beta, q.bias = bias;
    if (A2) q.A2 = A2, q.A2s = A2s, q.lda2 = lda, q.B2 = B2, q.B2s = B2s, q.ldb2 = ldb;
    sd::gemm(q, st);
  }

  void hvp(const float* v, float* hv, cudaStream_t st) {
    if (!have_batch) sd::fail(SD_STATE_ERROR, "mlp: set_batch was not called");
    const int Ln = L();
    // parameters and direction into padded buffers (+ tf32 residuals)
    for (int l = 0; l < Ln; ++l) {
      const long long nw = (long long)wp[l] * wp[l + 1];  // residuals over the padded block
      sd::k_pack<<<sd::blocks(nw), 256, 0, st>>>(theta, offW[l], w[l], w[l + 1], wp[l + 1], W[l]);
      sd::k_pack<<<sd::blocks(nw), 256, 0, st>>>(v, offW[l], w[l], w[l + 1], wp[l + 1], VW[l]);
      sd::k_pack<<<sd::blocks(wp[l + 1]), 256, 0, st>>>(theta, offb[l], 1, w[l + 1], wp[l + 1], b[l]);
      sd::k_pack<<<sd::blocks(wp[l + 1]), 256, 0, st>>>(v, offb[l], 1, w[l + 1], wp[l + 1], Vb[l]);
      SD_LAUNCHED("k_pack");
      sd::gpt_residual(W[l], Ws[l], nw, st);
      sd::gpt_residual(VW[l], VWs[l], nw, st);
    }
    // ---- forward with tangent
    for (int l = 0; l < Ln; ++l) {
      float* zo = l + 1 < Ln ? z[l] : a[Ln];
      float* dzo = l + 1 < Ln ? dz[l] : da[Ln];
      mm(n, wp[l + 1], wp[l], a[l], as[l], wp[l], false, W[l], Ws[l], wp[l + 1], true, zo, wp[l + 1], 0.0f, st,
         b[l]);
      if (l == 0) {  // da_0 = 0
        mm(n, wp[1], wp[0], a[0], as[0], wp[0], false, VW[0], VWs[0], wp[1], true, dzo, wp[1], 0.0f, st, Vb[0]);
      } else {
        mm(n, wp[l + 1], wp[l], da[l], das[l], wp[l], false, W[l], Ws[l], wp[l + 1], true, dzo, wp[l + 1], 0.0f, st,
           Vb[l], a[l], as[l], VW[l], VWs[l]);
      }
      if (l + 1 < Ln) {
        const long long ne = (long long)n * wp[l + 1];
        sd::k_tanh_fwd<<<sd::blocks(ne), 256, 0, st>>>(z[l], dz[l], a[l + 1], da[l + 1], ne);
        SD_LAUNCHED("k_tanh_fwd");
        sd::gpt_residual(a[l + 1], as[l + 1], ne, st);
        sd::gpt_residual(da[l + 1], das[l + 1], ne, st);
      }
    }
    // ---- loss and output adjoints
    const long long no = (long long)n * wp[Ln];
    const unsigned nb = sd::blocks(no);
    sd::k_mse<<<nb, 256, 0, st>>>(a[Ln], da[Ln], y, loss_scale, no, g, gd, loss_part);
    SD_LAUNCHED("k_mse");
    std::vector<double> parts(nb);
    // ---- backward with tangent
    for (int l = Ln - 1; l >= 0; --l) {
      const long long ne = (long long)n * wp[l + 1];
      float *gz = g, *gdz = gd;
      sd::gpt_residual(gz, gs, ne, st);
      sd::gpt_residual(gdz, gds, ne, st);
      // Hv_W = da_l^T gz + a_l^T gdz ; Hv_b = colsum(gdz)
      if (l == 0) {
        mm(wp[0], wp[1], n, a[0], as[0], wp[0], true, gdz, gds, wp[1], true, HW[0], wp[1], 0.0f, st);
      } else {
        mm(wp[l], wp[l + 1], n, da[l], das[l], wp[l], true, gz, gs, wp[l + 1], true, HW[l], wp[l + 1], 0.0f, st,
           nullptr, a[l], as[l], gdz, gds);
      }
      sd::gpt_colsum(gdz, n, wp[l + 1], wp[l + 1], Hb[l], red, st);
      if (l > 0) {
        // ga = gz W^T ; gda = gdz W^T + gz V_W^T
        mm(n, wp[l], wp[l + 1], gz, gs, wp[l + 1], false, W[l], Ws[l], wp[l + 1], false, ga, wp[l], 0.0f, st);
        mm(n, wp[l], wp[l + 1], gdz, gds, wp[l + 1], false, W[l], Ws[l], wp[l + 1], false, gda, wp[l], 0.0f, st,
           nullptr, gz, gs, VW[l], VWs[l]);
        const long long nh = (long long)n * wp[l];
        sd::k_tanh_bwd<<<sd::blocks(nh), 256, 0, st>>>(a[l], da[l], ga, gda, g, gd, nh);
        SD_LAUNCHED("k_tanh_bwd");
      }
    }
    for (int l = 0; l < Ln; ++l) {
      const long long nw = (long long)w[l] * w[l + 1];
      sd::k_unpack<<<sd::blocks(nw), 256, 0, st>>>(HW[l], w[l], w[l + 1], wp[l + 1], hv, offW[l]);
      sd::k_unpack<<<sd::blocks(w[l + 1]), 256, 0, st>>>(Hb[l], 1, w[l + 1], wp[l + 1], hv, offb[l]);
      SD_LAUNCHED("k_unpack");
    }
    SD_CUDA(cudaMemcpyAsync(parts.data(), loss_part, nb * sizeof(double), cudaMemcpyDeviceToHost, st));
    SD_CUDA(cudaStreamSynchronize(st));
    double acc = 0.0;
    for (double p : parts) acc += p;
    last_loss = acc * double(loss_scale);
  }
};

namespace {
struct MlpOpCtx {
  sd_mlp m;
  sd_comm comm;
};
sd_status mlp_apply(void* ctx, const void* x, void* y, sd_stream s) {
  auto* c = static_cast<MlpOpCtx*>(ctx);
  return sd::guard([&] {
    c->m->hvp(static_cast<const float*>(x), static_cast<float*>(y), (cudaStream_t)s);
    sd::comm_allreduce_f32(c->comm, static_cast<float*>(y), uint64_t(c->m->P), (cudaStream_t)s);
  });
}
int pad4(int x) { return (x + 3) & ~3; }
}  // namespace

extern "C" {

uint64_t sd_mlp_param_count(const uint64_t* widths, int n_widths) {
  if (!widths || n_widths < 2) return 0;
  uint64_t n = 0;
  for (int l = 0; l + 1 < n_widths; ++l) n += widths[l] * widths[l + 1] + widths[l + 1];
  return n;
}

sd_status sd_mlp_create(const uint64_t* widths, int n_widths, int n_max, const float* theta, sd_stream s,
                        sd_mlp* out) {
  return sd::guard([&] {
    (void)s;
    if (!widths || n_widths < 2) sd::fail(SD_CONFIG_ERROR, "mlp needs at least two widths");
    if (n_max < 1) sd::fail(SD_CONFIG_ERROR, "mlp batch capacity must be positive");
    if (!theta) sd::fail(SD_ARGUMENT_ERROR, "mlp parameters are null");
    auto m = std::make_unique<sd_mlp_s>();
    for (int l = 0; l < n_widths; ++l) {
      if (widths[l] < 1 || widths[l] > (1u << 20)) sd::fail(SD_CONFIG_ERROR, "mlp width out of range");
      m->w.push_back(int(widths[l]));
      m->wp.push_back(pad4(int(widths[l])));
    }
    m->theta = theta;
    m->n_max = n_max;
    long long off = 0;
    const int Ln = m->L();
    int wmax = 0;
    for (int l = 0; l <= Ln; ++l) wmax = std::max(wmax, m->wp[l]);
    for (int l = 0; l < Ln; ++l) {
      m->offW.push_back(off);
      off += (long long)m->w[l] * m->w[l + 1];
      m->offb.push_back(off);
      off += m->w[l + 1];
      // W buffers hold wp[l] rows (the K padding rows stay zero)
      const long long nwp = (long long)m->wp[l] * m->wp[l + 1];
      m->W.push_back(m->alloc(nwp)), m->Ws.push_back(m->alloc(nwp));
      m->VW.push_back(m->alloc(nwp)), m->VWs.push_back(m->alloc(nwp));
      m->HW.push_back(m->alloc((long long)m->wp[l] * m->wp[l + 1]));
      m->b.push_back(m->alloc(m->wp[l + 1])), m->Vb.push_back(m->alloc(m->wp[l + 1]));
      m->Hb.push_back(m->alloc(m->wp[l + 1]));
    }
    m->P = off;
    for (int l = 0; l <= Ln; ++l) {
      const long long na = (long long)n_max * m->wp[l];
      m->a.push_back(m->alloc(na)), m->as.push_back(m->alloc(na));
      m->da.push_back(m->alloc(na)), m->das.push_back(m->alloc(na));
      if (l < Ln) {  // pre-activation of layer l: width wp[l + 1]
        const long long nz = (long long)n_max * m->wp[l + 1];
        m->z.push_back(m->alloc(nz)), m->dz.push_back(m->alloc(nz));
      }
    }
    const long long nm = (long long)n_max * wmax;
    m->y = m->alloc((long long)n_max * m->wp[Ln]);
    m->g = m->alloc(nm), m->gs = m->alloc(nm), m->gd = m->alloc(nm), m->gds = m->alloc(nm);
    m->ga = m->alloc(nm), m->gda = m->alloc(nm);
    m->red = m->alloc(sd::kColredReserve + 2LL * 64 * wmax);
    SD_CUDA(cudaMemset(m->red, 0, sd::kColredReserve * sizeof(float)));  // column-reduction arrival counters
    void* lp = nullptr;
    SD_CUDA(cudaMalloc(&lp, size_t((nm + 255) / 256 + 1) * sizeof(double)));
    m->owned.push_back(lp);
    m->loss_part = static_cast<double*>(lp);
    *out = m.release();
  });
}

sd_status sd_mlp_set_batch(sd_mlp m, const float* x, const float* y, int n, float loss_scale, sd_stream s) {
  return sd::guard([&] {
    if (!m) sd::fail(SD_ARGUMENT_ERROR, "mlp handle is null");
    if (n < 1) sd::fail(SD_ARGUMENT_ERROR, "empty batch");
    if (n > m->n_max) sd::fail(SD_ARGUMENT_ERROR, "batch larger than the engine capacity");
    const int Ln = m->L();
    auto upload = [&](const float* src, int cols, int ldp, float* dst) {
      std::vector<float> h((size_t)n * ldp, 0.0f);
      for (int r = 0; r < n; ++r)
        for (int c = 0; c < cols; ++c) h[(size_t)r * ldp + c] = src[(size_t)r * cols + c];
      SD_CUDA(cudaMemcpyAsync(dst, h.data(), h.size() * sizeof(float), cudaMemcpyHostToDevice, (cudaStream_t)s));
      SD_CUDA(cudaStreamSynchronize((cudaStream_t)s));
    };
    upload(x, m->w[0], m->wp[0], m->a[0]);
    sd::gpt_residual(m->a[0], m->as[0], (long long)n * m->wp[0], (cudaStream_t)s);
    upload(y, m->w[Ln], m->wp[Ln], m->y);
    m->n = n;
    m->loss_scale = loss_scale;
    m->have_batch = true;
  });
}

sd_status sd_mlp_hvp(sd_mlp m, const float* v, float* hv, sd_stream s) {
  return sd::guard([&] {
    if (!m) sd::fail(SD_ARGUMENT_ERROR, "mlp handle is null");
    m->hvp(v, hv, (cudaStream_t)s);
  });
}

sd_status sd_mlp_last_loss(sd_mlp m, double* loss) {
  return sd::guard([&] {
    if (!m || !loss) sd::fail(SD_ARGUMENT_ERROR, "null argument");
    *loss = m->last_loss;
  });
}

sd_status sd_mlp_destroy(sd_mlp m) {
  return sd::guard([&] { delete m; });
}

sd_status sd_operator_mlp(sd_mlp m, sd_comm comm, sd_operator* out) {
  return sd::guard([&] {
    auto* ctx = new MlpOpCtx{m, comm};
    const sd_status st = sd_operator_custom(uint64_t(m->P), mlp_apply, ctx, out);
    if (st != SD_OK) {
      delete ctx;
      sd::fail(st, "operator_custom failed");
    }
    sd::operator_set_dtor(*out, [](void* p) { delete static_cast<MlpOpCtx*>(p); });
  });
}

}  // extern "C"

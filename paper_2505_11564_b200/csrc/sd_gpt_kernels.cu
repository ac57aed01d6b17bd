// Fused R-op (forward tangent) and double-backward elementwise kernels of the
// GPT decoder HVP (Pearlmutter: Hv = d/de grad L(theta + e v)). Every kernel
// computes a primal quantity together with its directional derivative along
// v, so each activation is read once per pass. Wherever an output feeds a
// tensor-core GEMM, the kernel also writes its tf32 residual
// (x - trunc_tf32(x)) for the 3xTF32 product.
//
// Notation: X primal, dX tangent (R-op), gX adjoint, gdX adjoint tangent.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <math.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>
#include <initializer_list>

#include "sd_common.cuh"
#include "sd_gpt.h"

namespace sd {

__device__ __forceinline__ float tf32_res(float x) { return x - __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

template <int NW>
__device__ __forceinline__ float block_sum(float v, float* red) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  v = warp_sum(v);
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  float t = 0.f;
#pragma unroll
  for (int i = 0; i < NW; ++i) t += red[i];
  return t;
}
template <int NW>
__device__ __forceinline__ float block_max(float v, float* red) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  v = warp_max(v);
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  float t = -INFINITY;
#pragma unroll
  for (int i = 0; i < NW; ++i) t = fmaxf(t, red[i]);
  return t;
}

// ------------------------------------------------------------- embedding
// x[t] = wte[tok] + wpe[s]; dx[t] = Vwte[tok] + Vwpe[s]
__global__ void k_embed(const int* __restrict__ tok, int S, int d, const float* __restrict__ wte,
                        const float* __restrict__ wpe, const float* __restrict__ vwte, const float* __restrict__ vwpe,
                        float* __restrict__ x, float* __restrict__ dx, long long n) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const long long t = i / d;
  const int e = int(i - t * d);
  const int s = int(t % S);
  const long long tk = tok[t];
  x[i] = wte[tk * d + e] + (wpe ? wpe[(long long)s * d + e] : 0.f);
  dx[i] = vwte[tk * d + e] + (vwpe ? vwpe[(long long)s * d + e] : 0.f);
}

// ------------------------------------------------------------- LayerNorm
// One warp per row. h = g*xh + b, xh = (x - mu) r, r = (var + eps)^-1/2;
// dxh = r (dx - mean(dx) - xh mean(xh dx)), dr = -r * mean(xh dx) (per-row
// tangent of r divided by r), dh = Vg*xh + g*dxh + Vb.
__global__ void k_ln_fwd(const float* __restrict__ x, const float* __restrict__ dx, const float* __restrict__ g,
                         const float* __restrict__ b, const float* __restrict__ vg, const float* __restrict__ vb,
                         int T, int d, float eps, float* __restrict__ h, float* __restrict__ hs,
                         float* __restrict__ dh, float* __restrict__ dhs, float* __restrict__ xh,
                         float* __restrict__ dxh, float* __restrict__ r_out, float* __restrict__ dr_out, int rms) {
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= T) return;
  const float* xr = x + (long long)row * d;
  const float* dxr = dx + (long long)row * d;
  float mu = 0.f, dmu = 0.f;  // RMSNorm: no centring
  if (!rms) {
    float s = 0.f, ds = 0.f;
    for (int e = lane; e < d; e += 32) {
      s += xr[e];
      ds += dxr[e];
    }
    mu = warp_sum(s) / d, dmu = warp_sum(ds) / d;
  }
  float v = 0.f;
  for (int e = lane; e < d; e += 32) {
    const float c = xr[e] - mu;
    v += c * c;
  }
  const float var = warp_sum(v) / d;
  const float r = rsqrtf(var + eps);
  float m2 = 0.f;
  for (int e = lane; e < d; e += 32) m2 += (xr[e] - mu) * r * (dxr[e] - dmu);
  const float mxd = warp_sum(m2) / d;  // mean(xh * dx) (dx centred; mean(xh) = 0)
  const long long o = (long long)row * d;
  for (int e = lane; e < d; e += 32) {
    const float xhv = (xr[e] - mu) * r;
    const float dxhv = r * (dxr[e] - dmu - xhv * mxd);
    const float hv = g[e] * xhv + (b ? b[e] : 0.f);
    const float dhv = vg[e] * xhv + g[e] * dxhv + (vb ? vb[e] : 0.f);
    xh[o + e] = xhv;
    dxh[o + e] = dxhv;
    h[o + e] = hv;
    hs[o + e] = tf32_res(hv);
    dh[o + e] = dhv;
    dhs[o + e] = tf32_res(dhv);
  }
  if (lane == 0) {
    r_out[row] = r;
    dr_out[row] = -r * mxd;  // dr / r
  }
}

// Register-resident forms for d = 128 NV <= 1024 (GPT-2 d = 768: NV = 6): one
// warp per row, lane l owns the float4 groups l, l + 32, ... of the row, which
// it loads ONCE (16-byte coalesced) and keeps in registers through every pass;
// same math as k_ln_fwd / k_ln_bwd.
template <int NV>
__global__ void __launch_bounds__(128) k_ln_fwd_reg(const float* __restrict__ x, const float* __restrict__ dx,
    const float* __restrict__ g, const float* __restrict__ b, const float* __restrict__ vg,
    const float* __restrict__ vb, int T, float eps, float* __restrict__ h, float* __restrict__ hs,
    float* __restrict__ dh, float* __restrict__ dhs, float* __restrict__ xh, float* __restrict__ dxh,
    float* __restrict__ r_out, float* __restrict__ dr_out, int rms) {
  pdl_wait();  // PDL: nothing global is touched before the previous kernel completes
  constexpr int d = 128 * NV;
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= T) return;
  const long long o4 = (long long)row * (d / 4);
  float4 xv[NV], dv[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    xv[i] = reinterpret_cast<const float4*>(x)[o4 + lane + 32 * i];
    dv[i] = reinterpret_cast<const float4*>(dx)[o4 + lane + 32 * i];
  }
  float mu = 0.f, dmu = 0.f;
  if (!rms) {
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      s1 += (xv[i].x + xv[i].y) + (xv[i].z + xv[i].w);
      s2 += (dv[i].x + dv[i].y) + (dv[i].z + dv[i].w);
    }
    mu = warp_sum(s1) / d, dmu = warp_sum(s2) / d;
  }
  float v = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const float a0 = xv[i].x - mu, a1 = xv[i].y - mu, a2 = xv[i].z - mu, a3 = xv[i].w - mu;
    v += (a0 * a0 + a1 * a1) + (a2 * a2 + a3 * a3);
  }
  const float r = rsqrtf(warp_sum(v) / d + eps);
  float m2 = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i)
    m2 += ((xv[i].x - mu) * r * (dv[i].x - dmu) + (xv[i].y - mu) * r * (dv[i].y - dmu)) +
          ((xv[i].z - mu) * r * (dv[i].z - dmu) + (xv[i].w - mu) * r * (dv[i].w - dmu));
  const float mxd = warp_sum(m2) / d;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c4 = lane + 32 * i;
    const float4 gg = reinterpret_cast<const float4*>(g)[c4], vgg = reinterpret_cast<const float4*>(vg)[c4];
    const float4 bb = b ? reinterpret_cast<const float4*>(b)[c4] : make_float4(0.f, 0.f, 0.f, 0.f);
    const float4 vbb = vb ? reinterpret_cast<const float4*>(vb)[c4] : make_float4(0.f, 0.f, 0.f, 0.f);
    float4 xo, dxo, ho, hso, dho, dhso;
#define SD_LN_LANE(f)                                              \
    {                                                              \
      const float xhv = (xv[i].f - mu) * r;                        \
      const float dxhv = r * (dv[i].f - dmu - xhv * mxd);          \
      const float hv = gg.f * xhv + bb.f;                          \
      const float dhv = vgg.f * xhv + gg.f * dxhv + vbb.f;         \
      xo.f = xhv, dxo.f = dxhv, ho.f = hv, hso.f = tf32_res(hv);   \
      dho.f = dhv, dhso.f = tf32_res(dhv);                         \
    }
    SD_LN_LANE(x) SD_LN_LANE(y) SD_LN_LANE(z) SD_LN_LANE(w)
#undef SD_LN_LANE
    reinterpret_cast<float4*>(xh)[o4 + c4] = xo;
    reinterpret_cast<float4*>(dxh)[o4 + c4] = dxo;
    reinterpret_cast<float4*>(h)[o4 + c4] = ho;
    reinterpret_cast<float4*>(hs)[o4 + c4] = hso;
    reinterpret_cast<float4*>(dh)[o4 + c4] = dho;
    reinterpret_cast<float4*>(dhs)[o4 + c4] = dhso;
  }
  if (lane == 0) {
    r_out[row] = r;
    dr_out[row] = -r * mxd;
  }
}

template <int NV>
__global__ void __launch_bounds__(256, NV <= 6 ? 2 : 1) k_ln_bwd_reg(const float* __restrict__ gy, const float* __restrict__ gdy,
    const float* __restrict__ g, const float* __restrict__ vg, const float* __restrict__ xh,
    const float* __restrict__ dxh, const float* __restrict__ rr, const float* __restrict__ drr, int T,
    float* __restrict__ gx, float* __restrict__ gdx, float* __restrict__ gxs, float* __restrict__ gdxs, int rms) {
  pdl_wait();  // PDL: nothing global is touched before the previous kernel completes
  constexpr int d = 128 * NV;
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= T) return;
  const long long o4 = (long long)row * (d / 4);
  float4 gq[NV], gdq[NV], xhv[NV], dxhv[NV];
  float s1 = 0.f, s2 = 0.f, s3 = 0.f, s4 = 0.f, s5 = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c4 = lane + 32 * i;
    const float4 a = reinterpret_cast<const float4*>(gy)[o4 + c4], ad = reinterpret_cast<const float4*>(gdy)[o4 + c4];
    const float4 gg = reinterpret_cast<const float4*>(g)[c4], vgg = reinterpret_cast<const float4*>(vg)[c4];
    xhv[i] = reinterpret_cast<const float4*>(xh)[o4 + c4];
    dxhv[i] = reinterpret_cast<const float4*>(dxh)[o4 + c4];
#define SD_LNB_LANE(f)                                  \
    gq[i].f = a.f * gg.f;                               \
    gdq[i].f = ad.f * gg.f + a.f * vgg.f;               \
    s1 += gq[i].f, s2 += gq[i].f * xhv[i].f, s3 += gdq[i].f; \
    s4 += gdq[i].f * xhv[i].f, s5 += gq[i].f * dxhv[i].f;
    SD_LNB_LANE(x) SD_LNB_LANE(y) SD_LNB_LANE(z) SD_LNB_LANE(w)
#undef SD_LNB_LANE
  }
  const float m_g = rms ? 0.f : warp_sum(s1) / d, m_gx = warp_sum(s2) / d, m_d = rms ? 0.f : warp_sum(s3) / d;
  const float m_dx = warp_sum(s4) / d, m_gdx = warp_sum(s5) / d;
  const float r = rr[row], dr = drr[row];
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c4 = lane + 32 * i;
    float4 ox = reinterpret_cast<const float4*>(gx)[o4 + c4], od = reinterpret_cast<const float4*>(gdx)[o4 + c4];
    float4 oxs, ods;
#define SD_LNB_OUT(f)                                                                              \
    {                                                                                              \
      const float base = gq[i].f - m_g - xhv[i].f * m_gx;                                          \
      ox.f = ox.f + r * base;                                                                      \
      od.f = od.f + dr * r * base + r * (gdq[i].f - m_d - dxhv[i].f * m_gx - xhv[i].f * (m_dx + m_gdx)); \
      oxs.f = tf32_res(ox.f), ods.f = tf32_res(od.f);                                              \
    }
    SD_LNB_OUT(x) SD_LNB_OUT(y) SD_LNB_OUT(z) SD_LNB_OUT(w)
#undef SD_LNB_OUT
    reinterpret_cast<float4*>(gx)[o4 + c4] = ox;
    reinterpret_cast<float4*>(gdx)[o4 + c4] = od;
    if (gxs) {
      reinterpret_cast<float4*>(gxs)[o4 + c4] = oxs;
      reinterpret_cast<float4*>(gdxs)[o4 + c4] = ods;
    }
  }
}

// Backward of LN with its tangent, accumulating into the residual adjoints:
//   gq = gy*g;      gdq = gdy*g + gy*Vg
//   gx += r (gq - mean(gq) - xh mean(gq xh))
//   gdx += dr*r*(gq - mean(gq) - xh mean(gq xh))
//        + r (gdq - mean(gdq) - dxh mean(gq xh) - xh (mean(gdq xh) + mean(gq dxh)))
__global__ void k_ln_bwd(const float* __restrict__ gy, const float* __restrict__ gdy, const float* __restrict__ g,
                         const float* __restrict__ vg, const float* __restrict__ xh, const float* __restrict__ dxh,
                         const float* __restrict__ rr, const float* __restrict__ drr, int T, int d,
                         float* __restrict__ gx, float* __restrict__ gdx, float* __restrict__ gxs,
                         float* __restrict__ gdxs, int rms) {
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= T) return;
  const long long o = (long long)row * d;
  float s1 = 0.f, s2 = 0.f, s3 = 0.f, s4 = 0.f, s5 = 0.f;
  for (int e = lane; e < d; e += 32) {
    const float gq = gy[o + e] * g[e];
    const float gdq = gdy[o + e] * g[e] + gy[o + e] * vg[e];
    s1 += gq;
    s2 += gq * xh[o + e];
    s3 += gdq;
    s4 += gdq * xh[o + e];
    s5 += gq * dxh[o + e];
  }
  const float m_g = rms ? 0.f : warp_sum(s1) / d, m_gx = warp_sum(s2) / d, m_d = rms ? 0.f : warp_sum(s3) / d;
  const float m_dx = warp_sum(s4) / d, m_gdx = warp_sum(s5) / d;
  const float r = rr[row], dr = drr[row];
  for (int e = lane; e < d; e += 32) {
    const float gq = gy[o + e] * g[e];
    const float gdq = gdy[o + e] * g[e] + gy[o + e] * vg[e];
    const float base = gq - m_g - xh[o + e] * m_gx;
    const float a = gx[o + e] + r * base;
    const float b = gdx[o + e] + dr * r * base +
                    r * (gdq - m_d - dxh[o + e] * m_gx - xh[o + e] * (m_dx + m_gdx));
    gx[o + e] = a;
    gdx[o + e] = b;
    if (gxs) {
      gxs[o + e] = tf32_res(a);
      gdxs[o + e] = tf32_res(b);
    }
  }
}

// Column reductions over the T token rows (bias and LN-parameter Hv), two
// deterministic stages: stage 1 = CTA (32 columns x row group) folds its rows
// with 8 row-lanes per column and a fixed shared-memory tree; stage 2 sums the
// row-group partials in ascending order.
constexpr int kRowGroups = 64;

// mode 0: sum a ; mode 1: sum (gdy*xh + gy*dxh) and sum gdy (two outputs)
template <int MODE>
__global__ void k_colred1(const float* __restrict__ a, const float* __restrict__ b, const float* __restrict__ c,
                          const float* __restrict__ e, int T, int n, long long lda, float* __restrict__ part,
                          unsigned* __restrict__ cnt, float* __restrict__ out0, float* __restrict__ out1, int acc) {
  __shared__ float s0[8][33], s1[8][33];
  __shared__ bool last;
  const int col = blockIdx.x * 32 + (threadIdx.x & 31);
  const int rl = threadIdx.x >> 5;
  const int rows = (T + gridDim.y - 1) / gridDim.y;
  const int r0 = blockIdx.y * rows, r1 = min(T, r0 + rows);
  float x0 = 0.f, x1 = 0.f;
  if (col < n)
    for (int t = r0 + rl; t < r1; t += 8) {
      const long long o = (long long)t * lda + col;
      if (MODE == 0) {
        x0 += a[o];
      } else {  // a = gy, b = gdy, c = xh, e = dxh
        x0 += b[o] * c[o] + a[o] * e[o];
        x1 += b[o];
      }
    }
  s0[rl][threadIdx.x & 31] = x0;
  s1[rl][threadIdx.x & 31] = x1;
  __syncthreads();
  if (rl == 0 && col < n) {
    float t0 = 0.f, t1 = 0.f;
    for (int i = 0; i < 8; ++i) {
      t0 += s0[i][threadIdx.x];
      t1 += s1[i][threadIdx.x];
    }
    part[(long long)blockIdx.y * n + col] = t0;
    if (MODE == 1) part[(long long)(gridDim.y + blockIdx.y) * n + col] = t1;
  }
  // stage 2 in the last-arriving row-group block of this column slab: the
  // row-group partials summed in ascending order (deterministic), then the
  // slab's arrival counter is reset for the next reduction
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(&cnt[blockIdx.x], 1u) == gridDim.y - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  // all eight warps take part: warp w loads the partials of groups w, w + 8, ...
  // (independent loads in flight), then lane-column sums run in group order
  {
    const int groups = gridDim.y;
    __shared__ float pg[2][kRowGroups][33];
    for (int g = rl; g < groups; g += 8) {
      pg[0][g][threadIdx.x & 31] = col < n ? __ldcg(&part[(long long)g * n + col]) : 0.f;
      if (MODE == 1) pg[1][g][threadIdx.x & 31] = col < n ? __ldcg(&part[(long long)(groups + g) * n + col]) : 0.f;
    }
    __syncthreads();
    if (rl == 0 && col < n) {
      float t0 = 0.f, t1 = 0.f;
      for (int g = 0; g < groups; ++g) t0 += pg[0][g][threadIdx.x];
      out0[col] = acc ? out0[col] + t0 : t0;  // acc: micro-batch accumulation (pipeline stages)
      if (MODE == 1 && out1) {
        for (int g = 0; g < groups; ++g) t1 += pg[1][g][threadIdx.x];
        out1[col] = acc ? out1[col] + t1 : t1;
      }
    }
  }
  if (threadIdx.x == 0) cnt[blockIdx.x] = 0u;
}

// k_colred1 with 16-byte loads: a CTA covers 128 columns (lane = 4 adjacent
// columns) x 8 row-lanes, so each load instruction moves 4x the bytes. Every
// column is summed in exactly k_colred1's order (row-lane strided fold, the 8
// row-lanes in order, then the row groups in order). Stage 2 runs in the
// last-arriving CTA: thread t folds one (output, column) over the groups.
// Needs n % 4 == 0, lda % 4 == 0 and 16-byte aligned operands.
template <int MODE>
__global__ void __launch_bounds__(256) k_colred4(const float* __restrict__ a, const float* __restrict__ b,
                                                 const float* __restrict__ c, const float* __restrict__ e, int T,
                                                 int n, long long lda, float* __restrict__ part,
                                                 unsigned* __restrict__ cnt, float* __restrict__ out0,
                                                 float* __restrict__ out1, int acc) {
  pdl_wait();  // PDL: nothing global is touched before the previous kernel completes
  __shared__ float4 s0[8][32], s1[8][32];
  __shared__ bool last;
  const int lane = threadIdx.x & 31, rl = threadIdx.x >> 5;
  const int col = blockIdx.x * 128 + lane * 4;
  const int rows = (T + gridDim.y - 1) / gridDim.y;
  const int r0 = blockIdx.y * rows, r1 = min(T, r0 + rows);
  float4 x0 = make_float4(0.f, 0.f, 0.f, 0.f), x1 = x0;
  if (col < n)
    for (int t = r0 + rl; t < r1; t += 8) {
      const long long o = ((long long)t * lda + col) >> 2;
      if (MODE == 0) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(a) + o);
        x0.x += v.x, x0.y += v.y, x0.z += v.z, x0.w += v.w;
      } else {  // a = gy, b = gdy, c = xh, e = dxh
        const float4 va = __ldg(reinterpret_cast<const float4*>(a) + o), vb = __ldg(reinterpret_cast<const float4*>(b) + o);
        const float4 vc = __ldg(reinterpret_cast<const float4*>(c) + o), ve = __ldg(reinterpret_cast<const float4*>(e) + o);
        x0.x += vb.x * vc.x + va.x * ve.x, x1.x += vb.x;
        x0.y += vb.y * vc.y + va.y * ve.y, x1.y += vb.y;
        x0.z += vb.z * vc.z + va.z * ve.z, x1.z += vb.z;
        x0.w += vb.w * vc.w + va.w * ve.w, x1.w += vb.w;
      }
    }
  s0[rl][lane] = x0;
  s1[rl][lane] = x1;
  __syncthreads();
  if (rl == 0 && col < n) {
    float4 t0 = make_float4(0.f, 0.f, 0.f, 0.f), t1 = t0;
    for (int i = 0; i < 8; ++i) {
      const float4 u = s0[i][lane], w = s1[i][lane];
      t0.x += u.x, t0.y += u.y, t0.z += u.z, t0.w += u.w;
      t1.x += w.x, t1.y += w.y, t1.z += w.z, t1.w += w.w;
    }
    reinterpret_cast<float4*>(part + (long long)blockIdx.y * n)[col >> 2] = t0;
    if (MODE == 1) reinterpret_cast<float4*>(part + (long long)(gridDim.y + blockIdx.y) * n)[col >> 2] = t1;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(&cnt[blockIdx.x], 1u) == gridDim.y - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  const int groups = gridDim.y;
  const int which = threadIdx.x >> 7;  // 0: out0, 1: out1
  const int cc = blockIdx.x * 128 + (threadIdx.x & 127);
  if ((MODE == 1 || which == 0) && cc < n && (which == 0 || out1)) {
    const float* p = part + (long long)which * groups * n + cc;
    float t = 0.f;
#pragma unroll 8
    for (int g = 0; g < groups; ++g) t += __ldcg(p + (long long)g * n);
    float* o = which ? out1 : out0;
    o[cc] = acc ? o[cc] + t : t;  // acc: micro-batch accumulation (pipeline stages)
  }
  if (threadIdx.x == 0) cnt[blockIdx.x] = 0u;
}

// ------------------------------------------------------------------ GELU
__device__ __forceinline__ void gelu_derivs(float x, float& y, float& d1, float& d2) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  const float x2 = x * x;
  const float u = k0 * (x + k1 * x2 * x);
  const float du = k0 * (1.f + 3.f * k1 * x2);
  const float ddu = k0 * 6.f * k1 * x;
  const float t = tanhf(u);
  const float sech2 = 1.f - t * t;
  y = 0.5f * x * (1.f + t);
  d1 = 0.5f * (1.f + t) + 0.5f * x * sech2 * du;
  d2 = sech2 * du + 0.5f * x * (-2.f * t * sech2 * du * du + sech2 * ddu);
}

// u = gelu(f), du = gelu'(f) df (+ residuals for the next GEMM)
__global__ void k_gelu_fwd(const float* __restrict__ f, const float* __restrict__ df, float* __restrict__ u,
                           float* __restrict__ us, float* __restrict__ du, float* __restrict__ dus, long long n) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  float y, d1, d2;
  gelu_derivs(f[i], y, d1, d2);
  const float dy = d1 * df[i];
  u[i] = y;
  us[i] = tf32_res(y);
  du[i] = dy;
  dus[i] = tf32_res(dy);
}

// k_gelu_fwd on 16-byte vectors (4 elements per thread, the same per-element
// arithmetic): more bytes in flight per load instruction
__global__ void k_gelu_fwd4(const float4* __restrict__ f, const float4* __restrict__ df, float4* __restrict__ u,
                            float4* __restrict__ us, float4* __restrict__ du, float4* __restrict__ dus, long long n4) {
  pdl_wait();  // PDL: nothing global is touched before the previous kernel completes
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n4) return;
  const float4 fv = __ldg(f + i), dv = __ldg(df + i);
  float4 y, s, dy, ds;
  float d1, d2;
#define SD_GF4(c)                       \
  gelu_derivs(fv.c, y.c, d1, d2);       \
  dy.c = d1 * dv.c;                     \
  s.c = tf32_res(y.c), ds.c = tf32_res(dy.c);
  SD_GF4(x) SD_GF4(y) SD_GF4(z) SD_GF4(w)
#undef SD_GF4
  u[i] = y, us[i] = s, du[i] = dy, dus[i] = ds;
}

// gf = gu g'(f); gdf = gdu g'(f) + gu g''(f) df   (in place over gu, gdu)
__global__ void k_gelu_bwd(const float* __restrict__ f, const float* __restrict__ df, float* __restrict__ gu,
                           float* __restrict__ gdu, float* __restrict__ gus, float* __restrict__ gdus, long long n) {
  pdl_wait();  // PDL: nothing global is touched before the previous kernel completes
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  float y, d1, d2;
  gelu_derivs(f[i], y, d1, d2);
  const float a = gu[i], b = gdu[i];
  const float gf = a * d1;
  const float gdf = b * d1 + a * d2 * df[i];
  gu[i] = gf;
  gdu[i] = gdf;
  gus[i] = tf32_res(gf);
  gdus[i] = tf32_res(gdf);
}

// --------------------------------------------------------- attention softmax
// Row (z, i) of the per-head score matrix (already scaled), causal: columns
// j <= i. P = softmax, dP = P (dS - sum_j P dS); masked entries -> 0.
// Causal score products are tiled in 128-row blocks (sd_gemm.cu BM, causal
// modes 1-3): entries right of the diagonal but inside the diagonal tile are
// read (as zeros), entries beyond the tile never are -- so they are not written.
constexpr int kCausalTile = 128;

__global__ void k_attn_softmax_fwd(float* __restrict__ Sm, float* __restrict__ dS, float* __restrict__ Ps,
                                   float* __restrict__ dPs, int S, long long rows) {
  const long long row = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const int i = int(row % S);
  float* s = Sm + row * S;
  float* ds = dS + row * S;
  float m = -INFINITY;
  for (int j = lane; j <= i; j += 32) m = fmaxf(m, s[j]);
  m = warp_max(m);
  float z = 0.f, zd = 0.f;
  for (int j = lane; j <= i; j += 32) {
    const float e = __expf(s[j] - m);
    z += e;
    zd += e * ds[j];
  }
  z = warp_sum(z);
  zd = warp_sum(zd);
  const float inv = 1.f / z, mean_d = zd * inv;
  float* ps = Ps + row * S;
  float* dps = dPs + row * S;
  // the causal GEMMs read P only up to the end of the row's 128-row tile
  const int jend = min(S, (i / kCausalTile + 1) * kCausalTile);
  for (int j = lane; j < jend; j += 32) {
    float p = 0.f, dp = 0.f;
    if (j <= i) {
      p = __expf(s[j] - m) * inv;
      dp = p * (ds[j] - mean_d);
    }
    s[j] = p;
    ds[j] = dp;
    if (Ps) {  // residual arrays only for consumers without on-chip residuals
      ps[j] = tf32_res(p);
      dps[j] = tf32_res(dp);
    }
  }
}

// Register-resident forms for S = 128 NV <= 1024 (rows 16-byte aligned): lane
// l owns the float4 groups l, l + 32, ... of its row; a row is read once into
// registers (only the groups up to the causal end), exponentials are formed
// once, and the writes stop at the end of the row's 128-row tile.
template <int NV>
__global__ void __launch_bounds__(128) k_attn_softmax_fwd_reg(float* __restrict__ Sm, float* __restrict__ dS,
                                                              long long rows) {
  pdl_wait();  // PDL: nothing global is touched before the previous kernel completes
  constexpr int S = 128 * NV;
  const long long row = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const int i = int(row % S);
  float4* s4 = reinterpret_cast<float4*>(Sm + row * S);
  float4* d4 = reinterpret_cast<float4*>(dS + row * S);
  float4 sv[NV], dv[NV];
  float m = -INFINITY;
#pragma unroll
  for (int t = 0; t < NV; ++t) {
    const int j0 = 4 * (lane + 32 * t);
    if (j0 <= i) {
      sv[t] = s4[lane + 32 * t];
      dv[t] = d4[lane + 32 * t];
      m = fmaxf(m, sv[t].x);
      if (j0 + 1 <= i) m = fmaxf(m, sv[t].y);
      if (j0 + 2 <= i) m = fmaxf(m, sv[t].z);
      if (j0 + 3 <= i) m = fmaxf(m, sv[t].w);
    }
  }
  m = warp_max(m);
  float z = 0.f, zd = 0.f;
#pragma unroll
  for (int t = 0; t < NV; ++t) {
    const int j0 = 4 * (lane + 32 * t);
    if (j0 <= i) {
#define SD_SMX(f, o)                                   \
      {                                                \
        const float e = j0 + o <= i ? __expf(sv[t].f - m) : 0.f; \
        sv[t].f = e;                                   \
        z += e;                                        \
        zd += e * dv[t].f;                             \
      }
      SD_SMX(x, 0) SD_SMX(y, 1) SD_SMX(z, 2) SD_SMX(w, 3)
#undef SD_SMX
    }
  }
  z = warp_sum(z);
  zd = warp_sum(zd);
  const float inv = 1.f / z, mean_d = zd * inv;
  const int jend = min(S, (i / kCausalTile + 1) * kCausalTile);
#pragma unroll
  for (int t = 0; t < NV; ++t) {
    const int j0 = 4 * (lane + 32 * t);
    if (j0 < jend) {
      float4 p = make_float4(0.f, 0.f, 0.f, 0.f), dp = p;
      if (j0 <= i) {  // masked entries hold e = 0
        p = make_float4(sv[t].x * inv, sv[t].y * inv, sv[t].z * inv, sv[t].w * inv);
        dp = make_float4(p.x * (dv[t].x - mean_d), p.y * (dv[t].y - mean_d), p.z * (dv[t].z - mean_d),
                         p.w * (dv[t].w - mean_d));
        if (j0 + 1 > i) dp.y = 0.f;
        if (j0 + 2 > i) dp.z = 0.f;
        if (j0 + 3 > i) dp.w = 0.f;
      }
      s4[lane + 32 * t] = p;
      d4[lane + 32 * t] = dp;
    }
  }
}

template <int NV>
__global__ void __launch_bounds__(128) k_attn_softmax_bwd_reg(const float* __restrict__ P,
                                                              const float* __restrict__ dP, float* __restrict__ gP,
                                                              float* __restrict__ gdP, long long rows) {
  pdl_wait();  // PDL: nothing global is touched before the previous kernel completes
  constexpr int S = 128 * NV;
  const long long row = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const int i = int(row % S);
  const float4* p4 = reinterpret_cast<const float4*>(P + row * S);
  const float4* dp4 = reinterpret_cast<const float4*>(dP + row * S);
  float4* g4 = reinterpret_cast<float4*>(gP + row * S);
  float4* gd4 = reinterpret_cast<float4*>(gdP + row * S);
  float4 pv[NV], dpv[NV], gv[NV], gdv[NV];
  float c = 0.f, dc = 0.f;
#pragma unroll
  for (int t = 0; t < NV; ++t) {
    const int j0 = 4 * (lane + 32 * t);
    if (j0 <= i) {  // P, dP are zero past the diagonal (written so by the forward)
      pv[t] = p4[lane + 32 * t], dpv[t] = dp4[lane + 32 * t];
      gv[t] = g4[lane + 32 * t], gdv[t] = gd4[lane + 32 * t];
#define SD_SMB(f)                                              \
      c += pv[t].f * gv[t].f;                                  \
      dc += dpv[t].f * gv[t].f + pv[t].f * gdv[t].f;
      SD_SMB(x) SD_SMB(y) SD_SMB(z) SD_SMB(w)
#undef SD_SMB
    }
  }
  c = warp_sum(c);
  dc = warp_sum(dc);
  const int jend = min(S, (i / kCausalTile + 1) * kCausalTile);
#pragma unroll
  for (int t = 0; t < NV; ++t) {
    const int j0 = 4 * (lane + 32 * t);
    if (j0 < jend) {
      float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a;
      if (j0 <= i) {
#define SD_SMB2(f)                                                                   \
        a.f = pv[t].f * (gv[t].f - c);                                               \
        b.f = dpv[t].f * (gv[t].f - c) + pv[t].f * (gdv[t].f - dc);
        SD_SMB2(x) SD_SMB2(y) SD_SMB2(z) SD_SMB2(w)
#undef SD_SMB2
      }
      g4[lane + 32 * t] = a;
      gd4[lane + 32 * t] = b;
    }
  }
}

// gS = P (gP - c), gdS = dP (gP - c) + P (gdP - dc),  c = sum P gP,
// dc = sum (dP gP + P gdP). In place over gP, gdP.
__global__ void k_attn_softmax_bwd(const float* __restrict__ P, const float* __restrict__ dP, float* __restrict__ gP,
                                   float* __restrict__ gdP, float* __restrict__ gPs, float* __restrict__ gdPs, int S,
                                   long long rows) {
  const long long row = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const int i = int(row % S);
  const long long o = row * S;
  float c = 0.f, dc = 0.f;
  for (int j = lane; j <= i; j += 32) {
    c += P[o + j] * gP[o + j];
    dc += dP[o + j] * gP[o + j] + P[o + j] * gdP[o + j];
  }
  c = warp_sum(c);
  dc = warp_sum(dc);
  const int jend = min(S, (i / kCausalTile + 1) * kCausalTile);
  for (int j = lane; j < jend; j += 32) {
    float a = 0.f, b = 0.f;
    if (j <= i) {
      const float gp = gP[o + j];
      a = P[o + j] * (gp - c);
      b = dP[o + j] * (gp - c) + P[o + j] * (gdP[o + j] - dc);
    }
    gP[o + j] = a;
    gdP[o + j] = b;
    if (gPs) {
      gPs[o + j] = tf32_res(a);
      gdPs[o + j] = tf32_res(b);
    }
  }
}

// --------------------------------------------------------- cross-entropy
// Row t of the logits: p = softmax(z); loss_t = logsumexp(z) - z[y];
// gz = (p - onehot(y)) * scale; gdz = p (dz - sum p dz) * scale. In place.
__global__ void __launch_bounds__(256) k_ce(float* __restrict__ z, float* __restrict__ dz, float* __restrict__ zs,
                                            float* __restrict__ dzs, const int* __restrict__ tgt, int V, long long ld,
                                            float scale, double* __restrict__ loss_rows) {
  __shared__ float rm[8], rs[8], rsd[8];
  const long long t = blockIdx.x;
  float* zr = z + t * ld;
  float* dzr = dz + t * ld;
  // one streaming pass for max, sum e^(z-m) and sum e^(z-m) dz (online
  // rescaling), then the write pass: the row is read twice, not three times
  float m = -INFINITY, s = 0.f, sd = 0.f;
  for (int j = threadIdx.x; j < V; j += 256) {
    const float zj = zr[j], dj = dzr[j];
    if (zj > m) {
      const float c = __expf(m - zj);
      s *= c;
      sd *= c;
      m = zj;
    }
    const float e = __expf(zj - m);
    s += e;
    sd += e * dj;
  }
  // warp then block combine of (m, s, sd)
  for (int o = 16; o > 0; o >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, m, o), s2 = __shfl_xor_sync(0xffffffffu, s, o),
                sd2 = __shfl_xor_sync(0xffffffffu, sd, o);
    const float mn = fmaxf(m, m2);
    const float c1 = m == -INFINITY ? 0.f : __expf(m - mn), c2 = m2 == -INFINITY ? 0.f : __expf(m2 - mn);
    s = s * c1 + s2 * c2;
    sd = sd * c1 + sd2 * c2;
    m = mn;
  }
  if ((threadIdx.x & 31) == 0) rm[threadIdx.x >> 5] = m, rs[threadIdx.x >> 5] = s, rsd[threadIdx.x >> 5] = sd;
  __syncthreads();
  m = rm[0];
  for (int w = 1; w < 8; ++w) m = fmaxf(m, rm[w]);
  s = 0.f, sd = 0.f;
  for (int w = 0; w < 8; ++w) {
    const float c = rm[w] == -INFINITY ? 0.f : __expf(rm[w] - m);
    s += rs[w] * c;
    sd += rsd[w] * c;
  }
  const float inv = 1.f / s, md = sd * inv;
  const int y = tgt[t];
  if (threadIdx.x == 0) loss_rows[t] = double(logf(s) + m - zr[y]);
  __syncthreads();
  for (int j = threadIdx.x; j < V; j += 256) {
    const float p = __expf(zr[j] - m) * inv;
    const float g = (p - (j == y ? 1.f : 0.f)) * scale;
    const float gd = p * (dzr[j] - md) * scale;
    zr[j] = g;
    dzr[j] = gd;
    zs[t * ld + j] = tf32_res(g);
    dzs[t * ld + j] = tf32_res(gd);
  }
}

// ------------------------------------------------------------------ RoPE
// Pair (i, i + dh/2) of every q and k head at position p = t % S rotates by
// p * base^(-2i/dh) (rotate-half convention); f64 angle and rotation, one
// rounding per stored value. inverse: the transpose (backward adjoint).
__global__ void k_rope(float* __restrict__ a, float* __restrict__ as, float* __restrict__ da, float* __restrict__ das,
                       int T, int S, int d, int dh, float base, int inverse) {
  const int half = dh / 2;
  const long long n = (long long)T * 2 * (d / 2);  // (t, q|k, head, i) pairs
  const long long id = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (id >= n) return;
  const int per_t = d;                             // 2 parts x H heads x half pairs = d
  const long long t = id / per_t;
  const int rem = int(id % per_t);
  const int part = rem / (d / 2), hp = rem % (d / 2);
  const int h = hp / half, i = hp % half;
  const int p = int(t % S);
  const double theta = pow(double(base), -2.0 * double(i) / double(dh));
  double sn, cs;
  sincos(double(p) * theta, &sn, &cs);
  if (inverse) sn = -sn;
  const long long o = t * 3LL * d + (long long)part * d + (long long)h * dh + i;
  const double x1 = a[o], x2 = a[o + half];
  const float y1 = float(x1 * cs - x2 * sn), y2 = float(x2 * cs + x1 * sn);
  a[o] = y1;
  a[o + half] = y2;
  if (as) as[o] = tf32_res(y1), as[o + half] = tf32_res(y2);
  const double u1 = da[o], u2 = da[o + half];
  const float w1 = float(u1 * cs - u2 * sn), w2 = float(u2 * cs + u1 * sn);
  da[o] = w1;
  da[o + half] = w2;
  if (das) das[o] = tf32_res(w1), das[o + half] = tf32_res(w2);
}

// ------------------------------------------------- grouped-query attention
__global__ void k_gqa_expand(const float* __restrict__ raw, const float* __restrict__ raws,
                             const float* __restrict__ draw, const float* __restrict__ draws, float* __restrict__ a,
                             float* __restrict__ as, float* __restrict__ da, float* __restrict__ das, int d, int dh,
                             int KV, int H, long long n) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int W = d + 2 * KV * dh;
  const long long t = i / (3LL * d);
  const int col = int(i % (3LL * d));
  int src;
  if (col < d) {
    src = col;
  } else {
    const int part = (col - d) / d, c2 = (col - d) % d;  // 0: k, 1: v
    const int h = c2 / dh, e = c2 % dh, kv = h / (H / KV);
    src = d + part * KV * dh + kv * dh + e;
  }
  const long long o = t * W + src;
  a[i] = raw[o], as[i] = raws[o], da[i] = draw[o], das[i] = draws[o];
}
__global__ void k_gqa_reduce(const float* __restrict__ ga, const float* __restrict__ gda, float* __restrict__ graw,
                             float* __restrict__ graws, float* __restrict__ gdraw, float* __restrict__ gdraws, int d,
                             int dh, int KV, int H, long long n) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int W = d + 2 * KV * dh, G = H / KV;
  const long long t = i / W;
  const int col = int(i % W);
  const float* gr = ga + t * 3LL * d;
  const float* gdr = gda + t * 3LL * d;
  float a, b;
  if (col < d) {
    a = gr[col], b = gdr[col];
  } else {
    const int part = (col - d) / (KV * dh), c2 = (col - d) % (KV * dh);
    const int kv = c2 / dh, e = c2 % dh;
    double sa = 0.0, sb = 0.0;  // the group's query heads in ascending order
    for (int g = 0; g < G; ++g) {
      const int mc = d + part * d + (kv * G + g) * dh + e;
      sa += gr[mc], sb += gdr[mc];
    }
    a = float(sa), b = float(sb);
  }
  graw[i] = a, graws[i] = tf32_res(a);
  gdraw[i] = b, gdraws[i] = tf32_res(b);
}

// --------------------------------------------------------------- SwiGLU
// s = silu(f) = f sig(f); s1 = silu'(f); s2 = silu''(f); a = s u.
__device__ __forceinline__ void silu_derivs(double f, double& s, double& s1, double& s2) {
  const double sg = 1.0 / (1.0 + exp(-f));
  s = f * sg;
  s1 = sg * (1.0 + f * (1.0 - sg));
  s2 = sg * (1.0 - sg) * (2.0 + f * (1.0 - 2.0 * sg));
}
__global__ void k_swiglu_fwd(const float* __restrict__ fu, const float* __restrict__ dfu, float* __restrict__ a,
                             float* __restrict__ as, float* __restrict__ da, float* __restrict__ das, int ff,
                             long long n) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const long long t = i / ff;
  const int e = int(i % ff);
  const long long og = t * 2LL * ff + e, ou = og + ff;
  double s, s1, s2;
  silu_derivs(fu[og], s, s1, s2);
  const double u = fu[ou];
  const float av = float(s * u);
  const float dv = float(s1 * double(dfu[og]) * u + s * double(dfu[ou]));
  a[i] = av, as[i] = tf32_res(av);
  da[i] = dv, das[i] = tf32_res(dv);
}
//   g_up = ga s ; g_gate = ga u s1
//   gd_up = gda s + ga s1 df ; gd_gate = gda u s1 + ga du s1 + ga u s2 df
__global__ void k_swiglu_bwd(const float* __restrict__ fu, const float* __restrict__ dfu, const float* __restrict__ ga,
                             const float* __restrict__ gda, float* __restrict__ gfu, float* __restrict__ gfus,
                             float* __restrict__ gdfu, float* __restrict__ gdfus, int ff, long long n) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const long long t = i / ff;
  const int e = int(i % ff);
  const long long og = t * 2LL * ff + e, ou = og + ff;
  double s, s1, s2;
  silu_derivs(fu[og], s, s1, s2);
  const double u = fu[ou], df = dfu[og], du = dfu[ou], g = ga[i], gd = gda[i];
  const float gu = float(g * s), gg = float(g * u * s1);
  const float gdu = float(gd * s + g * s1 * df);
  const float gdg = float(gd * u * s1 + g * du * s1 + g * u * s2 * df);
  gfu[og] = gg, gfu[ou] = gu;
  gfus[og] = tf32_res(gg), gfus[ou] = tf32_res(gu);
  gdfu[og] = gdg, gdfu[ou] = gdu;
  gdfus[og] = tf32_res(gdg), gdfus[ou] = tf32_res(gdu);
}

// ------------------------------------------------------ embedding backward
// Hv_wte[v] += sum over positions with token v of gdx (CSR by token, fixed
// order), one warp per (token, 32-column slab). Hv_wpe[s] = sum_b gdx[b,s].
__global__ void k_embed_bwd_wte(const int* __restrict__ uniq, const int* __restrict__ start,
                                const int* __restrict__ pos, const int* __restrict__ n_uniq_dev, int d,
                                const float* __restrict__ gdx, float* __restrict__ hv_wte) {
  const long long w = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  const int slabs = (d + 31) / 32;
  const int n_uniq = *n_uniq_dev;
  if (w >= (long long)n_uniq * slabs) return;
  const int u = int(w / slabs), slab = int(w % slabs);
  const int col = slab * 32 + lane;
  if (col >= d) return;
  float acc = 0.f;
  for (int p = start[u]; p < start[u + 1]; ++p) acc += gdx[(long long)pos[p] * d + col];
  float* dst = hv_wte + (long long)uniq[u] * d + col;
  *dst += acc;
}

__global__ void k_embed_bwd_wpe(const float* __restrict__ gdx, int B, int S, int d, float* __restrict__ hv_wpe,
                                int accumulate) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= (long long)S * d) return;
  const int s = int(i / d), e = int(i % d);
  float acc = 0.f;
  for (int b = 0; b < B; ++b) acc += gdx[((long long)b * S + s) * d + e];
  hv_wpe[i] = accumulate ? hv_wpe[i] + acc : acc;
}

__global__ void k_res(const float* __restrict__ x, float* __restrict__ xs, long long n) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) xs[i] = tf32_res(x[i]);
}
__global__ void k_res4(const float4* __restrict__ x, float4* __restrict__ xs, long long n4) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n4) return;
  const float4 v = __ldg(x + i);
  xs[i] = make_float4(tf32_res(v.x), tf32_res(v.y), tf32_res(v.z), tf32_res(v.w));
}

__global__ void k_fill(float* __restrict__ x, float v, long long n) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) x[i] = v;
}

// synthetic init theta[i] = base + scale * gaussian(seed, i) (float), per slot
__global__ void k_init_slot(float* __restrict__ th, long long off, long long n, uint64_t key, double base,
                            double scale, int bf16, long long th_base) {
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= n) return;
  const uint64_t i = uint64_t(off + e);  // global flat index (the counter): layout-invariant values
  double v = base;
  if (scale != 0.0) {
    const double u1 = __dadd_rn(__dmul_rn(double(keyed_counter_k(key, 2 * i) >> 11), 0x1p-53), 0x1p-54);
    const double u2 = __dadd_rn(__dmul_rn(double(keyed_counter_k(key, 2 * i + 1) >> 11), 0x1p-53), 0x1p-54);
    const double gsn = __dmul_rn(__dsqrt_rn(__dmul_rn(-2.0, log(u1))), cos(__dmul_rn(6.283185307179586, u2)));
    v = __dadd_rn(base, __dmul_rn(scale, gsn));
  }
  const float f = __double2float_rn(v);
  th[off + e - th_base] = bf16 ? __bfloat162float(__float2bfloat16_rn(f)) : f;  // bf16: the f32 value rounded RNE
}

// number of elements that are not bf16-valued (low 16 mantissa bits set)
__global__ void k_count_not_bf16(const float* __restrict__ x, long long n, unsigned long long* __restrict__ cnt) {
  unsigned long long c = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    c += (__float_as_uint(x[i]) & 0xFFFFu) != 0u;
  c = __reduce_add_sync(0xffffffffu, unsigned(c));
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(cnt, c);
}

// ------------------------------------------------------------- launchers
static unsigned g1(long long n, int t = 256) { return unsigned((n + t - 1) / t); }

void gpt_embed(const int* tok, int T, int S, int d, const float* wte, const float* wpe, const float* vwte,
               const float* vwpe, float* x, float* dx, cudaStream_t s) {
  const long long n = (long long)T * d;
  k_embed<<<g1(n), 256, 0, s>>>(tok, S, d, wte, wpe, vwte, vwpe, x, dx, n);
  SD_LAUNCHED("k_embed");
}

#define SD_LN_REG_CASES(X) X(2) X(4) X(6) X(8)
void gpt_ln_fwd(const LnArgs& a, cudaStream_t s) {
#define SD_LNF(NV)                                                                                                 \
  if (a.d == 128 * NV) {                                                                                           \
    launch_pdl(k_ln_fwd_reg<NV>, dim3(g1(a.T, 4)), dim3(128), 0, s, a.x, a.dx, a.g, a.b, a.vg, a.vb, a.T, a.eps, a.h, a.hs, a.dh, a.dhs, \
                                                a.xh, a.dxh, a.r, a.dr, a.rms);                                    \
    SD_LAUNCHED("k_ln_fwd_reg");                                                                                   \
    return;                                                                                                        \
  }
  SD_LN_REG_CASES(SD_LNF)
#undef SD_LNF
  k_ln_fwd<<<g1(a.T, 8), 256, 0, s>>>(a.x, a.dx, a.g, a.b, a.vg, a.vb, a.T, a.d, a.eps, a.h, a.hs, a.dh, a.dhs, a.xh,
                                      a.dxh, a.r, a.dr, a.rms);
  SD_LAUNCHED("k_ln_fwd");
}

// 16-byte path of the column reductions (k_colred4): n and lda multiples of 4,
// operands 16-byte aligned; SD_COLRED1=1 forces the scalar kernel (A/B)
static bool colred4_ok(int n, long long lda, std::initializer_list<const float*> ps) {
  static const bool off = [] {
    const char* e = std::getenv("SD_COLRED1");
    return e && e[0] == '1';
  }();
  if (off || (n & 3) || (lda & 3)) return false;
  for (const float* p : ps)
    if (reinterpret_cast<uintptr_t>(p) & 15) return false;
  return true;
}

void gpt_ln_bwd(const LnBwdArgs& a, cudaStream_t s) {
  bool done = false;
#define SD_LNB(NV)                                                                                                 \
  if (!done && a.d == 128 * NV) {                                                                                  \
    launch_pdl(k_ln_bwd_reg<NV>, dim3(g1(a.T, 8)), dim3(256), 0, s, a.gy, a.gdy, a.g, a.vg, a.xh, a.dxh, a.r, a.dr, a.T, a.gx, a.gdx,  \
                                                a.gxs, a.gdxs, a.rms);                                             \
    SD_LAUNCHED("k_ln_bwd_reg");                                                                                   \
    done = true;                                                                                                   \
  }
  SD_LN_REG_CASES(SD_LNB)
#undef SD_LNB
  if (!done) {
    k_ln_bwd<<<g1(a.T, 8), 256, 0, s>>>(a.gy, a.gdy, a.g, a.vg, a.xh, a.dxh, a.r, a.dr, a.T, a.d, a.gx, a.gdx, a.gxs,
                                        a.gdxs, a.rms);
    SD_LAUNCHED("k_ln_bwd");
  }
  const int groups = std::min(kRowGroups, std::max(1, a.T / 64));
  if (colred4_ok(a.d, a.d, {a.gy, a.gdy, a.xh, a.dxh})) {
    launch_pdl(k_colred4<1>, dim3(dim3(unsigned((a.d + 127) / 128), unsigned(groups))), dim3(256), 0, s, 
        a.gy, a.gdy, a.xh, a.dxh, a.T, a.d, a.d, a.scratch + kColredReserve, reinterpret_cast<unsigned*>(a.scratch),
        a.hv_g, a.hv_b, a.acc);
    SD_LAUNCHED("k_colred4");
    return;
  }
  k_colred1<1><<<dim3(unsigned((a.d + 31) / 32), unsigned(groups)), 256, 0, s>>>(
      a.gy, a.gdy, a.xh, a.dxh, a.T, a.d, a.d, a.scratch + kColredReserve, reinterpret_cast<unsigned*>(a.scratch),
      a.hv_g, a.hv_b, a.acc);
  SD_LAUNCHED("k_colred1");
}

void gpt_colsum(const float* a, int T, int n, long long lda, float* out, float* scratch, cudaStream_t s, int acc) {
  const int groups = std::min(kRowGroups, std::max(1, T / 64));
  if (colred4_ok(n, lda, {a})) {
    launch_pdl(k_colred4<0>, dim3(dim3(unsigned((n + 127) / 128), unsigned(groups))), dim3(256), 0, s, 
        a, nullptr, nullptr, nullptr, T, n, lda, scratch + kColredReserve, reinterpret_cast<unsigned*>(scratch), out,
        nullptr, acc);
    SD_LAUNCHED("k_colred4");
    return;
  }
  k_colred1<0><<<dim3(unsigned((n + 31) / 32), unsigned(groups)), 256, 0, s>>>(
      a, nullptr, nullptr, nullptr, T, n, lda, scratch + kColredReserve, reinterpret_cast<unsigned*>(scratch), out,
      nullptr, acc);
  SD_LAUNCHED("k_colred1");
}

void gpt_gelu_fwd(const float* f, const float* df, float* u, float* us, float* du, float* dus, long long n,
                  cudaStream_t s) {
  const bool v4 = n % 4 == 0 && ((reinterpret_cast<uintptr_t>(f) | reinterpret_cast<uintptr_t>(df) |
                                   reinterpret_cast<uintptr_t>(u) | reinterpret_cast<uintptr_t>(us) |
                                   reinterpret_cast<uintptr_t>(du) | reinterpret_cast<uintptr_t>(dus)) & 15) == 0;
  if (v4) {
    launch_pdl(k_gelu_fwd4, dim3(g1(n / 4)), dim3(256), 0, s, reinterpret_cast<const float4*>(f), reinterpret_cast<const float4*>(df),
                                          reinterpret_cast<float4*>(u), reinterpret_cast<float4*>(us),
                                          reinterpret_cast<float4*>(du), reinterpret_cast<float4*>(dus), n / 4);
    SD_LAUNCHED("k_gelu_fwd4");
    return;
  }
  k_gelu_fwd<<<g1(n), 256, 0, s>>>(f, df, u, us, du, dus, n);
  SD_LAUNCHED("k_gelu_fwd");
}

void gpt_gelu_bwd(const float* f, const float* df, float* gu, float* gdu, float* gus, float* gdus, long long n,
                  cudaStream_t s) {
  launch_pdl(k_gelu_bwd, dim3(g1(n)), dim3(256), 0, s, f, df, gu, gdu, gus, gdus, n);
  SD_LAUNCHED("k_gelu_bwd");
}

void gpt_attn_softmax_fwd(float* Sm, float* dS, float* Ps, float* dPs, int S, long long rows, cudaStream_t s) {
  if (!Ps && S % 128 == 0 && S <= 1024) {
    switch (S / 128) {
#define SD_SMF(NV)                                                                  \
  case NV:                                                                          \
    launch_pdl(k_attn_softmax_fwd_reg<NV>, dim3(g1(rows, 4)), dim3(128), 0, s, Sm, dS, rows);           \
    SD_LAUNCHED("k_attn_softmax_fwd_reg");                                          \
    return;
      SD_SMF(1) SD_SMF(2) SD_SMF(3) SD_SMF(4) SD_SMF(5) SD_SMF(6) SD_SMF(7) SD_SMF(8)
#undef SD_SMF
    }
  }
  k_attn_softmax_fwd<<<g1(rows, 8), 256, 0, s>>>(Sm, dS, Ps, dPs, S, rows);
  SD_LAUNCHED("k_attn_softmax_fwd");
}

void gpt_attn_softmax_bwd(const float* P, const float* dP, float* gP, float* gdP, float* gPs, float* gdPs, int S,
                          long long rows, cudaStream_t s) {
  if (!gPs && S % 128 == 0 && S <= 1024) {
    switch (S / 128) {
#define SD_SMBW(NV)                                                                 \
  case NV:                                                                          \
    launch_pdl(k_attn_softmax_bwd_reg<NV>, dim3(g1(rows, 4)), dim3(128), 0, s, P, dP, gP, gdP, rows);    \
    SD_LAUNCHED("k_attn_softmax_bwd_reg");                                          \
    return;
      SD_SMBW(1) SD_SMBW(2) SD_SMBW(3) SD_SMBW(4) SD_SMBW(5) SD_SMBW(6) SD_SMBW(7) SD_SMBW(8)
#undef SD_SMBW
    }
  }
  k_attn_softmax_bwd<<<g1(rows, 8), 256, 0, s>>>(P, dP, gP, gdP, gPs, gdPs, S, rows);
  SD_LAUNCHED("k_attn_softmax_bwd");
}

void gpt_ce(float* z, float* dz, float* zs, float* dzs, const int* tgt, int T, int V, long long ld, float scale,
            double* loss_rows, cudaStream_t s) {
  k_ce<<<unsigned(T), 256, 0, s>>>(z, dz, zs, dzs, tgt, V, ld, scale, loss_rows);
  SD_LAUNCHED("k_ce");
}

void gpt_embed_bwd(const int* uniq, const int* start, const int* pos, const int* n_uniq_dev, int B, int S, int d,
                   const float* gdx, float* hv_wte, float* hv_wpe, cudaStream_t s, int acc) {
  // one warp per (unique token, 32-column slab); the count of unique tokens
  // is device-resident (built by gpt_token_csr): size the grid for all T rows
  const long long warps = (long long)B * S * ((d + 31) / 32);
  if (warps > 0) {
    k_embed_bwd_wte<<<g1(warps, 8), 256, 0, s>>>(uniq, start, pos, n_uniq_dev, d, gdx, hv_wte);
    SD_LAUNCHED("k_embed_bwd_wte");
  }
  if (hv_wpe) {
    k_embed_bwd_wpe<<<g1((long long)S * d), 256, 0, s>>>(gdx, B, S, d, hv_wpe, acc);
    SD_LAUNCHED("k_embed_bwd_wpe");
  }
}

// ---- token -> positions CSR of the deterministic embedding backward, built
// on the device from the uploaded tokens (sd_gpt_set_batch): per micro-batch
// the distinct tokens in ascending order (uniq), the start of each one's run
// of positions (ustart, + T at n), the positions sorted stably by token
// (upos), and the distinct-token count (nuniq). One stable radix sort of the
// composite key m * V + token over all micro-batches, a head scan, a fill.
__global__ void k_csr_keys(const int* __restrict__ tok, int T, long long n, int V, int* __restrict__ keys,
                           int* __restrict__ vals) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int m = int(i / T);
  keys[i] = m * V + tok[i];
  vals[i] = int(i - (long long)m * T);
}
__global__ void k_csr_heads(const int* __restrict__ keys, int T, long long n, int* __restrict__ flag) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  flag[i] = (i % T == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
}
__global__ void k_csr_fill(const int* __restrict__ keys, const int* __restrict__ flag, const int* __restrict__ scan,
                           int T, long long n, int V, int* __restrict__ uniq, int* __restrict__ ustart,
                           int* __restrict__ nuniq) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int m = int(i / T), li = int(i - (long long)m * T);
  const long long seg = (long long)m * T;
  const int u = scan[i] - scan[seg];
  int* um = uniq + (long long)m * (T + 1);
  int* sm = ustart + (long long)m * (T + 1);
  if (flag[i]) {
    um[u] = keys[i] - m * V;
    sm[u] = li;
  }
  if (li == T - 1) {
    const int cnt = u + flag[i];
    nuniq[m] = cnt;
    sm[cnt] = T;
  }
}

size_t gpt_token_csr_scratch(int T, int M, int V) {
  const long long n = (long long)T * M;
  int end_bit = 1;
  while ((1LL << end_bit) < (long long)M * V) ++end_bit;
  size_t sort_bytes = 0, scan_bytes = 0;
  SD_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, (const int*)nullptr, (int*)nullptr,
                                          (const int*)nullptr, (int*)nullptr, int(n), 0, end_bit));
  SD_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, (const int*)nullptr, (int*)nullptr, int(n)));
  return size_t(n) * 5 * sizeof(int) + std::max(sort_bytes, scan_bytes) + 256;
}

void gpt_token_csr(const int* tok, int T, int M, int V, int* uniq, int* ustart, int* upos, int* nuniq,
                   void* scratch, size_t scratch_bytes, cudaStream_t s) {
  const long long n = (long long)T * M;
  int end_bit = 1;
  while ((1LL << end_bit) < (long long)M * V) ++end_bit;
  size_t sort_bytes = 0, scan_bytes = 0;
  SD_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, (const int*)nullptr, (int*)nullptr,
                                          (const int*)nullptr, (int*)nullptr, int(n), 0, end_bit, s));
  SD_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, (const int*)nullptr, (int*)nullptr, int(n), s));
  const size_t ints = size_t(n) * 5;  // keys, vals, keys_sorted, flag, scan
  if (scratch_bytes < ints * sizeof(int) + std::max(sort_bytes, scan_bytes) + 256)
    fail(SD_ARGUMENT_ERROR, "token CSR scratch too small");
  char* buf = static_cast<char*>(scratch);
  int* keys = reinterpret_cast<int*>(buf);
  int* vals = keys + n;
  int* ksorted = vals + n;
  int* flag = ksorted + n;
  int* scan = flag + n;
  void* temp = reinterpret_cast<void*>((reinterpret_cast<uintptr_t>(scan + n) + 255) & ~uintptr_t(255));
  k_csr_keys<<<g1(n), 256, 0, s>>>(tok, T, n, V, keys, vals);
  SD_LAUNCHED("k_csr_keys");
  SD_CUDA(cub::DeviceRadixSort::SortPairs(temp, sort_bytes, keys, ksorted, vals, upos, int(n), 0, end_bit, s));
  k_csr_heads<<<g1(n), 256, 0, s>>>(ksorted, T, n, flag);
  SD_LAUNCHED("k_csr_heads");
  SD_CUDA(cub::DeviceScan::ExclusiveSum(temp, scan_bytes, flag, scan, int(n), s));
  k_csr_fill<<<g1(n), 256, 0, s>>>(ksorted, flag, scan, T, n, V, uniq, ustart, nuniq);
  SD_LAUNCHED("k_csr_fill");
}

void llama_rope(float* a, float* as, float* da, float* das, int T, int S, int d, int dh, float base, int inverse,
                cudaStream_t s) {
  const long long n = (long long)T * d;
  k_rope<<<g1(n), 256, 0, s>>>(a, as, da, das, T, S, d, dh, base, inverse);
  SD_LAUNCHED("k_rope");
}

void llama_gqa_expand(const float* raw, const float* raws, const float* draw, const float* draws, float* a, float* as,
                      float* da, float* das, int T, int d, int dh, int KV, int H, cudaStream_t s) {
  const long long n = (long long)T * 3 * d;
  k_gqa_expand<<<g1(n), 256, 0, s>>>(raw, raws, draw, draws, a, as, da, das, d, dh, KV, H, n);
  SD_LAUNCHED("k_gqa_expand");
}

void llama_gqa_reduce(const float* ga, const float* gda, float* graw, float* graws, float* gdraw, float* gdraws, int T,
                      int d, int dh, int KV, int H, cudaStream_t s) {
  const long long n = (long long)T * (d + 2 * KV * dh);
  k_gqa_reduce<<<g1(n), 256, 0, s>>>(ga, gda, graw, graws, gdraw, gdraws, d, dh, KV, H, n);
  SD_LAUNCHED("k_gqa_reduce");
}

void llama_swiglu_fwd(const float* fu, const float* dfu, float* a, float* as, float* da, float* das, int T, int ff,
                      cudaStream_t s) {
  const long long n = (long long)T * ff;
  k_swiglu_fwd<<<g1(n), 256, 0, s>>>(fu, dfu, a, as, da, das, ff, n);
  SD_LAUNCHED("k_swiglu_fwd");
}

void llama_swiglu_bwd(const float* fu, const float* dfu, const float* ga, const float* gda, float* gfu, float* gfus,
                      float* gdfu, float* gdfus, int T, int ff, cudaStream_t s) {
  const long long n = (long long)T * ff;
  k_swiglu_bwd<<<g1(n), 256, 0, s>>>(fu, dfu, ga, gda, gfu, gfus, gdfu, gdfus, ff, n);
  SD_LAUNCHED("k_swiglu_bwd");
}

void gpt_residual(const float* x, float* xs, long long n, cudaStream_t s) {
  if (n <= 0) return;
  long long done = 0;
  if ((reinterpret_cast<uintptr_t>(x) & 15) == 0 && (reinterpret_cast<uintptr_t>(xs) & 15) == 0 && n >= 4) {
    const long long n4 = n / 4;
    k_res4<<<g1(n4), 256, 0, s>>>(reinterpret_cast<const float4*>(x), reinterpret_cast<float4*>(xs), n4);
    SD_LAUNCHED("k_res4");
    done = n4 * 4;
  }
  if (done < n) {
    k_res<<<g1(n - done), 256, 0, s>>>(x + done, xs + done, n - done);
    SD_LAUNCHED("k_res");
  }
}

void gpt_fill(float* x, float v, long long n, cudaStream_t s) {
  if (n <= 0) return;
  k_fill<<<g1(n), 256, 0, s>>>(x, v, n);
  SD_LAUNCHED("k_fill");
}

void gpt_init_slot(float* th, long long off, long long n, uint64_t seed, double base, double scale, cudaStream_t s,
                   bool bf16, long long th_base) {
  if (n <= 0) return;
  k_init_slot<<<g1(n), 256, 0, s>>>(th, off, n, mix64(seed), base, scale, bf16 ? 1 : 0, th_base);
  SD_LAUNCHED("k_init_slot");
}

unsigned long long gpt_count_not_bf16(const float* x, long long n, unsigned long long* scratch, cudaStream_t s) {
  SD_CUDA(cudaMemsetAsync(scratch, 0, sizeof(unsigned long long), s));
  if (n > 0) {
    k_count_not_bf16<<<unsigned(std::min<long long>(g1(n), 148 * 16)), 256, 0, s>>>(x, n, scratch);
    SD_LAUNCHED("k_count_not_bf16");
  }
  unsigned long long h = 0;
  SD_CUDA(cudaMemcpyAsync(&h, scratch, sizeof(h), cudaMemcpyDeviceToHost, s));
  SD_CUDA(cudaStreamSynchronize(s));
  return h;
}

}  // namespace sd

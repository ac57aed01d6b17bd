// Lanczos vector algebra on sm_100a: probe generation, ordered blocked dot
// partials, fused recurrence passes, classical Gram-Schmidt passes and the
// dense test operator. All floating-point work that the reference performs in
// f64 is done here in f64 with explicit _rn intrinsics (no FMA contraction),
// so every rounded element and every folded scalar is bit-identical to
// proj/src/sharded.cpp + proj/include/specden/reduction.hpp.
//
// Memory layout: a vector shard is one contiguous array (float or double);
// a Krylov basis is column-major, column i at Q + i*ldq. Reductions follow the
// reference's fixed 1024-element global grid: one thread folds one grid block
// serially (left fold from +0.0) after the block is staged through shared
// memory in 32-element chunks with coalesced 128 B loads.
#include <cuda_runtime.h>
#include <math.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <mutex>
#include <thread>
#include <vector>

#include "sd_common.cuh"

namespace sd {


// ------------------------------------------------------------------ probes
// draw_probe fill, proj/src/sharded.cpp:67-75 (normalisation composes later).
template <typename T>
__global__ void k_probe(T* x, uint64_t begin, uint64_t n, uint64_t key, int dist, uint64_t one_hot) {
  const uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (t >= n) return;
  const uint64_t i = begin + t;
  double v;
  if (dist == SD_RADEMACHER) {
    v = (keyed_counter_k(key, i) & 1ull) ? 1.0 : -1.0;
  } else if (dist == SD_ONE_HOT) {
    v = (i == one_hot) ? 1.0 : 0.0;
  } else {
    // SD_GAUSSIAN_DEVICE: Box-Muller on counters (2i, 2i+1), rng.hpp:37-41,
    // with CUDA's log/cos -- within 1-2 ulp of glibc's, not bitwise.
    // SD_GAUSSIAN itself is drawn on the host (gaussian_fill_host below).
    const double u1 = __dadd_rn(__dmul_rn(double(keyed_counter_k(key, 2 * i) >> 11), 0x1p-53), 0x1p-54);
    const double u2 = __dadd_rn(__dmul_rn(double(keyed_counter_k(key, 2 * i + 1) >> 11), 0x1p-53), 0x1p-54);
    const double two_pi = 6.283185307179586;  // 2.0 * std::numbers::pi (exact doubling)
    v = __dmul_rn(__dsqrt_rn(__dmul_rn(-2.0, log(u1))), cos(__dmul_rn(two_pi, u2)));
  }
  x[t] = round_to<T>(v);
}

// ------------------------------------------------- recurrence pass (fused)
// y = round(y + alpha*x) with alpha = -(*coef) (axpy, sharded.cpp:106-118),
// then the block folds of sum z[i]*y[i] (DOT=1) or y[i]*y[i] (DOT=2) over
// full grid blocks. One CTA = kUnits consecutive grid blocks; thread t folds
// block t. Elements are staged as [unit][33] tiles (conflict-free column walk).
// 16-byte vector view of T (float4 / double2) for streaming loads.
template <typename T>
struct V16;
template <>
struct V16<float> {
  using type = float4;
  static constexpr int W = 4;
};
template <>
struct V16<double> {
  using type = double2;
  static constexpr int W = 2;
};
template <typename T>
union VU {
  typename V16<T>::type v;
  T a[V16<T>::W];
};
__host__ __device__ __forceinline__ bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// One THREAD per full grid block: it streams its 1024 elements with 16 B
// loads (several in flight, unroll 4), applies the update element by element
// and continues the block's serial f64 fold in element order.
template <typename T, bool UPD, int DOT>
__global__ void __launch_bounds__(128) k_axpy_dot_units(const T* __restrict__ x, T* __restrict__ y,
                                                        const T* __restrict__ z, const double* coefp, uint64_t base,
                                                        uint64_t n_units, uint64_t local_end,
                                                        double* __restrict__ sums) {
  constexpr int W = V16<T>::W;
  using V = typename V16<T>::type;
  const uint64_t unit = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (unit >= n_units) return;
  const uint64_t e0 = base + unit * kBlock;
  const uint64_t n = (local_end - e0) < kBlock ? (local_end - e0) : kBlock;
  const double alpha = UPD ? -(*coefp) : 0.0;
  double acc = 0.0;
  T* yp = y + e0;
  const bool vec = n == kBlock && al16(yp) && (!UPD || al16(x + e0)) && (DOT != 1 || al16(z + e0));
  if (vec) {
#pragma unroll 4
    for (int i = 0; i < int(kBlock) / W; ++i) {
      VU<T> yv, xv, zv;
      yv.v = reinterpret_cast<const V*>(yp)[i];
      if (UPD) xv.v = __ldg(reinterpret_cast<const V*>(x + e0) + i);
      if (DOT == 1) zv.v = __ldg(reinterpret_cast<const V*>(z + e0) + i);
      if (UPD) {
#pragma unroll
        for (int k = 0; k < W; ++k) yv.a[k] = round_to<T>(__dadd_rn(double(yv.a[k]), __dmul_rn(alpha, double(xv.a[k]))));
        reinterpret_cast<V*>(yp)[i] = yv.v;
      }
      if (DOT != 0) {
#pragma unroll
        for (int k = 0; k < W; ++k) {
          const double a = double(yv.a[k]);
          acc = __dadd_rn(acc, __dmul_rn(DOT == 1 ? double(zv.a[k]) : a, a));
        }
      }
    }
  } else {
    for (uint64_t i = 0; i < n; ++i) {
      T yv = yp[i];
      if (UPD) {
        yv = round_to<T>(__dadd_rn(double(yv), __dmul_rn(alpha, double(x[e0 + i]))));
        yp[i] = yv;
      }
      if (DOT != 0) {
        const double a = double(yv);
        acc = __dadd_rn(acc, __dmul_rn(DOT == 1 ? double(z[e0 + i]) : a, a));
      }
    }
  }
  if (DOT != 0) sums[unit] = acc;
}

// Head/tail elements of a shard (straddled grid blocks): update and emit raw
// terms (reduction.hpp:60-69 "head"/"tail").
template <typename T, bool UPD, int DOT>
__global__ void k_axpy_dot_edges(const T* __restrict__ x, T* __restrict__ y, const T* __restrict__ z,
                                 const double* coefp, uint64_t n_head, uint64_t tail_begin, uint64_t n_tail,
                                 uint64_t tail_slot, double* __restrict__ partial) {
  const uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (t >= n_head + n_tail) return;
  const uint64_t li = t < n_head ? t : tail_begin + (t - n_head);
  const uint64_t slot = t < n_head ? t : tail_slot + (t - n_head);
  T yv = y[li];
  if (UPD) {
    yv = round_to<T>(__dadd_rn(double(yv), __dmul_rn(-(*coefp), double(x[li]))));
    y[li] = yv;
  }
  if (DOT == 1) partial[slot] = __dmul_rn(double(z[li]), double(yv));
  if (DOT == 2) partial[slot] = __dmul_rn(double(yv), double(yv));
}

// ------------------------------------------------------ Gram-Schmidt pass
// Reorthogonalisation runs as two kernels per pass: an element-parallel
// update (k_cgs_update) and a block-fold for the next pass's dots
// (k_cgs_dots_pairs for few columns, warp-staged k_cgs_dots for many).

// CGS update, element-parallel: every element applies the reference's j
// sequential axpys r = axpy(-c_i, q_i, r) (f64 product and sum, rounded to
// the storage type after each); 16 B vector loads of the j columns, several
// in flight per thread.
template <typename T>
__global__ void __launch_bounds__(256) k_cgs_update(const T* __restrict__ Q, uint64_t ldq, int j, T* __restrict__ r,
                                                    const double* __restrict__ coef, uint64_t n) {
  extern __shared__ double cs[];  // -coef[0..j)
  for (int i = threadIdx.x; i < j; i += blockDim.x) cs[i] = -coef[i];
  __syncthreads();
  constexpr int W = V16<T>::W;
  using V = typename V16<T>::type;
  const uint64_t e = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) * W;
  if (e >= n) return;
  if (e + W <= n && al16(r + e) && al16(Q + e) && ((ldq * sizeof(T)) & 15) == 0) {
    VU<T> rv;
    rv.v = *reinterpret_cast<const V*>(r + e);
    double v[W];
#pragma unroll
    for (int k = 0; k < W; ++k) v[k] = double(rv.a[k]);
#pragma unroll 4
    for (int i = 0; i < j; ++i) {
      VU<T> q;
      q.v = __ldg(reinterpret_cast<const V*>(Q + uint64_t(i) * ldq + e));
#pragma unroll
      for (int k = 0; k < W; ++k) v[k] = rround<T>((__dadd_rn(v[k], __dmul_rn(cs[i], double(q.a[k])))));
    }
#pragma unroll
    for (int k = 0; k < W; ++k) rv.a[k] = T(v[k]);
    *reinterpret_cast<V*>(r + e) = rv.v;
  } else {
    for (uint64_t m = e; m < n && m < e + W; ++m) {
      double v = double(r[m]);
      for (int i = 0; i < j; ++i) v = rround<T>((__dadd_rn(v, __dmul_rn(cs[i], double(Q[uint64_t(i) * ldq + m])))));
      r[m] = T(v);
    }
  }
}

// CGS dots for few columns (j < 24): one THREAD per (column, block) pair
// streams the column's 1024 block elements with 16 B loads and runs the
// serial f64 fold against r, staged once per block in shared memory.
template <typename T, int NB>
__global__ void __launch_bounds__(256) k_cgs_dots_pairs(const T* __restrict__ Q, uint64_t ldq, int j,
                                                        const T* __restrict__ r, uint64_t base, uint64_t n_units,
                                                        uint64_t local_end, uint64_t pstride, uint64_t head_n,
                                                        double* __restrict__ partials) {
  constexpr int W = V16<T>::W;
  using V = typename V16<T>::type;
  __shared__ __align__(16) T rs[NB][kBlock];
  const uint64_t u0 = uint64_t(blockIdx.x) * NB;
  for (int idx = threadIdx.x; idx < NB * int(kBlock); idx += blockDim.x) {
    const int b = idx / int(kBlock), o = idx % int(kBlock);
    const uint64_t e = base + (u0 + b) * kBlock + o;
    rs[b][o] = (u0 + b < n_units && e < local_end) ? r[e] : T(0);
  }
  __syncthreads();
  for (int p = threadIdx.x; p < NB * j; p += blockDim.x) {
    const int col = p % j, b = p / j;
    const uint64_t unit = u0 + b;
    if (unit >= n_units) continue;
    const uint64_t e0 = base + unit * kBlock;
    const uint64_t n = (local_end - e0) < kBlock ? (local_end - e0) : kBlock;
    const T* qp = Q + uint64_t(col) * ldq + e0;
    const T* rb = rs[b];
    double acc = 0.0;
    if (n == kBlock && al16(qp)) {
#pragma unroll 4
      for (int i = 0; i < int(kBlock) / W; ++i) {
        VU<T> q;
        q.v = __ldg(reinterpret_cast<const V*>(qp) + i);
#pragma unroll
        for (int k = 0; k < W; ++k) acc = __dadd_rn(acc, __dmul_rn(double(q.a[k]), double(rb[i * W + k])));
      }
    } else {
      for (uint64_t i = 0; i < n; ++i) acc = __dadd_rn(acc, __dmul_rn(double(qp[i]), double(rb[i])));
    }
    partials[uint64_t(col) * pstride + head_n + unit] = acc;
  }
}

// CGS dots over full grid blocks. One WARP per (block, group of 32 columns):
// per 32-element chunk the warp loads each column's chunk as one coalesced
// 128 B row into a per-warp [32][33] shared tile (no CTA barrier), then lane c
// continues the serial f64 fold of column c against the chunk of r.
template <typename T>
__global__ void __launch_bounds__(256) k_cgs_dots(const T* __restrict__ Q, uint64_t ldq, int j,
                                                  const T* __restrict__ r, uint64_t base, uint64_t n_units,
                                                  uint64_t local_end, uint64_t pstride, uint64_t head_n,
                                                  double* __restrict__ partials) {
  constexpr int WPC = sizeof(T) == 4 ? 8 : 4;  // warps per CTA (== blockDim.x / 32)
  __shared__ T tile[WPC][32][33];
  __shared__ T rbuf[WPC][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int groups = (j + 31) / 32;
  const uint64_t gw = uint64_t(blockIdx.x) * WPC + warp;
  const uint64_t unit = gw / groups;
  if (unit >= n_units) return;
  const int c0 = int(gw % groups) * 32;
  const int ncol = (j - c0) < 32 ? (j - c0) : 32;
  const uint64_t e0 = base + unit * kBlock;
  const uint64_t n = (local_end - e0) < kBlock ? (local_end - e0) : kBlock;
  const T* qb = Q + uint64_t(c0) * ldq + e0;
  T(*tl)[33] = tile[warp];
  double acc = 0.0;
  for (uint64_t off = 0; off < n; off += 32) {
    const int cnt = int((n - off) < 32 ? (n - off) : 32);
    const bool valid = lane < cnt;
    rbuf[warp][lane] = valid ? r[e0 + off + lane] : T(0);
#pragma unroll 8
    for (int c = 0; c < ncol; ++c) tl[c][lane] = valid ? __ldg(qb + uint64_t(c) * ldq + off + lane) : T(0);
    __syncwarp();
    if (lane < ncol) {
#pragma unroll 8
      for (int k = 0; k < cnt; ++k) acc = __dadd_rn(acc, __dmul_rn(double(tl[lane][k]), double(rbuf[warp][k])));
    }
    __syncwarp();
  }
  if (lane < ncol) partials[uint64_t(c0 + lane) * pstride + head_n + unit] = acc;
}

template <typename T, bool UPD, int MODE>
__global__ void k_cgs_edges(const T* __restrict__ Q, uint64_t ldq, int j, T* __restrict__ r,
                            const double* __restrict__ coef, uint64_t n_head, uint64_t tail_begin, uint64_t n_tail,
                            uint64_t tail_slot, uint64_t plen, double* __restrict__ partials) {
  const uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (t >= n_head + n_tail) return;
  const uint64_t li = t < n_head ? t : tail_begin + (t - n_head);
  const uint64_t slot = t < n_head ? t : tail_slot + (t - n_head);
  double v = double(r[li]);
  if (UPD) {
    for (int i = 0; i < j; ++i) v = rround<T>((__dadd_rn(v, __dmul_rn(-coef[i], double(Q[uint64_t(i) * ldq + li])))));
    r[li] = T(v);
  }
  if (MODE == 1)
    for (int i = 0; i < j; ++i) partials[uint64_t(i) * plen + slot] = __dmul_rn(double(Q[uint64_t(i) * ldq + li]), v);
  if (MODE == 2) partials[slot] = __dmul_rn(v, v);
}

// ------------------------------------------------------------- ordered fold
// combine_blocked (reduction.hpp:76-107) for m sequences at once: thread s
// folds sequence s across ranks in ascending rank order, resuming straddled
// grid blocks term by term. Partials are [rank][seq][plen_max].
struct RankTable {
  int n;
  uint64_t begin[64], end[64];
};
constexpr int kCombChunk = 2048;
__global__ void __launch_bounds__(256) k_combine(RankTable rt, uint64_t total, uint64_t m, uint64_t plen_max,
                                                 const double* __restrict__ partials, double* __restrict__ out,
                                                 int post_sqrt) {
  // One CTA per sequence: warps 1..7 stream the block sums into a shared
  // double buffer while thread 0 runs the (inherently serial) left fold.
  __shared__ double buf[2][kCombChunk];
  const uint64_t s = blockIdx.x;
  double closed = 0.0, open = 0.0;
  uint64_t at = 0;
  auto feed = [&](double t) {
    open = __dadd_rn(open, t);
    ++at;
    const uint64_t ge = ((at - 1) / kBlock + 1) * kBlock;
    if (at == (ge < total ? ge : total)) {
      closed = __dadd_rn(closed, open);
      open = 0.0;
    }
  };
  for (int rk = 0; rk < rt.n; ++rk) {
    const PartialShape ps = partial_shape(rt.begin[rk], rt.end[rk], total);
    const double* p = partials + (uint64_t(rk) * m + s) * plen_max;
    if (threadIdx.x == 0)
      for (uint64_t i = 0; i < ps.n_head; ++i) feed(p[i]);
    const double* sums = p + ps.n_head;
    const uint64_t nch = (ps.n_sums + kCombChunk - 1) / kCombChunk;
    // prologue: chunk 0
    for (uint64_t i = threadIdx.x; i < kCombChunk && i < ps.n_sums; i += blockDim.x) buf[0][i] = sums[i];
    __syncthreads();
    for (uint64_t c = 0; c < nch; ++c) {
      const uint64_t c0 = c * kCombChunk;
      const int len = int((ps.n_sums - c0) < uint64_t(kCombChunk) ? (ps.n_sums - c0) : kCombChunk);
      if (threadIdx.x == 0) {
        const double* b = buf[c & 1];
        int i = 0;
        for (; i + 8 <= len; i += 8) {
          double v[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) v[q] = b[i + q];
#pragma unroll
          for (int q = 0; q < 8; ++q) closed = __dadd_rn(closed, v[q]);
        }
        for (; i < len; ++i) closed = __dadd_rn(closed, b[i]);
      } else if (threadIdx.x >= 32 && c + 1 < nch) {
        const uint64_t n0 = c0 + kCombChunk;
        for (uint64_t i = threadIdx.x - 32; i < kCombChunk && n0 + i < ps.n_sums; i += blockDim.x - 32)
          buf[(c + 1) & 1][i] = sums[n0 + i];
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      at = ps.n_sums ? ((at + ps.n_sums * kBlock) < total ? at + ps.n_sums * kBlock : total) : at;
      const double* tail = sums + ps.n_sums;
      for (uint64_t t = 0; t < ps.n_tail; ++t) feed(tail[t]);
    }
  }
  if (threadIdx.x == 0) out[s] = post_sqrt ? __dsqrt_rn(closed) : closed;  // norm2 = sqrt(dot), sharded.cpp:102-104
}

// ------------------------------------------------------ elementwise kernels
template <typename T>
__global__ void k_axpy(const T* __restrict__ x, T* __restrict__ y, uint64_t n, const double* alphap, double sign) {
  const uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const double alpha = sign * (*alphap);
  y[i] = round_to<T>(__dadd_rn(double(y[i]), __dmul_rn(alpha, double(x[i]))));
}

// 16-byte vector forms of axpy / scale (one V16 group per thread; the
// reciprocal of scale is computed once per thread, not per element)
template <typename T>
__global__ void k_axpy_v(const T* __restrict__ x, T* __restrict__ y, uint64_t nv, const double* alphap, double sign) {
  using V = typename V16<T>::type;
  constexpr int W = V16<T>::W;
  const uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (i >= nv) return;
  const double alpha = sign * (*alphap);
  VU<T> yv, xv;
  yv.v = reinterpret_cast<const V*>(y)[i];
  xv.v = __ldg(reinterpret_cast<const V*>(x) + i);
#pragma unroll
  for (int k = 0; k < W; ++k) yv.a[k] = round_to<T>(__dadd_rn(double(yv.a[k]), __dmul_rn(alpha, double(xv.a[k]))));
  reinterpret_cast<V*>(y)[i] = yv.v;
}

template <typename T>
__global__ void k_scale_v(const T* __restrict__ x, T* __restrict__ out, uint64_t nv, const double* cp, int recip) {
  using V = typename V16<T>::type;
  constexpr int W = V16<T>::W;
  const uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (i >= nv) return;
  const double c = recip ? __ddiv_rn(1.0, *cp) : *cp;
  VU<T> xv;
  xv.v = __ldg(reinterpret_cast<const V*>(x) + i);
#pragma unroll
  for (int k = 0; k < W; ++k) xv.a[k] = round_to<T>(__dmul_rn(c, double(xv.a[k])));
  reinterpret_cast<V*>(out)[i] = xv.v;
}

template <typename T>
__global__ void k_scale(const T* __restrict__ x, T* __restrict__ out, uint64_t n, const double* cp, int recip) {
  const uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const double c = recip ? __ddiv_rn(1.0, *cp) : *cp;
  out[i] = round_to<T>(__dmul_rn(c, double(x[i])));
}

static unsigned grid_for(uint64_t n, unsigned threads) { return unsigned((n + threads - 1) / threads); }

template <typename T>
static void scale_t(const T* x, T* out, uint64_t n, const double* c, int recip, cudaStream_t s) {
  constexpr int W = V16<T>::W;
  uint64_t done = 0;
  if (al16(x) && al16(out) && n >= W) {
    const uint64_t nv = n / W;
    k_scale_v<T><<<grid_for(nv, 256), 256, 0, s>>>(x, out, nv, c, recip);
    SD_LAUNCHED("k_scale_v");
    done = nv * W;
  }
  if (done < n) {
    k_scale<T><<<grid_for(n - done, 256), 256, 0, s>>>(x + done, out + done, n - done, c, recip);
    SD_LAUNCHED("k_scale");
  }
}

template <typename T>
static void axpy_t(const T* x, T* y, uint64_t n, const double* alpha, double sign, cudaStream_t s) {
  constexpr int W = V16<T>::W;
  uint64_t done = 0;
  if (al16(x) && al16(y) && n >= W) {
    const uint64_t nv = n / W;
    k_axpy_v<T><<<grid_for(nv, 256), 256, 0, s>>>(x, y, nv, alpha, sign);
    SD_LAUNCHED("k_axpy_v");
    done = nv * W;
  }
  if (done < n) {
    k_axpy<T><<<grid_for(n - done, 256), 256, 0, s>>>(x + done, y + done, n - done, alpha, sign);
    SD_LAUNCHED("k_axpy");
  }
}


// dense_operator apply, operators.cpp:39-44: serial f64 fold over the full row.
template <typename T>
__global__ void k_dense_apply(const double* __restrict__ a, uint64_t n, const T* __restrict__ xf, T* __restrict__ y,
                              uint64_t row_begin, uint64_t row_end) {
  extern __shared__ double xs[];
  for (uint64_t k = threadIdx.x; k < n; k += blockDim.x) xs[k] = double(xf[k]);
  __syncthreads();
  const uint64_t i = row_begin + blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (i >= row_end) return;
  const double* row = a + i * n;
  double acc = 0.0;
  for (uint64_t k = 0; k < n; ++k) acc = __dadd_rn(acc, __dmul_rn(row[k], xs[k]));
  y[i - row_begin] = round_to<T>(acc);
}

// diagonal test operator: y = round(d*x), one rounding of the exact f64 product
template <typename T>
__global__ void k_diag_apply(const T* __restrict__ d, const T* __restrict__ x, T* __restrict__ y, uint64_t n) {
  const uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (i < n) y[i] = round_to<T>(__dmul_rn(double(d[i]), double(x[i])));
}

// ------------------------------------------------------------ launchers

template <typename T>
static void launch_axpy_dot(const void* x, void* y, const void* z, const double* coef, uint64_t begin, uint64_t end,
                            uint64_t total, double* partial, cudaStream_t s) {
  const PartialShape ps = partial_shape(begin, end, total);
  const uint64_t local_end = end - begin;
  const uint64_t tail_begin = ps.n_head + ps.n_sums * kBlock;
  const bool upd = x != nullptr;
  const int dot = partial == nullptr ? 0 : (z == nullptr ? 2 : 1);
  auto run = [&](auto upd_c, auto dot_c) {
    constexpr bool U = decltype(upd_c)::value;
    constexpr int D = decltype(dot_c)::value;
    if (ps.n_sums) {
      const unsigned g = unsigned((ps.n_sums + 127) / 128);
      k_axpy_dot_units<T, U, D><<<g, 128, 0, s>>>((const T*)x, (T*)y, (const T*)z, coef, ps.n_head, ps.n_sums,
                                                       local_end, partial ? partial + ps.n_head : nullptr);
      SD_LAUNCHED("k_axpy_dot_units");
    }
    if (ps.n_head + ps.n_tail) {
      k_axpy_dot_edges<T, U, D><<<grid_for(ps.n_head + ps.n_tail, 256), 256, 0, s>>>(
          (const T*)x, (T*)y, (const T*)z, coef, ps.n_head, tail_begin, ps.n_tail, ps.n_head + ps.n_sums, partial);
      SD_LAUNCHED("k_axpy_dot_edges");
    }
  };
  using TT = std::true_type;
  using FF = std::false_type;
  using D0 = std::integral_constant<int, 0>;
  using D1 = std::integral_constant<int, 1>;
  using D2 = std::integral_constant<int, 2>;
  if (upd) {
    if (dot == 0) {
      // update only: element-parallel (no block folds to keep in order)
      if (local_end) {
        axpy_t<T>((const T*)x, (T*)y, local_end, coef, -1.0, s);
      }
    } else if (dot == 1) run(TT{}, D1{});
    else run(TT{}, D2{});
  } else {
    if (dot == 0) fail(SD_ARGUMENT_ERROR, "axpy_dot with neither update nor dot");
    else if (dot == 1) run(FF{}, D1{});
    else run(FF{}, D2{});
  }
}

__device__ __forceinline__ double to_d_alu(float x) { return widen_f32(x); }
__device__ __forceinline__ double to_d_alu(double x) { return x; }

// Fused Gram-Schmidt pass over full grid blocks: one CTA per 1024-element
// block, walked in CH-element chunks that are double-buffered in shared
// memory with cp.async (one HBM read of the j basis columns per pass):
//   UPD : r[e] = axpy(-c_{j-1}, q_{j-1}, ... axpy(-c_0, q_0, r))[e]  (thread = element)
//   dots: continue the serial f64 fold of q_i . r_new (thread = column i)
// Same arithmetic and fold order as k_cgs_update + k_cgs_dots.
constexpr int kCgsChunk = 64;
constexpr int kCgsMaxCols = 2 * 128;  // columns per CTA (acc[2] per thread)

template <typename T>
struct CgsSmem {
  static constexpr int PAD = 16 / sizeof(T);  // row stride = CH + PAD: 16 B rows, conflict-free column walks
  static constexpr int STRIDE = kCgsChunk + PAD;
  static size_t bytes(int j) {
    return size_t((j + 1) & ~1) * sizeof(double) + size_t(kCgsChunk) * sizeof(double) +
           2 * size_t(j) * STRIDE * sizeof(T);
  }
};

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}

template <typename T, bool UPD>
__global__ void __launch_bounds__(128) k_cgs_block(const T* __restrict__ Q, uint64_t ldq, int j, T* __restrict__ r,
                                                   const double* __restrict__ coef, uint64_t base, uint64_t local_end,
                                                   uint64_t pstride, uint64_t head_n, double* __restrict__ partials) {
  using V = typename V16<T>::type;
  constexpr int W = V16<T>::W, CH = kCgsChunk, STRIDE = CgsSmem<T>::STRIDE, NV = CH / W;
  extern __shared__ __align__(16) unsigned char sm_raw[];
  double* cs = reinterpret_cast<double*>(sm_raw);
  double* rt = cs + ((j + 1) & ~1);  // r chunk, widened once per element
  T* qbuf = reinterpret_cast<T*>(rt + CH);  // [2][j][STRIDE]
  const int tid = threadIdx.x;
  const uint64_t unit = blockIdx.x;
  const uint64_t e0 = base + unit * kBlock;
  const int n = int((local_end - e0) < kBlock ? (local_end - e0) : kBlock);
  const bool vec = n == int(kBlock) && ((reinterpret_cast<uintptr_t>(Q + e0) | (ldq * sizeof(T))) & 15) == 0;
  if (UPD)
    for (int i = tid; i < j; i += blockDim.x) cs[i] = -coef[i];
  auto stage = [&](int c0, T* dst) {
    if (vec) {
      for (int idx = tid; idx < j * NV; idx += blockDim.x) {
        const int i = idx / NV, v = idx % NV;
        cp_async16(dst + i * STRIDE + v * W, Q + uint64_t(i) * ldq + e0 + c0 + v * W);
      }
    } else {
      const int cnt = (n - c0) < CH ? (n - c0) : CH;
      for (int idx = tid; idx < j * CH; idx += blockDim.x) {
        const int i = idx / CH, e = idx % CH;
        if (e < cnt) dst[i * STRIDE + e] = Q[uint64_t(i) * ldq + e0 + c0 + e];
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  double acc0 = 0.0, acc1 = 0.0;
  stage(0, qbuf);
  for (int c0 = 0, it = 0; c0 < n; c0 += CH, ++it) {
    const int cnt = (n - c0) < CH ? (n - c0) : CH;
    T* qt = qbuf + (it & 1) * j * STRIDE;
    // prefetch the next chunk into the other buffer (its readers finished at
    // the previous iteration's trailing barrier)
    if (c0 + CH < n) {
      stage(c0 + CH, qbuf + ((it + 1) & 1) * j * STRIDE);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    if (tid < cnt) {
      T rv = r[e0 + c0 + tid];
      if (UPD) {
        double v = double(rv);
        // widening of the staged column entries on the integer pipe (the XU
        // pipe carries the f64 -> f32 rounding and the dot phase's widening)
        for (int i = 0; i < j; ++i) v = rround<T>((__dadd_rn(v, __dmul_rn(cs[i], to_d_alu(qt[i * STRIDE + tid])))));
        rv = T(v);
        r[e0 + c0 + tid] = rv;
        rt[tid] = v;
      } else {
        rt[tid] = double(rv);
      }
    }
    __syncthreads();
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int col = tid + 128 * h;
      if (col < j) {
        const T* qr = qt + col * STRIDE;
        double a = h ? acc1 : acc0;
        if (cnt == CH) {
#pragma unroll 4
          for (int e = 0; e < CH; e += W) {
            VU<T> q;
            q.v = *reinterpret_cast<const V*>(qr + e);
#pragma unroll
            for (int k = 0; k < W; ++k) a = __dadd_rn(a, __dmul_rn(double(q.a[k]), rt[e + k]));
          }
        } else {
          for (int e = 0; e < cnt; ++e) a = __dadd_rn(a, __dmul_rn(double(qr[e]), rt[e]));
        }
        if (h) acc1 = a;
        else acc0 = a;
      }
    }
    __syncthreads();  // rt and this buffer are free for the next iteration
  }
  if (tid < j) partials[uint64_t(tid) * pstride + head_n + unit] = acc0;
  if (tid + 128 < j) partials[uint64_t(tid + 128) * pstride + head_n + unit] = acc1;
}

static uint64_t fused_update_max_cols() {
  static const uint64_t v = [] {
    const char* e = std::getenv("SD_CGS_FUSED_UPDATE_MAX");
    return e ? uint64_t(std::strtoull(e, nullptr, 10)) : uint64_t(40);
  }();
  return v;
}

template <typename T>
static bool launch_cgs_fused(const void* Q, uint64_t ldq, uint64_t j, void* r, const double* coef, int mode,
                             const PartialShape& ps, uint64_t local_end, uint64_t plen, double* partials,
                             cudaStream_t s) {
  static const bool enabled = [] {
    const char* e = std::getenv("SD_CGS_FUSED");
    return !(e && e[0] == '0');
  }();
  constexpr size_t kMaxSmem = 100 * 1024;
  const size_t smem = CgsSmem<T>::bytes(int(j));
  if (!enabled || mode != 1 || j > uint64_t(kCgsMaxCols) || smem > kMaxSmem) return false;
  // the in-CTA update is a j-long dependent chain per element: beyond ~40
  // columns the element-parallel k_cgs_update followed by the block dots is
  // faster than the fused single read (measured in round 1; the tree mode, sd_lanczos_tree.cu, is the fast path)
  if (coef != nullptr && j >= fused_update_max_cols()) {
    constexpr int W = V16<T>::W;
    const uint64_t threads = (local_end + W - 1) / W;
    k_cgs_update<T><<<unsigned((threads + 255) / 256), 256, size_t(j) * sizeof(double), s>>>(
        (const T*)Q, ldq, int(j), (T*)r, coef, local_end);
    SD_LAUNCHED("k_cgs_update");
    coef = nullptr;
  }
  static const bool attr = [] {
    SD_CUDA(cudaFuncSetAttribute(k_cgs_block<T, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kMaxSmem)));
    SD_CUDA(cudaFuncSetAttribute(k_cgs_block<T, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kMaxSmem)));
    return true;
  }();
  (void)attr;
  const uint64_t tail_begin = ps.n_head + ps.n_sums * kBlock;
  const bool upd = coef != nullptr;
  if (ps.n_sums) {
    auto kern = upd ? k_cgs_block<T, true> : k_cgs_block<T, false>;
    kern<<<unsigned(ps.n_sums), 128, smem, s>>>((const T*)Q, ldq, int(j), (T*)r, coef, ps.n_head, local_end, plen,
                                                ps.n_head, partials);
    SD_LAUNCHED("k_cgs_block");
  }
  if (ps.n_head + ps.n_tail) {
    auto kern = upd ? k_cgs_edges<T, true, 1> : k_cgs_edges<T, false, 1>;
    kern<<<grid_for(ps.n_head + ps.n_tail, 128), 128, 0, s>>>((const T*)Q, ldq, int(j), (T*)r, coef, ps.n_head,
                                                              tail_begin, ps.n_tail, ps.n_head + ps.n_sums, plen,
                                                              partials);
    SD_LAUNCHED("k_cgs_edges");
  }
  return true;
}

template <typename T>
static void launch_cgs(const void* Q, uint64_t ldq, uint64_t j, void* r, const double* coef, int mode, uint64_t begin,
                       uint64_t end, uint64_t total, double* partials, uint64_t pstride, cudaStream_t s) {
  if (j == 0) return;
  const PartialShape ps = partial_shape(begin, end, total);
  const uint64_t local_end = end - begin, plen = pstride ? pstride : ps.len();
  const uint64_t tail_begin = ps.n_head + ps.n_sums * kBlock;
  const bool upd = coef != nullptr;
  if (!upd && mode == 0) fail(SD_ARGUMENT_ERROR, "cgs with neither update nor dots");
  if (launch_cgs_fused<T>(Q, ldq, j, r, coef, mode, ps, local_end, plen, partials, s)) return;
  // (1) the j sequential axpys, element-parallel and streaming
  if (upd) {
    constexpr int W = V16<T>::W;
    const uint64_t threads = (local_end + W - 1) / W;
    k_cgs_update<T><<<unsigned((threads + 255) / 256), 256, size_t(j) * sizeof(double), s>>>(
        (const T*)Q, ldq, int(j), (T*)r, coef, local_end);
    SD_LAUNCHED("k_cgs_update");
  }
  // (2) the dots against the updated r
  if (mode == 1) {
    if (ps.n_sums) {
      if (j < 24) {
        constexpr int NB = sizeof(T) == 4 ? 8 : 4;  // 32 KB of staged r
        k_cgs_dots_pairs<T, NB><<<unsigned((ps.n_sums + NB - 1) / NB), 256, 0, s>>>(
            (const T*)Q, ldq, int(j), (const T*)r, ps.n_head, ps.n_sums, local_end, plen, ps.n_head, partials);
      } else {
        const uint64_t warps = ps.n_sums * ((j + 31) / 32);
        constexpr unsigned WPC = sizeof(T) == 4 ? 8 : 4;
        k_cgs_dots<T><<<unsigned((warps + WPC - 1) / WPC), 32 * WPC, 0, s>>>(
            (const T*)Q, ldq, int(j), (const T*)r, ps.n_head, ps.n_sums, local_end, plen, ps.n_head, partials);
      }
      SD_LAUNCHED("k_cgs_dots");
    }
    if (ps.n_head + ps.n_tail) {
      k_cgs_edges<T, false, 1><<<grid_for(ps.n_head + ps.n_tail, 128), 128, 0, s>>>(
          (const T*)Q, ldq, int(j), (T*)r, nullptr, ps.n_head, tail_begin, ps.n_tail, ps.n_head + ps.n_sums, plen,
          partials);
      SD_LAUNCHED("k_cgs_edges");
    }
  } else if (mode == 2) {
    launch_axpy_dot<T>(nullptr, r, nullptr, nullptr, begin, end, total, partials, s);
  }
}

void combine_device(uint64_t nranks, const uint64_t* begins, const uint64_t* ends, uint64_t total, uint64_t m,
                    uint64_t plen_max, const double* partials, double* out, cudaStream_t s, int post_sqrt) {
  if (nranks == 0 || nranks > 64) fail(SD_ARGUMENT_ERROR, "combine: 1..64 ranks");
  RankTable rt;
  rt.n = int(nranks);
  uint64_t at = 0;
  for (uint64_t r = 0; r < nranks; ++r) {
    if (begins[r] != at) fail(SD_PROTOCOL_ERROR, "blocked partials are not contiguous in worker order");
    rt.begin[r] = begins[r];
    rt.end[r] = ends[r];
    at = ends[r];
  }
  if (at != total) fail(SD_PROTOCOL_ERROR, "blocked partials do not cover the vector");
  k_combine<<<unsigned(m), 256, 0, s>>>(rt, total, m, plen_max, partials, out, post_sqrt);
  SD_LAUNCHED("k_combine");
}

void axpy_dot(const void* x, void* y, const void* z, const double* coef, uint64_t begin, uint64_t end, uint64_t total,
              int prec, double* partial, cudaStream_t s) {
  if (prec == SD_F32) launch_axpy_dot<float>(x, y, z, coef, begin, end, total, partial, s);
  else launch_axpy_dot<double>(x, y, z, coef, begin, end, total, partial, s);
}

void cgs(const void* Q, uint64_t ldq, uint64_t j, void* r, const double* coef, int mode, uint64_t begin, uint64_t end,
         uint64_t total, int prec, double* partials, uint64_t pstride, cudaStream_t s) {
  if (prec == SD_F32) launch_cgs<float>(Q, ldq, j, r, coef, mode, begin, end, total, partials, pstride, s);
  else launch_cgs<double>(Q, ldq, j, r, coef, mode, begin, end, total, partials, pstride, s);
}

// Bit-exact Gaussian draws (rng.hpp:37-41). Box-Muller needs libm's log and
// cos, and the reference's values are glibc's, whose last ulp no device
// implementation reproduces (CUDA's differ for ~0.2% of draws; glibc is not
// correctly rounded either). So SD_GAUSSIAN probes are generated on the host
// with the reference's own expression -- the integer counter hash, the same
// libm calls, no FMA contraction (this file is built -ffp-contract=off) --
// by all host threads into two pinned staging chunks that are uploaded
// asynchronously while the next chunk is drawn. A one-time cost per probe
// (~0.1 s per 10^8 elements on 16 cores), not part of the Lanczos step.
namespace {
struct Staging {
  std::mutex m;
  void* buf[2] = {nullptr, nullptr};
  cudaEvent_t done[2] = {nullptr, nullptr};
  size_t bytes = 0;
};
Staging& staging() {
  static Staging st;
  return st;
}
inline double gaussian_host(uint64_t key, uint64_t i) {
  const double u1 = double(keyed_counter_k(key, 2 * i) >> 11) * 0x1p-53 + 0x1p-54;
  const double u2 = double(keyed_counter_k(key, 2 * i + 1) >> 11) * 0x1p-53 + 0x1p-54;
  constexpr double kTwoPi = 6.283185307179586;  // 2.0 * std::numbers::pi (exact doubling)
  return std::sqrt(-2.0 * std::log(u1)) * std::cos(kTwoPi * u2);
}
template <typename T>
void draw_range(T* out, uint64_t first, uint64_t n, uint64_t key) {
  for (uint64_t t = 0; t < n; ++t) out[t] = T(gaussian_host(key, first + t));  // round_elem
}
}  // namespace

static void gaussian_fill_host(void* x, uint64_t begin, uint64_t n, uint64_t seed, int prec, cudaStream_t s) {
  constexpr uint64_t kChunk = uint64_t(1) << 22;
  const size_t es = prec == SD_F32 ? 4 : 8;
  Staging& st = staging();
  std::lock_guard<std::mutex> lk(st.m);
  if (st.bytes < kChunk * es) {
    for (int b = 0; b < 2; ++b) {
      if (st.buf[b]) SD_CUDA(cudaFreeHost(st.buf[b]));
      SD_CUDA(cudaMallocHost(&st.buf[b], kChunk * es));
      if (!st.done[b]) SD_CUDA(cudaEventCreateWithFlags(&st.done[b], cudaEventDisableTiming));
    }
    st.bytes = kChunk * es;
  }
  const uint64_t key = mix64(seed);
  const unsigned nt = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  for (uint64_t c0 = 0, it = 0; c0 < n; c0 += kChunk, ++it) {
    const int b = int(it & 1);
    const uint64_t len = std::min(kChunk, n - c0);
    SD_CUDA(cudaEventSynchronize(st.done[b]));  // the buffer's previous upload has landed
    std::vector<std::thread> th;
    const uint64_t per = (len + nt - 1) / nt;
    for (unsigned t = 0; t < nt; ++t) {
      const uint64_t a = uint64_t(t) * per, e = std::min(len, a + per);
      if (a >= e) break;
      th.emplace_back([&, a, e] {
        if (prec == SD_F32) draw_range(static_cast<float*>(st.buf[b]) + a, begin + c0 + a, e - a, key);
        else draw_range(static_cast<double*>(st.buf[b]) + a, begin + c0 + a, e - a, key);
      });
    }
    for (auto& t : th) t.join();
    SD_CUDA(cudaMemcpyAsync(static_cast<char*>(x) + c0 * es, st.buf[b], len * es, cudaMemcpyHostToDevice, s));
    SD_CUDA(cudaEventRecord(st.done[b], s));
  }
  SD_CUDA(cudaStreamSynchronize(s));
}

void probe_fill(void* x, uint64_t begin, uint64_t end, uint64_t seed, int dist, uint64_t one_hot, int prec,
                cudaStream_t s) {
  const uint64_t n = end - begin;
  if (n == 0) return;
  if (dist != SD_GAUSSIAN && dist != SD_RADEMACHER && dist != SD_ONE_HOT && dist != SD_GAUSSIAN_DEVICE)
    fail(SD_CONFIG_ERROR, "unknown probe distribution");
  if (dist == SD_GAUSSIAN) {
    gaussian_fill_host(x, begin, n, seed, prec, s);
    return;
  }
  const uint64_t key = mix64(seed);
  if (prec == SD_F32) k_probe<float><<<grid_for(n, 256), 256, 0, s>>>((float*)x, begin, n, key, dist, one_hot);
  else k_probe<double><<<grid_for(n, 256), 256, 0, s>>>((double*)x, begin, n, key, dist, one_hot);
  SD_LAUNCHED("k_probe");
}

void scale(const void* x, void* out, uint64_t n, const double* c, int recip, int prec, cudaStream_t s) {
  if (n == 0) return;
  if (prec == SD_F32) scale_t((const float*)x, (float*)out, n, c, recip, s);
  else scale_t((const double*)x, (double*)out, n, c, recip, s);
}

void axpy(const void* x, void* y, uint64_t n, const double* alpha, double sign, int prec, cudaStream_t s) {
  if (n == 0) return;
  if (prec == SD_F32) axpy_t((const float*)x, (float*)y, n, alpha, sign, s);
  else axpy_t((const double*)x, (double*)y, n, alpha, sign, s);
}

void dense_apply(const double* a, uint64_t n, const void* xf, void* y, uint64_t rb, uint64_t re, int prec,
                 cudaStream_t s) {
  if (re <= rb) return;
  const size_t smem = size_t(n) * sizeof(double);
  if (prec == SD_F32)
    k_dense_apply<float><<<grid_for(re - rb, 128), 128, smem, s>>>(a, n, (const float*)xf, (float*)y, rb, re);
  else
    k_dense_apply<double><<<grid_for(re - rb, 128), 128, smem, s>>>(a, n, (const double*)xf, (double*)y, rb, re);
  SD_LAUNCHED("k_dense_apply");
}

void diag_apply(const void* d, const void* x, void* y, uint64_t n, int prec, cudaStream_t s) {
  if (n == 0) return;
  if (prec == SD_F32)
    k_diag_apply<float><<<grid_for(n, 256), 256, 0, s>>>((const float*)d, (const float*)x, (float*)y, n);
  else
    k_diag_apply<double><<<grid_for(n, 256), 256, 0, s>>>((const double*)d, (const double*)x, (double*)y, n);
  SD_LAUNCHED("k_diag_apply");
}

// ------------------------------------------------------ column statistics
// column_report (SPEC.md column_probe): strict threshold counts |x| < t_k and
// max |x| in one pass; then a histogram of |x| over [0, max] in `bins`
// uniform bins, bin = min(bins - 1, floor(|x| / max * bins)) in f64 (max == 0:
// everything in bin 0). Integer counts: layout-invariant and bit-exact.
constexpr int kMaxThr = 32;
template <typename T>
__global__ void __launch_bounds__(256) k_abs_stats(const T* __restrict__ x, uint64_t n, const double* __restrict__ thr,
                                                   int n_thr, unsigned long long* __restrict__ counts,
                                                   unsigned long long* __restrict__ max_bits) {
  __shared__ unsigned int sc[kMaxThr];
  __shared__ unsigned long long smax;
  if (threadIdx.x < kMaxThr) sc[threadIdx.x] = 0;
  if (threadIdx.x == 0) smax = 0;
  __syncthreads();
  unsigned int c[kMaxThr];
#pragma unroll
  for (int k = 0; k < kMaxThr; ++k) c[k] = 0;
  double m = 0.0;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
    const double a = fabs(double(x[i]));
    m = fmax(m, a);
#pragma unroll
    for (int k = 0; k < kMaxThr; ++k)
      if (k < n_thr && a < thr[k]) ++c[k];
  }
  for (int k = 0; k < n_thr; ++k) atomicAdd(&sc[k], c[k]);
  atomicMax(&smax, static_cast<unsigned long long>(__double_as_longlong(m)));
  __syncthreads();
  if (threadIdx.x < n_thr) atomicAdd(&counts[threadIdx.x], (unsigned long long)sc[threadIdx.x]);
  if (threadIdx.x == 0) atomicMax(max_bits, smax);
}

template <typename T>
__global__ void __launch_bounds__(256) k_abs_hist(const T* __restrict__ x, uint64_t n, double mx, int bins,
                                                  unsigned long long* __restrict__ counts) {
  extern __shared__ unsigned int sh[];
  for (int b = threadIdx.x; b < bins; b += blockDim.x) sh[b] = 0;
  __syncthreads();
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
    int b = 0;
    if (mx > 0.0) {
      const double t = floor(__dmul_rn(__ddiv_rn(fabs(double(x[i])), mx), double(bins)));
      b = t >= double(bins - 1) ? bins - 1 : int(t);
    }
    atomicAdd(&sh[b], 1u);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < bins; b += blockDim.x)
    if (sh[b]) atomicAdd(&counts[b], (unsigned long long)sh[b]);
}

unsigned stats_grid(uint64_t n) {
  const uint64_t g = (n + 255) / 256;
  return unsigned(g < 148 * 8 ? (g ? g : 1) : 148 * 8);
}

void abs_stats(const void* x, uint64_t n, int prec, const double* thr_host, int n_thr, uint64_t* counts_host,
               double* max_host, cudaStream_t s) {
  if (n_thr < 0 || n_thr > kMaxThr) fail(SD_ARGUMENT_ERROR, "column stats: 0..32 thresholds");
  void* buf = nullptr;
  const size_t bytes = sizeof(double) * kMaxThr + sizeof(unsigned long long) * (kMaxThr + 1);
  SD_CUDA(cudaMallocAsync(&buf, bytes, s));
  double* thr = static_cast<double*>(buf);
  auto* cnt = reinterpret_cast<unsigned long long*>(thr + kMaxThr);
  SD_CUDA(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long) * (kMaxThr + 1), s));
  if (n_thr) SD_CUDA(cudaMemcpyAsync(thr, thr_host, sizeof(double) * n_thr, cudaMemcpyHostToDevice, s));
  if (n) {
    if (prec == SD_F32)
      k_abs_stats<float><<<stats_grid(n), 256, 0, s>>>((const float*)x, n, thr, n_thr, cnt, cnt + kMaxThr);
    else
      k_abs_stats<double><<<stats_grid(n), 256, 0, s>>>((const double*)x, n, thr, n_thr, cnt, cnt + kMaxThr);
    SD_LAUNCHED("k_abs_stats");
  }
  unsigned long long h[kMaxThr + 1];
  SD_CUDA(cudaMemcpyAsync(h, cnt, sizeof(h), cudaMemcpyDeviceToHost, s));
  SD_CUDA(cudaFreeAsync(buf, s));
  SD_CUDA(cudaStreamSynchronize(s));
  for (int k = 0; k < n_thr; ++k) counts_host[k] = h[k];
  *max_host = __builtin_bit_cast(double, h[kMaxThr]);
}

void abs_hist(const void* x, uint64_t n, int prec, double mx, int bins, uint64_t* counts_host, cudaStream_t s) {
  if (bins < 1 || bins > 4096) fail(SD_ARGUMENT_ERROR, "column histogram: 1..4096 bins");
  if (!(mx >= 0.0) || !std::isfinite(mx)) fail(SD_ARGUMENT_ERROR, "column histogram: max must be finite");
  void* buf = nullptr;
  SD_CUDA(cudaMallocAsync(&buf, sizeof(unsigned long long) * bins, s));
  auto* cnt = static_cast<unsigned long long*>(buf);
  SD_CUDA(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long) * bins, s));
  if (n) {
    const size_t sm = sizeof(unsigned int) * bins;
    if (prec == SD_F32)
      k_abs_hist<float><<<stats_grid(n), 256, sm, s>>>((const float*)x, n, mx, bins, cnt);
    else
      k_abs_hist<double><<<stats_grid(n), 256, sm, s>>>((const double*)x, n, mx, bins, cnt);
    SD_LAUNCHED("k_abs_hist");
  }
  std::vector<unsigned long long> h(bins);
  SD_CUDA(cudaMemcpyAsync(h.data(), cnt, sizeof(unsigned long long) * bins, cudaMemcpyDeviceToHost, s));
  SD_CUDA(cudaFreeAsync(buf, s));
  SD_CUDA(cudaStreamSynchronize(s));
  for (int b = 0; b < bins; ++b) counts_host[b] = h[b];
}

}  // namespace sd

// ------------------------------------------------------------------ C-ABI
using namespace sd;

extern "C" {

sd_status sd_k_probe_fill(void* x, uint64_t begin, uint64_t end, uint64_t seed, int dist, uint64_t one_hot,
                          int prec, sd_stream s) {
  return guard([&] {
    if (end < begin) fail(SD_LAYOUT_ERROR, "probe range end < begin");
    probe_fill(x, begin, end, seed, dist, one_hot, prec, (cudaStream_t)s);
  });
}

sd_status sd_k_dot_partial(const void* a, const void* b, uint64_t begin, uint64_t end, uint64_t total, int prec,
                           double* partial, sd_stream s) {
  return guard([&] {
    // dot(a, b) partial: no update, terms b*a (commutative, exact in f64)
    axpy_dot(nullptr, const_cast<void*>(b), a, nullptr, begin, end, total, prec, partial, (cudaStream_t)s);
  });
}

sd_status sd_k_combine(uint64_t nranks, const uint64_t* begins, const uint64_t* ends, uint64_t total, uint64_t m,
                       const double* partials, double* out, sd_stream s) {
  return guard([&] {
    uint64_t plen_max = 0;
    for (uint64_t r = 0; r < nranks; ++r) {
      const uint64_t l = partial_shape(begins[r], ends[r], total).len();
      plen_max = l > plen_max ? l : plen_max;
    }
    combine_device(nranks, begins, ends, total, m, plen_max, partials, out, (cudaStream_t)s, 0);
  });
}

sd_status sd_k_axpy(const void* x, void* y, uint64_t n, const double* alpha_dev, double sign, int prec, sd_stream s) {
  return guard([&] { axpy(x, y, n, alpha_dev, sign, prec, (cudaStream_t)s); });
}

sd_status sd_k_scale(const void* x, void* out, uint64_t n, const double* c_dev, int reciprocal, int prec,
                     sd_stream s) {
  return guard([&] { scale(x, out, n, c_dev, reciprocal, prec, (cudaStream_t)s); });
}

sd_status sd_k_axpy_dot(const void* x, void* y, const void* z, const double* coef, uint64_t begin, uint64_t end,
                        uint64_t total, int prec, double* partial, sd_stream s) {
  return guard([&] { axpy_dot(x, y, z, coef, begin, end, total, prec, partial, (cudaStream_t)s); });
}

sd_status sd_k_cgs(const void* Q, uint64_t ldq, uint64_t j, void* r, const double* coef, int mode, uint64_t begin,
                   uint64_t end, uint64_t total, int prec, double* partials, sd_stream s) {
  return guard([&] { cgs(Q, ldq, j, r, coef, mode, begin, end, total, prec, partials, 0, (cudaStream_t)s); });
}

sd_status sd_k_abs_stats(const void* x, uint64_t n, int prec, const double* thresholds, int n_thresholds,
                         uint64_t* counts, double* max_abs, sd_stream s) {
  return guard([&] { abs_stats(x, n, prec, thresholds, n_thresholds, counts, max_abs, (cudaStream_t)s); });
}

sd_status sd_k_abs_histogram(const void* x, uint64_t n, int prec, double max_abs, int bins, uint64_t* counts,
                             sd_stream s) {
  return guard([&] { abs_hist(x, n, prec, max_abs, bins, counts, (cudaStream_t)s); });
}

sd_status sd_k_dense_apply(const double* a, uint64_t n, const void* x_full, void* y, uint64_t row_begin,
                           uint64_t row_end, int prec, sd_stream s) {
  return guard([&] { dense_apply(a, n, x_full, y, row_begin, row_end, prec, (cudaStream_t)s); });
}

}  // extern "C"

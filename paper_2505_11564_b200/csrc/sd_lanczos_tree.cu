// Tree-mode Lanczos passes (sd_lanczos_config.reduction = SD_REDUCE_TREE):
// the recurrence and full/selective reorthogonalisation as three fused,
// HBM-streaming GEMV passes over a TMA-staged Krylov basis, with the alpha /
// beta / Gram-Schmidt coefficient dots as warp-shuffle + block reductions in
// a fixed order (deterministic run to run; not the reference's 1024-block
// fold -- that is the ordered mode, which stays the parity mode).
//
// One step (j = stored columns, q_k and q_{k-1} among them):
//   pass 0: r' = r - beta_{k-1} q_{k-1}   (axpy semantics, one rounding)
//           c  = Q^T r'                   (alpha_k = c_k)
//   pass 1: r1 = r' - Q c                 (f64 accumulation, one rounding)
//           c' = Q^T r1
//   pass 2: r2 = r1 - Q c'; beta_k = ||r2||
// The first classical Gram-Schmidt pass against Q (which contains q_k)
// subsumes the reference's separate r -= alpha q_k: in exact
// arithmetic Q^T(r' - alpha q_k) = c - alpha e_k, so r' - alpha q_k - Q(c -
// alpha e_k) = r' - Q c; the difference is second order in the loss of
// orthogonality and is corrected by the second pass. Without reorthogonal-
// isation pass 0 runs over {q_{k-1}, q_k} and pass 2 over {q_k} alone
// (r -= alpha q_k; beta = ||r||). Per step that is 3 reads of the basis plus
// 3 read-writes of r: 4 P (3 j + 6) bytes, the algorithmic minimum of a
// two-pass classical Gram-Schmidt.
//
// Kernel shape: persistent, one 256-thread CTA per SM, tiles of TE elements x
// jb columns staged by one 2-D TMA box (plus the r tile) into an NS-deep
// mbarrier ring. Warp w owns a contiguous block of CPW columns; lane l owns
// EPL consecutive elements of the tile (16-byte shared loads). Update phase:
// each warp's partial sum over its columns, combined across the 8 warps in
// warp order, then one rounding to the storage type. Dot phase: per-lane f64
// accumulators per column across all of the CTA's tiles, warp-shuffle reduced
// at the end; the last CTA to finish folds the per-CTA sums in CTA order.
// f32 storage (measured: f32 -> f64 conversions of every staged element, on
// the 16-lane XU pipe or as integer widening, bounded the first version at
// 2.3-4.3 TB/s): the Gram-Schmidt update sums the small-coefficient columns
// in f32 (FFMA) and applies the dominant column -- q_k, whose coefficient is
// alpha in the first pass -- exactly in f64, then rounds once; the dots sum
// each lane's EPL exact-input products in f32 and accumulate those in f64
// across tiles. f64 storage runs everything in f64 (DFMA).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <string>
#include <vector>

#include "sd_common.cuh"

namespace sd {
namespace tree {

constexpr int kThreads = 256, kWarps = 8, kMaxCols = 256, kSMs = 148, kMaxPerSM = 2, kGrid = kSMs * kMaxPerSM;
constexpr uint64_t kChunk = uint64_t(1) << 30;  // elements per launch (TMA coordinates are int32)

struct Params {
  void* r;
  uint64_t n;          // elements of this launch's chunk
  int jb;              // columns in the box
  const double* coef;  // MODE 0: &beta (or null: no update); MODE 1/2: jb coefficients
  int ucol;            // MODE 0: column updated with -coef[0]
  int xcol;            // MODE 1/2, f32 storage: the dominant column, applied in f64 (-1: none)
  double* part;        // [parts][kMaxCols] per-CTA sums (this launch: rows part0 + blockIdx.x)
  int part0, nparts;   // first row of this launch, rows of the whole pass (final fold)
  unsigned* counter;   // CTAs finished over the whole pass (reset by the last one)
  unsigned expected;   // total CTAs of the pass
  double* out;         // jb (MODE 0/1) or 1 (MODE 2) results
  double* alpha_out;   // copy of out[alpha_col] (may be null)
  int alpha_col;
  int post_sqrt;
  int ntiles;
  int ns;              // ring depth
};

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

template <typename T>
__device__ __forceinline__ double xu_d(T v) {
  return double(v);  // F2F.F64.F32 (XU) for float
}
template <typename T>
__device__ __forceinline__ double alu_d(T v);
template <>
__device__ __forceinline__ double alu_d<float>(float v) {
  return widen_f32(v);
}
template <>
__device__ __forceinline__ double alu_d<double>(double v) {
  return v;
}

template <typename T, int EPL>
struct Vec;
template <>
struct Vec<float, 4> {
  using V = float4;
};
template <>
struct Vec<float, 2> {
  using V = float2;
};
template <>
struct Vec<double, 2> {
  using V = double2;
};
template <>
struct Vec<double, 1> {
  using V = double;
};
template <typename T, int EPL>
union VU {
  typename Vec<T, EPL>::V v;
  T a[EPL];
};

template <typename T, int MODE, int EPL, int CPW>
__global__ void __launch_bounds__(kThreads, 2) k_gs_tree(const __grid_constant__ CUtensorMap tq,
                                                         const __grid_constant__ CUtensorMap tr, Params p) {
  constexpr int TE = 32 * EPL;
  extern __shared__ __align__(128) unsigned char smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int jb = p.jb;
  const size_t stage_bytes = (size_t(jb + 1) * TE * sizeof(T) + 127) & ~size_t(127);
  unsigned char* ring = smem;
  double* sp = reinterpret_cast<double*>(ring + p.ns * stage_bytes);  // [kWarps][TE]
  double* rt = sp + kWarps * TE;                                        // [TE]
  double* cs = rt + TE;                                                 // [kMaxCols]
  double* red = cs + kMaxCols;                                          // [kWarps]
  float* spf = reinterpret_cast<float*>(sp);                            // f32 storage: [kWarps][TE]
  float* rtf = reinterpret_cast<float*>(rt);                            // f32 storage: [TE]
  float* cs32 = reinterpret_cast<float*>(cs + kMaxCols / 2);            // f32 storage: [kMaxCols]
  constexpr bool kF32 = sizeof(T) == 4;
  uint64_t* bar = reinterpret_cast<uint64_t*>(red + kWarps);            // [ns]
  int& s_last = *reinterpret_cast<int*>(bar + p.ns);

  const int G = gridDim.x;
  const int my_tiles = p.ntiles > int(blockIdx.x) ? (p.ntiles - int(blockIdx.x) + G - 1) / G : 0;
  const uint32_t tx = uint32_t(size_t(jb + 1) * TE * sizeof(T));
  if (tid == 0) {
    for (int s = 0; s < p.ns; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar + s)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (MODE != 0) {
    if (kF32) {
      for (int i = tid; i < jb; i += kThreads) cs32[i] = i == p.xcol ? 0.0f : float(p.coef[i]);
    } else {
      for (int i = tid; i < jb; i += kThreads) cs[i] = p.coef[i];
    }
  }
  const double xc = (MODE != 0 && p.xcol >= 0) ? p.coef[p.xcol] : 0.0;
  __syncthreads();
  auto issue = [&](int s, int tile) {
    unsigned char* dst = ring + s * stage_bytes;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar + s)), "r"(tx) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            su32(dst)),
        "l"(&tq), "r"(su32(bar + s)), "r"(tile * TE), "r"(0)
        : "memory");
    asm volatile(
        "cp.async.bulk.tensor.1d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3}], [%2];" ::"r"(
            su32(dst + size_t(jb) * TE * sizeof(T))),
        "l"(&tr), "r"(su32(bar + s)), "r"(tile * TE)
        : "memory");
  };
  if (tid == 0)
    for (int s = 0; s < p.ns && s < my_tiles; ++s) issue(s, int(blockIdx.x) + s * G);

  using V = typename Vec<T, EPL>::V;
  const int col0 = warp * CPW;
  double acc[CPW];
#pragma unroll
  for (int c = 0; c < CPW; ++c) acc[c] = 0.0;
  double nrm = 0.0;
  T* rg = static_cast<T*>(p.r);
  const double beta = (MODE == 0 && p.coef) ? -p.coef[0] : 0.0;

  for (int k = 0; k < my_tiles; ++k) {
    const int s = k % p.ns;
    const uint32_t parity = uint32_t(k / p.ns) & 1u;
    asm volatile(
        "{\n\t.reg .pred P1;\n\tW_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W_%=;\n\t}" ::"r"(su32(bar + s)),
        "r"(parity)
        : "memory");
    const T* qt = reinterpret_cast<const T*>(ring + s * stage_bytes);
    const T* rtile = qt + size_t(jb) * TE;
    const uint64_t e0 = uint64_t(int(blockIdx.x) + k * G) * TE;
    // ---- update phase
    if (MODE == 0) {
      if (tid < TE) {
        double v = double(rtile[tid]);
        if (p.coef) {
          v = rround<T>(__dadd_rn(v, __dmul_rn(beta, double(qt[p.ucol * TE + tid]))));  // axpy (sharded.cpp:106-118)
          if (e0 + tid < p.n) rg[e0 + tid] = T(v);
        }
        if constexpr (kF32) rtf[tid] = float(v);
        else rt[tid] = v;
      }
    } else if constexpr (kF32) {
      // f32 storage: the small Gram-Schmidt terms on the FP32 pipe (f32
      // coefficients, FFMA), the dominant column (q_k: alpha in the first
      // pass) exactly in f64, combined in f64 and rounded once to f32
      float S[EPL];
#pragma unroll
      for (int e = 0; e < EPL; ++e) S[e] = 0.0f;
#pragma unroll
      for (int c = 0; c < CPW; ++c) {
        const int col = col0 + c;
        if (col < jb) {
          VU<T, EPL> q;
          q.v = *reinterpret_cast<const V*>(qt + size_t(col) * TE + lane * EPL);
          const float cc = cs32[col];
#pragma unroll
          for (int e = 0; e < EPL; ++e) S[e] = fmaf(cc, q.a[e], S[e]);
        }
      }
#pragma unroll
      for (int e = 0; e < EPL; ++e) spf[warp * TE + lane * EPL + e] = S[e];
      __syncthreads();
      if (tid < TE) {
        double sum = p.xcol >= 0 ? xc * double(qt[p.xcol * TE + tid]) : 0.0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) sum += double(spf[w * TE + tid]);
        const float v = float(double(rtile[tid]) - sum);
        if (e0 + tid < p.n) rg[e0 + tid] = v;
        rtf[tid] = v;
        if (MODE == 2) nrm = fma(double(v), double(v), nrm);
      }
    } else {
      double S[EPL];
#pragma unroll
      for (int e = 0; e < EPL; ++e) S[e] = 0.0;
#pragma unroll
      for (int c = 0; c < CPW; ++c) {
        const int col = col0 + c;
        if (col < jb) {
          VU<T, EPL> q;
          q.v = *reinterpret_cast<const V*>(qt + size_t(col) * TE + lane * EPL);
          const double cc = cs[col];
#pragma unroll
          for (int e = 0; e < EPL; ++e) S[e] = fma(cc, double(q.a[e]), S[e]);
        }
      }
#pragma unroll
      for (int e = 0; e < EPL; ++e) sp[warp * TE + lane * EPL + e] = S[e];
      __syncthreads();
      if (tid < TE) {
        double sum = sp[tid];
#pragma unroll
        for (int w = 1; w < kWarps; ++w) sum += sp[w * TE + tid];
        const double v = double(rtile[tid]) - sum;
        if (e0 + tid < p.n) rg[e0 + tid] = T(v);
        rt[tid] = v;
        if (MODE == 2) nrm = fma(v, v, nrm);
      }
    }
    __syncthreads();
    // ---- dot phase: acc[c] += q_col . r_new over this lane's elements
    if constexpr (MODE != 2) {
      if constexpr (kF32) {
        // exact f32 inputs; the lane's EPL products summed on the FP32 pipe,
        // then accumulated in f64 across tiles (one conversion per EPL terms)
        VU<T, EPL> rv;
        rv.v = *reinterpret_cast<const V*>(rtf + lane * EPL);
#pragma unroll
        for (int c = 0; c < CPW; ++c) {
          const int col = col0 + c;
          if (col < jb) {
            VU<T, EPL> q;
            q.v = *reinterpret_cast<const V*>(qt + size_t(col) * TE + lane * EPL);
            float t = q.a[0] * rv.a[0];
#pragma unroll
            for (int e = 1; e < EPL; ++e) t = fmaf(q.a[e], rv.a[e], t);
            acc[c] += double(t);
          }
        }
      } else {
        double rv[EPL];
#pragma unroll
        for (int e = 0; e < EPL; ++e) rv[e] = rt[lane * EPL + e];
#pragma unroll
        for (int c = 0; c < CPW; ++c) {
          const int col = col0 + c;
          if (col < jb) {
            VU<T, EPL> q;
            q.v = *reinterpret_cast<const V*>(qt + size_t(col) * TE + lane * EPL);
#pragma unroll
            for (int e = 0; e < EPL; ++e) acc[c] = fma(double(q.a[e]), rv[e], acc[c]);
          }
        }
      }
    }
    __syncthreads();  // stage s and rt are free
    if (tid == 0 && k + p.ns < my_tiles) issue(s, int(blockIdx.x) + (k + p.ns) * G);
  }

  // ---- per-CTA sums (fixed shuffle pattern), then the last CTA folds them
  double* myrow = p.part + size_t(p.part0 + blockIdx.x) * kMaxCols;
  if (MODE != 2) {
#pragma unroll
    for (int c = 0; c < CPW; ++c) {
      double v = acc[c];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0 && col0 + c < jb) myrow[col0 + c] = v;
    }
  } else {
    double v = nrm;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[warp] = v;
    __syncthreads();
    if (tid == 0) {
      double t = red[0];
      for (int w = 1; w < kWarps; ++w) t += red[w];
      myrow[0] = t;
    }
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = atomicAdd(p.counter, 1u) == p.expected - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const int m = MODE == 2 ? 1 : jb;
  for (int col = tid; col < m; col += kThreads) {
    double t = 0.0;
    for (int g = 0; g < p.nparts; ++g) t += __ldcg(p.part + size_t(g) * kMaxCols + col);
    if (p.post_sqrt) t = __dsqrt_rn(t);
    p.out[col] = t;
    if (p.alpha_out && col == p.alpha_col) *p.alpha_out = t;
  }
  if (tid == 0) *p.counter = 0;
}

// rank-ordered fold of per-rank results: out[c] = sum_r recv[r][c] (r ascending)
__global__ void k_rank_fold(const double* __restrict__ recv, int nranks, int m, double* __restrict__ out,
                            int post_sqrt, double* alpha_out, int alpha_col) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= m) return;
  double t = recv[c];
  for (int r = 1; r < nranks; ++r) t += recv[size_t(r) * m + c];
  if (post_sqrt) t = __dsqrt_rn(t);
  out[c] = t;
  if (alpha_out && c == alpha_col) *alpha_out = t;
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeFn encoder() {
  static EncodeFn fn = [] {
    void* q = nullptr;
    cudaDriverEntryPointQueryResult r;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &q, cudaEnableDefault, &r) != cudaSuccess ||
        r != cudaDriverEntryPointSuccess)
      q = nullptr;
    return reinterpret_cast<EncodeFn>(q);
  }();
  if (!fn) fail(SD_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
  return fn;
}

struct Shape {
  int epl, ns, te;
};
// tile width and ring depth for jb columns: the widest tile whose ring of
// >= 2 stages fits ~200 KB of shared memory
template <typename T>
static Shape pick(int jb) {
  const int epl_max = sizeof(T) == 4 ? 4 : 2;
  for (int epl = epl_max; epl >= epl_max / 2; epl /= 2) {
    const int te = 32 * epl;
    const size_t stage = (size_t(jb + 1) * te * sizeof(T) + 127) & ~size_t(127);
    const size_t fixed = sizeof(double) * (kWarps * te + te + kMaxCols + kWarps) + 64;
    for (int ns = 3; ns >= 2; --ns)
      if (ns * stage + fixed <= 200 * 1024) return {epl, ns, te};
  }
  fail(SD_CONFIG_ERROR, "tree-mode pass: too many basis columns for the shared-memory ring");
}
template <typename T>
static size_t smem_bytes(const Shape& sh, int jb) {
  const size_t stage = (size_t(jb + 1) * sh.te * sizeof(T) + 127) & ~size_t(127);
  return sh.ns * stage + sizeof(double) * (kWarps * sh.te + sh.te + kMaxCols + kWarps) + 8 * sh.ns + 16;
}

template <typename T, int MODE, int EPL, int CPW>
static void launch_one(const CUtensorMap& tq, const CUtensorMap& tr, const Params& p, int grid, size_t smem,
                       cudaStream_t s) {
  auto kern = k_gs_tree<T, MODE, EPL, CPW>;
  static bool attr = false;
  if (!attr) {
    SD_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    attr = true;
  }
  kern<<<grid, kThreads, smem, s>>>(tq, tr, p);
  SD_LAUNCHED("k_gs_tree");
}

template <typename T, int MODE, int EPL>
static void dispatch_cpw(int cpw, const CUtensorMap& tq, const CUtensorMap& tr, const Params& p, int grid,
                         size_t smem, cudaStream_t s) {
  if (cpw <= 1) launch_one<T, MODE, EPL, 1>(tq, tr, p, grid, smem, s);
  else if (cpw <= 2) launch_one<T, MODE, EPL, 2>(tq, tr, p, grid, smem, s);
  else if (cpw <= 4) launch_one<T, MODE, EPL, 4>(tq, tr, p, grid, smem, s);
  else if (cpw <= 8) launch_one<T, MODE, EPL, 8>(tq, tr, p, grid, smem, s);
  else if (cpw <= 16) launch_one<T, MODE, EPL, 16>(tq, tr, p, grid, smem, s);
  else launch_one<T, MODE, EPL, 32>(tq, tr, p, grid, smem, s);
}

template <typename T, int MODE>
static void dispatch(const Shape& sh, int cpw, const CUtensorMap& tq, const CUtensorMap& tr, const Params& p, int grid,
                     size_t smem, cudaStream_t s) {
  constexpr int E_HI = sizeof(T) == 4 ? 4 : 2, E_LO = E_HI / 2;
  if (sh.epl == E_HI) dispatch_cpw<T, MODE, E_HI>(cpw, tq, tr, p, grid, smem, s);
  else dispatch_cpw<T, MODE, E_LO>(cpw, tq, tr, p, grid, smem, s);
}

template <typename T>
static void pass_t(int mode, const void* Q, uint64_t ldq, int jb, void* r, uint64_t n, const double* coef, int ucol,
                   int xcol, double* part, unsigned* counter, double* out, double* alpha_out, int alpha_col, int post_sqrt,
                   cudaStream_t s) {
  if (jb < 1 || jb > kMaxCols) fail(SD_CONFIG_ERROR, "tree-mode pass: 1..256 basis columns");
  if (n == 0) fail(SD_ARGUMENT_ERROR, "tree-mode pass over an empty shard");
  if ((reinterpret_cast<uintptr_t>(Q) | reinterpret_cast<uintptr_t>(r)) & 15)
    fail(SD_ARGUMENT_ERROR, "tree-mode pass: vectors must be 16-byte aligned");
  if ((ldq * sizeof(T)) % 16) fail(SD_ARGUMENT_ERROR, "tree-mode pass: basis column stride must be 16-byte aligned");
  const Shape sh = pick<T>(jb);
  const size_t smem = smem_bytes<T>(sh, jb);
  const int cpw = (jb + kWarps - 1) / kWarps;
  // two CTAs per SM when their rings fit (227 KB per SM): one CTA's update
  // phase overlaps the other's dot phase and barriers
  static const int max_per_sm = [] {
    const char* e = std::getenv("SD_TREE_CTAS_PER_SM");
    return e ? std::max(1, std::min(kMaxPerSM, std::atoi(e))) : kMaxPerSM;
  }();
  const int per_sm = (2 * (smem + 1024) <= 227 * 1024) ? max_per_sm : 1;
  const uint64_t nchunks = (n + kChunk - 1) / kChunk;
  // CTAs of every chunk launch, so the last one knows it is last
  std::vector<int> grids(nchunks), tiles(nchunks);
  int nparts = 0;
  for (uint64_t c = 0; c < nchunks; ++c) {
    const uint64_t len = std::min<uint64_t>(kChunk, n - c * kChunk);
    tiles[c] = int((len + sh.te - 1) / sh.te);
    grids[c] = std::min(tiles[c], kSMs * per_sm);
    nparts += grids[c];
  }
  const CUtensorMapDataType dt = sizeof(T) == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64;
  int part0 = 0;
  for (uint64_t c = 0; c < nchunks; ++c) {
    const uint64_t off = c * kChunk, len = std::min<uint64_t>(kChunk, n - off);
    CUtensorMap tq, tr;
    cuuint64_t qd[2] = {cuuint64_t(len), cuuint64_t(jb)}, qs[1] = {cuuint64_t(ldq * sizeof(T))};
    cuuint32_t qb[2] = {cuuint32_t(sh.te), cuuint32_t(jb)}, one[2] = {1, 1};
    CUresult e = encoder()(&tq, dt, 2, const_cast<T*>(static_cast<const T*>(Q) + off), qd, qs, qb, one,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (e != CUDA_SUCCESS) fail(SD_CUDA_ERROR, "cuTensorMapEncodeTiled (basis) failed (" + std::to_string(int(e)) + ")");
    cuuint64_t rd[1] = {cuuint64_t(len)}, rs[1] = {cuuint64_t(len * sizeof(T))};
    cuuint32_t rb[1] = {cuuint32_t(sh.te)};
    e = encoder()(&tr, dt, 1, static_cast<T*>(r) + off, rd, rs, rb, one, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (e != CUDA_SUCCESS) fail(SD_CUDA_ERROR, "cuTensorMapEncodeTiled (r) failed (" + std::to_string(int(e)) + ")");
    Params p{};
    p.r = static_cast<T*>(r) + off;
    p.n = len;
    p.jb = jb;
    p.coef = coef;
    p.ucol = ucol;
    p.xcol = xcol;
    p.part = part;
    p.part0 = part0;
    p.nparts = nparts;
    p.counter = counter;
    p.expected = unsigned(nparts);
    p.out = out;
    p.alpha_out = alpha_out;
    p.alpha_col = alpha_col;
    p.post_sqrt = post_sqrt;
    p.ntiles = tiles[c];
    p.ns = sh.ns;
    if (mode == 0) dispatch<T, 0>(sh, cpw, tq, tr, p, grids[c], smem, s);
    else if (mode == 1) dispatch<T, 1>(sh, cpw, tq, tr, p, grids[c], smem, s);
    else dispatch<T, 2>(sh, cpw, tq, tr, p, grids[c], smem, s);
    part0 += grids[c];
  }
}

}  // namespace tree

uint64_t tree_part_rows(uint64_t n) {
  const uint64_t nchunks = (n + tree::kChunk - 1) / tree::kChunk;
  return nchunks * tree::kGrid;
}
uint64_t tree_part_bytes(uint64_t n) { return tree_part_rows(n) * tree::kMaxCols * sizeof(double) + 256; }

void tree_pass(int prec, int mode, const void* Q, uint64_t ldq, int jb, void* r, uint64_t n, const double* coef,
               int ucol, int xcol, double* part, unsigned* counter, double* out, double* alpha_out, int alpha_col,
               int post_sqrt, cudaStream_t s) {
  if (prec == SD_F32)
    tree::pass_t<float>(mode, Q, ldq, jb, r, n, coef, ucol, xcol, part, counter, out, alpha_out, alpha_col, post_sqrt,
                        s);
  else
    tree::pass_t<double>(mode, Q, ldq, jb, r, n, coef, ucol, xcol, part, counter, out, alpha_out, alpha_col, post_sqrt,
                         s);
}

void tree_rank_fold(const double* recv, int nranks, int m, double* out, int post_sqrt, double* alpha_out,
                    int alpha_col, cudaStream_t s) {
  tree::k_rank_fold<<<(m + 127) / 128, 128, 0, s>>>(recv, nranks, m, out, post_sqrt, alpha_out, alpha_col);
  SD_LAUNCHED("k_rank_fold");
}

}  // namespace sd

// fp32-faithful GEMM on the 5th-generation tensor cores (sm_100a).
//
//   C[z] = alpha * op(A[z]) . op(B[z]) + beta * C[z] (+ bias)   (fp32 in/out)
//
// 3xTF32: every operand x is consumed as its raw fp32 bits (the tensor core
// reads the top 19 bits, i.e. trunc_tf32(x)) plus a precomputed residual
// x_s = x - trunc_tf32(x); the product is accumulated in TMEM as
//   A.B ~= A_b.B_b + A_b.B_s + A_s.B_b        (3 tcgen05.mma kind::tf32)
// which carries ~21-22 significant bits per product (fp32-faithful).
//
// Persistent warp-specialised kernel, one CTA per SM, 128 x BN output tiles
// walked in a static round-robin schedule:
//   warp 0   : TMA producer (cp.async.bulk.tensor) into a STAGES-deep smem
//              ring (full/empty mbarriers), running ahead across tiles;
//   warp 1   : TMEM allocator + single-thread tcgen05.mma issuer;
//   warps 2-3: residual warps: with on-chip residuals (GemmArgs::onchip)
//              they write x - trunc_tf32(x) of each landed raw tile into its
//              residual slot (half the bytes through L2/TMA, no residual
//              arrays in HBM), then release the stage to the MMA (conv[s]);
//   warps 4-11: epilogue: drain TMEM chunks (tcgen05.ld 32x32b) into
//              round-to-nearest fp32 registers, then alpha/beta/bias,
//              residual and store — overlapped with the next tile's MMAs.
// Source structures per launch: one product; dual (C = A B + A2 B2, one
// accumulator); twin (C = A B and C2 = A2 B + A B2 -- a weight's primal and
// tangent products -- as two tile sets of one launch, C2's first); split
// (the 64-wide attention pairs, below).
// Operand majors: A is K-major (row-major M x K) or MN-major (row-major K x M);
// B is K-major (row-major N x K) or MN-major (row-major K x N). A batch index
// z decomposes as (z1 = z % Z1, z2 = z / Z1) with independent strides, which
// covers per-head attention slices of a packed QKV activation.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <atomic>
#include <mutex>
#include <vector>

#include "sd_common.cuh"
#include "sd_gemm.h"
#include "sd_gemm_dev.cuh"

namespace sd {

namespace gk {
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encoder() {
  static EncodeFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<EncodeFn>(p);
  }();
  if (!fn) fail(SD_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
  return fn;
}

// 4-D map over a row-major operand: inner extent `inner` (contiguous),
// `outer` rows of stride ld, then two batch dims.
void make_map(CUtensorMap* m, const float* base, long long inner, long long outer, long long ld, int Z1,
              long long s1, int Z2, long long s2, int box_inner, int box_outer, bool mn_major) {
  if ((reinterpret_cast<uintptr_t>(base) & 15) != 0) fail(SD_ARGUMENT_ERROR, "gemm operand not 16-byte aligned");
  if ((ld * 4) % 16 != 0 || (Z1 > 1 && (s1 * 4) % 16) || (Z2 > 1 && (s2 * 4) % 16))
    fail(SD_ARGUMENT_ERROR, "gemm operand strides must be multiples of 16 bytes");
  cuuint64_t dims[4] = {cuuint64_t(inner), cuuint64_t(outer), cuuint64_t(Z1), cuuint64_t(Z2)};
  const long long whole = ((ld * outer * 4 + 15) / 16) * 16;  // stride of a size-1 batch dim
  cuuint64_t strides[3] = {cuuint64_t(ld * 4), cuuint64_t(Z1 > 1 ? s1 * 4 : whole), cuuint64_t(Z2 > 1 ? s2 * 4 : whole)};
  cuuint32_t box[4] = {cuuint32_t(box_inner), cuuint32_t(box_outer), 1, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  const CUresult r = encoder()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(base), dims, strides, box, es,
                               CU_TENSOR_MAP_INTERLEAVE_NONE,
                               mn_major ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_64B,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(SD_CUDA_ERROR, "cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
}

bool sd_gemm_tma_store_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("SD_GEMM_TMA_STORE");
    return !(e && e[0] == '0');
  }();
  return on;
}
bool sd_gemm_tmem_a_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("SD_GEMM_TMEM_A");
    return !(e && e[0] == '0');  // SD_GEMM_TMEM_A=0: A from shared memory (bit-identical results)
  }();
  return on;
}

bool tma_store_ok(const GemmArgs& g, int splits, int bias_cols, bool allow_add) {
  // beta 1 without a residual output: the tile is added in place by a TMA reduce-add store
  const bool beta_ok = g.beta == 0.0f || (allow_add && g.beta == 1.0f && !g.Cs);
  return sd_gemm_tma_store_enabled() && splits == 1 && beta_ok &&
         (reinterpret_cast<uintptr_t>(g.C) & 15) == 0 && (g.ldc % 4) == 0 &&
         (!g.Cs || (reinterpret_cast<uintptr_t>(g.Cs) & 15) == 0) &&
         (!g.bias || ((reinterpret_cast<uintptr_t>(g.bias) & 15) == 0 && g.N % bias_cols == 0)) &&
         (g.Z1 * g.Z2 == 1 || ((g.Z1 == 1 || g.sc1 % 4 == 0) && (g.Z2 == 1 || g.sc2 % 4 == 0)));
}

void make_store_map(CUtensorMap* m, float* C, const GemmArgs& g, int box_cols) {
  cuuint64_t dims[4] = {cuuint64_t(g.N), cuuint64_t(g.M), cuuint64_t(g.Z1), cuuint64_t(g.Z2)};
  const long long whole = ((g.ldc * (long long)g.M * 4 + 15) / 16) * 16;
  cuuint64_t strides[3] = {cuuint64_t(g.ldc * 4), cuuint64_t(g.Z1 > 1 ? g.sc1 * 4 : whole),
                           cuuint64_t(g.Z2 > 1 ? g.sc2 * 4 : whole)};
  cuuint32_t box[4] = {cuuint32_t(box_cols), 32, 1, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  const CUresult r = encoder()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, C, dims, strides, box, es,
                               CU_TENSOR_MAP_INTERLEAVE_NONE,
                               box_cols == 32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(SD_CUDA_ERROR, "cuTensorMapEncodeTiled (C) failed (" + std::to_string(int(r)) + ")");
}

// The eight operand maps of a launch: A, A_small, B, B_small, then the same
// for the second product of a dual-source GEMM (copies of the first if none).
// K-major tiles are box_m (A) / box_n (B) rows of BK elements; MN-major tiles
// are loaded as 32-element chunks of BK rows.
// MN-major operand whose extent is a multiple of 32: one 5-D box loads the
// whole tile -- dims (32 elements, K rows, 32-element chunks, z1, z2), box
// (32, BK, chunks, 1, 1) lands chunk-major, exactly the 2 KB-per-chunk
// SWIZZLE_128B_ATOM_32B layout the UMMA descriptors expect (one TMA
// instruction instead of one per chunk).
void make_map_mn5(CUtensorMap* m, const float* base, long long extent, long long K, long long ld, int Z1, long long s1,
                  int Z2, long long s2, int chunks) {
  if ((reinterpret_cast<uintptr_t>(base) & 15) != 0) fail(SD_ARGUMENT_ERROR, "gemm operand not 16-byte aligned");
  if ((ld * 4) % 16 != 0 || (Z1 > 1 && (s1 * 4) % 16) || (Z2 > 1 && (s2 * 4) % 16))
    fail(SD_ARGUMENT_ERROR, "gemm operand strides must be multiples of 16 bytes");
  cuuint64_t dims[5] = {32, cuuint64_t(K), cuuint64_t((extent + 31) / 32), cuuint64_t(Z1), cuuint64_t(Z2)};
  const long long whole = ((ld * K * 4 + 15) / 16) * 16;
  cuuint64_t strides[4] = {cuuint64_t(ld * 4), 128, cuuint64_t(Z1 > 1 ? s1 * 4 : whole),
                           cuuint64_t(Z2 > 1 ? s2 * 4 : whole)};
  cuuint32_t box[5] = {32, cuuint32_t(BK), cuuint32_t(chunks), 1, 1};
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  const CUresult r = encoder()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, const_cast<float*>(base), dims, strides, box, es,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(SD_CUDA_ERROR, "cuTensorMapEncodeTiled (mn5) failed (" + std::to_string(int(r)) + ")");
}

bool sd_gemm_mn5_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("SD_GEMM_MN5");
    return !(e && e[0] == '0');
  }();
  return on;
}

void operand_maps(const GemmArgs& g, bool a_mn, bool b_mn, bool three, int box_n, CUtensorMap* m, int* mn5) {
  // (an extent that is not a multiple of 32 is fine when the rows have room for
  // the last chunk: the extra columns only feed output rows/columns >= M/N,
  // which the epilogue never stores)
  const auto r32 = [](long long x) { return (x + 31) / 32 * 32; };
  const bool a5 = a_mn && (g.M % 32 == 0 || g.lda >= r32(g.M)) && (!g.A2 || g.M % 32 == 0 || g.lda2 >= r32(g.M)) &&
                  sd_gemm_mn5_enabled();
  const bool b5 = b_mn && (g.N % 32 == 0 || g.ldb >= r32(g.N)) && (!g.A2 || g.N % 32 == 0 || g.ldb2 >= r32(g.N)) &&
                  sd_gemm_mn5_enabled();
  if (mn5) *mn5 = (a5 ? 1 : 0) | (b5 ? 2 : 0);
  auto amap = [&](CUtensorMap* o, const float* p, long long ld, long long s1, long long s2) {
    if (a5) make_map_mn5(o, p, g.M, g.K, ld, g.Z1, s1, g.Z2, s2, BM / 32);
    else if (a_mn) make_map(o, p, g.M, g.K, ld, g.Z1, s1, g.Z2, s2, 32, BK, true);
    else make_map(o, p, g.K, g.M, ld, g.Z1, s1, g.Z2, s2, BK, BM, false);
  };
  auto bmap = [&](CUtensorMap* o, const float* p, long long ld, long long s1, long long s2) {
    if (b5) make_map_mn5(o, p, g.N, g.K, ld, g.Z1, s1, g.Z2, s2, box_n / 32);
    else if (b_mn) make_map(o, p, g.N, g.K, ld, g.Z1, s1, g.Z2, s2, 32, BK, true);
    else make_map(o, p, g.K, g.N, ld, g.Z1, s1, g.Z2, s2, BK, box_n, false);
  };
  // residual maps only when the residuals come from memory (not on chip)
  const bool mem_res = three && !g.onchip;
  amap(&m[0], g.A, g.lda, g.sa1, g.sa2);
  amap(&m[1], mem_res ? g.As : g.A, g.lda, g.sa1, g.sa2);
  bmap(&m[2], g.B, g.ldb, g.sb1, g.sb2);
  bmap(&m[3], mem_res ? g.Bs : g.B, g.ldb, g.sb1, g.sb2);
  if (g.A2) {
    if (!g.B2 || (mem_res && (!g.A2s || !g.B2s)))
      fail(SD_ARGUMENT_ERROR, "dual-source gemm needs A2, B2 (and their residuals for 3xTF32)");
    amap(&m[4], g.A2, g.lda2, g.sa1_2, g.sa2_2);
    amap(&m[5], mem_res ? g.A2s : g.A2, g.lda2, g.sa1_2, g.sa2_2);
    bmap(&m[6], g.B2, g.ldb2, g.sb1_2, g.sb2_2);
    bmap(&m[7], mem_res ? g.B2s : g.B2, g.ldb2, g.sb1_2, g.sb2_2);
  } else {
    for (int i = 0; i < 4; ++i) m[4 + i] = m[i];
  }
}

// Split-K count: minimise the modelled time
//   ceil(tiles s / units) * ceil(kb / s) * t_kb          (waves x k-blocks)
//   + 2 s * out_bytes / HBM + launch                      (partials + reduce)
// where t_kb is the time one worker spends on one k-block of one tile and kb
// counts the k-blocks of all sources; every split keeps >= 16 k-blocks.
int choose_splits(int tiles, int units, int total_kb, int nsrc, double t_kb, double out_bytes) {
  auto cost = [&](int s) {
    const double waves = double(((long long)tiles * s + units - 1) / units);
    const double kb = double((total_kb * nsrc + s - 1) / s);
    return waves * kb * t_kb + (s > 1 ? 2.0 * s * out_bytes / 6.0e12 + 5e-6 : 0.0);
  };
  int best_s = 1;
  double best = cost(1);
  for (int s = 2; s <= 16 && total_kb / s >= 16; ++s) {
    const double c = cost(s);
    if (c < best * 0.97) {
      best = c;
      best_s = s;
    }
  }
  return best_s;
}

// Split count of a twin launch: its units are the C2 tiles (two sources,
// first) and the C tiles (one source) of every split, dealt boustrophedon to
// the cluster slots (deal_unit); the modelled time is the busiest slot's k-blocks plus the
// split-K partial traffic (as choose_splits).
int choose_splits_twin(int tiles, int units, int total_kb, double t_kb, double out_bytes) {
  int best_s = 1;
  double best = 0.0;
  std::vector<long long> load(units);
  for (int s = 1; s <= 16 && (s == 1 || total_kb / s >= 16); ++s) {
    const long long kb = (total_kb + s - 1) / s, n = (long long)tiles * s;
    std::fill(load.begin(), load.end(), 0);
    for (long long t = 0; t < 2 * n; ++t) {  // the boustrophedon deal of deal_unit
      const long long r = t / units, p = t % units;
      load[(r & 1) ? units - 1 - p : p] += (t < n ? 2 : 1) * kb;
    }
    const double c = double(*std::max_element(load.begin(), load.end())) * t_kb +
                     (s > 1 ? 2.0 * s * out_bytes / 6.0e12 + 5e-6 : 0.0);
    if (s == 1 || c < best * 0.97) {
      best = c;
      best_s = s;
    }
  }
  return best_s;
}

// C = alpha * sum_split partial[split] + beta * C + bias (fixed split order)
__device__ __forceinline__ float tf32_residual(float r) {
  return r - __uint_as_float(__float_as_uint(r) & 0xFFFFE000u);
}
// grid (column groups of 4 x 128 threads, M, batch): no integer division
__global__ void __launch_bounds__(128) k_splitk_reduce(const float* __restrict__ ws, int splits, int zc, int Z1, int M,
                                                      int N, float* __restrict__ C, long long ldc, long long sc1,
                                                      long long sc2, float alpha, float beta,
                                                      const float* __restrict__ bias, float* __restrict__ Cs, int vec) {
  pdl_wait();  // PDL: nothing global is touched before the previous kernel completes
  const int col = 4 * (blockIdx.x * blockDim.x + threadIdx.x);
  if (col >= N) return;
  const int row = blockIdx.y, z = blockIdx.z;
  const long long mn = (long long)M * N;
  const float* p = ws + (long long)z * mn + (long long)row * N + col;
  const long long off = (z % Z1) * sc1 + (z / Z1) * sc2 + (long long)row * ldc + col;
  if (vec) {
    float4 acc = *reinterpret_cast<const float4*>(p);
    for (int sp = 1; sp < splits; ++sp) {
      const float4 v = *reinterpret_cast<const float4*>(p + sp * zc * mn);
      acc.x += v.x, acc.y += v.y, acc.z += v.z, acc.w += v.w;
    }
    float4 r = make_float4(alpha * acc.x, alpha * acc.y, alpha * acc.z, alpha * acc.w);
    if (beta != 0.0f) {
      const float4 o = *reinterpret_cast<const float4*>(C + off);
      r.x += beta * o.x, r.y += beta * o.y, r.z += beta * o.z, r.w += beta * o.w;
    }
    if (bias) r.x += bias[col], r.y += bias[col + 1], r.z += bias[col + 2], r.w += bias[col + 3];
    *reinterpret_cast<float4*>(C + off) = r;
    if (Cs)
      *reinterpret_cast<float4*>(Cs + off) =
          make_float4(tf32_residual(r.x), tf32_residual(r.y), tf32_residual(r.z), tf32_residual(r.w));
    return;
  }
  for (int j = 0; j < 4 && col + j < N; ++j) {
    float acc = p[j];
    for (int sp = 1; sp < splits; ++sp) acc += p[sp * zc * mn + j];
    float r = alpha * acc;
    if (beta != 0.0f) r += beta * C[off + j];
    if (bias) r += bias[col + j];
    C[off + j] = r;
    if (Cs) Cs[off + j] = tf32_residual(r);
  }
}

// Split-K scratch: lazily grown device buffers per (issuing thread, device).
// The GEMMs one thread issues go to one stream in program order, so its
// consecutive calls never overlap; in-process workers (one thread each) get
// their own buffers, released when the thread exits.
namespace {
struct SplitScratch {
  float* ws = nullptr;
  size_t cap = 0;
};
struct ThreadScratch {
  std::vector<SplitScratch> per_dev;
  ~ThreadScratch() {  // errors ignored: at process exit the runtime may be gone
    for (size_t d = 0; d < per_dev.size(); ++d)
      if (per_dev[d].ws && cudaSetDevice(int(d)) == cudaSuccess) (void)cudaFree(per_dev[d].ws);
  }
};
SplitScratch& split_scratch() {
  thread_local ThreadScratch t;
  int dev = 0;
  SD_CUDA(cudaGetDevice(&dev));
  if (t.per_dev.size() <= size_t(dev)) t.per_dev.resize(dev + 1);
  return t.per_dev[dev];
}
}  // namespace
std::atomic<uint64_t> g_scratch_gen{0};
float* splitk_workspace(size_t floats) {
  SplitScratch& sc = split_scratch();
  if (floats > sc.cap) {
    g_scratch_gen.fetch_add(1);
    if (sc.ws) SD_CUDA(cudaFree(sc.ws));
    SD_CUDA(cudaMalloc(&sc.ws, floats * sizeof(float)));
    sc.cap = floats;
  }
  return sc.ws;
}

// Optional per-launch CUDA-event timing of every GEMM (bench.py roofline):
// events are recorded on the launching stream around each kernel.
struct Prof {
  bool on = false;
  std::vector<cudaEvent_t> ev;
  std::vector<double> flops;
  std::vector<std::string> tags;  // "M,N,K,batch,a_mn,b_mn,causal,splits" per launch
  size_t used = 0;
  std::string next_tag;
};
Prof& prof() {
  static Prof p;
  return p;
}
void prof_begin(cudaStream_t s) {
  Prof& p = prof();
  if (!p.on) return;
  if (p.used + 2 > p.ev.size()) {
    const size_t n = p.ev.size();
    p.ev.resize(n + 4096);
    for (size_t i = n; i < p.ev.size(); ++i) SD_CUDA(cudaEventCreate(&p.ev[i]));
  }
  SD_CUDA(cudaEventRecord(p.ev[p.used], s));
}
void prof_end(cudaStream_t s, double flops) {
  Prof& p = prof();
  if (!p.on) return;
  SD_CUDA(cudaEventRecord(p.ev[p.used + 1], s));
  p.flops.push_back(flops);
  p.tags.push_back(p.next_tag);
  p.used += 2;
}
bool prof_on() { return prof().on; }
bool pdl_on() {
  static const bool on = [] {
    const char* e = std::getenv("SD_GEMM_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}
void prof_tag(const std::string& tag) { prof().next_tag = tag; }

void launch_splitk_reduce(const float* ws, int splits, int zc, const GemmArgs& g, cudaStream_t s) {
  const bool vec = g.N % 4 == 0 && g.ldc % 4 == 0 && (zc == 1 || (g.sc1 % 4 == 0 && g.sc2 % 4 == 0)) &&
                   (reinterpret_cast<uintptr_t>(g.C) & 15) == 0 && (!g.Cs || (reinterpret_cast<uintptr_t>(g.Cs) & 15) == 0);
  const dim3 grid(unsigned((g.N + 511) / 512), unsigned(g.M), unsigned(zc));
  launch_pdl(k_splitk_reduce, dim3(grid), dim3(128), 0, s, ws, splits, zc, g.Z1, g.M, g.N, g.C, g.ldc, g.sc1, g.sc2, g.alpha, g.beta, g.bias,
                                       g.Cs, int(vec));
  SD_LAUNCHED("k_splitk_reduce");
}

}  // namespace gk

namespace {
using namespace gk;

// TA: the A operand (K-major, 64-wide attention products with on-chip
// residuals) goes to tensor memory instead of being re-read from shared memory
// by every MMA: four residual warps (one per TMEM lane quarter) read each
// landed A row once, write its tf32 high part and residual into a per-stage
// TMEM slot (tcgen05.st), and the MMAs take A from there.
template <bool TA>
constexpr int kThreadsFor() { return TA ? 32 * (2 + 4 + 8) : NUM_THREADS; }

template <bool A_MN, bool B_MN, bool THREE, int BN_, bool CAUSAL, bool TA = false>
__global__ void __launch_bounds__(kThreadsFor<TA>(), 1)
    k_gemm_tf32(const __grid_constant__ CUtensorMap mA, const __grid_constant__ CUtensorMap mAs,
                const __grid_constant__ CUtensorMap mB, const __grid_constant__ CUtensorMap mBs,
                const __grid_constant__ CUtensorMap mA2, const __grid_constant__ CUtensorMap mAs2,
                const __grid_constant__ CUtensorMap mB2, const __grid_constant__ CUtensorMap mBs2,
                const __grid_constant__ CUtensorMap mC, const __grid_constant__ CUtensorMap mCs,
                const __grid_constant__ CUtensorMap mC2, const __grid_constant__ CUtensorMap mCs2, int K,
                EpiParams ep) {
  using Cf = Cfg<BN_>;
  constexpr int BN = Cf::BN, STAGES = Cf::STAGES, EC = Cf::EC;
  constexpr int A_BYTES = Cf::A_BYTES, B_BYTES = Cf::B_BYTES;
  static_assert(!TA || (THREE && (BN_ == 64 || BN_ == 128)), "TMEM-A: 3xTF32, 64- or 128-wide tiles");
  constexpr int CONV = TA ? 4 : kConvWarps;
  constexpr uint32_t TA_COL0 = 2 * BN_;                       // A slots after the two accumulators
  constexpr uint32_t TMEM_COLS = TA ? 512 : Cf::TMEM_COLS;   // TA: 128 + STAGES x (16 hi + 16 lo)
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1024-byte aligned ring: per stage [A | As | B | Bs]
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int STAGE_BYTES = (THREE ? 2 : 1) * (A_BYTES + B_BYTES);
  // [ring | 8 epilogue staging boxes of 4 KB (TMA store) | barriers]
  float* epi_stage = reinterpret_cast<float*>(smem + STAGES * STAGE_BYTES);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES + 8 * 4096);
  uint64_t* empty = full + STAGES;
  uint64_t* conv = empty + STAGES;   // [STAGES] residual tiles ready
  uint64_t* tfull = conv + STAGES;   // [2]
  uint64_t* tempty = tfull + 2;      // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
      mbar_init(&conv[s], TA ? 4 : 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  // programmatic dependent launch: the set-up above (barriers, TMEM) overlaps
  // the previous kernel's tail; no global memory is read or written before
  // the previous grid has completed. Dependents may be scheduled right away
  // (every CTA of this persistent grid is resident).
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  if (warp == 0) {
    {  // whole warp; elected lane issues (no waterfall loops around TMA)
      asm volatile("prefetch.tensormap [%0];" ::"l"(&mA) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&mB) : "memory");
      uint32_t g = 0;  // global k-block counter (ring position)
      for (int t = blockIdx.x; t < ep.n_tiles; t += gridDim.x) {
        const TileInfo ti = tile_info<BN, CAUSAL>(ep, t, K);
        if (ti.skip) continue;
        const int z1 = ti.z % ep.Z1, z2 = ti.z / ep.Z1;
        for (int kk = 0; kk < ti.nsrc * ti.num_kb; ++kk, ++g) {
          const int s = g % STAGES;
          const uint32_t ph = (g / STAGES) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          unsigned char* st = smem + s * STAGE_BYTES;
          // dual source: the second product's k-blocks follow the first's, (A, B)
          // then (A2, B2); twin C2 tiles: (A2, B) then (A, B2); split pairs:
          // interleaved, and source 2 multiplies B, not B2
          const bool src2 = ep.split ? (kk & 1) != 0 : kk >= ti.num_kb;
          const bool useA2 = ti.tan ? !src2 : src2, useB2 = src2 && !ep.split;
          const bool bex = THREE && !ep.res && ((ep.bexact >> (src2 ? 1 : 0)) & 1);
          mbar_expect_tx_e(&full[s], ep.split ? A_BYTES + (src2 ? B_BYTES / 2 : B_BYTES)
                                              : (ep.res ? A_BYTES + B_BYTES : STAGE_BYTES - (bex ? B_BYTES : 0)));
          const int kb = ep.split ? kk >> 1 : (src2 ? kk - ti.num_kb : kk);
          const CUtensorMap* pA = useA2 ? &mA2 : &mA;
          const CUtensorMap* pAs = useA2 ? &mAs2 : &mAs;
          const CUtensorMap* pB = useB2 ? &mB2 : &mB;
          const CUtensorMap* pBs = useB2 ? &mBs2 : &mBs;
          const int k0 = (ti.kb0 + kb) * BK;
          if (A_MN && (ep.mn5 & 1)) {
            tma_load_5d_e(pA, &full[s], st, 0, k0, ti.m0 / 32, z1, z2);
            if (THREE && !ep.res) tma_load_5d_e(pAs, &full[s], st + A_BYTES, 0, k0, ti.m0 / 32, z1, z2);
          } else if (A_MN) {
#pragma unroll
            for (int c = 0; c < BM / 32; ++c) {
              tma_load_4d_e(pA, &full[s], st + c * 2048, ti.m0 + 32 * c, k0, z1, z2);
              if (THREE && !ep.res) tma_load_4d_e(pAs, &full[s], st + A_BYTES + c * 2048, ti.m0 + 32 * c, k0, z1, z2);
            }
          } else {
            tma_load_4d_e(pA, &full[s], st, k0, ti.m0, z1, z2);
            if (THREE && !ep.res) tma_load_4d_e(pAs, &full[s], st + A_BYTES, k0, ti.m0, z1, z2);
          }
          unsigned char* sb = st + (THREE ? 2 : 1) * A_BYTES;
          if (B_MN && ep.split) {
            // [B | B2] as two 64-wide 5-D boxes (2 chunks each); source 2: B only
            tma_load_5d_e(pB, &full[s], sb, 0, k0, 0, z1, z2);
            if (!src2) tma_load_5d_e(&mB2, &full[s], sb + B_BYTES / 2, 0, k0, 0, z1, z2);
          } else if (B_MN && (ep.mn5 & 2)) {
            tma_load_5d_e(pB, &full[s], sb, 0, k0, ti.n0 / 32, z1, z2);
            if (THREE && !ep.res && !bex) tma_load_5d_e(pBs, &full[s], sb + B_BYTES, 0, k0, ti.n0 / 32, z1, z2);
          } else if (B_MN) {
#pragma unroll
            for (int c = 0; c < BN / 32; ++c) {
              tma_load_4d_e(pB, &full[s], sb + c * 2048, ti.n0 + 32 * c, k0, z1, z2);
              if (THREE && !ep.res && !bex) tma_load_4d_e(pBs, &full[s], sb + B_BYTES + c * 2048, ti.n0 + 32 * c, k0, z1, z2);
            }
          } else {
            tma_load_4d_e(pB, &full[s], sb, k0, ti.n0, z1, z2);
            if (THREE && !ep.res && !bex) tma_load_4d_e(pBs, &full[s], sb + B_BYTES, k0, ti.n0, z1, z2);
          }
        }
      }
    }
  } else if (TA && warp >= 2 && warp < 2 + CONV) {
    // TMEM-A residual warps: warp w owns TMEM lanes / A rows 32 (w % 4) .. +31
    // and a quarter of the B tile; every stage goes through all four
    const int q = warp & 3, m = 32 * q + lane;
    uint32_t g = 0;
    for (int t = blockIdx.x; t < ep.n_tiles; t += gridDim.x) {
      const TileInfo ti = tile_info<BN, CAUSAL>(ep, t, K);
      if (ti.skip) continue;
      for (int kk = 0; kk < ti.nsrc * ti.num_kb; ++kk, ++g) {
        const int s = g % STAGES;
        mbar_wait(&full[s], (g / STAGES) & 1);
        unsigned char* st = smem + s * STAGE_BYTES;
        uint32_t hi[16], lo[16];
        if (!A_MN) {
          // row m of the K-major A tile: 64 B, SWIZZLE_64B (16 B chunk c at c ^ ((m >> 1) & 3))
          const uint32_t row = smem_u32(st + m * 64);
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const float4 v = lds128(row + 16u * uint32_t(c ^ ((m >> 1) & 3)));
            const float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const uint32_t h = __float_as_uint(e[u]) & 0xFFFFE000u;
              hi[4 * c + u] = h;
              lo[4 * c + u] = __float_as_uint(e[u] - __uint_as_float(h));
            }
          }
        } else {
          // MN-major A tile: 32-row chunk q (= this warp) at q * 2048, k-row k of
          // 128 B, 32 B granule (m % 32) / 8 swizzled with k & 3 (SWIZZLE_128B_ATOM_32B)
          const uint32_t ch = smem_u32(st + q * 2048 + (lane & 7) * 4);
#pragma unroll
          for (int k = 0; k < 16; ++k) {
            const float x = lds32(ch + uint32_t(k * 128 + (((lane >> 3) ^ (k & 3)) << 5)));
            const uint32_t h = __float_as_uint(x) & 0xFFFFE000u;
            hi[k] = h;
            lo[k] = __float_as_uint(x - __uint_as_float(h));
          }
        }
        const uint32_t ta = tmem + (uint32_t(32 * q) << 16) + TA_COL0 + uint32_t(s) * 32u;
        tmem_st16(ta, hi);
        tmem_st16(ta + 16, lo);
        stage_residual(st + 2 * A_BYTES + q * (B_BYTES / 4), st + 2 * A_BYTES + B_BYTES + q * (B_BYTES / 4),
                       B_BYTES / 4, lane, 32);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        fence_proxy_async_smem();
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&conv[s]);
      }
    }
  } else if (!TA && warp >= 2 && warp < 2 + kConvWarps) {
    // residual warps: once a stage lands, write x - trunc_tf32(x) of the raw
    // A and B tiles into their residual slots (3xTF32 without residual arrays
    // in memory: half the operand bytes through L2 and TMA), then release it
    // (warp w takes the stages with g % kConvWarps == w - 2: two stages in flight)
    const int cw = warp - 2;
    uint32_t g = 0;
    if (THREE && ep.res)
      for (int t = blockIdx.x; t < ep.n_tiles; t += gridDim.x) {
        const TileInfo ti = tile_info<BN, CAUSAL>(ep, t, K);
        if (ti.skip) continue;
        for (int kk = 0; kk < ti.nsrc * ti.num_kb; ++kk, ++g) {
          if (int(g % kConvWarps) != cw) continue;
          const int s = g % STAGES;
          mbar_wait(&full[s], (g / STAGES) & 1);
          unsigned char* st = smem + s * STAGE_BYTES;
          stage_residual(st, st + A_BYTES, A_BYTES, lane, 32);
          stage_residual(st + 2 * A_BYTES, st + 2 * A_BYTES + B_BYTES, B_BYTES, lane, 32);
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) mbar_arrive(&conv[s]);
        }
      }
  } else if (warp == 1) {
    constexpr uint32_t idesc = make_idesc(TA ? false : A_MN, B_MN, BN);  // TMEM A: lane = row, column = k
    constexpr uint32_t idesc_half = make_idesc(TA ? false : A_MN, B_MN, BN / 2);  // split: source 2
    uint32_t g = 0, chunk = 0;
    for (int t = blockIdx.x; t < ep.n_tiles; t += gridDim.x) {
      const TileInfo ti = tile_info<BN, CAUSAL>(ep, t, K);
      if (ti.skip) continue;
      const int nkb = ti.nsrc * ti.num_kb;
      for (int kb = 0; kb < nkb; ++kb, ++g) {
        const int s = g % STAGES;
        const uint32_t ph = (g / STAGES) & 1;
        const bool first = (kb % KC) == 0;
        const bool last = (kb % KC) == KC - 1 || kb == nkb - 1;
        const uint32_t buf = chunk & 1;
        if (first && chunk >= 2) mbar_wait(&tempty[buf], ((chunk >> 1) - 1) & 1);
        mbar_wait(ep.res ? &conv[s] : &full[s], ph);  // stage landed (and its residuals written)
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        {  // whole warp: uniform descriptor math, one elect.sync-elected lane issues (a lane-0
           // branch here makes the compiler wrap every MMA in a waterfall loop)
          const uint32_t d = tmem + buf * BN;
          const uint32_t st = smem_u32(smem + s * STAGE_BYTES);
          const uint32_t a = st, as = st + A_BYTES;
          const uint32_t b = st + (THREE ? 2 : 1) * A_BYTES, bs = b + B_BYTES;
          const bool bex = THREE && !ep.res && ((ep.bexact >> (kb >= ti.num_kb ? 1 : 0)) & 1);
#pragma unroll
          for (int ks = 0; ks < BK / 8; ++ks) {
            const uint32_t acc0 = (first && ks == 0) ? 0u : 1u;
            if (TA) {
              const uint32_t ta = tmem + TA_COL0 + uint32_t(s) * 32u + uint32_t(ks) * 8u;
              // split pair, source 2: N = BN/2 into accumulator columns BN/2.. (a chunk
              // always starts with a source-1 k-block, so acc0 is 0 only there)
              const bool half = ep.split && (kb & 1);
              const uint32_t dd = half ? d + uint32_t(BN / 2) : d, id = half ? idesc_half : idesc;
              mma_tf32_ta_e(dd, ta + 16, tile_desc<B_MN>(b, ks), id, acc0);
              mma_tf32_ta_e(dd, ta, tile_desc<B_MN>(bs, ks), id, 1u);
              mma_tf32_ta_e(dd, ta, tile_desc<B_MN>(b, ks), id, 1u);
            } else if (THREE) {
              mma_tf32_e(d, tile_desc<A_MN>(as, ks), tile_desc<B_MN>(b, ks), idesc, acc0);
              if (!bex) mma_tf32_e(d, tile_desc<A_MN>(a, ks), tile_desc<B_MN>(bs, ks), idesc, 1u);
              mma_tf32_e(d, tile_desc<A_MN>(a, ks), tile_desc<B_MN>(b, ks), idesc, 1u);
            } else {
              mma_tf32_e(d, tile_desc<A_MN>(a, ks), tile_desc<B_MN>(b, ks), idesc, acc0);
            }
          }
          mma_commit_e(&empty[s]);
          if (last) mma_commit_e(&tfull[buf]);
        }
        __syncwarp();
        if (last) ++chunk;
      }
    }
  } else {
    // epilogue: 8 warps (4-11); warp w drains TMEM lanes 32*(w%4) .. +31 (its
    // sub-partition) and the column half (w-4)/4 of the tile: thread = one
    // output row, EC = BN/2 fp32 accumulators in registers.
    const int sub = warp & 3;
    const int cb = ((warp - 2 - CONV) >> 2) * EC;
    uint32_t chunk = 0;
    for (int t = blockIdx.x; t < ep.n_tiles; t += gridDim.x) {
      const TileInfo ti = tile_info<BN, CAUSAL>(ep, t, K);
      if (ti.skip) continue;
      const int row = ti.m0 + sub * 32 + lane;
      float acc[EC];
#pragma unroll
      for (int j = 0; j < EC; ++j) acc[j] = 0.0f;
      const int nchunks = (ti.nsrc * ti.num_kb + KC - 1) / KC;
      for (int c = 0; c < nchunks; ++c, ++chunk) {
        const uint32_t buf = chunk & 1;
        mbar_wait(&tfull[buf], (chunk >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
        for (int c0 = 0; c0 < EC; c0 += 32) {
          uint32_t v[32];
          tmem_ld32(tmem + (uint32_t(sub * 32) << 16) + buf * BN + uint32_t(cb + c0), v);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int j = 0; j < 32; ++j) acc[c0 + j] += __uint_as_float(v[j]);
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[buf]);
      }
      if (ep.tma_store) {
        const int ew = warp - 2 - CONV;                 // 0..7: its staging box
        const bool second = ep.split && cb >= BN / 2;  // split pair: columns BN/2.. are C2's
        const bool t2 = ti.tan || second;               // twin: C2's tile
        const CUtensorMap* pcs = t2 ? (ep.Cs2 ? &mCs2 : nullptr) : (ep.Cs ? &mCs : nullptr);
        warp_tma_store<EC>(t2 ? &mC2 : &mC, pcs, epi_stage + ew * 1024, acc, ti.tan ? ep.alpha2 : ep.alpha,
                           ti.tan ? ep.bias2 : ep.bias, lane, ti.m0 + sub * 32, ti.n0 + cb - (second ? BN / 2 : 0),
                           ti.z % ep.Z1, ti.z / ep.Z1, false);
        if (lane == 0) bulk_wait_read0();  // staging box free for the next tile
        __syncwarp();
      } else if (ti.tan) {
        EpiParams e2 = ep;  // twin: C2's tile
        e2.C = ep.C2, e2.Cs = ep.Cs2, e2.alpha = ep.alpha2, e2.beta = ep.beta2, e2.bias = ep.bias2, e2.ws = ep.ws2;
        store_row<EC>(e2, ti, row, ti.n0 + cb, acc);
      } else if (ep.split && cb >= BN / 2) {
        EpiParams e2 = ep;  // columns BN/2.. of the split pair: the second output
        e2.C = ep.C2, e2.Cs = ep.Cs2;
        store_row<EC>(e2, ti, row, ti.n0 + cb - BN / 2, acc);
      } else {
        store_row<EC>(ep, ti, row, ti.n0 + cb, acc);
      }
    }
  }
  if (ep.tma_store && lane == 0) bulk_wait0();  // (no-op for non-epilogue warps: nothing committed)
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
  }
}

// residual x - trunc_tf32(x) (the tensor core reads trunc_tf32 of the raw bits)
__global__ void k_split_tf32(const float* __restrict__ x, float* __restrict__ s, long long n, int mode) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float v = x[i];
  float hi;
  if (mode == 0) {
    hi = __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
  } else {
    uint32_t t;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(t) : "f"(v));
    hi = __uint_as_float(t);
  }
  s[i] = v - hi;
}

// ------------------------------------------------------------- tensor maps
template <bool A_MN, bool B_MN, bool THREE, int BN>
void launch(const GemmArgs& g, cudaStream_t s) {
  using Cf = Cfg<BN>;
  CUtensorMap maps[8];
  int mn5 = 0;
  operand_maps(g, A_MN, B_MN, THREE, BN, maps, &mn5);
  const bool dual = g.A2 != nullptr;
  const int zc = g.Z1 * g.Z2;
  const int tn = (g.N + BN - 1) / BN, tm = (g.M + BM - 1) / BM;
  int tiles = tn * tm * zc;
  if (g.causal == 1 && BN == BM) {
    if (tn != tm) fail(SD_ARGUMENT_ERROR, "causal score product must be square");
    tiles = tm * (tm + 1) / 2 * zc;  // lower-triangle tiles only (tile_info)
  }
  const int total_kb = (g.K + BK - 1) / BK;
  // split-K when the output grid cannot fill the 148 SMs and K is long (the
  // Hv weight products reduce over all T tokens): partial tiles go to a
  // workspace and are summed in a fixed order by k_splitk_reduce.
  // Choose the split count minimising waves-per-unit-of-work
  // ceil(tiles*s/148)/s (each split keeps >= 16 k-blocks), smallest s on ties.
  // one worker: 128 x BN x BK per k-block at ~200 TF/s (algorithmic) per 148 SMs
  const double t_kb = 2.0 * BM * BN * BK / (2.0e14 / kNumSMs) / (THREE ? 1.0 : 3.0);
  const bool twin = g.twin;
  int splits = g.causal == 0 ? (twin ? choose_splits_twin(tiles, kNumSMs, total_kb, t_kb, 8.0 * zc * g.M * g.N)
                                     : choose_splits(tiles, kNumSMs, total_kb, dual ? 2 : 1, t_kb, 4.0 * zc * g.M * g.N))
                             : 1;
  const int kb_per = (total_kb + splits - 1) / splits;
  splits = (total_kb + kb_per - 1) / kb_per;
  const size_t part = size_t(splits) * zc * size_t(g.M) * g.N;
  float* ws = nullptr;
  if (splits > 1) ws = splitk_workspace((twin ? 2 : 1) * part);
  EpiParams ep{g.C, g.ldc, g.sc1, g.sc2, g.M, g.N, g.Z1, g.alpha, g.beta, g.bias, g.Cs, g.dbg, zc, kb_per, ws,
               g.causal, tn, tm, tiles * splits * (twin ? 2 : 1), dual ? 2 : 1, g.onchip ? 1 : 0};
  GemmArgs g2 = g;  // twin: C2's epilogue
  g2.C = g.C2, g2.Cs = g.Cs2, g2.alpha = g.alpha2, g2.beta = g.beta2, g2.bias = g.bias2;
  if (twin) {
    ep.twin = 1, ep.tiles1 = tiles * splits;
    ep.C2 = g.C2, ep.Cs2 = g.Cs2, ep.alpha2 = g.alpha2, ep.beta2 = g.beta2, ep.bias2 = g.bias2;
    ep.ws2 = ws ? ws + part : nullptr;
  }
  const size_t smem = 1024 + size_t(Cf::STAGES) * (THREE ? 2 : 1) * (Cf::A_BYTES + Cf::B_BYTES) + 8 * 4096 + 512;
  // TMA-store epilogue: plain C = alpha op(A) op(B) tiles (no accumulate/bias/residual/split)
  CUtensorMap mC = maps[0], mCs = maps[0], mC2 = maps[0], mCs2 = maps[0];
  const bool tma_store = tma_store_ok(g, splits, 32) && (!twin || tma_store_ok(g2, splits, 32));
  if (tma_store) {
    make_store_map(&mC, g.C, g);
    if (g.Cs) make_store_map(&mCs, g.Cs, g);
    if (twin) {
      make_store_map(&mC2, g2.C, g2);
      if (g2.Cs) make_store_map(&mCs2, g2.Cs, g2);
    }
  }
  ep.tma_store = tma_store ? 1 : 0;
  ep.mn5 = mn5;
  if (!g.causal) ep.group = walk_group(g, BM, BN, tm, tn, THREE);
  ep.bexact = (g.b_exact ? 1 : 0) | (g.b2_exact ? 2 : 0);
  auto kern = g.causal ? k_gemm_tf32<A_MN, B_MN, THREE, BN, true> : k_gemm_tf32<A_MN, B_MN, THREE, BN, false>;
  int threads = NUM_THREADS;
  static bool attr_set = false;
  if (!attr_set) {
    SD_CUDA(cudaFuncSetAttribute(k_gemm_tf32<A_MN, B_MN, THREE, BN, true>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    SD_CUDA(cudaFuncSetAttribute(k_gemm_tf32<A_MN, B_MN, THREE, BN, false>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    attr_set = true;
  }
  if constexpr (THREE && BN == 64) {
    // on-chip residuals: A through tensor memory (SD_GEMM_TMEM_A=0 disables)
    if (g.onchip && sd_gemm_tmem_a_enabled()) {
      kern = g.causal ? k_gemm_tf32<A_MN, B_MN, THREE, BN, true, true> : k_gemm_tf32<A_MN, B_MN, THREE, BN, false, true>;
      threads = kThreadsFor<true>();
      static bool attr_ta = false;
      if (!attr_ta) {
        SD_CUDA(cudaFuncSetAttribute(k_gemm_tf32<A_MN, B_MN, THREE, BN, true, true>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        SD_CUDA(cudaFuncSetAttribute(k_gemm_tf32<A_MN, B_MN, THREE, BN, false, true>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        attr_ta = true;
      }
    }
  }
  const int grid = std::min(ep.n_tiles, kNumSMs);
  // (the twin score products keep the plain round robin: their one- and
  // two-source tiles cost about the same -- the epilogue bounds them -- and
  // the boustrophedon deal measured 1.6% slower there)
  if (prof().on)
    prof().next_tag = std::to_string(g.M) + "," + std::to_string(g.N) + "," + std::to_string(g.K) + "," +
                      std::to_string(zc) + "," + std::to_string(int(A_MN)) + "," + std::to_string(int(B_MN)) + "," +
                      std::to_string(g.causal) + "," + std::to_string(splits) + (twin ? ",twin" : dual ? ",2" : ",1");
  prof_begin(s);
  launch_gemm_kernel(kern, unsigned(grid), unsigned(threads), smem, s, maps[0], maps[1], maps[2], maps[3], maps[4],
                     maps[5], maps[6], maps[7], mC, mCs, mC2, mCs2, g.K, ep);
  SD_LAUNCHED("k_gemm_tf32");
  if (splits > 1) {
    launch_splitk_reduce(ws, splits, zc, g, s);
    if (twin) launch_splitk_reduce(ws + part, splits, zc, g2, s);
  }
  prof_end(s, (twin ? 6.0 : dual ? 4.0 : 2.0) * double(g.M) * g.N * g.K * g.Z1 * g.Z2);
}

// Merged pair of 64-wide products sharing A (GemmArgs::split): one 1-CTA
// launch with a 128-wide TMEM accumulator and A from tensor memory. Per
// k-block: source 1 (A) against [B | B2] (N = 128: 3 MMAs), source 2 (A2)
// against B into columns 64-127 (N = 64: 3 MMAs) -- the MMA work of the two
// separate products, but each A tile is staged and split once and every MMA
// of source 1 is 128 wide (the 64-wide tf32 MMA is issue-bound).
template <bool A_MN>
void launch_split(const GemmArgs& g, cudaStream_t s) {
  constexpr int BN = 128;
  using Cf = Cfg<BN>;
  if (g.N != 64 || !g.b_mn || !g.A2 || !g.B2 || !g.C2) fail(SD_ARGUMENT_ERROR, "split gemm: 64-wide MN-major pair");
  GemmArgs m = g;  // maps: A, A2; B and B2 as 64-wide 5-D boxes
  m.ldb2 = g.ldb, m.sb1_2 = g.sb1, m.sb2_2 = g.sb2;
  m.As = m.Bs = m.A2s = m.B2s = nullptr;
  m.onchip = true;
  CUtensorMap maps[8];
  int mn5 = 0;
  operand_maps(m, A_MN, true, true, 64, maps, &mn5);
  if (!(mn5 & 2)) fail(SD_ARGUMENT_ERROR, "split gemm: B needs 32-element chunks");
  const int zc = g.Z1 * g.Z2;
  const int tm = (g.M + BM - 1) / BM;
  const int total_kb = (g.K + BK - 1) / BK;
  EpiParams ep{g.C, g.ldc, g.sc1, g.sc2, g.M, g.N, g.Z1, g.alpha, g.beta, g.bias, g.Cs, g.dbg, zc, total_kb, nullptr,
               g.causal, 1, tm, tm * zc, 2, 1};
  ep.mn5 = mn5;
  ep.bexact = 0;
  ep.split = 1;
  ep.C2 = g.C2, ep.Cs2 = g.Cs2;
  ep.group = 0;
  // TMA-store epilogue: each output's 64 columns as two 32-wide boxes
  // (SD_SPLIT_TMA_STORE=0: row stores)
  static const bool tma_on = [] {
    const char* e = std::getenv("SD_SPLIT_TMA_STORE");
    return !(e && e[0] == '0');
  }();
  GemmArgs g2 = g;
  g2.C = g.C2, g2.Cs = g.Cs2;
  CUtensorMap mC = maps[0], mCs = maps[0], mC2 = maps[0], mCs2 = maps[0];
  ep.tma_store = tma_on && tma_store_ok(g, 1, 32) && tma_store_ok(g2, 1, 32);
  if (ep.tma_store) {
    make_store_map(&mC, g.C, g);
    make_store_map(&mC2, g.C2, g2);
    if (g.Cs) make_store_map(&mCs, g.Cs, g);
    if (g.Cs2) make_store_map(&mCs2, g.Cs2, g2);
  }
  const size_t smem = 1024 + size_t(Cf::STAGES) * 2 * (Cf::A_BYTES + Cf::B_BYTES) + 8 * 4096 + 512;
  auto kern = g.causal ? k_gemm_tf32<A_MN, true, true, BN, true, true> : k_gemm_tf32<A_MN, true, true, BN, false, true>;
  static bool attr = false;
  if (!attr) {
    SD_CUDA(cudaFuncSetAttribute(k_gemm_tf32<A_MN, true, true, BN, true, true>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    SD_CUDA(cudaFuncSetAttribute(k_gemm_tf32<A_MN, true, true, BN, false, true>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    attr = true;
  }
  const int grid = std::min(ep.n_tiles, kNumSMs);
  if (g.causal == 2 || g.causal == 3) {  // K-trimmed row tiles, longest first: boustrophedon deal
    ep.ncl = grid, ep.units = ep.n_tiles;
    ep.n_tiles = (ep.n_tiles + ep.ncl - 1) / ep.ncl * ep.ncl;
  }
  if (prof().on)
    prof().next_tag = std::to_string(g.M) + "," + std::to_string(2 * g.N) + "," + std::to_string(g.K) + "," +
                      std::to_string(zc) + "," + std::to_string(int(A_MN)) + ",1," + std::to_string(g.causal) +
                      ",1,split";
  prof_begin(s);
  launch_gemm_kernel(kern, unsigned(grid), unsigned(kThreadsFor<true>()), smem, s, maps[0], maps[1], maps[2], maps[3],
                     maps[4], maps[5], maps[6], maps[7], mC, mCs, mC2, mCs2, g.K, ep);
  SD_LAUNCHED("k_gemm_tf32_split");
  // algorithmic flops of the pair: A B + A B2 + A2 B
  prof_end(s, 6.0 * double(g.M) * g.N * g.K * g.Z1 * g.Z2);
}

bool env_on(const char* name) {
  const char* e = std::getenv(name);
  return !(e && e[0] == '0');
}
bool sd_gemm_wide_enabled() {
  static const bool on = env_on("SD_GEMM_WIDE");
  return on;
}
bool sd_gemm_pair_enabled() {
  static const bool on = env_on("SD_GEMM_PAIR");
  return on;
}

}  // namespace

bool twin_enabled() {  // SD_GEMM_TWIN=0: twin products as two launches
  static const bool on = [] {
    const char* e = std::getenv("SD_GEMM_TWIN");
    return !(e && e[0] == '0');
  }();
  return on;
}

void gemm(const GemmArgs& g_in, cudaStream_t s) {
  if (g_in.M <= 0 || g_in.N <= 0 || g_in.K <= 0) return;
  if (g_in.twin) {
    if (!g_in.A2 || !g_in.B2 || !g_in.C2 || g_in.split) fail(SD_ARGUMENT_ERROR, "twin gemm needs A2, B2 and C2");
    // one launch for the weight products (K = d or ff; pair kernel) and the
    // per-head score products (causal 1, 128-wide tiles; k_gemm_tf32); the
    // LM-head adjoint (K = vocab: the logits-sized A operands dominate, and
    // the twin walk re-streams them: 23 vs 15 GB measured) stays two launches
    // (measured with the boustrophedon deal: GPT-2-small at 8192 tokens
    // -3.5 ms per step, the C3 micro-batches of 2048 tokens -1.5%, the C4
    // stage's 1024-token micro-batches -0.3%)
    static const int min_m = [] {  // SD_GEMM_TWIN_MIN_M: shortest token panel for pair twins
      const char* e = std::getenv("SD_GEMM_TWIN_MIN_M");
      return e ? std::atoi(e) : 1024;
    }();
    const bool pair_ok = g_in.causal == 0 && g_in.M >= std::max(256, min_m) && g_in.N >= 256 && g_in.K <= 16384 &&
                         sd_gemm_pair_enabled();
    const bool score_ok = g_in.causal == 1 && g_in.N > 64 && g_in.M == g_in.N;
    // on-chip residuals (an operand without its residual array, e.g. the probe
    // under SD_GPT_NO_PROBE_RESIDUAL) would extend to the primal product and
    // drop its exact-B 2-MMA path: two launches then
    const bool one = twin_enabled() && (pair_ok || score_ok) && !g_in.onchip;
    if (!one) {  // C = alpha A B + beta C ; C2 = alpha2 (A2 B + A B2) + beta2 C2
      GemmArgs p = g_in;
      p.twin = false, p.A2 = p.A2s = p.B2 = p.B2s = nullptr, p.b2_exact = false, p.C2 = p.Cs2 = nullptr;
      gemm(p, s);
      GemmArgs t = g_in;
      t.twin = false;
      t.A = g_in.A2, t.As = g_in.A2s, t.lda = g_in.lda2, t.sa1 = g_in.sa1_2, t.sa2 = g_in.sa2_2;
      t.A2 = g_in.A, t.A2s = g_in.As, t.lda2 = g_in.lda, t.sa1_2 = g_in.sa1, t.sa2_2 = g_in.sa2;
      t.C = g_in.C2, t.Cs = g_in.Cs2, t.alpha = g_in.alpha2, t.beta = g_in.beta2, t.bias = g_in.bias2;
      t.C2 = t.Cs2 = nullptr;
      gemm(t, s);
      return;
    }
  }
  GemmArgs g = g_in;
  // tf32-exact B operands: their (zero) residual is never loaded; the B map
  // stands in for the residual map so the 3xTF32 path applies
  if (g.b_exact && g.As && !g.Bs) g.Bs = g.B;
  if (g.A2 && g.b2_exact && g.A2s && !g.B2s) g.B2s = g.B2;
  if (!g.A2) g.b2_exact = false;
  if (g.split) return g.a_mn ? launch_split<true>(g, s) : launch_split<false>(g, s);
  const bool pair = g.causal == 0 && g.M >= 256 && g.N >= 256 && sd_gemm_pair_enabled();
  // On-chip residuals (onchip = allowed): they halve the operand bytes through
  // L2 and TMA but add a shared-memory read + write of every staged tile, and
  // measured slower wherever residual arrays exist (K-major pair products 258
  // -> 162 TF/s; the dual weight products 176 -> 158, round-1 A/B, profiles/r01_*).
  // So they are used where arrays do not exist (attention P, dP, gS, gdS).
  (void)pair;
  if (g.onchip) {
    const bool have = g.As && g.Bs && (!g.A2 || (g.A2s && g.B2s));
    const bool prefer = false;
    if (have && !prefer) g.onchip = false;
    else g.As = g.Bs = g.A2s = g.B2s = nullptr;
  }
  const bool three = (g.As != nullptr && g.Bs != nullptr) || g.onchip;
  // large non-causal products: 256 x 256 tiles on CTA pairs (half the
  // operand bytes per flop per SM)
  if (pair) return gemm_pair(g, s);
  const bool narrow = g.N <= 64;  // head-dimension outputs: 64-wide tiles
  // 256-wide tiles halve the shared-memory operand traffic per MMA flop (the
  // tf32 SS-MMA at N=128 is shared-memory-bandwidth bound) when there are
  // enough output tiles to fill the machine.
  const long long t256 = (long long)((g.N + 255) / 256) * ((g.M + BM - 1) / BM) * g.Z1 * g.Z2;
  const bool wide = g.N >= 256 && t256 >= 2 * kNumSMs && g.causal == 0 && sd_gemm_wide_enabled();
#define SD_GEMM_CASE(AM, BMJ, TH)                                  \
  if (g.a_mn == AM && g.b_mn == BMJ && three == TH) {              \
    if (narrow) return launch<AM, BMJ, TH, 64>(g, s);              \
    if (wide) return launch<AM, BMJ, TH, 256>(g, s);               \
    return launch<AM, BMJ, TH, 128>(g, s);                         \
  }
  SD_GEMM_CASE(false, false, true)
  SD_GEMM_CASE(false, true, true)
  SD_GEMM_CASE(true, false, true)
  SD_GEMM_CASE(true, true, true)
  SD_GEMM_CASE(false, false, false)
  SD_GEMM_CASE(false, true, false)
  SD_GEMM_CASE(true, false, false)
  SD_GEMM_CASE(true, true, false)
#undef SD_GEMM_CASE
}

void split_tf32(const float* x, float* small, long long n, int mode, cudaStream_t s) {
  if (n <= 0) return;
  k_split_tf32<<<unsigned((n + 255) / 256), 256, 0, s>>>(x, small, n, mode);
  SD_LAUNCHED("k_split_tf32");
}

uint64_t gemm_scratch_generation() { return gk::g_scratch_gen.load(); }
bool gemm_profiling() { return gk::prof_on(); }

}  // namespace sd

namespace {
sd::GemmArgs args_from(const sd_gemm_desc* d) {
  sd::GemmArgs g;
  g.M = d->m;
  g.N = d->n;
  g.K = d->k;
  g.A = d->a;
  g.As = d->a_small;
  g.lda = d->lda;
  g.a_mn = d->a_mn != 0;
  g.B = d->b;
  g.Bs = d->b_small;
  g.ldb = d->ldb;
  g.b_mn = d->b_mn != 0;
  g.C = d->c;
  g.ldc = d->ldc;
  g.alpha = d->alpha;
  g.beta = d->beta;
  g.Z1 = d->z1 > 0 ? d->z1 : 1;
  g.Z2 = d->z2 > 0 ? d->z2 : 1;
  g.sa1 = d->sa1;
  g.sa2 = d->sa2;
  g.sb1 = d->sb1;
  g.sb2 = d->sb2;
  g.sc1 = d->sc1;
  g.sc2 = d->sc2;
  return g;
}
}  // namespace

extern "C" {


sd_status sd_gemm_tf32(const sd_gemm_desc* d, sd_stream s) {
  return sd::guard([&] { sd::gemm(args_from(d), (cudaStream_t)s); });
}

// Extended entry: optional dual source (d2) and flags (SD_GEMM_ONCHIP_RESIDUAL:
// 3xTF32 with the residual tiles computed in shared memory, a_small/b_small
// ignored). C = alpha (op(A1) op(B1) [+ op(A2) op(B2)]) + beta C, one launch.
sd_status sd_gemm_tf32_ex(const sd_gemm_desc* d1, const sd_gemm_desc* d2, int flags, sd_stream s) {
  return sd::guard([&] {
    if (!d1) sd::fail(SD_ARGUMENT_ERROR, "null gemm descriptor");
    const bool onchip = (flags & SD_GEMM_ONCHIP_RESIDUAL) != 0;
    sd::GemmArgs g = args_from(d1);
    g.onchip = onchip;
    g.b_exact = (flags & SD_GEMM_B_EXACT) != 0;
    g.b2_exact = (flags & SD_GEMM_B2_EXACT) != 0;
    if (onchip) g.As = g.Bs = nullptr;
    if (d2) {
      if (d1->m != d2->m || d1->n != d2->n || d1->k != d2->k || d1->a_mn != d2->a_mn || d1->b_mn != d2->b_mn ||
          (!onchip && ((d1->a_small == nullptr) != (d2->a_small == nullptr) ||
                       (d1->b_small == nullptr && !g.b_exact) != (d2->b_small == nullptr && !g.b2_exact))))
        sd::fail(SD_ARGUMENT_ERROR, "dual gemm: both products need the same shape, majors and precision");
      g.A2 = d2->a, g.lda2 = d2->lda;
      g.B2 = d2->b, g.ldb2 = d2->ldb;
      if (!onchip) g.A2s = d2->a_small, g.B2s = d2->b_small;
      g.sa1_2 = d2->sa1, g.sa2_2 = d2->sa2, g.sb1_2 = d2->sb1, g.sb2_2 = d2->sb2;
    }
    sd::gemm(g, (cudaStream_t)s);
  });
}

// Dual-source product C = alpha (op(A1) op(B1) + op(A2) op(B2)) + beta C in
// one launch (one TMEM accumulation); d2 supplies the second operand pair.
sd_status sd_gemm_tf32_dual(const sd_gemm_desc* d1, const sd_gemm_desc* d2, sd_stream s) {
  if (!d2) {
    sd::set_last_error("null gemm descriptor");
    return SD_ARGUMENT_ERROR;
  }
  return sd_gemm_tf32_ex(d1, d2, 0, s);
}

// GEMM profiling window: begin() clears; end() synchronises and returns the
// summed kernel time (ms), algorithmic flops (2MNK per launch) and launches.
sd_status sd_gemm_profile_begin(void) {
  return sd::guard([] {
    auto& p = sd::prof();
    p.on = true;
    p.used = 0;
    p.flops.clear();
    p.tags.clear();
  });
}

sd_status sd_gemm_profile_end(double* ms, double* flops, uint64_t* launches) {
  return sd::guard([&] {
    auto& p = sd::prof();
    p.on = false;
    double t = 0, f = 0;
    for (size_t i = 0; i + 1 < p.used; i += 2) {
      SD_CUDA(cudaEventSynchronize(p.ev[i + 1]));
      float x = 0;
      SD_CUDA(cudaEventElapsedTime(&x, p.ev[i], p.ev[i + 1]));
      t += x;
    }
    for (double x : p.flops) f += x;
    *ms = t;
    *flops = f;
    *launches = p.flops.size();
  });
}

// Per-launch record of the last profiling window as CSV lines
// "M,N,K,batch,a_mn,b_mn,causal,splits,ms,flops" (call after profile_end).
sd_status sd_gemm_profile_dump(const char* path) {
  return sd::guard([&] {
    auto& p = sd::prof();
    FILE* f = std::fopen(path, "w");
    if (!f) sd::fail(SD_ARGUMENT_ERROR, "cannot open profile dump path");
    std::fprintf(f, "M,N,K,batch,a_mn,b_mn,causal,splits,nsrc,ms,flops\n");
    for (size_t i = 0; i + 1 < p.used; i += 2) {
      float x = 0;
      SD_CUDA(cudaEventElapsedTime(&x, p.ev[i], p.ev[i + 1]));
      std::fprintf(f, "%s,%.6f,%.0f\n", p.tags[i / 2].c_str(), x, p.flops[i / 2]);
    }
    std::fclose(f);
  });
}

sd_status sd_split_tf32(const float* x, float* small, uint64_t n, int mode, sd_stream s) {
  return sd::guard([&] { sd::split_tf32(x, small, (long long)n, mode, (cudaStream_t)s); });
}

}  // extern "C"

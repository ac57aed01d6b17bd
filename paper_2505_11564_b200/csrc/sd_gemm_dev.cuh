// Device helpers shared by the 1-CTA and CTA-pair tcgen05 GEMM kernels
// (sd_gemm.cu, sd_gemm_pair.cu): mbarriers, TMA, UMMA descriptors, TMEM
// loads, epilogue parameters and the persistent tile walk.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <string>
#include <utility>

#include "sd_common.cuh"
#include "sd_gemm.h"

namespace sd {
namespace gk {


// BK = 16 fp32 (64 B) per stage keeps a 6-deep ring of 4 operand tiles in
// 192 KB of shared memory: enough bytes in flight to cover TMA latency.
constexpr int BM = 128, BK = 16;
constexpr int NUM_THREADS = 384;  // producer, MMA, 2 residual warps, 8 epilogue warps
constexpr int kConvWarps = 2;     // warps 2-3: on-chip tf32 residuals of the staged operands
constexpr int kNumSMs = 148;

// Tile-width dependent constants: BN = 128 for general products, BN = 64 for
// the per-head attention products whose N is the head dimension (64).
template <int BN_>
struct Cfg {
  static constexpr int BN = BN_;
  static constexpr int A_BYTES = BM * BK * 4;         // 8 KB per A tile
  static constexpr int B_BYTES = BN_ * BK * 4;        // 8 / 4 KB per B tile
  static constexpr int STAGES = BN_ == 256 ? 4 : (BN_ == 128 ? 6 : 8);  // <= 192 KB ring
  static constexpr uint32_t TMEM_COLS = 2 * BN_;      // two accumulation buffers
  static constexpr int EC = BN_ / 2;                  // accumulator columns per epilogue thread
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t"
      ".reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t"
      "}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Warp-wide producer forms: every lane runs the loop, one elected lane issues.
__device__ __forceinline__ void mbar_expect_tx_e(uint64_t* bar, uint32_t bytes) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n\t}" ::"r"(smem_u32(bar)),
      "r"(bytes)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d_e(const CUtensorMap* map, uint64_t* bar, void* dst, int c0, int c1,
                                              int c2, int c3) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], "
      "[%2];\n\t}" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
__device__ __forceinline__ void tma_load_5d_e(const CUtensorMap* map, uint64_t* bar, void* dst, int c0, int c1,
                                              int c2, int c3, int c4) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, "
      "%7}], [%2];\n\t}" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
      : "memory");
}

// UMMA shared-memory matrix descriptor. Layout codes: 4 = SWIZZLE_64B (K-major
// tiles), 1 = SWIZZLE_128B_BASE32B (MN-major tf32 tiles: the only MN-major
// smem layout the tf32 MMA accepts).
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= uint64_t((saddr >> 4) & 0x3FFF);
  d |= uint64_t((lbo >> 4) & 0x3FFF) << 16;
  d |= uint64_t((sbo >> 4) & 0x3FFF) << 32;
  d |= uint64_t(1) << 46;  // descriptor version (sm_100)
  d |= uint64_t(layout) << 61;
  return d;
}

// Instruction descriptor: kind::tf32, fp32 accumulate, M=128, N=bn.
__host__ __device__ constexpr uint32_t make_idesc(bool a_mn, bool b_mn, int bn, int m = BM) {
  return (1u << 4)                 // D format F32
         | (2u << 7)               // A format TF32
         | (2u << 10)              // B format TF32
         | (uint32_t(a_mn) << 15)  // A major
         | (uint32_t(b_mn) << 16)  // B major
         | (uint32_t(bn >> 3) << 17) | (uint32_t(m >> 4) << 24);
}

// 16 consecutive 32-bit TMEM columns of this thread's lane (warp = its 32-lane quarter)
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}

// Warp-wide issue forms: every lane runs the (uniform) descriptor math and one
// elected lane issues -- no per-instruction waterfall around divergent code.
__device__ __forceinline__ void mma_tf32_e(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t"
      ".reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t"
      "}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
// A operand from tensor memory (M lanes x 8 tf32 columns at a_tmem), B from shared memory
__device__ __forceinline__ void mma_tf32_ta_e(uint32_t tmem_d, uint32_t a_tmem, uint64_t db, uint32_t idesc,
                                              uint32_t acc) {
  asm volatile(
      "{\n\t"
      ".reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t"
      "}" ::"r"(tmem_d),
      "r"(a_tmem), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit_e(uint64_t* bar) {
  asm volatile(
      "{\n\t"
      ".reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t"
      "}" ::"r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}

struct EpiParams {
  float* C;
  long long ldc, sc1, sc2;
  int M, N, Z1;
  float alpha, beta;
  const float* bias;  // per output column, may be null
  float* Cs;          // residual output, may be null
  float* dbg;         // debug hook (unused by the persistent kernel)
  int zcount, kb_per;  // batch count; k-blocks per split
  float* ws;           // split-K: raw partial tiles [split][z][M][N] (else null)
  int causal;          // 0 none, 1 lower output, 2 lower-triangular A, 3 upper-triangular A
  int n_tiles_n, n_tiles_m, n_tiles;  // tile grid (n fastest), n_tiles over all (split, z)
  int nsrc;                           // 1, or 2 for a dual-source product
  int res;                            // 3xTF32 residuals computed on chip from the staged raw tiles
  int tma_store;                      // C = alpha acc written by TMA from smem (beta 0, no bias/Cs/split)
  int mn5;                            // bit 0 / 1: MN-major A / B tile as one 5-D TMA box
  int bexact;                         // bit 0 / 1: source 1 / 2 B operand exact in tf32 (bf16-valued
                                      // weights): no B residual load, no A.B_lo MMA
  int split;                          // merged 64-wide pair (GemmArgs::split): source 1 fills the
                                      // 128 accumulator columns [A B | A B2], source 2 adds A2 B into
                                      // columns 64-127; k-blocks interleave 1, 2, 1, 2, ...
  float *C2, *Cs2;                    // split: output of columns 64-127
  int tma_add;                        // TMA-store epilogue, bit 0 / 1: C / C2 accumulate (beta 1) by reduce-add
  int group;                          // grouped tile walk (raster_group): > 0 groups of `group` m tiles,
                                      // m fastest inside a group; < 0 groups of -group n tiles, n fastest
                                      // inside; 0 n fastest over the whole grid
  int twin, tiles1;                   // twin products (GemmArgs::twin): tiles [0, tiles1) are C2's
                                      // (sources A2 B, A B2), [tiles1, 2 tiles1) C's (source A B)
  float alpha2, beta2;                // twin: C2's epilogue
  const float* bias2;
  float* ws2;                         // twin: C2's split-K partials
  int ncl, units;                     // boustrophedon deal (deal_unit): worker slots of the launch
                                      // (CTAs / clusters) and the real units; n_tiles is then padded
                                      // to whole rounds; ncl 0: plain round robin
};

// Launches whose units differ in cost -- a twin launch's two-source C2 tiles
// then one-source C tiles, the causal K-trimmed attention products' row tiles
// from the longest to the shortest -- deal them to the persistent workers in
// boustrophedon order: round r of the static round robin walks the workers
// forward for even r and backward for odd r, so the workers that drew the
// last expensive units draw the first cheap ones (e.g. 96 + 96 twin units on
// 74 clusters: busiest worker 4 instead of 5 unit-costs). Returns the unit of
// slot t, or -1 past the last unit.
__device__ __forceinline__ int deal_unit(const EpiParams& ep, int t) {
  if (ep.ncl == 0) return t;
  const int r = t / ep.ncl, p = t - r * ep.ncl;
  const int u = r * ep.ncl + ((r & 1) ? ep.ncl - 1 - p : p);
  return u < ep.units ? u : -1;
}

// Rasterisation. A persistent wave of clusters works on consecutive tile
// indices, so the walk order decides which operand stays in L2: with n
// fastest, every m row re-streams the whole B panel from HBM unless B stays
// cached. When A is the smaller operand, raster_group walks groups of G row
// tiles, m fastest inside a group, with G row panels filling a ~40 MB slice
// of the 126 MB L2 (SD_GEMM_L2_MB): B is then streamed ceil(tiles_m / G)
// times instead of tiles_m times. E.g. the LM-head product (A = 8192 x 768
// activations + tangents, B = 50257 x 768 tied embedding + its tangent, with
// tf32 residuals) walks groups of 12 of its 32 row tiles: 21.9 -> 8.7 GB of
// DRAM traffic (ncu). When B is the smaller operand the n-fastest walk
// already streams A once and keeps B hot.
inline int raster_group(long long M, long long N, long long K, int BMr, int tiles_m, int tiles_n, int a_copies,
                        int b_copies) {
  static const double budget = [] {
    const char* e = std::getenv("SD_GEMM_L2_MB");
    return (e ? std::atof(e) : 40.0) * 1024 * 1024;
  }();
  const double a_total = double(M) * K * 4.0 * a_copies, b_total = double(N) * K * 4.0 * b_copies;
  // B the smaller operand: the plain n-fastest walk keeps the B panel hot
  // while the A rows stream through once
  if (b_total < a_total || tiles_m < 2 || tiles_n < 2) return 0;
  const double panel = double(BMr) * K * 4.0 * a_copies;
  return int(std::max(1.0, std::min(double(tiles_m), budget / panel)));
}
inline int walk_group(const GemmArgs& g, int BMr, int BNc, int tiles_m, int tiles_n, bool three) {
  static const int on = [] {
    const char* e = std::getenv("SD_GEMM_RASTER");  // 0: always n fastest (the round-1 walk)
    return !(e && e[0] == '0');
  }();
  if (!on) return 0;
  const int dual = g.A2 ? 2 : 1;
  const int ac = dual * ((three && g.As) ? 2 : 1);
  const int bc = dual * ((three && g.Bs && !g.b_exact) ? 2 : 1);
  (void)BNc;
  return raster_group(g.M, g.N, g.K, BMr, tiles_m, tiles_n, ac, bc);
}
// tile t of the (m, n) grid (zz = batch/split index) under the grouped walk
__device__ __forceinline__ void walk_tile(const EpiParams& ep, int t, int& mt, int& nt, int& zz) {
  const int tm = ep.n_tiles_m, tn = ep.n_tiles_n, per = tm * tn;
  zz = t / per;
  const int r0 = t - zz * per;
  if (ep.group > 0) {
    const int G = ep.group, g = r0 / (G * tn), r = r0 - g * G * tn, gm = min(G, tm - g * G);
    mt = g * G + r % gm;
    nt = r / gm;
  } else if (ep.group < 0) {
    const int G = -ep.group, g = r0 / (G * tm), r = r0 - g * G * tm, gn = min(G, tn - g * G);
    nt = g * G + r % gn;
    mt = r / gn;
  } else {
    nt = r0 % tn;
    mt = r0 / tn;
  }
}

__device__ __forceinline__ void fence_proxy_async_smem_decl() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// TMA store of a staged 32 x 32 fp32 box (128B-swizzled smem) to C
__device__ __forceinline__ void tma_store_4d(const CUtensorMap* map, const void* src, int c0, int c1, int c2, int c3) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(map),
               "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
               : "memory");
}
// ... or added element-wise to C in place (fp32 reduce-add, one writer per element)
__device__ __forceinline__ void tma_store_add_4d(const CUtensorMap* map, const void* src, int c0, int c1, int c2,
                                                 int c3) {
  asm volatile("cp.reduce.async.bulk.tensor.4d.global.shared::cta.add.tile.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(map),
               "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// explicit shared-space vector accesses (a generic pointer into the dynamic
// smem ring compiles to LD.E / ST.E through the L1TEX long-scoreboard path)
__device__ __forceinline__ float4 lds128(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts128(uint32_t a, float4 v) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}
__device__ __forceinline__ float lds32(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
  return v;
}

// One warp's 32 rows x EC columns (thread = row) of o = alpha*acc (+ bias)
// -- and, if requested, the tf32 residual of o into Cs -- through a 4 KB
// 128B-swizzled staging box and TMA stores (full lines; OOB clipped).
// BOXC = 32 (128 B rows, SWIZZLE_128B: chunk c of row r at c ^ (r & 7)) or
// 16 (64 B rows, SWIZZLE_64B: chunk c at c ^ ((r >> 1) & 3)).
template <int EC, int BOXC = 32>
__device__ __forceinline__ void warp_tma_store(const CUtensorMap* mC, const CUtensorMap* mCs, float* stage,
                                               const float (&acc)[EC], float alpha, const float* bias, int lane,
                                               int row0, int col0, int z1, int z2, bool add) {
  constexpr int NQ = BOXC / 4;  // 16 B chunks per staged row
  const int sw = BOXC == 32 ? (lane & 7) : ((lane >> 1) & 3);
  const uint32_t rowa = smem_u32(stage + lane * BOXC);
  bool pending = false;
#pragma unroll
  for (int c0 = 0; c0 < EC; c0 += BOXC) {
    float o[BOXC];
#pragma unroll
    for (int q = 0; q < BOXC; ++q) o[q] = alpha * acc[c0 + q];
    if (bias) {
      const float4* b4 = reinterpret_cast<const float4*>(bias + col0 + c0);
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const float4 bb = b4[q];
        o[4 * q] += bb.x, o[4 * q + 1] += bb.y, o[4 * q + 2] += bb.z, o[4 * q + 3] += bb.w;
      }
    }
#pragma unroll
    for (int pass = 0; pass < 2; ++pass) {
      if (pass == 1 && !mCs) break;
      if (pending) {  // the previous box must have left the staging buffer
        if (lane == 0) bulk_wait_read0();
        __syncwarp();
      }
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        float4 v = make_float4(o[4 * q], o[4 * q + 1], o[4 * q + 2], o[4 * q + 3]);
        if (pass == 1) {
          v.x -= __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u);
          v.y -= __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u);
          v.z -= __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u);
          v.w -= __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u);
        }
        sts128(rowa + 16u * uint32_t(q ^ sw), v);
      }
      fence_proxy_async_smem_decl();
      __syncwarp();
      if (lane == 0) {
        if (add && pass == 0) tma_store_add_4d(mC, stage, col0 + c0, row0, z1, z2);  // C += o (beta 1)
        else tma_store_4d(pass ? mCs : mC, stage, col0 + c0, row0, z1, z2);
        bulk_commit();
      }
      pending = true;
    }
  }
}

// x - trunc_tf32(x) over a staged operand tile (any smem layout: the residual
// is elementwise), written to the tile's residual slot; threads t of nt.
__device__ __forceinline__ void stage_residual(const unsigned char* src, unsigned char* dst, int bytes, int t, int nt) {
  const uint32_t s0 = smem_u32(src), d0 = smem_u32(dst);
#pragma unroll 4
  for (int i = t; i < bytes / 16; i += nt) {
    const float4 v = lds128(s0 + 16u * i);
    float4 r;
    r.x = v.x - __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u);
    r.y = v.y - __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u);
    r.z = v.z - __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u);
    r.w = v.w - __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u);
    sts128(d0 + 16u * i, r);
  }
}
// generic-proxy smem writes -> visible to the tensor core (async proxy)
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Descriptor of k-step `ks` (8 tf32 = 32 B of K) of an operand tile.
// K-major: 128 rows x 64 B, SWIZZLE_64B in 8-row (512 B) atoms: advance 32 B
// per k-step, SBO = 512 B. MN-major: four 32-element chunks of [16 k-rows x
// 128 B] swizzled in 4-row (512 B) atoms of 32 B granules: advance 8 rows =
// 1024 B per k-step, LBO = 2048 B between MN chunks, SBO = 512 B.
template <bool MN>
__device__ __forceinline__ uint64_t tile_desc(uint32_t base, int ks) {
  if (MN) return make_desc(base + ks * 1024, 2048, 512, 1);
  return make_desc(base + ks * 32, 16, 512, 4);
}

// The tensor core's fp32 accumulation is not round-to-nearest (its error grows
// ~linearly with the number of accumulated MMAs). To stay fp32-faithful at
// K = 8192 the K loop is cut into chunks of KC k-blocks: each chunk
// accumulates in one of two TMEM buffers, and the epilogue warps drain every
// finished chunk into round-to-nearest fp32 registers while the MMA warp
// fills the other buffer (chunks continue across the tiles of a CTA).
constexpr int KC = 8;  // k-blocks (8 x 16 = 128 of K) per TMEM chunk
static_assert(KC % 2 == 0, "split products interleave the two sources: a chunk must start with source 1");

struct TileInfo {
  int n0, m0, z, split, kb0, num_kb;
  bool skip;
  bool tan = false;  // twin: a C2 (two-source) tile
  int nsrc = 1;      // sources of this tile
};

template <int BN, bool CAUSAL>
__device__ __forceinline__ TileInfo tile_info(const EpiParams& ep, int t, int K) {
  TileInfo ti;
  int nt, mt, zz;
  t = deal_unit(ep, t);
  if (t < 0) {
    ti.skip = true;
    return ti;
  }
  // twin (causal 0 / 1 only): units [0, tiles1) are C2's tiles, then C's
  ti.tan = ep.twin && t < ep.tiles1;
  if (ep.twin && !ti.tan) t -= ep.tiles1;
  if (CAUSAL && ep.causal == 1 && BN == BM) {
    // only the tm (tm + 1) / 2 lower-triangle tiles of each square head are
    // enumerated: every CTA of the round-robin gets equal work
    const int per = ep.n_tiles_m * (ep.n_tiles_m + 1) / 2;
    const int q = t % per;
    zz = t / per;
    int m = int((sqrtf(8.0f * q + 1.0f) - 1.0f) * 0.5f);
    while ((m + 1) * (m + 2) / 2 <= q) ++m;
    while (m * (m + 1) / 2 > q) --m;
    mt = m;
    nt = q - m * (m + 1) / 2;
  } else if (CAUSAL && (ep.causal == 2 || ep.causal == 3)) {
    // K range grows (2) / shrinks (3) with the row tile: walk the row tiles
    // from the longest to the shortest, so that each round-robin wave holds
    // tiles of (nearly) equal cost
    const int per = (ep.ncl ? ep.units : ep.n_tiles) / ep.n_tiles_m;  // n tiles x (split, z)
    const int mi = t / per, rem = t % per;
    mt = ep.causal == 2 ? ep.n_tiles_m - 1 - mi : mi;
    nt = rem % ep.n_tiles_n;
    zz = rem / ep.n_tiles_n;
  } else {
    walk_tile(ep, t, mt, nt, zz);
  }
  ti.nsrc = ep.twin ? (ti.tan ? 2 : 1) : ep.nsrc;
  ti.n0 = nt * BN;
  ti.m0 = mt * BM;
  ti.z = zz % ep.zcount;
  ti.split = zz / ep.zcount;
  ti.kb0 = ti.split * ep.kb_per;
  ti.num_kb = min(ep.kb_per, (K + BK - 1) / BK - ti.kb0);
  // Causal attention structure (square S x S per head, tile-aligned):
  //  1: C[i][j] is only needed for j <= i -> tiles strictly above the diagonal skip;
  //  2: A[i][k] is zero for k > i  -> K range [0, m0 + BM);
  //  3: A[i][k] is zero for k < i  -> K range [m0, K).
  ti.skip = false;
  if (CAUSAL) {
    ti.skip = (ep.causal == 1 && ti.n0 > ti.m0 + BM - 1);
    if (ep.causal == 2) ti.num_kb = min(ti.num_kb, (ti.m0 + BM + BK - 1) / BK - ti.kb0);
    if (ep.causal == 3) {
      const int lo = ti.m0 / BK;
      ti.num_kb -= max(0, lo - ti.kb0);
      ti.kb0 = max(ti.kb0, lo);
    }
  }
  if (ti.num_kb <= 0) ti.skip = true;
  return ti;
}


// Epilogue of one output row segment [n0, n0 + EC) held by one thread:
// C = alpha acc + beta C + bias (and the tf32 residual Cs of the result), or
// the raw split-K partial.
template <int EC>
__device__ __forceinline__ void store_row(const EpiParams& ep, const TileInfo& ti, int row, int n0,
                                          const float (&acc)[EC]) {
  if (row >= ep.M) return;
  const int z1 = ti.z % ep.Z1, z2 = ti.z / ep.Z1;
  const int nvalid = ep.N - n0;
  if (nvalid <= 0) return;
  if (ep.ws) {
    // split-K partial: raw accumulator, dense [M][N] per (split, z)
    float* prow = ep.ws + ((long long)ti.split * ep.zcount + ti.z) * ((long long)ep.M * ep.N) +
                  (long long)row * ep.N + n0;
    if (nvalid >= EC && (ep.N & 3) == 0) {
#pragma unroll
      for (int j = 0; j < EC; j += 4)
        *reinterpret_cast<float4*>(prow + j) = make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
    } else {
#pragma unroll
      for (int j = 0; j < EC; ++j)
        if (j < nvalid) prow[j] = acc[j];
    }
    return;
  }
  const long long off = z1 * ep.sc1 + z2 * ep.sc2 + (long long)row * ep.ldc + n0;
  float* crow = ep.C + off;
  float* srow = ep.Cs ? ep.Cs + off : nullptr;
  const float* brow = ep.bias ? ep.bias + n0 : nullptr;
  const bool vec = nvalid >= EC && ((reinterpret_cast<uintptr_t>(crow) & 15) == 0) &&
                   (!srow || (reinterpret_cast<uintptr_t>(srow) & 15) == 0);
  if (vec) {
#pragma unroll
    for (int j = 0; j < EC; j += 4) {
      float4 o = make_float4(ep.alpha * acc[j], ep.alpha * acc[j + 1], ep.alpha * acc[j + 2], ep.alpha * acc[j + 3]);
      if (ep.beta != 0.0f) {
        const float4 old = *reinterpret_cast<const float4*>(crow + j);
        o.x += ep.beta * old.x;
        o.y += ep.beta * old.y;
        o.z += ep.beta * old.z;
        o.w += ep.beta * old.w;
      }
      if (brow) {
        o.x += brow[j];
        o.y += brow[j + 1];
        o.z += brow[j + 2];
        o.w += brow[j + 3];
      }
      *reinterpret_cast<float4*>(crow + j) = o;
      if (srow) {
        const float4 r = make_float4(o.x - __uint_as_float(__float_as_uint(o.x) & 0xFFFFE000u),
                                     o.y - __uint_as_float(__float_as_uint(o.y) & 0xFFFFE000u),
                                     o.z - __uint_as_float(__float_as_uint(o.z) & 0xFFFFE000u),
                                     o.w - __uint_as_float(__float_as_uint(o.w) & 0xFFFFE000u));
        *reinterpret_cast<float4*>(srow + j) = r;
      }
    }
  } else {
#pragma unroll
    for (int j = 0; j < EC; ++j) {
      if (j < nvalid) {
        float r = ep.alpha * acc[j];
        if (ep.beta != 0.0f) r += ep.beta * crow[j];
        if (brow) r += brow[j];
        crow[j] = r;
        if (srow) srow[j] = r - __uint_as_float(__float_as_uint(r) & 0xFFFFE000u);
      }
    }
  }
}

// ---- host helpers (sd_gemm.cu)
void make_map(CUtensorMap* m, const float* base, long long inner, long long outer, long long ld, int Z1,
              long long s1, int Z2, long long s2, int box_inner, int box_outer, bool mn_major);
// box_cols x 32 fp32 boxes (32: 128B swizzle, 16: 64B): the epilogue's TMA store map of C
void make_store_map(CUtensorMap* m, float* C, const GemmArgs& g, int box_cols = 32);
// whether a product may take the TMA-store epilogue (beta 0, aligned C/Cs/bias, no split)
bool tma_store_ok(const GemmArgs& g, int splits, int bias_cols, bool allow_add = false);
float* splitk_workspace(size_t floats);
int choose_splits(int tiles, int units, int total_kb, int nsrc, double t_kb, double out_bytes);
int choose_splits_twin(int tiles, int units, int total_kb, double t_kb, double out_bytes);
void operand_maps(const GemmArgs& g, bool a_mn, bool b_mn, bool three, int box_n, CUtensorMap* m, int* mn5);
bool prof_on();
void prof_tag(const std::string& tag);
void prof_begin(cudaStream_t s);
void prof_end(cudaStream_t s, double flops);
void launch_splitk_reduce(const float* ws, int splits, int zc, const GemmArgs& g, cudaStream_t s);
// CTA-pair (cta_group::2) 256 x 256 tiles (sd_gemm_pair.cu)
void gemm_pair(const GemmArgs& g, cudaStream_t s);

// GEMM launches carry the programmatic-stream-serialization attribute (PDL):
// the kernel's prologue may start during the previous kernel's tail and waits
// (griddepcontrol.wait) before touching global memory. SD_GEMM_PDL=0 turns it off.
bool pdl_on();
template <typename... P, typename... A>
void launch_gemm_kernel(void (*kern)(P...), unsigned grid, unsigned threads, size_t smem, cudaStream_t s,
                        A&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_on() ? 1 : 0;
  SD_CUDA(cudaLaunchKernelEx(&cfg, kern, std::forward<A>(args)...));
}

}  // namespace gk
}  // namespace sd

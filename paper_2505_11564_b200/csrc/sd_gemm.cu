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
// Persistent warp-specialised kernel, one CTA per SM, 128 x 128 output tiles
// walked in a static round-robin schedule:
//   warp 0   : TMA producer (cp.async.bulk.tensor) into a STAGES-deep smem
//              ring (full/empty mbarriers), running ahead across tiles;
//   warp 1   : TMEM allocator + single-thread tcgen05.mma issuer;
//   warps 2-5: epilogue: drain TMEM chunks (tcgen05.ld 32x32b) into
//              round-to-nearest fp32 registers, then alpha/beta/bias,
//              residual and store — overlapped with the next tile's MMAs.
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
#include <mutex>
#include <vector>

#include "sd_common.cuh"
#include "sd_gemm.h"

namespace sd {

namespace {

// BK = 16 fp32 (64 B) per stage keeps a 6-deep ring of 4 operand tiles in
// 192 KB of shared memory: enough bytes in flight to cover TMA latency.
constexpr int BM = 128, BK = 16;
constexpr int NUM_THREADS = 320;  // producer, MMA, 8 epilogue warps
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
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
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

__device__ __forceinline__ void tma_load_4d(const CUtensorMap* map, uint64_t* bar, void* dst, int c0, int c1, int c2,
                                            int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];" ::
          "r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
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
__host__ __device__ constexpr uint32_t make_idesc(bool a_mn, bool b_mn, int bn) {
  return (1u << 4)                 // D format F32
         | (2u << 7)               // A format TF32
         | (2u << 10)              // B format TF32
         | (uint32_t(a_mn) << 15)  // A major
         | (uint32_t(b_mn) << 16)  // B major
         | (uint32_t(bn >> 3) << 17) | (uint32_t(BM >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t"
      ".reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t"
      "}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
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
};

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

struct TileInfo {
  int n0, m0, z, split, kb0, num_kb;
  bool skip;
};

template <int BN>
__device__ __forceinline__ TileInfo tile_info(const EpiParams& ep, int t, int K) {
  TileInfo ti;
  const int nt = t % ep.n_tiles_n;
  const int mt = (t / ep.n_tiles_n) % ep.n_tiles_m;
  const int zz = t / (ep.n_tiles_n * ep.n_tiles_m);
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
  ti.skip = (ep.causal == 1 && ti.n0 > ti.m0 + BM - 1);
  if (ep.causal == 2) ti.num_kb = min(ti.num_kb, (ti.m0 + BM + BK - 1) / BK - ti.kb0);
  if (ep.causal == 3) {
    const int lo = ti.m0 / BK;
    ti.num_kb -= max(0, lo - ti.kb0);
    ti.kb0 = max(ti.kb0, lo);
  }
  if (ti.num_kb <= 0) ti.skip = true;
  return ti;
}

template <bool A_MN, bool B_MN, bool THREE, int BN_>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    k_gemm_tf32(const __grid_constant__ CUtensorMap mA, const __grid_constant__ CUtensorMap mAs,
                const __grid_constant__ CUtensorMap mB, const __grid_constant__ CUtensorMap mBs, int K, EpiParams ep) {
  using Cf = Cfg<BN_>;
  constexpr int BN = Cf::BN, STAGES = Cf::STAGES, EC = Cf::EC;
  constexpr int A_BYTES = Cf::A_BYTES, B_BYTES = Cf::B_BYTES;
  constexpr uint32_t TMEM_COLS = Cf::TMEM_COLS;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1024-byte aligned ring: per stage [A | As | B | Bs]
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int STAGE_BYTES = (THREE ? 2 : 1) * (A_BYTES + B_BYTES);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;  // [2]
  uint64_t* tempty = tfull + 2;      // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
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

  if (warp == 0) {
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&mA) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&mB) : "memory");
      uint32_t g = 0;  // global k-block counter (ring position)
      for (int t = blockIdx.x; t < ep.n_tiles; t += gridDim.x) {
        const TileInfo ti = tile_info<BN>(ep, t, K);
        if (ti.skip) continue;
        const int z1 = ti.z % ep.Z1, z2 = ti.z / ep.Z1;
        for (int kb = 0; kb < ti.num_kb; ++kb, ++g) {
          const int s = g % STAGES;
          const uint32_t ph = (g / STAGES) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          unsigned char* st = smem + s * STAGE_BYTES;
          mbar_expect_tx(&full[s], STAGE_BYTES);
          const int k0 = (ti.kb0 + kb) * BK;
          if (A_MN) {
#pragma unroll
            for (int c = 0; c < BM / 32; ++c) {
              tma_load_4d(&mA, &full[s], st + c * 2048, ti.m0 + 32 * c, k0, z1, z2);
              if (THREE) tma_load_4d(&mAs, &full[s], st + A_BYTES + c * 2048, ti.m0 + 32 * c, k0, z1, z2);
            }
          } else {
            tma_load_4d(&mA, &full[s], st, k0, ti.m0, z1, z2);
            if (THREE) tma_load_4d(&mAs, &full[s], st + A_BYTES, k0, ti.m0, z1, z2);
          }
          unsigned char* sb = st + (THREE ? 2 : 1) * A_BYTES;
          if (B_MN) {
#pragma unroll
            for (int c = 0; c < BN / 32; ++c) {
              tma_load_4d(&mB, &full[s], sb + c * 2048, ti.n0 + 32 * c, k0, z1, z2);
              if (THREE) tma_load_4d(&mBs, &full[s], sb + B_BYTES + c * 2048, ti.n0 + 32 * c, k0, z1, z2);
            }
          } else {
            tma_load_4d(&mB, &full[s], sb, k0, ti.n0, z1, z2);
            if (THREE) tma_load_4d(&mBs, &full[s], sb + B_BYTES, k0, ti.n0, z1, z2);
          }
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = make_idesc(A_MN, B_MN, BN);
    uint32_t g = 0, chunk = 0;
    for (int t = blockIdx.x; t < ep.n_tiles; t += gridDim.x) {
      const TileInfo ti = tile_info<BN>(ep, t, K);
      if (ti.skip) continue;
      for (int kb = 0; kb < ti.num_kb; ++kb, ++g) {
        const int s = g % STAGES;
        const uint32_t ph = (g / STAGES) & 1;
        const bool first = (kb % KC) == 0;
        const bool last = (kb % KC) == KC - 1 || kb == ti.num_kb - 1;
        const uint32_t buf = chunk & 1;
        if (first && chunk >= 2) mbar_wait(&tempty[buf], ((chunk >> 1) - 1) & 1);
        mbar_wait(&full[s], ph);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (lane == 0) {
          const uint32_t d = tmem + buf * BN;
          const uint32_t st = smem_u32(smem + s * STAGE_BYTES);
          const uint32_t a = st, as = st + A_BYTES;
          const uint32_t b = st + (THREE ? 2 : 1) * A_BYTES, bs = b + B_BYTES;
#pragma unroll
          for (int ks = 0; ks < BK / 8; ++ks) {
            const uint32_t acc0 = (first && ks == 0) ? 0u : 1u;
            if (THREE) {
              mma_tf32(d, tile_desc<A_MN>(as, ks), tile_desc<B_MN>(b, ks), idesc, acc0);
              mma_tf32(d, tile_desc<A_MN>(a, ks), tile_desc<B_MN>(bs, ks), idesc, 1u);
              mma_tf32(d, tile_desc<A_MN>(a, ks), tile_desc<B_MN>(b, ks), idesc, 1u);
            } else {
              mma_tf32(d, tile_desc<A_MN>(a, ks), tile_desc<B_MN>(b, ks), idesc, acc0);
            }
          }
          mma_commit(&empty[s]);
          if (last) mma_commit(&tfull[buf]);
        }
        __syncwarp();
        if (last) ++chunk;
      }
    }
  } else {
    // epilogue: 8 warps; warp w drains TMEM lanes 32*(w%4) .. +31 (its
    // sub-partition) and the column half (w-2)/4 of the tile: thread = one
    // output row, EC = BN/2 fp32 accumulators in registers.
    const int sub = warp & 3;
    const int cb = ((warp - 2) >> 2) * EC;
    uint32_t chunk = 0;
    for (int t = blockIdx.x; t < ep.n_tiles; t += gridDim.x) {
      const TileInfo ti = tile_info<BN>(ep, t, K);
      if (ti.skip) continue;
      const int row = ti.m0 + sub * 32 + lane;
      float acc[EC];
#pragma unroll
      for (int j = 0; j < EC; ++j) acc[j] = 0.0f;
      const int nchunks = (ti.num_kb + KC - 1) / KC;
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
      if (row >= ep.M) continue;
      const int z1 = ti.z % ep.Z1, z2 = ti.z / ep.Z1;
      const int n0 = ti.n0 + cb;
      const int nvalid = ep.N - n0;
      if (nvalid <= 0) continue;
      if (ep.ws) {
        // split-K partial: raw accumulator, dense [M][N] per (split, z)
        float* prow = ep.ws + ((long long)ti.split * ep.zcount + ti.z) * ((long long)ep.M * ep.N) +
                      (long long)row * ep.N + n0;
#pragma unroll
        for (int j = 0; j < EC; ++j)
          if (j < nvalid) prow[j] = acc[j];
        continue;
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
  }
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

// C = alpha * sum_split partial[split] + beta * C + bias (fixed split order)
__global__ void k_splitk_reduce(const float* __restrict__ ws, int splits, int zc, int Z1, int M, int N,
                                float* __restrict__ C, long long ldc, long long sc1, long long sc2, float alpha,
                                float beta, const float* __restrict__ bias, float* __restrict__ Cs) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long mn = (long long)M * N;
  if (i >= (long long)zc * mn) return;
  const int z = int(i / mn);
  const long long rc = i - z * mn;
  const int row = int(rc / N), col = int(rc % N);
  float acc = 0.f;
  for (int sp = 0; sp < splits; ++sp) acc += ws[((long long)sp * zc + z) * mn + rc];
  float* c = C + (z % Z1) * sc1 + (z / Z1) * sc2 + (long long)row * ldc + col;
  float r = alpha * acc;
  if (beta != 0.0f) r += beta * *c;
  if (bias) r += bias[col];
  *c = r;
  if (Cs) Cs[c - C] = r - __uint_as_float(__float_as_uint(r) & 0xFFFFE000u);
}

// Split-K scratch: one lazily grown device buffer. GEMMs of this library are
// issued on one stream in program order, so consecutive calls never overlap.
float* splitk_workspace(size_t floats) {
  static float* buf = nullptr;
  static size_t cap = 0;
  if (floats > cap) {
    if (buf) SD_CUDA(cudaFree(buf));
    SD_CUDA(cudaMalloc(&buf, floats * sizeof(float)));
    cap = floats;
  }
  return buf;
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

template <bool A_MN, bool B_MN, bool THREE, int BN>
void launch(const GemmArgs& g, cudaStream_t s) {
  using Cf = Cfg<BN>;
  CUtensorMap mA, mAs, mB, mBs;
  // A logical M x K. K-major: rows = M (ld = lda), inner = K. MN-major: rows = K, inner = M.
  if (A_MN) {
    make_map(&mA, g.A, g.M, g.K, g.lda, g.Z1, g.sa1, g.Z2, g.sa2, 32, BK, true);
    make_map(&mAs, THREE ? g.As : g.A, g.M, g.K, g.lda, g.Z1, g.sa1, g.Z2, g.sa2, 32, BK, true);
  } else {
    make_map(&mA, g.A, g.K, g.M, g.lda, g.Z1, g.sa1, g.Z2, g.sa2, BK, BM, false);
    make_map(&mAs, THREE ? g.As : g.A, g.K, g.M, g.lda, g.Z1, g.sa1, g.Z2, g.sa2, BK, BM, false);
  }
  if (B_MN) {
    make_map(&mB, g.B, g.N, g.K, g.ldb, g.Z1, g.sb1, g.Z2, g.sb2, 32, BK, true);
    make_map(&mBs, THREE ? g.Bs : g.B, g.N, g.K, g.ldb, g.Z1, g.sb1, g.Z2, g.sb2, 32, BK, true);
  } else {
    make_map(&mB, g.B, g.K, g.N, g.ldb, g.Z1, g.sb1, g.Z2, g.sb2, BK, BN, false);
    make_map(&mBs, THREE ? g.Bs : g.B, g.K, g.N, g.ldb, g.Z1, g.sb1, g.Z2, g.sb2, BK, BN, false);
  }
  const int zc = g.Z1 * g.Z2;
  const int tn = (g.N + BN - 1) / BN, tm = (g.M + BM - 1) / BM;
  const int tiles = tn * tm * zc;
  const int total_kb = (g.K + BK - 1) / BK;
  // split-K when the output grid cannot fill the 148 SMs and K is long (the
  // Hv weight products reduce over all T tokens): partial tiles go to a
  // workspace and are summed in a fixed order by k_splitk_reduce.
  // Choose the split count minimising waves-per-unit-of-work
  // ceil(tiles*s/148)/s (each split keeps >= 16 k-blocks), smallest s on ties.
  int splits = 1;
  if (g.causal == 0 && tiles < kNumSMs && total_kb >= 32) {
    double best = 1.0;
    for (int s2 = 2; s2 <= 16 && total_kb / s2 >= 16; ++s2) {
      const double cost = double((tiles * s2 + kNumSMs - 1) / kNumSMs) / s2 + 0.04 * s2;  // + reduce traffic
      if (cost < best - 1e-9) {
        best = cost;
        splits = s2;
      }
    }
  }
  const int kb_per = (total_kb + splits - 1) / splits;
  splits = (total_kb + kb_per - 1) / kb_per;
  float* ws = nullptr;
  if (splits > 1) ws = splitk_workspace(size_t(splits) * zc * size_t(g.M) * g.N);
  EpiParams ep{g.C, g.ldc, g.sc1, g.sc2, g.M, g.N, g.Z1, g.alpha, g.beta, g.bias, g.Cs, g.dbg, zc, kb_per, ws,
               g.causal, tn, tm, tiles * splits};
  const size_t smem = 1024 + size_t(Cf::STAGES) * (THREE ? 2 : 1) * (Cf::A_BYTES + Cf::B_BYTES) + 256;
  auto kern = k_gemm_tf32<A_MN, B_MN, THREE, BN>;
  static bool attr_set = false;
  if (!attr_set) {
    SD_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    attr_set = true;
  }
  const int grid = std::min(ep.n_tiles, kNumSMs);
  if (prof().on)
    prof().next_tag = std::to_string(g.M) + "," + std::to_string(g.N) + "," + std::to_string(g.K) + "," +
                      std::to_string(zc) + "," + std::to_string(int(A_MN)) + "," + std::to_string(int(B_MN)) + "," +
                      std::to_string(g.causal) + "," + std::to_string(splits);
  prof_begin(s);
  kern<<<grid, NUM_THREADS, smem, s>>>(mA, mAs, mB, mBs, g.K, ep);
  SD_LAUNCHED("k_gemm_tf32");
  if (splits > 1) {
    const long long n = (long long)zc * g.M * g.N;
    k_splitk_reduce<<<unsigned((n + 255) / 256), 256, 0, s>>>(ws, splits, zc, g.Z1, g.M, g.N, g.C, g.ldc, g.sc1, g.sc2,
                                                              g.alpha, g.beta, g.bias, g.Cs);
    SD_LAUNCHED("k_splitk_reduce");
  }
  prof_end(s, 2.0 * double(g.M) * g.N * g.K * g.Z1 * g.Z2);
}

bool sd_gemm_wide_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("SD_GEMM_WIDE");
    return !(e && e[0] == '0');
  }();
  return on;
}

}  // namespace

void gemm(const GemmArgs& g, cudaStream_t s) {
  if (g.M <= 0 || g.N <= 0 || g.K <= 0) return;
  const bool three = g.As != nullptr && g.Bs != nullptr;
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

}  // namespace sd

extern "C" {

sd_status sd_gemm_tf32(const sd_gemm_desc* d, sd_stream s) {
  return sd::guard([&] {
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
    sd::gemm(g, (cudaStream_t)s);
  });
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
    std::fprintf(f, "M,N,K,batch,a_mn,b_mn,causal,splits,ms,flops\n");
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

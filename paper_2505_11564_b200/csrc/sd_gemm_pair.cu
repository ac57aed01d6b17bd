// CTA-pair variant of the fp32-faithful tcgen05 GEMM (sm_100a).
//
// Two CTAs of a cluster (two SMs of one TPC) compute one 256 x 256 output
// tile with tcgen05.mma.cta_group::2 (M = 256): CTA r stages rows
// [m0 + 128 r, +128) of A and columns [n0 + 128 r, +128) of B, and holds rows
// [m0 + 128 r, +128) x all 256 columns of the accumulator in its TMEM. Each
// SM therefore moves half the operand bytes per flop of the single-CTA
// 128 x 256 tile: the 3xTF32 products (raw + residual operands, 2x the bytes
// of a plain GEMM) are otherwise bound by L2 -> SM bandwidth.
//
// Roles per CTA: warp 0 TMA producer (own stage, own full barrier), warp 1
// TMEM allocator + (leader only) MMA issuer, warps 2-3 residual warps (write
// the tf32 residual tiles on chip, then arrive on the leader's conv barrier),
// warps 4..19 epilogue (16 warps: lane quadrant warp % 4, 64 columns each).
// Same 3xTF32 scheme, chunked round-to-nearest drain (KC), dual-source, twin
// and split-K support as the single-CTA kernel in sd_gemm.cu.
#include <algorithm>
#include <cstdlib>
#include <string>
#include <vector>

#include "sd_gemm_dev.cuh"

namespace sd {
namespace gk {
namespace {

constexpr int kPairM = 256;                           // pair tile M (each CTA stages 128 rows of A)
constexpr int kEpiWarps = 16;
constexpr int kPairThreads = 32 * (2 + kConvWarps + kEpiWarps);  // producer, MMA, residual, epilogue
constexpr int PA_BYTES = BM * BK * 4;                 // 8 KB
constexpr int kPairStages = 6;
// Pair tile width PN in {256, 192}: each CTA stages PN/2 columns of B; the
// narrower tile is chosen when it quantises into fuller waves (gemm_pair()).
template <int PN>
struct PairCfg {
  static constexpr int HALF = PN / 2;
  static constexpr int PB_BYTES = HALF * BK * 4;      // 8 / 6 KB
  static constexpr uint32_t TMEM_COLS = 512;          // two accumulation buffers (2 PN <= 512)
  static constexpr int EC = PN / (kEpiWarps / 4);     // 64 / 48 accumulator columns per epilogue thread
};

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// shared::cluster address of the same variable in the leader CTA (rank 0)
__device__ __forceinline__ uint32_t leader_addr(const void* p) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(smem_u32(p)));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void tma_load_4d_pair_e(const CUtensorMap* map, uint32_t bar, void* dst, int c0, int c1,
                                                   int c2, int c3) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4, %5, %6}], [%2];\n\t}" ::"r"(smem_u32(dst)),
      "l"(map), "r"(bar), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
__device__ __forceinline__ void tma_load_5d_pair_e(const CUtensorMap* map, uint32_t bar, void* dst, int c0, int c1,
                                                   int c2, int c3, int c4) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e cp.async.bulk.tensor.5d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4, %5, %6, %7}], [%2];\n\t}" ::"r"(smem_u32(dst)),
      "l"(map), "r"(bar), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
      : "memory");
}
// arrive on the barrier at this offset in BOTH CTAs of the pair once the
// leader's previously issued MMAs complete
// warp-wide issue: uniform descriptor math on every lane, one elected lane issues
__device__ __forceinline__ void mma_tf32_pair_e(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                                uint32_t acc) {
  asm volatile(
      "{\n\t"
      ".reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t"
      "}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit_pair_e(uint64_t* bar) {
  asm volatile(
      "{\n\t"
      ".reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t"
      "}" ::"r"(smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}

template <int PN>
__device__ __forceinline__ TileInfo pair_tile(const EpiParams& ep, int t, int K) {
  TileInfo ti;
  int mt, nt, zz;
  t = deal_unit(ep, t);
  if (t < 0) {
    ti.skip = true;
    return ti;
  }
  ti.tan = ep.twin && t < ep.tiles1;
  ti.nsrc = ep.twin ? (ti.tan ? 2 : 1) : ep.nsrc;
  walk_tile(ep, (ep.twin && !ti.tan) ? t - ep.tiles1 : t, mt, nt, zz);
  ti.n0 = nt * PN;
  ti.m0 = mt * kPairM;
  ti.z = zz % ep.zcount;
  ti.split = zz / ep.zcount;
  ti.kb0 = ti.split * ep.kb_per;
  ti.num_kb = min(ep.kb_per, (K + BK - 1) / BK - ti.kb0);
  ti.skip = ti.num_kb <= 0;
  return ti;
}

template <bool A_MN, bool B_MN, bool THREE, int PN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kPairThreads, 1)
    k_gemm_pair(const __grid_constant__ CUtensorMap mA, const __grid_constant__ CUtensorMap mAs,
                const __grid_constant__ CUtensorMap mB, const __grid_constant__ CUtensorMap mBs,
                const __grid_constant__ CUtensorMap mA2, const __grid_constant__ CUtensorMap mAs2,
                const __grid_constant__ CUtensorMap mB2, const __grid_constant__ CUtensorMap mBs2,
                const __grid_constant__ CUtensorMap mC, const __grid_constant__ CUtensorMap mCs,
                const __grid_constant__ CUtensorMap mC2, const __grid_constant__ CUtensorMap mCs2, int K,
                EpiParams ep) {
  using PC = PairCfg<PN>;
  constexpr int STAGES = kPairStages, EC = PC::EC, kHalfB = PC::HALF, PB_BYTES = PC::PB_BYTES;
  constexpr int kPairN = PN;
  constexpr uint32_t kPairTmemCols = PC::TMEM_COLS;
  constexpr int STAGE_BYTES = (THREE ? 2 : 1) * (PA_BYTES + PB_BYTES);
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  // [ring | 16 epilogue staging boxes of 2 KB (TMA store, 16 x 32 fp32) | barriers]
  float* epi_stage = reinterpret_cast<float*>(smem + STAGES * STAGE_BYTES);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES + kEpiWarps * 2048);
  uint64_t* empty = full + STAGES;
  uint64_t* conv = empty + STAGES;   // [STAGES] (leader) both CTAs' stage s landed + residuals written
  uint64_t* tfull = conv + STAGES;   // [2]
  uint64_t* tempty = tfull + 2;      // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
      mbar_init(&conv[s], 2);  // one residual warp of each CTA per stage
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 2 * kEpiWarps);  // every epilogue warp of both CTAs
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(kPairTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync();  // both CTAs' barriers initialised and TMEM allocated
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
      const uint32_t full_leader = leader_addr(full);
      uint32_t g = 0;
      for (int t = cid; t < ep.n_tiles; t += ncl) {
        const TileInfo ti = pair_tile<PN>(ep, t, K);
        if (ti.skip) continue;
        const int z1 = ti.z % ep.Z1, z2 = ti.z / ep.Z1;
        const int m_own = ti.m0 + int(rank) * BM, n_own = ti.n0 + int(rank) * kHalfB;
        for (int kk = 0; kk < ti.nsrc * ti.num_kb; ++kk, ++g) {
          const int s = g % STAGES;
          const uint32_t ph = (g / STAGES) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          unsigned char* st = smem + s * STAGE_BYTES;
          // residuals from memory: both CTAs' bytes land on the leader's full
          // barrier. On chip: each CTA's raw bytes land on its own barrier and
          // its residual warp releases the stage to the leader (conv[s]).
          // dual: (A, B) then (A2, B2); twin C2 tiles: (A2, B) then (A, B2)
          const bool second = kk >= ti.num_kb;
          const bool useA2 = ti.tan ? !second : second, useB2 = second;
          const bool bex = THREE && !ep.res && ((ep.bexact >> (useB2 ? 1 : 0)) & 1);
          uint32_t bar;
          if (ep.res) {
            mbar_expect_tx_e(&full[s], PA_BYTES + PB_BYTES);
            bar = smem_u32(&full[s]);
          } else {
            if (rank == 0) mbar_expect_tx_e(&full[s], 2 * (STAGE_BYTES - (bex ? PB_BYTES : 0)));
            bar = full_leader + 8u * s;
          }
          const int kb = second ? kk - ti.num_kb : kk;
          const CUtensorMap* pA = useA2 ? &mA2 : &mA;
          const CUtensorMap* pAs = useA2 ? &mAs2 : &mAs;
          const CUtensorMap* pB = useB2 ? &mB2 : &mB;
          const CUtensorMap* pBs = useB2 ? &mBs2 : &mBs;
          const int k0 = (ti.kb0 + kb) * BK;
          if (A_MN && (ep.mn5 & 1)) {
            tma_load_5d_pair_e(pA, bar, st, 0, k0, m_own / 32, z1, z2);
            if (THREE && !ep.res) tma_load_5d_pair_e(pAs, bar, st + PA_BYTES, 0, k0, m_own / 32, z1, z2);
          } else if (A_MN) {
#pragma unroll
            for (int c = 0; c < BM / 32; ++c) {
              tma_load_4d_pair_e(pA, bar, st + c * 2048, m_own + 32 * c, k0, z1, z2);
              if (THREE && !ep.res) tma_load_4d_pair_e(pAs, bar, st + PA_BYTES + c * 2048, m_own + 32 * c, k0, z1, z2);
            }
          } else {
            tma_load_4d_pair_e(pA, bar, st, k0, m_own, z1, z2);
            if (THREE && !ep.res) tma_load_4d_pair_e(pAs, bar, st + PA_BYTES, k0, m_own, z1, z2);
          }
          unsigned char* sb = st + (THREE ? 2 : 1) * PA_BYTES;
          if (B_MN && (ep.mn5 & 2)) {
            tma_load_5d_pair_e(pB, bar, sb, 0, k0, n_own / 32, z1, z2);
            if (THREE && !ep.res && !bex) tma_load_5d_pair_e(pBs, bar, sb + PB_BYTES, 0, k0, n_own / 32, z1, z2);
          } else if (B_MN) {
#pragma unroll
            for (int c = 0; c < kHalfB / 32; ++c) {
              tma_load_4d_pair_e(pB, bar, sb + c * 2048, n_own + 32 * c, k0, z1, z2);
              if (THREE && !ep.res && !bex) tma_load_4d_pair_e(pBs, bar, sb + PB_BYTES + c * 2048, n_own + 32 * c, k0, z1, z2);
            }
          } else {
            tma_load_4d_pair_e(pB, bar, sb, k0, n_own, z1, z2);
            if (THREE && !ep.res && !bex) tma_load_4d_pair_e(pBs, bar, sb + PB_BYTES, k0, n_own, z1, z2);
          }
        }
      }
    }
  } else if (warp >= 2 && warp < 2 + kConvWarps) {
    // residual warps (both CTAs): stage landed -> residual tiles -> tell the leader
    // (warp w takes the stages with g % kConvWarps == w - 2: two stages in flight)
    const int cw = warp - 2;
    const uint32_t conv_leader = leader_addr(conv);
    uint32_t g = 0;
    if (THREE && ep.res)
      for (int t = cid; t < ep.n_tiles; t += ncl) {
        const TileInfo ti = pair_tile<PN>(ep, t, K);
        if (ti.skip) continue;
        for (int kk = 0; kk < ti.nsrc * ti.num_kb; ++kk, ++g) {
          if (int(g % kConvWarps) != cw) continue;
          const int s = g % STAGES;
          mbar_wait(&full[s], (g / STAGES) & 1);
          unsigned char* st = smem + s * STAGE_BYTES;
          stage_residual(st, st + PA_BYTES, PA_BYTES, lane, 32);
          stage_residual(st + 2 * PA_BYTES, st + 2 * PA_BYTES + PB_BYTES, PB_BYTES, lane, 32);
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) mbar_arrive_remote(conv_leader + 8u * s);
        }
      }
  } else if (warp == 1) {
    if (rank == 0) {
      constexpr uint32_t idesc = make_idesc(A_MN, B_MN, kPairN, kPairM);
      uint32_t g = 0, chunk = 0;
      for (int t = cid; t < ep.n_tiles; t += ncl) {
        const TileInfo ti = pair_tile<PN>(ep, t, K);
        if (ti.skip) continue;
        const int nkb = ti.nsrc * ti.num_kb;
        for (int kb = 0; kb < nkb; ++kb, ++g) {
          const int s = g % STAGES;
          const uint32_t ph = (g / STAGES) & 1;
          const bool first = (kb % KC) == 0;
          const bool last = (kb % KC) == KC - 1 || kb == nkb - 1;
          const uint32_t buf = chunk & 1;
          if (first && chunk >= 2) mbar_wait(&tempty[buf], ((chunk >> 1) - 1) & 1);
          mbar_wait(ep.res ? &conv[s] : &full[s], ph);  // both CTAs' stage s (and residuals) ready
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          {  // whole warp: elected issue
            const uint32_t d = tmem + buf * kPairN;
            const uint32_t st = smem_u32(smem + s * STAGE_BYTES);
            const uint32_t a = st, as = st + PA_BYTES;
            const uint32_t b = st + (THREE ? 2 : 1) * PA_BYTES, bs = b + PB_BYTES;
            const bool bex = THREE && !ep.res && ((ep.bexact >> (kb >= ti.num_kb ? 1 : 0)) & 1);
#pragma unroll
            for (int ks = 0; ks < BK / 8; ++ks) {
              const uint32_t acc0 = (first && ks == 0) ? 0u : 1u;
              if (THREE) {
                mma_tf32_pair_e(d, tile_desc<A_MN>(as, ks), tile_desc<B_MN>(b, ks), idesc, acc0);
                if (!bex) mma_tf32_pair_e(d, tile_desc<A_MN>(a, ks), tile_desc<B_MN>(bs, ks), idesc, 1u);
                mma_tf32_pair_e(d, tile_desc<A_MN>(a, ks), tile_desc<B_MN>(b, ks), idesc, 1u);
              } else {
                mma_tf32_pair_e(d, tile_desc<A_MN>(a, ks), tile_desc<B_MN>(b, ks), idesc, acc0);
              }
            }
            mma_commit_pair_e(&empty[s]);
            if (last) mma_commit_pair_e(&tfull[buf]);
          }
          __syncwarp();
          if (last) ++chunk;
        }
      }
    }
  } else {
    // epilogue: warp w drains TMEM lanes 32 (w % 4) .. +31 and the column
    // group (w - 2) / 4 (EC = 64 columns) of this CTA's 128 accumulator rows
    const int sub = warp & 3;
    const int cb = ((warp - 2 - kConvWarps) >> 2) * EC;
    const uint32_t tempty_leader = leader_addr(tempty);
    uint32_t chunk = 0;
    for (int t = cid; t < ep.n_tiles; t += ncl) {
      const TileInfo ti = pair_tile<PN>(ep, t, K);
      if (ti.skip) continue;
      const int row = ti.m0 + int(rank) * BM + sub * 32 + lane;
      float acc[EC];
#pragma unroll
      for (int j = 0; j < EC; ++j) acc[j] = 0.0f;
      const int nchunks = (ti.nsrc * ti.num_kb + KC - 1) / KC;
      for (int c = 0; c < nchunks; ++c, ++chunk) {
        const uint32_t buf = chunk & 1;
        mbar_wait(&tfull[buf], (chunk >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
        for (int c0 = 0; c0 < EC; c0 += 16) {
          uint32_t v[16];
          tmem_ld16(tmem + (uint32_t(sub * 32) << 16) + buf * kPairN + uint32_t(cb + c0), v);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int j = 0; j < 16; ++j) acc[c0 + j] += __uint_as_float(v[j]);
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(tempty_leader + 8u * buf);
      }
      if (ep.tma_store && ep.ws) {
        // split-K partial (raw accumulator) through the workspace maps: [split][z][M][N]
        const int ew = warp - 2 - kConvWarps;
        warp_tma_store<EC, 16>(ti.tan ? &mC2 : &mC, nullptr, epi_stage + ew * 512, acc, 1.0f, nullptr, lane,
                               ti.m0 + int(rank) * BM + sub * 32, ti.n0 + cb, ti.split * ep.zcount + ti.z, 0, false);
        if (lane == 0) bulk_wait_read0();
        __syncwarp();
      } else if (ep.tma_store) {
        const int ew = warp - 2 - kConvWarps;  // 0..15: its staging box
        const bool t2 = ti.tan;  // twin: C2's tile
        const CUtensorMap* pcs = t2 ? (ep.Cs2 ? &mCs2 : nullptr) : (ep.Cs ? &mCs : nullptr);
        warp_tma_store<EC, 16>(t2 ? &mC2 : &mC, pcs, epi_stage + ew * 512, acc, t2 ? ep.alpha2 : ep.alpha,
                               t2 ? ep.bias2 : ep.bias, lane, ti.m0 + int(rank) * BM + sub * 32, ti.n0 + cb,
                               ti.z % ep.Z1, ti.z / ep.Z1, (ep.tma_add >> (t2 ? 1 : 0)) & 1);
        if (lane == 0) bulk_wait_read0();  // staging box free for the next tile
        __syncwarp();
      } else if (ti.tan) {
        EpiParams e2 = ep;  // twin: C2's tile
        e2.C = ep.C2, e2.Cs = ep.Cs2, e2.alpha = ep.alpha2, e2.beta = ep.beta2, e2.bias = ep.bias2, e2.ws = ep.ws2;
        store_row<EC>(e2, ti, row, ti.n0 + cb, acc);
      } else {
        store_row<EC>(ep, ti, row, ti.n0 + cb, acc);
      }
    }
  }
  if (ep.tma_store && lane == 0) bulk_wait0();
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync();  // no CTA leaves while its peer may still touch its smem / barriers
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kPairTmemCols));
  }
}

int max_clusters(const void* kern, size_t smem) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2 * kNumSMs);
  cfg.blockDim = dim3(kPairThreads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  SD_CUDA(cudaOccupancyMaxActiveClusters(&n, kern, &cfg));
  return n;
}

bool sd_gemm_partials_tma() {  // SD_GEMM_PARTIALS_TMA=0: split-K partials by row stores
  static const bool on = [] {
    const char* e = std::getenv("SD_GEMM_PARTIALS_TMA");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <bool A_MN, bool B_MN, bool THREE, int PN>
void launch_pair_t(const GemmArgs& g, cudaStream_t s) {
  using PC = PairCfg<PN>;
  constexpr int kPairN = PN, kHalfB = PC::HALF, PB_BYTES = PC::PB_BYTES;
  CUtensorMap maps[8];
  int mn5 = 0;
  operand_maps(g, A_MN, B_MN, THREE, kHalfB, maps, &mn5);
  const bool twin = g.twin;
  const bool dual = g.A2 != nullptr && !twin;
  const int zc = g.Z1 * g.Z2;
  const int tn = (g.N + kPairN - 1) / kPairN, tm = (g.M + kPairM - 1) / kPairM;
  const int tiles = tn * tm * zc;
  const size_t smem = 1024 + size_t(kPairStages) * (THREE ? 2 : 1) * (PA_BYTES + PB_BYTES) + kEpiWarps * 2048 + 512;
  auto kern = k_gemm_pair<A_MN, B_MN, THREE, PN>;
  static int clusters = 0;
  if (!clusters) {
    SD_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    clusters = std::max(1, max_clusters(reinterpret_cast<const void*>(kern), smem));
  }
  // split-K as in the single-CTA launcher, over the cluster (pair) slots
  const int total_kb = (g.K + BK - 1) / BK;
  const double t_kb = 2.0 * kPairM * kPairN * BK / (2.0e14 / clusters) / (THREE ? 1.0 : 3.0);
  int splits = twin ? choose_splits_twin(tiles, clusters, total_kb, t_kb, 8.0 * zc * g.M * g.N)
                    : choose_splits(tiles, clusters, total_kb, dual ? 2 : 1, t_kb, 4.0 * zc * g.M * g.N);
  const int kb_per = (total_kb + splits - 1) / splits;
  splits = (total_kb + kb_per - 1) / kb_per;
  const size_t part = size_t(splits) * zc * size_t(g.M) * g.N;
  float* ws = nullptr;
  if (splits > 1) ws = splitk_workspace((twin ? 2 : 1) * part);
  EpiParams ep{g.C, g.ldc, g.sc1, g.sc2, g.M, g.N, g.Z1, g.alpha, g.beta, g.bias, g.Cs, g.dbg, zc, kb_per, ws,
               0, tn, tm, tiles * splits * (twin ? 2 : 1), dual ? 2 : 1, g.onchip ? 1 : 0};
  if (twin) {
    ep.twin = 1, ep.tiles1 = tiles * splits;
    ep.C2 = g.C2, ep.Cs2 = g.Cs2, ep.alpha2 = g.alpha2, ep.beta2 = g.beta2, ep.bias2 = g.bias2;
    ep.ws2 = ws ? ws + part : nullptr;
  }
  ep.group = walk_group(g, kPairM, PN, tm, tn, THREE);
  const int grid = 2 * std::min(ep.n_tiles, clusters);
  if (twin) {  // boustrophedon deal over the cluster slots (deal_unit)
    ep.ncl = grid / 2, ep.units = ep.n_tiles;
    ep.n_tiles = (ep.n_tiles + ep.ncl - 1) / ep.ncl * ep.ncl;
  }
  if (prof_on())
    prof_tag(std::to_string(g.M) + "," + std::to_string(g.N) + "," + std::to_string(g.K) + "," + std::to_string(zc) +
             "," + std::to_string(int(A_MN)) + "," + std::to_string(int(B_MN)) + ",pair," + std::to_string(splits) +
             (twin ? ",twin" : dual ? ",2" : ",1"));
  prof_begin(s);
  ep.mn5 = mn5;
  ep.bexact = (g.b_exact ? 1 : 0) | (g.b2_exact ? 2 : 0);
  CUtensorMap mC = maps[0], mCs = maps[0], mC2 = maps[0], mCs2 = maps[0];
  GemmArgs g2 = g;  // twin: C2's epilogue
  g2.C = g.C2, g2.Cs = g.Cs2, g2.alpha = g.alpha2, g2.beta = g.beta2, g2.bias = g.bias2;
  if (tma_store_ok(g, splits, 16, true) && (!twin || tma_store_ok(g2, splits, 16, true))) {
    ep.tma_add = (g.beta != 0.0f ? 1 : 0) | (twin && g2.beta != 0.0f ? 2 : 0);
    make_store_map(&mC, g.C, g, 16);
    if (g.Cs) make_store_map(&mCs, g.Cs, g, 16);
    if (twin) {
      make_store_map(&mC2, g2.C, g2, 16);
      if (g2.Cs) make_store_map(&mCs2, g2.Cs, g2, 16);
    }
    ep.tma_store = 1;
  } else if (splits > 1 && g.N % 4 == 0 && sd_gemm_partials_tma()) {
    // split-K partials through TMA stores: the workspace as a [split * z][M][N] tensor
    GemmArgs gw = g;
    gw.ldc = g.N, gw.Z1 = splits * zc, gw.sc1 = (long long)g.M * g.N, gw.Z2 = 1, gw.sc2 = 0;
    make_store_map(&mC, ws, gw, 16);
    if (twin) make_store_map(&mC2, ws + part, gw, 16);
    ep.tma_store = 1;
  }
  launch_gemm_kernel(kern, unsigned(grid), unsigned(kPairThreads), size_t(smem), s, maps[0], maps[1], maps[2], maps[3],
                     maps[4], maps[5], maps[6], maps[7], mC, mCs, mC2, mCs2, g.K, ep);
  SD_LAUNCHED("k_gemm_pair");
  if (splits > 1) {
    launch_splitk_reduce(ws, splits, zc, g, s);
    if (twin) launch_splitk_reduce(ws + part, splits, zc, g2, s);
  }
  prof_end(s, (twin ? 6.0 : dual ? 4.0 : 2.0) * double(g.M) * g.N * g.K * g.Z1 * g.Z2);
}

}  // namespace

// Wave-quantisation-aware tile width: the modelled time of each candidate
// (waves x k-blocks x per-k-block time, relative per-SM rate of the narrower
// tile 0.95) -- e.g. 8192 x 3072 outputs: 384 tiles of 256 (5.2 -> 6 waves)
// vs 512 of 192 (6.9 -> 7 waves, 5% less work per wave slot).
int pick_pair_n(const GemmArgs& g) {
  static const int forced = [] {
    const char* e = std::getenv("SD_GEMM_PAIR_N");
    return e ? std::atoi(e) : 0;
  }();
  if (forced == 256 || forced == 192) return forced;
  // measured on the GPT-2-small HVP: choosing 192 by this model made the step
  // slower (122.7 vs 118.4 ms), so 256 stays unless SD_GEMM_PAIR_N forces 192
  if (!forced) return 256;
  const int zc = g.Z1 * g.Z2, tm = (g.M + kPairM - 1) / kPairM;
  const int units = kNumSMs / 2;
  const int total_kb = (g.K + BK - 1) / BK * (g.A2 ? 2 : 1);
  double best = 1e30;
  int best_n = 256;
  for (int pn : {256, 192}) {
    const long long tiles = (long long)tm * ((g.N + pn - 1) / pn) * zc;
    const double rate = pn == 256 ? 1.0 : 0.95;
    const double t = double((tiles + units - 1) / units) * total_kb * (double(pn) / 256.0) / rate;
    if (t < best * 0.98) {
      best = t;
      best_n = pn;
    }
  }
  return best_n;
}

void gemm_pair(const GemmArgs& g, cudaStream_t s) {
  const bool three = (g.As != nullptr && g.Bs != nullptr) || g.onchip;
  const int pn = pick_pair_n(g);
#define SD_PAIR_CASE(AM, BMJ, TH)                                                                         \
  if (g.a_mn == AM && g.b_mn == BMJ && three == TH)                                                       \
    return pn == 192 ? launch_pair_t<AM, BMJ, TH, 192>(g, s) : launch_pair_t<AM, BMJ, TH, 256>(g, s);
  SD_PAIR_CASE(false, false, true)
  SD_PAIR_CASE(false, true, true)
  SD_PAIR_CASE(true, false, true)
  SD_PAIR_CASE(true, true, true)
  SD_PAIR_CASE(false, false, false)
  SD_PAIR_CASE(false, true, false)
  SD_PAIR_CASE(true, false, false)
  SD_PAIR_CASE(true, true, false)
#undef SD_PAIR_CASE
}

}  // namespace gk
}  // namespace sd

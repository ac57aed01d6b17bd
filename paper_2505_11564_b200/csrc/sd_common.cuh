// Shared device/host helpers for libspecden_b200 (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

#include "specden_b200.h"

namespace sd {

// Exception carrying an sd_status; converted at the C-ABI edge.
struct Error : std::runtime_error {
  sd_status code;
  Error(sd_status c, const std::string& w) : std::runtime_error(w), code(c) {}
};
[[noreturn]] inline void fail(sd_status c, const std::string& w) { throw Error(c, w); }

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(SD_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
}
#define SD_CUDA(call) ::sd::cuda_check((call), #call)
// every kernel launch of the library passes through here: it is checked and
// counted (sd_launch_count, reported as gpu_launches by bench.py)
void count_launch();
void add_launches(uint64_t n);  // kernels a replayed CUDA graph runs
#define SD_LAUNCHED(name) (::sd::count_launch(), ::sd::cuda_check(cudaGetLastError(), name))

void set_last_error(const std::string& m);

// Programmatic dependent launch (PDL) for the kernels that follow GEMMs: the
// launch carries cudaLaunchAttributeProgrammaticStreamSerialization and the
// kernel calls pdl_wait() before its first global-memory access, so its
// launch overlaps the previous kernel's tail (GEMMs trigger their dependents
// once every CTA is resident). SD_GEMM_PDL=0 turns it off (gk::pdl_on).
namespace gk {
bool pdl_on();
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
template <typename... P, typename... A>
void launch_pdl(void (*kern)(P...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, A&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = gk::pdl_on() ? 1 : 0;
  cuda_check(cudaLaunchKernelEx(&cfg, kern, static_cast<P>(args)...), "cudaLaunchKernelEx");
}

// Every C-ABI body runs inside this guard.
template <class F>
sd_status guard(F&& f) {
  try {
    f();
    return SD_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return SD_CUDA_ERROR;
  }
}

constexpr uint64_t kBlock = 1024;  // reduction grid, reduction.hpp:30

// Shape of a rank's BlockedPartial over [begin, end) (reduction.hpp:50-71).
struct PartialShape {
  uint64_t n_head, n_sums, n_tail;
  uint64_t len() const { return n_head + n_sums + n_tail; }
};
__host__ __device__ inline PartialShape partial_shape(uint64_t begin, uint64_t end, uint64_t total) {
  PartialShape p{0, 0, 0};
  const uint64_t first_full = (begin + kBlock - 1) / kBlock;
  uint64_t head_end = first_full * kBlock;
  if (head_end > end) head_end = end;
  p.n_head = head_end - begin;
  if (head_end < end) {
    if (end == total) {
      p.n_sums = (end - head_end + kBlock - 1) / kBlock;
    } else {
      p.n_sums = (end - head_end) / kBlock;
      p.n_tail = (end - head_end) % kBlock;
    }
  }
  return p;
}

// ---- counter RNG, proj/include/specden/rng.hpp:17-52 (bit-identical integer path)
__host__ __device__ inline uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
__host__ __device__ inline uint64_t keyed_counter_k(uint64_t key, uint64_t ctr) {
  return mix64(key ^ (ctr * 0x9e3779b97f4a7c15ull));
}

// Exact fp32 -> f64 widening on the integer pipe (normal numbers; zeros,
// subnormals, inf and nan take the conversion instruction). The f64 <-> f32
// conversions issue on the 16-lane XU pipe, which the reorthogonalisation
// update (one rounding per basis column per element) otherwise saturates.
__device__ __forceinline__ double widen_f32(float f) {
  const uint32_t u = __float_as_uint(f);
  const uint32_t a = u & 0x7fffffffu;
  if (a - 0x00800000u >= 0x7f000000u) return double(f);
  return __hiloint2double(int((u & 0x80000000u) | ((a >> 3) + 0x38000000u)), int(u << 29));
}

template <typename T>
__device__ __forceinline__ T round_to(double v);
template <>
__device__ __forceinline__ float round_to<float>(double v) {
  return __double2float_rn(v);
}
template <>
__device__ __forceinline__ double round_to<double>(double v) {
  return v;
}
// round_to<T>, returned as f64 (exact)
template <typename T>
__device__ __forceinline__ double rround(double v);
template <>
__device__ __forceinline__ double rround<float>(double v) {
  return widen_f32(__double2float_rn(v));
}
template <>
__device__ __forceinline__ double rround<double>(double v) {
  return v;
}

}  // namespace sd

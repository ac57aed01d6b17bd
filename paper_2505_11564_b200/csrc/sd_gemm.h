// Internal GEMM interface (see sd_gemm.cu).
#pragma once
#include <cuda_runtime.h>

namespace sd {
struct GemmArgs {
  int M = 0, N = 0, K = 0;
  const float* A = nullptr;   // raw fp32 operand
  const float* As = nullptr;  // residual (3xTF32); nullptr -> 1xTF32 (unless onchip)
  bool onchip = false;        // 3xTF32 with on-chip residuals allowed (required if As/Bs are null)
  long long lda = 0;
  bool a_mn = false;          // false: A row-major M x K; true: row-major K x M
  const float* B = nullptr;
  const float* Bs = nullptr;
  long long ldb = 0;
  bool b_mn = false;          // false: B row-major N x K; true: row-major K x N
  float* C = nullptr;
  long long ldc = 0;
  float alpha = 1.0f, beta = 0.0f;
  int Z1 = 1, Z2 = 1;         // batch z = z1 + Z1 * z2
  const float* bias = nullptr;  // per-column bias added in the epilogue
  float* Cs = nullptr;          // optional tf32 residual of the final C (same strides as C)
  float* dbg = nullptr;
  int causal = 0;  // causal attention structure, see k_gemm_tf32
  long long sa1 = 0, sa2 = 0, sb1 = 0, sb2 = 0, sc1 = 0, sc2 = 0;  // element strides
  // optional second product accumulated into the same tile (dual source):
  //   C = alpha (op(A) op(B) + op(A2) op(B2)) + beta C ; same M, N, K, majors
  const float *A2 = nullptr, *A2s = nullptr, *B2 = nullptr, *B2s = nullptr;
  long long lda2 = 0, ldb2 = 0, sa1_2 = 0, sa2_2 = 0, sb1_2 = 0, sb2_2 = 0;
  // B (B2) holds tf32-exact values (bf16-valued weights): its residual is zero,
  // so 3xTF32 needs neither its residual array nor the A . B_lo product
  bool b_exact = false, b2_exact = false;
  // merged pair of 64-wide products sharing A (the per-head attention
  // R-op products): C = alpha (A B), C2 = alpha (A B2 + A2 B), both N = 64,
  // B and B2 MN-major with the same strides (ldb, sb1, sb2), C2 / Cs2 with C's
  // strides; one launch with a 128-wide accumulator (A staged once for both)
  bool split = false;
  float *C2 = nullptr, *Cs2 = nullptr;
  // twin products sharing A and B (the primal and tangent products of one
  // weight in the R-op forward and adjoint): C = alpha A B + beta C (+bias,
  // Cs) and C2 = alpha2 (A2 B + A B2) + beta2 C2 (+bias2, Cs2), C2 with C's
  // strides; one launch whose tile list holds both outputs' tiles (C2's, the
  // two-source ones, first), or two launches where the pair kernel does not
  // apply
  bool twin = false;
  float alpha2 = 1.0f, beta2 = 0.0f;
  const float* bias2 = nullptr;
};
void gemm(const GemmArgs& g, cudaStream_t s);
// bumped whenever a split-K workspace is (re)allocated: a captured CUDA graph
// holding the old pointer must be re-captured
uint64_t gemm_scratch_generation();
// per-GEMM event profiling on (events cannot sit inside a replayed graph)
bool gemm_profiling();
void split_tf32(const float* x, float* small, long long n, int mode, cudaStream_t s);
}  // namespace sd

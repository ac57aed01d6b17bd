// Dependent f64 add latency on sm_100a (one thread): chain of __dadd_rn from
// registers, from shared memory (8 loads then 8 adds), and the clock rate.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, int n) {
  __shared__ double b[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) b[i] = 1e-3 * i;
  __syncthreads();
  if (threadIdx.x) return;
  double c = out[0], t = 1.0000001;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int q = 0; q < 16; ++q) c = __dadd_rn(c, t);
  }
  long long t1 = clock64();
  double d = out[1];
  for (int r = 0; r < n / 256; ++r)
    for (int i = 0; i < 4096; i += 8) {
      double v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = b[i + q];
#pragma unroll
      for (int q = 0; q < 8; ++q) d = __dadd_rn(d, v[q]);
    }
  long long t2 = clock64();
  out[2] = c + d;
  cyc[0] = t1 - t0;
  cyc[1] = t2 - t1;
}
int main() {
  double* o; long long* c;
  cudaMalloc(&o, 64); cudaMalloc(&c, 16); cudaMemset(o, 0, 64);
  int n = 1 << 14;
  k<<<1, 256>>>(o, c, n);
  cudaDeviceSynchronize();
  long long h[2];
  cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost);
  printf("register chain: %.2f cycles/DADD\n", double(h[0]) / (16.0 * n));
  printf("smem 8+8 chain: %.2f cycles/DADD\n", double(h[1]) / (double(n / 256) * 4096));
  return 0;
}

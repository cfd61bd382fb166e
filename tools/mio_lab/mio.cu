// Do shared-memory transposes and warp shuffles share one bandwidth?
// kernel mode 0: smem only, 1: shfl only, 2: both (same per-op counts as 0 and 1 together)
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int mode, int iters, double* out) {
  __shared__ double xb[4][16 * 34];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double v[16];
  for (int i = 0; i < 16; ++i) v[i] = lane * 0.5 + i;
  double* x = xb[w];
  for (int it = 0; it < iters; ++it) {
    if (mode != 1) {
      __syncwarp();
#pragma unroll
      for (int q = 0; q < 16; ++q) x[q * 34 + lane] = v[q];
      __syncwarp();
#pragma unroll
      for (int m = 0; m < 16; ++m) v[m] = x[(lane >> 1) * 34 + (lane & 1) + 2 * m] + 1e-9;
    }
    if (mode != 0) {
#pragma unroll
      for (int m = 0; m < 16; ++m) v[m] = __shfl_xor_sync(0xffffffffu, v[m], (m & 7) + 1) + 1e-9;
    }
  }
  double s = 0;
  for (int i = 0; i < 16; ++i) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  double* out;
  cudaMalloc(&out, 148 * 8 * 128 * 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 2000;
  for (int mode = 0; mode < 3; ++mode) {
    k<<<148 * 8, 128>>>(mode, 10, out);
    cudaEventRecord(a);
    k<<<148 * 8, 128>>>(mode, iters, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    // bytes moved per op class: smem 2 * 16 * 8 B * threads * iters; shfl 16 * 8 B * threads * iters
    const double thr = 148.0 * 8 * 128 * iters;
    printf("mode %d: %.3f ms  smem %.1f TB/s  shfl %.1f TB/s\n", mode, ms,
           mode != 1 ? 2 * 16 * 8 * thr / ms / 1e9 : 0.0, mode != 0 ? 16 * 8 * thr / ms / 1e9 : 0.0);
  }
  return 0;
}

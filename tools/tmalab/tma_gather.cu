// Microbenchmark: per-warp row gathers of a column-major intermediate with a
// TMA tensor box (16-byte inner extent, 8 KB row stride) versus contiguous
// 1-D bulk copies of a row-major intermediate.  Same bytes moved.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include "../../paper_2103_07706_b200/csrc/async_copy.cuh"
using namespace pswe;

constexpr int NX = 512, KY = 171, NF = 5, NP = 8;

// it: fields (0,1) (3,0) (4,1) (2,-)
__device__ int fa_of(int it) { return it == 0 ? 0 : (it == 1 ? 3 : (it == 2 ? 4 : 2)); }
__device__ int fb_of(int it) { return it == 0 ? 1 : (it == 1 ? 0 : (it == 2 ? 1 : -1)); }

// cp.async (LDGSTS) gather: lanes copy the row's 16-byte elements themselves
__global__ void __launch_bounds__(128) rows_ldgsts(const double2* I, double* out) {
  __shared__ __align__(128) double2 pre[4][2][176];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double acc = 0;
  const int ntask = NP * NX;
  for (int task = blockIdx.x * 4 + warp; task < ntask; task += gridDim.x * 4) {
    const int p = task / NX, x = task % NX;
    for (int it = 0; it < 4; ++it) {
      const int fa = fa_of(it), fb = fb_of(it);
      const double2* ga = I + ((size_t)(p * NF + fa) * KY) * NX + x;
      for (int j = lane; j < KY; j += 32) {
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(&pre[warp][0][j])), "l"(ga + (size_t)j * NX) : "memory");
      }
      if (fb >= 0) {
        const double2* gb = I + ((size_t)(p * NF + fb) * KY) * NX + x;
        for (int j = lane; j < KY; j += 32)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(&pre[warp][1][j])), "l"(gb + (size_t)j * NX) : "memory");
      }
      asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
      __syncwarp();
      for (int j = lane; j < KY; j += 32) acc += pre[warp][0][j].x + pre[warp][1][j].y;
      __syncwarp();
    }
  }
  out[blockIdx.x * 128 + threadIdx.x] = acc;
}

template <bool GATHER>
__global__ void __launch_bounds__(128) rows_kernel(const __grid_constant__ CUtensorMap map, const double2* I, double* out) {
  __shared__ __align__(128) double2 pre[4][2][176];
  __shared__ __align__(8) uint64_t bars[4];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint64_t* bar = &bars[warp];
  if (lane == 0) { mbar_init(bar, 1); fence_mbar_init(); }
  __syncthreads();
  double acc = 0;
  int ph = 0;
  const int ntask = NP * NX;
  for (int task = blockIdx.x * 4 + warp; task < ntask; task += gridDim.x * 4) {
    const int p = task / NX, x = task % NX;
    for (int it = 0; it < 4; ++it) {
      const int fa = fa_of(it), fb = fb_of(it);
      if (lane == 0) {
        const uint32_t seg = KY * 16;
        mbar_arrive_expect_tx(bar, fb >= 0 ? 2 * seg : seg);
        if (GATHER) {
          tma_load_4d(pre[warp][0], &map, 0, x, 0, fa + NF * p, bar);
          if (fb >= 0) tma_load_4d(pre[warp][1], &map, 0, x, 0, fb + NF * p, bar);
        } else {
          const double2* row = I + ((size_t)p * NX + x) * NF * KY;
          bulk_g2s(pre[warp][0], row + fa * KY, seg, bar);
          if (fb >= 0) bulk_g2s(pre[warp][1], row + fb * KY, seg, bar);
        }
      }
      mbar_wait(bar, ph);
      ph ^= 1;
      for (int j = lane; j < KY; j += 32) acc += pre[warp][0][j].x + pre[warp][1][j].y;
      __syncwarp();
    }
  }
  out[blockIdx.x * 128 + threadIdx.x] = acc;
}

int main() {
  const size_t n = (size_t)NP * NF * KY * NX;
  double2* I;
  double* out;
  cudaMalloc(&I, n * sizeof(double2));
  cudaMalloc(&out, 1 << 20);
  cudaMemset(I, 0, n * sizeof(double2));
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  if (!enc) { printf("no encode\n"); return 1; }
  CUtensorMap map;
  // column-major [p*f][j][x] of complex = doubles (2, x, j, pf)
  cuuint64_t dims[4] = {2, NX, KY, (cuuint64_t)NP * NF};
  cuuint64_t strides[3] = {16, (cuuint64_t)NX * 16, (cuuint64_t)NX * KY * 16};
  cuuint32_t box[4] = {2, 1, KY, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, I, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int grid : {148 * 3, 148 * 6, 148 * 12}) {
    for (int g = 0; g < 3; ++g) {
      float best = 1e9;
      for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(a);
        if (g == 1) rows_kernel<true><<<grid, 128>>>(map, I, out);
        else if (g == 2) rows_ldgsts<<<grid, 128>>>(I, out);
        else rows_kernel<false><<<grid, 128>>>(map, I, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
      }
      const double bytes = (double)NP * NX * 7 * KY * 16;
      printf("grid %d %s: %.3f us  %.1f GB/s  (%.2f us per phase)\n", grid, g == 1 ? "tensor-gather" : (g == 2 ? "ldgsts-gather" : "bulk-contig"), best * 1e3,
             bytes / (best * 1e-3) / 1e9, best * 1e3 / NP);
    }
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}

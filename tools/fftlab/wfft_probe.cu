// Static-SASS probe for the warp FFT: one kernel per (N, type, direction).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -cubin wfft_probe.cu; cuobjdump -sass
#include "../../paper_2103_07706_b200/csrc/wfft.cuh"
using namespace pswe;

template <int N, int TYPE, bool INV>
__global__ void __launch_bounds__(128) probe(const double2* __restrict__ in, double2* __restrict__ out,
                                             const double2* __restrict__ tw) {
  __shared__ double xbuf[4 * WF<N>::GPW * WF<N>::XBUF];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int t = lane % WF<N>::T, g = lane / WF<N>::T;
  double* xb = xbuf + (warp * WF<N>::GPW + g) * WF<N>::XBUF;
  double2 v[WF<N>::P];
  const size_t base = ((size_t)blockIdx.x * 128 + threadIdx.x) * WF<N>::P;
#pragma unroll
  for (int i = 0; i < WF<N>::P; ++i) v[i] = in[base + i];
  const WLane wl = wlane<N>(WTab{tw}, t);
  if (TYPE == 1)
    wfft_t1<N, INV>(v, t, xb, wl);
  else
    wfft_t2<N, INV>(v, t, xb, wl);
#pragma unroll
  for (int i = 0; i < WF<N>::P; ++i) out[base + i] = v[i];
}

template __global__ void probe<512, 1, true>(const double2*, double2*, const double2*);
template __global__ void probe<512, 2, false>(const double2*, double2*, const double2*);
template __global__ void probe<256, 1, true>(const double2*, double2*, const double2*);
template __global__ void probe<256, 2, false>(const double2*, double2*, const double2*);

// Snapshot diagnostics on the device: energy, mass and maximum speed of a
// state (diagnostics.py:58-78, integrator.py:124-135), from physical fields
// obtained by a full (unpruned) 2-D C2R of u, v, eta and b:
//   diag_cols  Hermitian projection (what real(ifft2(.)) does, grid.py:173)
//              + inverse x-FFT of the ky >= 0 columns  -> D[f][j][x]
//   diag_rows  per physical row: y-C2R of the packed pairs (u, v), (eta, b),
//              pointwise energy/mass/speed^2, reduced over the row in a fixed
//              order -> part[x][3]; the host sums the rows in order.
#pragma once
#include "wfft.cuh"
#include "pswe_kernels.cuh"

namespace pswe {

template <int NX>
__global__ void __launch_bounds__(128) diag_cols_kernel(GridDev G, const double2* __restrict__ u,
                                                        const double2* __restrict__ v,
                                                        const double2* __restrict__ e,
                                                        const double2* __restrict__ b, double2* __restrict__ D) {
  constexpr int T = WF<NX>::T, P = WF<NX>::P, GPW = WF<NX>::GPW;
  __shared__ double xbuf[4 * GPW * WF<NX>::XBUF];
  const int ny = G.ny, nyh = ny / 2 + 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int t = lane % T, g = lane / T;
  const int task = (blockIdx.x * 4 + warp) * GPW + g;  // f * nyh + j
  const bool active = task < 4 * nyh;
  const int f = active ? task / nyh : 0, j = active ? task % nyh : 0;
  const double2* c = f == 0 ? u : (f == 1 ? v : (f == 2 ? e : b));
  const int jm = (ny - j) % ny;
  double2 w[P];
#pragma unroll
  for (int n1 = 0; n1 < P; ++n1) {
    const int ix = t + T * n1, im = (NX - ix) % NX;
    if (active) {
      const double2 a = c[(size_t)ix * ny + j], m = c[(size_t)im * ny + jm];
      w[n1] = cmk(0.5 * (a.x + m.x), 0.5 * (a.y - m.y));
    } else {
      w[n1] = czero();
    }
  }
  const WLane wl = wlane<NX>(G.twx, t);
  wfft_t1<NX, true>(w, t, xbuf + (size_t)(warp * GPW + g) * WF<NX>::XBUF, wl);
  if (active) {
    double2* o = D + ((size_t)f * nyh + j) * NX;
#pragma unroll
    for (int i = 0; i < P; ++i) o[t1_pos<NX>(t, i)] = cscale(G.inv_n2, w[i]);
  }
}

// type-1 input of the packed pair A + iB at y position k from the x-row of the
// half spectra (columns j = 0..ny/2 of D for fields fa, fb); the Hermitian
// mirror supplies k > ny/2, the DC and Nyquist bins keep their real parts.
template <int NY>
__device__ __forceinline__ double2 diag_pair(const double2* D, int fa, int fb, int k, int x, int nx) {
  constexpr int NYH = NY / 2 + 1;
  const bool lo = k <= NY / 2;
  const int kk = lo ? k : NY - k;
  double2 A = D[((size_t)fa * NYH + kk) * nx + x], B = D[((size_t)fb * NYH + kk) * nx + x];
  if (kk == 0 || kk == NY / 2) {
    A.y = 0.0;
    B.y = 0.0;
  }
  if (!lo) {
    A.y = -A.y;
    B.y = -B.y;
  }
  return cmk(A.x - B.y, A.y + B.x);
}

// part: [nx][3] row partials; phys (optional): [3][nx][ny] physical u, v, eta
template <int NY>
__global__ void __launch_bounds__(128) diag_rows_kernel(GridDev G, const double2* __restrict__ D, double H,
                                                        double grav, double* __restrict__ part,
                                                        double* __restrict__ phys) {
  constexpr int T = WF<NY>::T, P = WF<NY>::P, GPW = WF<NY>::GPW;
  __shared__ double xbuf[4 * GPW * WF<NY>::XBUF];
  const int nx = G.nx;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int t = lane % T, g = lane / T;
  const int x = (blockIdx.x * 4 + warp) * GPW + g;
  const bool active = x < nx;
  const int xr = active ? x : 0;
  double* xb = xbuf + (size_t)(warp * GPW + g) * WF<NY>::XBUF;
  const WLane wl = wlane<NY>(G.twy, t);
  double2 uv[P], eb[P];
#pragma unroll
  for (int n1 = 0; n1 < P; ++n1) uv[n1] = diag_pair<NY>(D, 0, 1, t + T * n1, xr, nx);
  wfft_t1<NY, true>(uv, t, xb, wl);
#pragma unroll
  for (int n1 = 0; n1 < P; ++n1) eb[n1] = diag_pair<NY>(D, 2, 3, t + T * n1, xr, nx);
  wfft_t1<NY, true>(eb, t, xb, wl);
  if (phys != nullptr && active) {
    const size_t nxy = (size_t)nx * NY;
    double* pr = phys + (size_t)x * NY;
#pragma unroll
    for (int i = 0; i < P; ++i) {
      const int y = t1_pos<NY>(t, i);
      pr[y] = uv[i].x;
      pr[nxy + y] = uv[i].y;
      pr[2 * nxy + y] = eb[i].x;
    }
  }
  double se = 0.0, sm = 0.0, vmax = 0.0;
#pragma unroll
  for (int i = 0; i < P; ++i) {
    const double uu = uv[i].x, vv = uv[i].y, eta = eb[i].x, bb = eb[i].y;
    const double depth = H + eta - bb;
    const double s2 = uu * uu + vv * vv;
    se += 0.5 * depth * s2 + 0.5 * grav * eta * (eta + 2.0 * H);
    sm += depth;
    vmax = fmax(vmax, s2);
  }
  // fixed-order butterfly over the T lanes of the row
#pragma unroll
  for (int o = 1; o < T; o <<= 1) {
    se += __shfl_xor_sync(0xffffffffu, se, o, T);
    sm += __shfl_xor_sync(0xffffffffu, sm, o, T);
    vmax = fmax(vmax, __shfl_xor_sync(0xffffffffu, vmax, o, T));
  }
  if (active && t == 0) {
    part[3 * (size_t)x + 0] = se;
    part[3 * (size_t)x + 1] = sm;
    part[3 * (size_t)x + 2] = vmax;
  }
}

}  // namespace pswe

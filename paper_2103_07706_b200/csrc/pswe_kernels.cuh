// sm_100a kernels for the phase-averaged nonlinear tendency and the
// transformed SSPRK3 stepper.
//
// Data layouts (all fp64 complex, double2):
//   full    : one (nx, ny) array per field, row-major, numpy fft2 order
//             (grid.py:3-8).  Used at the API boundary and by the stepper.
//   compact : U[f][j][r], f in {u, v, eta}, j = ky index 0..KYM (ky >= 0 half),
//             r = compact kx index 0..Kx-1 (wx = r for r <= KXM, r - Kx after).
//             Only the 2/3 band |wx| <= nx/3, |wy| <= ny/3 (grid.py:102-103)
//             is stored; the ky < 0 half is the conjugate mirror.
//   I (chunk intermediates): I[p][f][j][x], p = phase in chunk, f in 0..4,
//             j = 0..KYM, x = 0..nx-1 (physical x, spectral y).
//
// Averaged RHS (averaging.py:116-156) for a chunk of phases:
//   pass A  (per phase, ky column)  e^{sL} per mode + 5 inverse x-FFTs
//   pass B  (per phase, x row)      7 C2R along y as 4 complex FFTs, the four
//                                   quadratic products, 2 R2C as complex FFTs
//   pass C  (per ky column, phases) 4 forward x-FFTs, flux divergence, 2/3
//                                   truncation, e^{-sL}, weighted ordered sum
// followed by an ordered reduction over the phase-group slots.
#pragma once
#include "fft_reg.cuh"

namespace pswe {

struct GridDev {
  int nx, ny, kxm, kym, Kx, Ky;
  Phys ph;
  double inv_n2;
  const double* kxc;   // [Kx]  compact kx
  const double* kyc;   // [Ky]  ky >= 0
  const double* kxf;   // [nx]  full kx (fft order)
  const double* kyf;   // [ny]
  const double2* twx;  // [nx]  exp(-2 pi i k/nx)
  const double2* twy;  // [ny]
  const double2* bc;   // [Ky][Kx] compact (Hermitian-projected) topography
};

struct PhaseDev {
  const double* s;  // [P] live node shifts, ascending k
  const double* w;  // [P] weights
  int P;
};

// compact kx index of FFT position k (0..nx-1), or -1 outside the band
__device__ __forceinline__ int band_r(int k, int n, int kxm, int Kx) {
  if (k <= kxm) return k;
  if (k >= n - kxm) return k - n + Kx;
  return -1;
}

__device__ __forceinline__ size_t cidx(const GridDev& G, int f, int j, int r) {
  return ((size_t)f * G.Ky + j) * G.Kx + r;
}

// ============================================================================
// pass A: e^{s L} + inverse x-FFT of u, v, eta-b, ikx u, ikx v for one column
// ============================================================================
template <int NX, int GPC>
__global__ void __launch_bounds__(GPC* NX / 8)
    passA_kernel(GridDev G, Prop pr, PhaseDev ph, int p0, int np, const double2* __restrict__ Uc,
                 double2* __restrict__ I) {
  constexpr int T = NX / 8;
  constexpr int PAD = FFTSize<NX>::PAD;
  __shared__ double2 sm[GPC][PAD];
  const int gid = threadIdx.x / T, t = threadIdx.x % T;
  const int task = blockIdx.x * GPC + gid;
  const bool active = task < np * G.Ky;
  const int pl = active ? task / G.Ky : 0;
  const int j = active ? task % G.Ky : 0;
  const double s = active ? ph.s[p0 + pl] : 0.0;
  const double ky = G.kyc[j];

  double2 uu[8], vv[8], dd[8];
  double kxv[8];
#pragma unroll
  for (int m = 0; m < 8; ++m) {
    const int r = band_r(t + m * T, NX, G.kxm, G.Kx);
    uu[m] = vv[m] = dd[m] = czero();
    kxv[m] = 0.0;
    if (active && r >= 0) {
      C3 q = {Uc[cidx(G, 0, j, r)], Uc[cidx(G, 1, j, r)], Uc[cidx(G, 2, j, r)]};
      const double kx = G.kxc[r];
      q = expL(s, q, G.ph, kx, ky, pr);
      const double2 b = G.bc[(size_t)j * G.Kx + r];
      uu[m] = cscale(G.inv_n2, q.u);
      vv[m] = cscale(G.inv_n2, q.v);
      dd[m] = cscale(G.inv_n2, csub(q.e, b));
      kxv[m] = kx;
    }
  }
  double2* out = I + ((size_t)pl * 5 * G.Ky + j) * NX;
  const size_t fstride = (size_t)G.Ky * NX;
#pragma unroll 1
  for (int f = 0; f < 5; ++f) {
    double2 v[8];
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      switch (f) {
        case 0: v[m] = uu[m]; break;
        case 1: v[m] = vv[m]; break;
        case 2: v[m] = dd[m]; break;
        case 3: v[m] = cik(kxv[m], uu[m]); break;
        default: v[m] = cik(kxv[m], vv[m]); break;
      }
    }
    fft_reg<NX, true>(v, t, sm[gid], gid, G.twx);
    if (active) {
#pragma unroll
      for (int m = 0; m < 8; ++m) out[f * fstride + t + m * T] = v[m];
    }
  }
}

// ============================================================================
// pass B: per physical row x: y-C2R of the 7 fields (paired by physical
// dimension: (u,v), (ux,uy), (vx,vy), (depth,0)), quadratic products, y-R2C
// of (A,B) and (C,D), keep ky = 0..KYM.  In place on I (fields 0..3 out).
// ============================================================================
template <int NY>
__device__ __forceinline__ void load_pair(double2* v, int t, const double2* tile, int G, int g,
                                          int Ky, int kym, int fa, int fb, int deriv_b,
                                          const double* __restrict__ kyc) {
  // Z[k] = A[k] + i B[k] (k <= KYM), conj(A[-k]) + i conj(B[-k]) (k >= NY-KYM)
  // fa, fb: tile field indices (fb < 0: B = 0); deriv_b: B = i ky * tile[fb].
  constexpr int T = NY / 8;
#pragma unroll
  for (int m = 0; m < 8; ++m) {
    const int k = t + m * T;
    int jj;
    bool cj;
    if (k <= kym) {
      jj = k;
      cj = false;
    } else if (k >= NY - kym) {
      jj = NY - k;
      cj = true;
    } else {
      v[m] = czero();
      continue;
    }
    double2 A = tile[((size_t)fa * Ky + jj) * G + g];
    double2 B = czero();
    if (fb >= 0) {
      B = tile[((size_t)fb * Ky + jj) * G + g];
      if (deriv_b) B = cik(__ldg(kyc + jj), B);
    }
    if (jj == 0) {
      v[m] = cmk(A.x, B.x);  // Hermitian projection of the y-mean bin
    } else if (!cj) {
      v[m] = cmk(A.x - B.y, A.y + B.x);
    } else {
      v[m] = cmk(A.x + B.y, B.x - A.y);
    }
  }
}

template <int NY, int G>
__global__ void __launch_bounds__(G* NY / 8)
    passB_kernel(GridDev Gd, int np, double2* __restrict__ I) {
  constexpr int T = NY / 8;
  constexpr int PAD = FFTSize<NY>::PAD;
  extern __shared__ double2 dsm[];
  const int Ky = Gd.Ky, NX = Gd.nx;
  double2* tile = dsm;                        // [5][Ky][G]
  double2* xs = dsm + (size_t)5 * Ky * G;     // [G][PAD]
  const int gid = threadIdx.x / T, t = threadIdx.x % T;
  const int ntask = np * NX;
  const size_t fstride = (size_t)Ky * NX;

  // cooperative, x-contiguous load of the 5 input fields for G rows
  for (int idx = threadIdx.x; idx < 5 * Ky * G; idx += blockDim.x) {
    const int g = idx % G, fj = idx / G;
    const int f = fj / Ky, jj = fj % Ky;
    const int task = blockIdx.x * G + g;
    double2 val = czero();
    if (task < ntask) {
      const int pl = task / NX, x = task % NX;
      val = I[((size_t)pl * 5 + f) * fstride + (size_t)jj * NX + x];
    }
    tile[idx] = val;
  }
  __syncthreads();

  double2* sm = xs + (size_t)gid * PAD;
  double pu[8], pv[8], pa[8], pb[8];
  double2 v[8];
  // (u, v)
  load_pair<NY>(v, t, tile, G, gid, Ky, Gd.kym, 0, 1, 0, Gd.kyc);
  fft_reg<NY, true>(v, t, sm, gid, Gd.twy);
#pragma unroll
  for (int m = 0; m < 8; ++m) { pu[m] = v[m].x; pv[m] = v[m].y; }
  // (ux, uy): A = -(u ux + v uy)
  load_pair<NY>(v, t, tile, G, gid, Ky, Gd.kym, 3, 0, 1, Gd.kyc);
  fft_reg<NY, true>(v, t, sm, gid, Gd.twy);
#pragma unroll
  for (int m = 0; m < 8; ++m) pa[m] = -(pu[m] * v[m].x + pv[m] * v[m].y);
  // (vx, vy): B = -(u vx + v vy)
  load_pair<NY>(v, t, tile, G, gid, Ky, Gd.kym, 4, 1, 1, Gd.kyc);
  fft_reg<NY, true>(v, t, sm, gid, Gd.twy);
#pragma unroll
  for (int m = 0; m < 8; ++m) pb[m] = -(pu[m] * v[m].x + pv[m] * v[m].y);
  // (depth, 0): C = u depth, D = v depth
  load_pair<NY>(v, t, tile, G, gid, Ky, Gd.kym, 2, -1, 0, Gd.kyc);
  fft_reg<NY, true>(v, t, sm, gid, Gd.twy);
  double2 z2[8];
#pragma unroll
  for (int m = 0; m < 8; ++m) z2[m] = cmk(pu[m] * v[m].x, pv[m] * v[m].x);
  __syncthreads();  // every group is done reading the input tile
  double2* otile = tile;  // [4][Ky][G]

  // forward transforms of A + iB and C + iD, split into the two real spectra
#pragma unroll 1
  for (int pass = 0; pass < 2; ++pass) {
    if (pass == 0) {
#pragma unroll
      for (int m = 0; m < 8; ++m) v[m] = cmk(pa[m], pb[m]);
    } else {
#pragma unroll
      for (int m = 0; m < 8; ++m) v[m] = z2[m];
    }
    fft_reg<NY, false>(v, t, sm, gid, Gd.twy);
    group_sync<NY>(gid);
#pragma unroll
    for (int m = 0; m < 8; ++m) sm[pidx(t + m * T)] = v[m];
    group_sync<NY>(gid);
    for (int jj = t; jj < Ky; jj += T) {
      const double2 a = sm[pidx(jj)];
      const double2 b = sm[pidx((NY - jj) & (NY - 1))];
      // X = (a + conj b)/2, Y = (a - conj b)/(2i)
      const double2 X = cmk(0.5 * (a.x + b.x), 0.5 * (a.y - b.y));
      const double2 Y = cmk(0.5 * (a.y + b.y), -0.5 * (a.x - b.x));
      otile[((size_t)(2 * pass) * Ky + jj) * G + gid] = X;
      otile[((size_t)(2 * pass + 1) * Ky + jj) * G + gid] = Y;
    }
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < 4 * Ky * G; idx += blockDim.x) {
    const int g = idx % G, fj = idx / G;
    const int f = fj / Ky, jj = fj % Ky;
    const int task = blockIdx.x * G + g;
    if (task < ntask) {
      const int pl = task / NX, x = task % NX;
      I[((size_t)pl * 5 + f) * fstride + (size_t)jj * NX + x] = otile[idx];
    }
  }
}

// ============================================================================
// pass C: forward x-FFT of the 4 product spectra of one ky column, flux
// divergence, 2/3 truncation, e^{-sL}, weighted sum over this group's phases
// in ascending order onto the group's slot (averaging.py:148-155).
// ============================================================================
template <int NX, int GPC>
__global__ void __launch_bounds__(GPC* NX / 8)
    passC_kernel(GridDev G, Prop pr, PhaseDev ph, int p0, int np, int Gc, const double2* __restrict__ I,
                 double2* __restrict__ slots, int first_chunk) {
  constexpr int T = NX / 8;
  constexpr int PAD = FFTSize<NX>::PAD;
  extern __shared__ double2 dsm[];
  const int Kx = G.Kx, Ky = G.Ky;
  const int gid = threadIdx.x / T, t = threadIdx.x % T;
  const int per_group = PAD + 7 * Kx;
  double2* sm = dsm + (size_t)gid * per_group;  // exchange
  double2* F = sm + PAD;                          // [4][Kx]
  double2* acc = F + 4 * Kx;                      // [3][Kx]
  const int task = blockIdx.x * GPC + gid;
  const bool active = task < Ky * Gc;
  const int j = active ? task % Ky : 0;
  const int g = active ? task / Ky : 0;
  const int lo = (int)(((long long)g * np) / Gc), hi = (int)(((long long)(g + 1) * np) / Gc);
  const double ky = G.kyc[j];
  const size_t KyKx = (size_t)Ky * Kx;
  double2* slot = slots + (size_t)g * 3 * KyKx;

  for (int r = t; r < Kx; r += T) {
#pragma unroll
    for (int f = 0; f < 3; ++f)
      acc[f * Kx + r] = (active && !first_chunk) ? slot[f * KyKx + (size_t)j * Kx + r] : czero();
  }
  const size_t fstride = (size_t)Ky * NX;
#pragma unroll 1
  for (int pl = lo; pl < hi; ++pl) {
    const double2* in = I + ((size_t)pl * 5 * Ky + j) * NX;
#pragma unroll 1
    for (int f = 0; f < 4; ++f) {
      double2 v[8];
#pragma unroll
      for (int m = 0; m < 8; ++m) v[m] = in[f * fstride + t + m * T];
      fft_reg<NX, false>(v, t, sm, gid, G.twx);
#pragma unroll
      for (int m = 0; m < 8; ++m) {
        const int r = band_r(t + m * T, NX, G.kxm, Kx);
        if (r >= 0) F[f * Kx + r] = v[m];
      }
    }
    group_sync<NX>(gid);
    const double s = ph.s[p0 + pl], w = ph.w[p0 + pl];
    for (int r = t; r < Kx; r += T) {
      const double kx = G.kxc[r];
      const double2 fx = F[2 * Kx + r], fy = F[3 * Kx + r];
      const double2 gx = cik(kx, fx), gy = cik(ky, fy);
      C3 q = {F[r], F[Kx + r], cmk(-(gx.x + gy.x), -(gx.y + gy.y))};
      q = expL(-s, q, G.ph, kx, ky, pr);
      acc[r] = cadd(acc[r], cscale(w, q.u));
      acc[Kx + r] = cadd(acc[Kx + r], cscale(w, q.v));
      acc[2 * Kx + r] = cadd(acc[2 * Kx + r], cscale(w, q.e));
    }
    // F is rewritten by the next phase only after the next FFTs' barriers
  }
  if (active) {
    for (int r = t; r < Kx; r += T) {
#pragma unroll
      for (int f = 0; f < 3; ++f) slot[f * KyKx + (size_t)j * Kx + r] = acc[f * Kx + r];
    }
  }
}

// ordered sum of the phase-group slots -> compact tendency
__global__ void reduce_slots_kernel(const double2* __restrict__ slots, int Gc, size_t n,
                                    double2* __restrict__ out) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    double2 a = slots[i];
    for (int g = 1; g < Gc; ++g) a = cadd(a, slots[(size_t)g * n + i]);
    out[i] = a;
  }
}

// ============================================================================
// layout conversion full <-> compact
// ============================================================================
// pack with Hermitian projection (c(k) + conj c(-k))/2, which is what the
// reference's real(ifft2(.)) does to a field (grid.py:173-174).
__global__ void pack_kernel(GridDev G, const double2* __restrict__ u, const double2* __restrict__ v,
                            const double2* __restrict__ e, double2* __restrict__ Uc) {
  const size_t KyKx = (size_t)G.Ky * G.Kx;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < 3 * KyKx; i += (size_t)gridDim.x * blockDim.x) {
    const int f = (int)(i / KyKx);
    const int rem = (int)(i % KyKx);
    const int j = rem / G.Kx, r = rem % G.Kx;
    const int wx = r <= G.kxm ? r : r - G.Kx;
    const int ix = (wx + G.nx) % G.nx, jx = (G.nx - ix) % G.nx;
    const int jy = j, my = (G.ny - j) % G.ny;
    const double2* c = f == 0 ? u : (f == 1 ? v : e);
    const double2 a = c[(size_t)ix * G.ny + jy];
    const double2 b = c[(size_t)jx * G.ny + my];
    Uc[i] = cmk(0.5 * (a.x + b.x), 0.5 * (a.y - b.y));
  }
}

__device__ __forceinline__ bool full_to_compact(const GridDev& G, int ix, int jy, int& j, int& r, bool& cj) {
  int wx = ix < G.nx / 2 ? ix : ix - G.nx;
  int wy = jy < G.ny / 2 ? jy : jy - G.ny;
  if (abs(wx) > G.kxm || abs(wy) > G.kym) return false;
  cj = wy < 0;
  if (cj) { wx = -wx; wy = -wy; }
  j = wy;
  r = wx >= 0 ? wx : wx + G.Kx;
  return true;
}

__device__ __forceinline__ C3 compact_at(const GridDev& G, const double2* __restrict__ Ac, int ix, int jy) {
  int j, r;
  bool cj;
  if (!full_to_compact(G, ix, jy, j, r, cj)) return c3zero();
  C3 q = {Ac[cidx(G, 0, j, r)], Ac[cidx(G, 1, j, r)], Ac[cidx(G, 2, j, r)]};
  return cj ? c3conj(q) : q;
}

__global__ void unpack_kernel(GridDev G, const double2* __restrict__ Ac, double2* __restrict__ u,
                              double2* __restrict__ v, double2* __restrict__ e) {
  const size_t n = (size_t)G.nx * G.ny;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int ix = (int)(i / G.ny), jy = (int)(i % G.ny);
    C3 q = compact_at(G, Ac, ix, jy);
    u[i] = q.u;
    v[i] = q.v;
    e[i] = q.e;
  }
}

// ============================================================================
// full-layout per-mode kernels (apply_linear, propagate, SSPRK3 stages)
// ============================================================================
struct Full3 {
  const double2* u;
  const double2* v;
  const double2* e;
};
struct Full3w {
  double2* u;
  double2* v;
  double2* e;
};
__device__ __forceinline__ C3 ld3(const Full3& a, size_t i) { return {a.u[i], a.v[i], a.e[i]}; }
__device__ __forceinline__ void st3(const Full3w& a, size_t i, const C3& q) {
  a.u[i] = q.u;
  a.v[i] = q.v;
  a.e[i] = q.e;
}

__global__ void linear_full_kernel(GridDev G, Full3 in, Full3w out) {
  const size_t n = (size_t)G.nx * G.ny;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int ix = (int)(i / G.ny), jy = (int)(i % G.ny);
    st3(out, i, lin(ld3(in, i), G.ph, G.kxf[ix], G.kyf[jy]));
  }
}

__global__ void propagate_full_kernel(GridDev G, Prop pr, double t, Full3 in, Full3w out) {
  const size_t n = (size_t)G.nx * G.ny;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int ix = (int)(i / G.ny), jy = (int)(i % G.ny);
    st3(out, i, expL(t, ld3(in, i), G.ph, G.kxf[ix], G.kyf[jy], pr));
  }
}

// per-field non-finite bits: bit (3*(stage-1) + field)
__device__ __forceinline__ void flag_nonfinite(const C3& q, int stage, int* flags) {
  int bits = 0;
  if (!finite2(q.u)) bits |= 1 << (3 * (stage - 1) + 0);
  if (!finite2(q.v)) bits |= 1 << (3 * (stage - 1) + 1);
  if (!finite2(q.e)) bits |= 1 << (3 * (stage - 1) + 2);
  bits = __reduce_or_sync(0xffffffffu, bits);
  if (bits && (threadIdx.x & 31) == 0) atomicOr(flags, bits);
}

// stage 1 (integrator.py:96-98): e_dt = E(dt) U;  u1 = e_dt + dt * E(dt) A(U)
__global__ void stage1_kernel(GridDev G, Prop pr, double dt, Full3 U, const double2* __restrict__ Ac,
                              Full3w edt, Full3w u1, int* flags) {
  const size_t n = (size_t)G.nx * G.ny;
  for (size_t i0 = blockIdx.x * (size_t)blockDim.x; i0 < n; i0 += (size_t)gridDim.x * blockDim.x) {
    const size_t i = i0 + threadIdx.x;
    C3 o = c3zero();
    if (i < n) {
      const int ix = (int)(i / G.ny), jy = (int)(i % G.ny);
      const double kx = G.kxf[ix], ky = G.kyf[jy];
      const C3 e = expL(dt, ld3(U, i), G.ph, kx, ky, pr);
      const C3 ea = expL(dt, compact_at(G, Ac, ix, jy), G.ph, kx, ky, pr);
      o = c3add(e, c3scale(dt, ea));
      st3(edt, i, e);
      st3(u1, i, o);
    }
    flag_nonfinite(o, 1, flags);
  }
}

// stage 2 (integrator.py:99-100): u2 = 3/4 E(dt/2) U + 1/4 E(-dt/2) (u1 + dt A(u1))
__global__ void stage2_kernel(GridDev G, Prop pr, double dt, Full3 U, Full3 u1, const double2* __restrict__ Ac,
                              Full3w u2, int* flags) {
  const size_t n = (size_t)G.nx * G.ny;
  const double h = 0.5 * dt;
  for (size_t i0 = blockIdx.x * (size_t)blockDim.x; i0 < n; i0 += (size_t)gridDim.x * blockDim.x) {
    const size_t i = i0 + threadIdx.x;
    C3 o = c3zero();
    if (i < n) {
      const int ix = (int)(i / G.ny), jy = (int)(i % G.ny);
      const double kx = G.kxf[ix], ky = G.kyf[jy];
      const C3 a = expL(h, ld3(U, i), G.ph, kx, ky, pr);
      const C3 y = c3add(ld3(u1, i), c3scale(dt, compact_at(G, Ac, ix, jy)));
      const C3 b = expL(-h, y, G.ph, kx, ky, pr);
      o = c3add(c3scale(0.75, a), c3scale(0.25, b));
      st3(u2, i, o);
    }
    flag_nonfinite(o, 2, flags);
  }
}

// stage 3 (integrator.py:101-102): out = 1/3 e_dt + 2/3 E(dt/2) (u2 + dt A(u2))
__global__ void stage3_kernel(GridDev G, Prop pr, double dt, Full3 edt, Full3 u2, const double2* __restrict__ Ac,
                              Full3w out, int* flags) {
  const size_t n = (size_t)G.nx * G.ny;
  const double h = 0.5 * dt;
  for (size_t i0 = blockIdx.x * (size_t)blockDim.x; i0 < n; i0 += (size_t)gridDim.x * blockDim.x) {
    const size_t i = i0 + threadIdx.x;
    C3 o = c3zero();
    if (i < n) {
      const int ix = (int)(i / G.ny), jy = (int)(i % G.ny);
      const double kx = G.kxf[ix], ky = G.kyf[jy];
      const C3 y = c3add(ld3(u2, i), c3scale(dt, compact_at(G, Ac, ix, jy)));
      const C3 b = expL(h, y, G.ph, kx, ky, pr);
      o = c3add(c3scale(1.0 / 3.0, ld3(edt, i)), c3scale(2.0 / 3.0, b));
      st3(out, i, o);
    }
    flag_nonfinite(o, 3, flags);
  }
}

__global__ void twiddle_kernel(double2* tw, int n) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    double s, c;
    sincospi(2.0 * k / n, &s, &c);
    tw[k] = cmk(c, -s);
  }
}

}  // namespace pswe

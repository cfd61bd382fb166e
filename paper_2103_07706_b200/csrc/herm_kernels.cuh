// The Hermitian-symmetry gate of the reference's to_physical (grid.py:140-180):
// a spectral field must satisfy c(-k) = conj c(k) to HERMITIAN_RTOL = 1e-12
// (grid.py:31) relative to max(largest coefficient, scale), otherwise
//   ValueError("non-Hermitian spectral field: mode (kx index i, ky index j)
//               has asymmetry A (relative R)")
// naming the most offending mode (first in row-major order on ties).
//
// Inside apply_nonlinear (dynamics.py:159-169) the gate sees, at every
// averaging node s, the dealiased fields u', v', eta' - b of e^{sL} U with
// one scale = their common maximum (the derivative fields then pass
// whenever u and v pass: their defect is |k| times u's, their reference
// scale_k = scale * max|k| is larger by more than that).
//
// Fast path (every full-layout call, no host round trip):
//   pack   -> max over the band of |D_f(k)|^2, D = c(k) - conj c(-k), per field
//   pass A -> per phase, max over the band of |e^{sL} U_h - b_h|_f^2 on the
//             Hermitian part it propagates anyway
//   herm_eval_block (by block 0 of the kernel that consumes the RHS -- the
//             stage kernel or unpack): e^{sL} is unitary in the energy norm
//             |x|_W^2 = H(|u|^2 + |v|^2) + g |eta|^2, so every propagated
//             defect is at most d = |D|_W / sqrt(min(H, g)) + max|D_b| and the
//             true scale is at least scale_h(s) - d / 2: when d < 1e-12
//             (scale_h(s) - d / 2) for every phase no node can fail -- the
//             common case (numpy's fft2 leaves ~1e-16 relative asymmetry).
//             Otherwise a flag is raised and the host runs the exact check.
// Exact path (flagged calls only): herm_node_kernel recomputes, per node,
// the propagated band fields at k and -k exactly as the reference forms
// them and reduces scale, worst defect and its mode; the host applies the
// reference's test in node order (averaging.py:130-141 wraps the message).
#pragma once
#include "pswe_kernels.cuh"

namespace pswe {

// block reduction of (max, first index) pairs and nonneg maxima
struct HermAcc {
  double scale;   // max |F_f| over the fields
  double def[3];  // worst defect per field
  long long idx[3];
  int nonfinite;
};

__device__ __forceinline__ void herm_take(HermAcc& a, int f, double d, long long i) {
  if (d > a.def[f] || (d == a.def[f] && i < a.idx[f])) {
    a.def[f] = d;
    a.idx[f] = i;
  }
}

template <int NT>
__device__ void herm_block_reduce(HermAcc& a, double* out) {
  __shared__ double ssc[NT / 32], sdef[3][NT / 32];
  __shared__ long long sidx[3][NT / 32];
  __shared__ int snf[NT / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int o = 16; o; o >>= 1) {
    a.scale = fmax(a.scale, __shfl_xor_sync(0xffffffffu, a.scale, o));
    a.nonfinite |= __shfl_xor_sync(0xffffffffu, a.nonfinite, o);
#pragma unroll
    for (int f = 0; f < 3; ++f) {
      const double d = __shfl_xor_sync(0xffffffffu, a.def[f], o);
      const long long i = __shfl_xor_sync(0xffffffffu, a.idx[f], o);
      herm_take(a, f, d, i);
    }
  }
  if (lane == 0) {
    ssc[w] = a.scale;
    snf[w] = a.nonfinite;
    for (int f = 0; f < 3; ++f) {
      sdef[f][w] = a.def[f];
      sidx[f][w] = a.idx[f];
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < NT / 32; ++k) {
      a.scale = fmax(a.scale, ssc[k]);
      a.nonfinite |= snf[k];
      for (int f = 0; f < 3; ++f) herm_take(a, f, sdef[f][k], sidx[f][k]);
    }
    out[0] = a.scale;
    for (int f = 0; f < 3; ++f) {
      out[1 + 2 * f] = a.def[f];
      out[2 + 2 * f] = (double)a.idx[f];
    }
    out[7] = a.nonfinite;
  }
}

// Exact gate of one averaging node per CTA (error path): the dealiased
// fields F = (u', v', eta' - b) of e^{s L} U (the identity for s = 0, as
// averaging.py:133-134) at every band mode k and its mirror -k, exactly as
// the reference forms them; out[node][8] = scale, (defect, flat index) of
// u, v, depth, nonfinite flag.
template <int NT>
__global__ void __launch_bounds__(NT) herm_node_kernel(GridDev G, Prop pr, const double* __restrict__ s,
                                                       const double2* __restrict__ u, const double2* __restrict__ v,
                                                       const double2* __restrict__ e,
                                                       const double2* __restrict__ b, double* __restrict__ out) {
  const double t = s[blockIdx.x];
  const int nx = G.nx, ny = G.ny;
  const int bw = 2 * G.kym + 1;  // band columns
  const long long nb = (long long)(2 * G.kxm + 1) * bw;
  HermAcc a;
  a.scale = 0.0;
  a.nonfinite = 0;
  for (int f = 0; f < 3; ++f) {
    a.def[f] = 0.0;
    a.idx[f] = LLONG_MAX;
  }
  for (long long m = threadIdx.x; m < nb; m += NT) {
    const int wx = (int)(m / bw) - G.kxm, wy = (int)(m % bw) - G.kym;
    const int ix = (wx + nx) % nx, jy = (wy + ny) % ny;
    const int mx = (nx - ix) % nx, my = (ny - jy) % ny;
    const size_t i = (size_t)ix * ny + jy, im = (size_t)mx * ny + my;
    C3 q = {u[i], v[i], e[i]}, qm = {u[im], v[im], e[im]};
    if (t != 0.0) {
      q = expL(t, q, G.ph, G.kxf[ix], G.kyf[jy], pr);
      qm = expL(t, qm, G.ph, G.kxf[mx], G.kyf[my], pr);
    }
    if (b) {
      q.e = csub(q.e, b[i]);
      qm.e = csub(qm.e, b[im]);
    }
    const double2 F[3] = {q.u, q.v, q.e}, Fm[3] = {qm.u, qm.v, qm.e};
#pragma unroll
    for (int f = 0; f < 3; ++f) {
      const double mag = hypot(F[f].x, F[f].y);
      if (!isfinite(mag)) a.nonfinite = 1;
      a.scale = fmax(a.scale, mag);
      // c(k) - conj(c(-k)), as numpy evaluates coeffs - np.conj(_reflect(coeffs))
      herm_take(a, f, hypot(F[f].x - Fm[f].x, F[f].y + Fm[f].y), (long long)i);
    }
  }
  herm_block_reduce<NT>(a, out + (size_t)blockIdx.x * 8);
}

// Exact full-grid gate of up to three fields per CTA group (snapshot
// diagnostics and to_physical: the fields as given, no dealiasing,
// integrator.py:124-135, diagnostics.py:21-25, io.py:41-46): CTA f reduces
// field f: out[f][8] = max|c|, defect/index in slot 0, nonfinite flag.
template <int NT>
__global__ void __launch_bounds__(NT) herm_full_kernel(int nx, int ny, const double2* __restrict__ f0,
                                                       const double2* __restrict__ f1,
                                                       const double2* __restrict__ f2,
                                                       const double2* __restrict__ f3, double* __restrict__ out) {
  const double2* c = blockIdx.x == 0 ? f0 : (blockIdx.x == 1 ? f1 : (blockIdx.x == 2 ? f2 : f3));
  HermAcc a;
  a.scale = 0.0;
  a.nonfinite = 0;
  for (int f = 0; f < 3; ++f) {
    a.def[f] = 0.0;
    a.idx[f] = LLONG_MAX;
  }
  const long long n = (long long)nx * ny;
  for (long long i = threadIdx.x; i < n; i += NT) {
    const int ix = (int)(i / ny), jy = (int)(i % ny);
    const size_t im = (size_t)((nx - ix) % nx) * ny + (ny - jy) % ny;
    const double2 x = c[i], y = c[im];
    const double mag = hypot(x.x, x.y);
    if (!isfinite(mag)) a.nonfinite = 1;
    a.scale = fmax(a.scale, mag);
    herm_take(a, 0, hypot(x.x - y.x, x.y + y.y), i);
  }
  herm_block_reduce<NT>(a, out + (size_t)blockIdx.x * 8);
}

}  // namespace pswe

// Small grids (n <= 64): the whole averaged-RHS term of a phase in ONE CTA.
//
// The three-pass pipeline (passes A, B, C) moves ~0.5 MB of intermediates
// per phase through HBM at 64^2 and pays three launches plus their fill /
// drain per evaluation: at n <= 64 an evaluation is latency-bound (SURVEY.md
// section 2 note on K2-K4, section 7 step 5).  Here a CTA owns a contiguous
// group of phases and runs, per phase, entirely in shared memory:
//
//   A  e^{sL} U per compact mode (phase table or Chebyshev), then the five
//      inverse x-FFTs (u, v, eta - b, ikx u, ikx v) of every ky column into
//      I[f][j][x]                                     (pass A of pswe_kernels)
//   B  per physical row x: the y-C2R of the dimension-matched pairs, the four
//      quadratic products, the two y-R2C, written back over the row's
//      consumed inputs I[0..3][j][x]                   (pass B)
//   C  forward x-FFT of every product column, 2/3 truncation, flux
//      divergence, e^{-sL}, weight, accumulated in registers     (pass C)
//
// and writes its phase group's sum once (slot g), followed by the ordered
// slot reduction -- or directly the output when one CTA holds every phase.
// The arithmetic per value is that of the three passes (same transforms,
// same pairing, same formulas), so the results agree with them to round-off.
// Window batches (MW): a group spanning several windows flushes its sum into
// slot [g][window] at every window boundary (slots zeroed first).
#pragma once
#include "pswe_kernels.cuh"

namespace pswe {

template <int N>
struct FusedW {
  static constexpr int T = WF<N>::T, P = WF<N>::P, GPW = WF<N>::GPW;
  static constexpr int K = N / 3, Kx = 2 * K + 1, Ky = K + 1, KyKx = Ky * Kx;
  // warps: enough groups for one round of stage B (one row per group)
  static constexpr int WARPS = N == 64 ? 8 : (N == 32 ? 4 : (N == 16 ? 2 : 1));
  static constexpr int NT = WARPS * 32;
  static constexpr int LD = N + 1;  // column stride of I (complex): conflict-free row reads
  static constexpr int CPT = (KyKx + NT - 1) / NT;  // combine modes per thread
  static constexpr size_t I_BYTES = (size_t)5 * Ky * LD * sizeof(double2);
  static constexpr size_t EU_BYTES = (size_t)3 * KyKx * sizeof(double2);
  static constexpr size_t XB_BYTES = (size_t)WARPS * GPW * WF<N>::XBUF * sizeof(double);
  static constexpr size_t R_BYTES = EU_BYTES > XB_BYTES ? EU_BYTES : XB_BYTES;
  // exchange buffers of the idle groups of a last, partial round (their results are discarded)
  static constexpr size_t SCR_BYTES = (size_t)GPW * WF<N>::XBUF * sizeof(double);
  // I | R (stage A: e^{sL} U compact [3][Ky][Kx]; stage B: exchange buffers) | ACC [3][Ky][Kx]
  // (the group's weighted sum; each thread owns its modes) | ky | idle scratch
  static constexpr size_t KY_BYTES = ((size_t)Ky * sizeof(double) + 15) / 16 * 16;
  static constexpr size_t bytes() { return I_BYTES + R_BYTES + EU_BYTES + KY_BYTES + SCR_BYTES; }
  // a column's own storage serves as its transform's exchange buffer
  static_assert(WF<N>::XBUF <= 2 * LD, "exchange buffer must fit in a column");
};

// y-transform input of the packed pair (A + iB) at position k = t + T N1 of
// row x, read from the column-major I with stride LD (cf. pair_val)
template <int N, int N1, bool HAS_B, bool DERIV>
__device__ __forceinline__ double2 fused_pair_val(int t, const double2* pA, const double2* pB, const double* kys) {
  constexpr int T = WF<N>::T, KYM = N / 3, LD = FusedW<N>::LD;
  constexpr int kmin = T * N1, kmax = T * N1 + T - 1;
  if constexpr (kmin > KYM && kmax < N - KYM) {
    return czero();
  } else {
    const int k = t + kmin;
    bool lo;
    if constexpr (kmax <= KYM) {
      lo = true;
    } else if constexpr (kmin >= N - KYM) {
      lo = false;
    } else {
      lo = k <= KYM;
      if (!lo && k < N - KYM) return czero();
    }
    const int jj = lo ? k : N - k;
    const double2 A = pA[(size_t)jj * LD];
    double2 B = czero();
    if constexpr (HAS_B) {
      B = pB[(size_t)jj * LD];
      if constexpr (DERIV) B = cik(kys[jj], B);
    }
    if constexpr (N1 == 0) {
      if (t == 0) return cmk(A.x, B.x);  // Hermitian projection of the y-mean bin
    }
    return lo ? cmk(A.x - B.y, A.y + B.x) : cmk(A.x + B.y, B.x - A.y);
  }
}

template <int N, bool HAS_B, bool DERIV, int N1 = 0>
__device__ __forceinline__ void fused_pair(double2* v, int t, const double2* pA, const double2* pB,
                                           const double* kys) {
  if constexpr (N1 < WF<N>::P) {
    v[N1] = fused_pair_val<N, N1, HAS_B, DERIV>(t, pA, pB, kys);
    fused_pair<N, HAS_B, DERIV, N1 + 1>(v, t, pA, pB, kys);
  }
}

template <int N, bool MW>
__global__ void __launch_bounds__(FusedW<N>::NT)
    fused_kernel(GridDev G, Prop pr, PhaseDev ph, int Gc, const double2* __restrict__ Uc,
                 const double2* __restrict__ ctab, double2* __restrict__ out, double* __restrict__ pscale) {
  // the dependency wait is below, after the part that reads nothing the kernels before this one wrote
  using W = FusedW<N>;
  constexpr int T = W::T, P = W::P, GPW = W::GPW, Ky = W::Ky, Kx = W::Kx, KyKx = W::KyKx, LD = W::LD;
  constexpr int CPT = W::CPT, NT = W::NT;
  extern __shared__ __align__(128) unsigned char sbytes[];
  double2* I = reinterpret_cast<double2*>(sbytes);                    // [5][Ky][LD]
  double2* EU = reinterpret_cast<double2*>(sbytes + W::I_BYTES);      // [3][Ky][Kx] (stage A)
  double* XB = reinterpret_cast<double*>(sbytes + W::I_BYTES);        // exchange buffers (stage B)
  double2* ACC = reinterpret_cast<double2*>(sbytes + W::I_BYTES + W::R_BYTES);  // [3][Ky][Kx]
  double* kys = reinterpret_cast<double*>(sbytes + W::I_BYTES + W::R_BYTES + W::EU_BYTES);
  double* idle = reinterpret_cast<double*>(sbytes + W::I_BYTES + W::R_BYTES + W::EU_BYTES + W::KY_BYTES);
  const int g = blockIdx.x;
  const int lo = (int)(((long long)g * ph.P) / Gc), hi = (int)(((long long)(g + 1) * ph.P) / Gc);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int t = lane % T, gi = lane / T;         // lane in its transform group, group in the warp
  const int grp = warp * GPW + gi, ngrp = W::WARPS * GPW;
  const bool tab = ctab != nullptr;
  const WLane wlx = wlane<N>(G.twx, t), wly = wlane<N>(G.twy, t);
  for (int i = threadIdx.x; i < Ky; i += NT) kys[i] = G.kyc[i];

  auto zero_acc = [&]() {
    for (int idx = threadIdx.x; idx < 3 * KyKx; idx += NT) ACC[idx] = czero();
  };
  auto flush = [&](int win, bool add) {  // the thread's own modes: no barrier needed
    double2* slot = out + ((size_t)g * ph.W + win) * 3 * KyKx;
    for (int idx = threadIdx.x; idx < 3 * KyKx; idx += NT) slot[idx] = add ? cadd(slot[idx], ACC[idx]) : ACC[idx];
  };
  zero_acc();
  griddep_wait();  // Uc, the gate scale and the slots belong to the kernels before this one
  // only now: the next kernel (a stage kernel when the slot reduction is skipped) reads states written
  // two kernels back before its own wait, so it must not start until this kernel has waited
  griddep_launch();
  int wcur = MW && lo < hi ? ph.win[lo] : 0;

#pragma unroll 1
  for (int p = lo; p < hi; ++p) {
    if constexpr (MW) {
      if (ph.win[p] != wcur) {
        flush(wcur, true);
        zero_acc();
        wcur = ph.win[p];
      }
    }
    const double s = ph.s[p], w = ph.w[p];
    const double2* U = Uc + (MW ? (size_t)ph.win[p] * ph.ustride : 0);
    const double2* ct = tab ? ctab + (size_t)p * KyKx : nullptr;
    // ---- stage A: e^{sL} U per compact mode, scaled by 1/(nx ny)
    double gmax = 0.0;
    for (int idx = threadIdx.x; idx < KyKx; idx += NT) {
      const int j = idx / Kx, r = idx % Kx;
      const C3 q0 = {U[idx], U[KyKx + idx], U[2 * KyKx + idx]};
      const double kx = __ldg(G.kxc + r), ky = kys[j];
      const C3 q = tab ? exp_c12(ct[idx], q0, G.ph, kx, ky) : expL(s, q0, G.ph, kx, ky, pr);
      const double2 dep = csub(q.e, G.bc[idx]);
      EU[idx] = cscale(G.inv_n2, q.u);
      EU[KyKx + idx] = cscale(G.inv_n2, q.v);
      EU[2 * KyKx + idx] = cscale(G.inv_n2, dep);
      if (pscale) gmax = nanmax(gmax, nanmax(nanmax(abs2(q.u), abs2(q.v)), abs2(dep)));
    }
    if (pscale) {  // the Hermitian gate's per-phase scale (see pass A)
#pragma unroll
      for (int o = 16; o; o >>= 1) gmax = nanmax(gmax, __shfl_xor_sync(0xffffffffu, gmax, o));
      if (lane == 0)
        atomicMax(reinterpret_cast<unsigned long long*>(pscale + p), (unsigned long long)__double_as_longlong(gmax));
    }
    __syncthreads();
    // inverse x-FFTs of the 5 fields per ky column into I[f][j][.]; the
    // destination column is the exchange buffer until the result is stored
    // (loops advance warp-uniformly: every lane takes part in the transforms'
    // warp-wide exchanges; a group past the end computes on zeros, stores nothing)
#pragma unroll 1
    for (int base = warp * GPW; base < 5 * Ky; base += ngrp) {
      const int task = base + gi;
      const bool active = task < 5 * Ky;
      const int f = active ? task / Ky : 0, j = active ? task % Ky : 0;
      const int fi = f < 3 ? f : f - 3;
      double2 v[P];
      band_gather<N>(v, t, EU + (size_t)fi * KyKx + (size_t)j * Kx, active);
      if (f >= 3) {
#pragma unroll
        for (int n1 = 0; n1 < P; ++n1) {
          const int r = band_r(t + T * n1, N, N / 3, Kx);
          if (r >= 0) v[n1] = cik(__ldg(G.kxc + r), v[n1]);
        }
      }
      double2* col = I + (size_t)task * LD;
      wfft_t1<N, true, true>(v, t, active ? reinterpret_cast<double*>(col) : idle + (size_t)gi * WF<N>::XBUF, wlx);
      __syncwarp();
      if (active) store_t1_strided<N>(v, t, col, 1);
    }
    __syncthreads();
    // ---- stage B: one physical row per group
#pragma unroll 1
    for (int base = warp * GPW; base < N; base += ngrp) {  // warp-uniform, like stages A and C
      const int xg = base + gi;
      const bool active = xg < N;
      const int x = active ? xg : 0;
      double* xb = XB + (size_t)grp * WF<N>::XBUF;
      const double2* row = I + x;
      auto fld = [&](int f) { return row + (size_t)f * Ky * LD; };
      double2 v[P], uv[P];
      double pa[P];
      fused_pair<N, true, false>(v, t, fld(0), fld(1), kys);  // (u, v)
      wfft_t1<N, true, true>(v, t, xb, wly);
#pragma unroll
      for (int i = 0; i < P; ++i) uv[i] = v[i];
      fused_pair<N, true, true>(v, t, fld(3), fld(0), kys);  // (ux, i ky u)
      wfft_t1<N, true, true>(v, t, xb, wly);
#pragma unroll
      for (int i = 0; i < P; ++i) pa[i] = ndot(uv[i], v[i]);  // A = -(u ux + v uy)
      fused_pair<N, true, true>(v, t, fld(4), fld(1), kys);  // (vx, i ky v)
      wfft_t1<N, true, true>(v, t, xb, wly);
#pragma unroll
      for (int i = 0; i < P; ++i) v[i] = cmk(pa[i], ndot(uv[i], v[i]));  // + iB
      wfft_t2<N, false>(v, t, xb, wly);
      __syncwarp();  // the row's (u, v) inputs were read by every lane of the group
      unpack_store<N>(v, t, const_cast<double2*>(fld(0)), const_cast<double2*>(fld(1)), Ky, LD, active);
      fused_pair<N, false, false>(v, t, fld(2), nullptr, kys);  // depth
      wfft_t1<N, true, true>(v, t, xb, wly);
#pragma unroll
      for (int i = 0; i < P; ++i) v[i] = cmk(uv[i].x * v[i].x, uv[i].y * v[i].x);  // C + iD = u d + i v d
      wfft_t2<N, false>(v, t, xb, wly);
      __syncwarp();
      unpack_store<N>(v, t, const_cast<double2*>(fld(2)), const_cast<double2*>(fld(3)), Ky, LD, active);
    }
    __syncthreads();
    // ---- stage C: forward x-FFT of the 4 product columns, band kept in place
#pragma unroll 1
    for (int base = warp * GPW; base < 4 * Ky; base += ngrp) {
      const int task = base + gi;
      const bool active = task < 4 * Ky;
      double2* col = I + (size_t)(active ? task : 0) * LD;
      double2 v[P];
#pragma unroll
      for (int n1 = 0; n1 < P; ++n1) v[n1] = active ? col[t + T * n1] : czero();
      __syncwarp();
      wfft_t1<N, false>(v, t, active ? reinterpret_cast<double*>(col) : idle + (size_t)gi * WF<N>::XBUF, wlx);
      __syncwarp();
      if (active) {
#pragma unroll
        for (int i = 0; i < P; ++i) {
          const int r = band_r(t1_pos<N>(t, i), N, N / 3, Kx);
          if (r >= 0) col[r] = v[i];
        }
      }
    }
    __syncthreads();
    // combine: flux divergence, e^{-sL}, weight; ascending phase order per mode
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      const int idx = threadIdx.x + c * NT;
      if (idx < KyKx) {
        const int j = idx / Kx, r = idx % Kx;
        const double2* F = I + (size_t)j * LD + r;  // field f at + f Ky LD
        const double kx = __ldg(G.kxc + r), ky = kys[j];
        const double2 gx = cik(kx, F[2 * Ky * LD]), gy = cik(ky, F[3 * Ky * LD]);
        C3 q = {F[0], F[Ky * LD], cmk(-(gx.x + gy.x), -(gx.y + gy.y))};
        if (tab) {
          double2 c12 = ct[idx];
          c12.x = -c12.x;  // e^{-sL}: c1(-s) = -c1(s), c2(-s) = c2(s)
          q = exp_c12(c12, q, G.ph, kx, ky);
        } else {
          q = expL(-s, q, G.ph, kx, ky, pr);
        }
        const C3 a = c3add({ACC[idx], ACC[KyKx + idx], ACC[2 * KyKx + idx]}, c3scale(w, q));
        ACC[idx] = a.u;
        ACC[KyKx + idx] = a.v;
        ACC[2 * KyKx + idx] = a.e;
      }
    }
    __syncthreads();  // I is rewritten by the next phase's stage A
  }
  if (MW) {
    if (lo < hi) flush(wcur, true);
  } else {
    flush(0, false);
  }
}

}  // namespace pswe

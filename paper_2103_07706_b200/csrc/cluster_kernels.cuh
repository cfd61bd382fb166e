// 64^2: one THREAD-BLOCK CLUSTER per phase group (C CTAs on C SMs), the
// three passes of a phase in distributed shared memory.
//
// At 64^2 a phase is too much work for one CTA's latency (fused_kernels.cuh
// measured slower than the three-pass pipeline there) and too little for
// three HBM round trips and four launches.  Here the cluster splits it:
//
//   A  CTA r owns the ky columns j = r, r + C, ... (its share of I[f][j][x]
//      in its own shared memory): e^{sL} U of those columns' modes and their
//      five inverse x-FFTs                                          (pass A)
//   -- cluster barrier --
//   B  CTA r owns the physical rows [r N/C, (r+1) N/C): four warps per row
//      group run the four inverse y-transforms at once (u, v), (ux, i ky u),
//      (vx, i ky v), (depth), reading the row's spectra from every CTA's
//      columns through distributed shared memory; the physical values meet
//      in a local stash; two warps run the forward transforms (A + iB),
//      (C + iD) and store the ky >= 0 half back into the owners' columns
//      (remote stores)                               (passB_split_kernel)
//   -- cluster barrier --
//   C  CTA r: forward x-FFTs of its product columns in place, flux
//      divergence, e^{-sL}, weight, summed into its modes       (pass C)
//
// Phase groups loop inside the cluster; each CTA writes its columns' part
// of the group's slot, followed by the ordered slot reduction.  Same
// transforms and formulas as the passes: results agree to round-off.
#pragma once
#include <cooperative_groups.h>

#include "pswe_kernels.cuh"

namespace pswe {

namespace cg = cooperative_groups;

template <int N, int C>
struct CFusedW {
  static constexpr int T = WF<N>::T, P = WF<N>::P, GPW = WF<N>::GPW;
  static constexpr int K = N / 3, Kx = 2 * K + 1, Ky = K + 1, KyKx = Ky * Kx;
  static constexpr int JL = (Ky + C - 1) / C;  // columns per CTA (at most)
  static constexpr int LD = N + 1;
  static constexpr int ROWS = N / C;           // physical rows per CTA
  static constexpr int RG = ROWS / GPW;        // row groups per CTA (four warps each)
  static constexpr int WARPS = 4 * RG;
  static constexpr int NT = WARPS * 32;
  static_assert(ROWS % GPW == 0 && RG >= 1, "whole row groups per CTA");
  static constexpr size_t I_BYTES = (size_t)5 * JL * LD * sizeof(double2);
  static constexpr size_t EU_BYTES = (size_t)3 * JL * Kx * sizeof(double2);
  static constexpr size_t STASH_BYTES = (size_t)RG * 4 * P * 32 * sizeof(double2);
  static constexpr size_t R_BYTES = EU_BYTES > STASH_BYTES ? EU_BYTES : STASH_BYTES;
  static constexpr size_t XB_BYTES = (size_t)WARPS * GPW * WF<N>::XBUF * sizeof(double);
  static constexpr size_t ACC_BYTES = (size_t)3 * JL * Kx * sizeof(double2);
  static constexpr size_t KY_BYTES = ((size_t)Ky * sizeof(double) + 15) / 16 * 16;
  static constexpr size_t SCR_BYTES = (size_t)GPW * WF<N>::XBUF * sizeof(double);
  // my modes' U (u, v, eta) and b, cached once per kernel (one window), and kx
  static constexpr size_t UC_BYTES = (size_t)4 * JL * Kx * sizeof(double2);
  static constexpr size_t KX_BYTES = ((size_t)Kx * sizeof(double) + 15) / 16 * 16;
  static constexpr int MI = (JL * Kx + NT - 1) / NT;  // modes per thread (at most)
  // stage A's outputs pushed to the row owners: [5][Ky][RLD], my rows
  static constexpr int RLD = ROWS + 1;
  static constexpr size_t IR_BYTES = (size_t)5 * Ky * RLD * sizeof(double2);
  // I | R (stage A: e^{sL} U; stage B: physical stash) | exchange buffers | ACC | ky | idle scratch | U, b | kx
  static constexpr size_t bytes() {
    return I_BYTES + R_BYTES + XB_BYTES + ACC_BYTES + KY_BYTES + SCR_BYTES + UC_BYTES + KX_BYTES + IR_BYTES;
  }
  static_assert(WF<N>::XBUF <= 2 * LD, "exchange buffer must fit in a column");
};

template <int N, int C, bool MW>
__global__ void __launch_bounds__(CFusedW<N, C>::NT, 1)
    cfused_kernel(GridDev G, Prop pr, PhaseDev ph, int Gc, const double2* __restrict__ Uc,
                  const double2* __restrict__ ctab, double2* __restrict__ out, double* __restrict__ pscale) {
  // the dependency wait is below, after the part that reads nothing the kernels before this one wrote
  using W = CFusedW<N, C>;
  constexpr int T = W::T, P = W::P, GPW = W::GPW, Ky = W::Ky, Kx = W::Kx, KyKx = W::KyKx, LD = W::LD;
  constexpr int JL = W::JL, NT = W::NT;
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  extern __shared__ __align__(128) unsigned char sbytes[];
  double2* I = reinterpret_cast<double2*>(sbytes);  // [5][JL][LD], my columns
  unsigned char* q = sbytes + W::I_BYTES;
  double2* EU = reinterpret_cast<double2*>(q);      // [3][JL][Kx] (stage A)
  double2* stash = reinterpret_cast<double2*>(q);   // [RG][4][P][32] (stage B)
  q += W::R_BYTES;
  double* XB = reinterpret_cast<double*>(q);
  q += W::XB_BYTES;
  double2* ACC = reinterpret_cast<double2*>(q);     // [3][JL][Kx]
  q += W::ACC_BYTES;
  double* kys = reinterpret_cast<double*>(q);
  q += W::KY_BYTES;
  double* idle = reinterpret_cast<double*>(q);
  q += W::SCR_BYTES;
  double2* UCc = reinterpret_cast<double2*>(q);  // [4][JL][Kx]: u, v, eta, b of my modes
  q += W::UC_BYTES;
  double* kxs = reinterpret_cast<double*>(q);
  q += W::KX_BYTES;
  // stage B's inputs, my rows of every column: stage A's CTAs store them
  // here remotely (distributed shared memory stores do not stall the
  // writer), so stage B reads locally instead of issuing remote loads
  double2* IR = reinterpret_cast<double2*>(q);  // [5][Ky][RLD]
  constexpr int RLD = W::RLD, ROWS = W::ROWS;
  // every CTA's columns, by rank (distributed shared memory)
  // column (f, j) of its owner CTA (mapa per access: no per-rank pointer table in local memory)
  auto colp = [&](int f, int j) -> double2* {
    return cluster.map_shared_rank(I + ((size_t)f * JL + j / C) * LD, (unsigned)(j % C));
  };

  const int g = blockIdx.x / C;  // phase group = cluster
  const int lo = (int)(((long long)g * ph.P) / Gc), hi = (int)(((long long)(g + 1) * ph.P) / Gc);
  const int jl_n = (Ky - rank + C - 1) / C;  // my columns: j = rank + C jl, jl < jl_n
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int t = lane % T, gi = lane / T;
  const int grp = warp * GPW + gi, ngrp = W::WARPS * GPW;
  const bool tab = ctab != nullptr;
  const WLane wlx = wlane<N>(G.twx, t), wly = wlane<N>(G.twy, t);
  for (int i = threadIdx.x; i < Ky; i += NT) kys[i] = G.kyc[i];
  for (int i = threadIdx.x; i < Kx; i += NT) kxs[i] = G.kxc[i];
  griddep_wait();  // Uc, the gate scale and the slots belong to the kernels before this one
  // only now: the next kernel (a stage kernel when the slot reduction is skipped) reads states written
  // two kernels back before its own wait, so it must not start until this kernel has waited
  griddep_launch();
  const int nmode = jl_n * Kx;  // my compact modes
  constexpr int MI = W::MI;
  // one window: my modes' U and b stay in shared memory for all phases
  // (window batches read each phase's window state from global memory)
  if constexpr (!MW) {
    for (int m = threadIdx.x; m < nmode; m += NT) {
      const int jl = m / Kx, r = m % Kx, idx = (rank + C * jl) * Kx + r;
      const size_t e = (size_t)jl * Kx + r;
      UCc[e] = Uc[idx];
      UCc[JL * Kx + e] = Uc[KyKx + idx];
      UCc[2 * JL * Kx + e] = Uc[2 * KyKx + idx];
      UCc[3 * JL * Kx + e] = G.bc[idx];
    }
  }
  // each thread's modes m = tid + k NT: their (c1, c2) phase-table entries
  // for the next phase are loaded a whole phase ahead (and reused by the
  // combine), so no table load sits on a phase's critical path
  double2 c12n[MI];
  auto load_c12 = [&](int p) {
#pragma unroll
    for (int k = 0; k < MI; ++k) {
      const int m = threadIdx.x + k * NT;
      c12n[k] = czero();
      if (ctab && p < hi && m < nmode) {
        const int jl = m / Kx, r = m % Kx;
        c12n[k] = __ldg(ctab + (size_t)p * KyKx + (size_t)(rank + C * jl) * Kx + r);
      }
    }
  };

  auto zero_acc = [&]() {
    for (int idx = threadIdx.x; idx < 3 * JL * Kx; idx += NT) ACC[idx] = czero();
  };
  auto flush = [&](int win, bool add) {  // my columns of slot [g][win]
    double2* slot = out + ((size_t)g * ph.W + win) * 3 * KyKx;
    for (int idx = threadIdx.x; idx < 3 * nmode; idx += NT) {
      const int f = idx / nmode, m = idx % nmode, jl = m / Kx, r = m % Kx;
      double2* d = slot + (size_t)f * KyKx + (size_t)(rank + C * jl) * Kx + r;
      const double2 v = ACC[((size_t)f * JL + jl) * Kx + r];
      *d = add ? cadd(*d, v) : v;
    }
  };
  zero_acc();
  int wcur = MW && lo < hi ? ph.win[lo] : 0;
  load_c12(lo);
  __syncthreads();

#pragma unroll 1
  for (int p = lo; p < hi; ++p) {
    if constexpr (MW) {
      if (ph.win[p] != wcur) {
        flush(wcur, true);
        __syncthreads();  // flush reads ACC in another thread order than zero_acc writes it
        zero_acc();
        wcur = ph.win[p];
      }
    }
    const double s = ph.s[p], w = ph.w[p];
    const double2* U = Uc + (MW ? (size_t)ph.win[p] * ph.ustride : 0);
    double2 c12c[MI];
#pragma unroll
    for (int k = 0; k < MI; ++k) c12c[k] = c12n[k];
    load_c12(p + 1);
    // ---- A: e^{sL} U of my columns' modes, scaled by 1/(nx ny)
    double gmax = 0.0;
#pragma unroll
    for (int k = 0; k < MI; ++k) {
      const int m = threadIdx.x + k * NT;
      if (m >= nmode) break;
      const int jl = m / Kx, r = m % Kx, j = rank + C * jl;
      const int idx = j * Kx + r;
      const size_t e = (size_t)jl * Kx + r;
      const C3 q0 = MW ? C3{U[idx], U[KyKx + idx], U[2 * KyKx + idx]}
                       : C3{UCc[e], UCc[JL * Kx + e], UCc[2 * JL * Kx + e]};
      const double kx = kxs[r], ky = kys[j];
      const C3 qe = tab ? exp_c12(c12c[k], q0, G.ph, kx, ky) : expL(s, q0, G.ph, kx, ky, pr);
      const double2 dep = csub(qe.e, MW ? G.bc[idx] : UCc[3 * JL * Kx + e]);
      EU[e] = cscale(G.inv_n2, qe.u);
      EU[JL * Kx + e] = cscale(G.inv_n2, qe.v);
      EU[2 * JL * Kx + e] = cscale(G.inv_n2, dep);
      if (pscale) gmax = fmax(gmax, fmax(fmax(abs2(qe.u), abs2(qe.v)), abs2(dep)));
    }
    if (pscale) {  // the Hermitian gate's per-phase scale (see pass A)
#pragma unroll
      for (int o = 16; o; o >>= 1) gmax = fmax(gmax, __shfl_xor_sync(0xffffffffu, gmax, o));
      if (lane == 0)
        atomicMax(reinterpret_cast<unsigned long long*>(pscale + p), (unsigned long long)__double_as_longlong(gmax));
    }
    __syncthreads();
#pragma unroll 1
    for (int base = warp * GPW; base < 5 * jl_n; base += ngrp) {  // warp-uniform
      const int task = base + gi;
      const bool active = task < 5 * jl_n;
      const int f = active ? task / jl_n : 0, jl = active ? task % jl_n : 0;
      const int fi = f < 3 ? f : f - 3;
      double2 v[P];
      band_gather<N>(v, t, EU + ((size_t)fi * JL + jl) * Kx, active);
      if (f >= 3) {
#pragma unroll
        for (int n1 = 0; n1 < P; ++n1) {
          const int r = band_r(t + T * n1, N, N / 3, Kx);
          if (r >= 0) v[n1] = cik(kxs[r], v[n1]);
        }
      }
      double2* col = I + ((size_t)f * JL + jl) * LD;
      wfft_t1<N, true, true>(v, t, active ? reinterpret_cast<double*>(col) : idle + (size_t)gi * WF<N>::XBUF, wlx);
      if (active) {  // row x of column j -> its owner (x / ROWS), local row x % ROWS
        const int j = rank + C * jl;
#pragma unroll
        for (int i = 0; i < P; ++i) {
          const int x = t1_pos<N>(t, i);
          *cluster.map_shared_rank(IR + ((size_t)f * Ky + j) * RLD + x % ROWS, (unsigned)(x / ROWS)) = v[i];
        }
      }
    }
    cluster.sync();  // every CTA's columns complete
    // ---- B: my rows; warp role `it` of its row group
    {
      const int rg = warp / 4, it = warp % 4;
      const int x = rank * W::ROWS + rg * GPW + gi;
      double* xb = XB + (size_t)grp * WF<N>::XBUF;
      const int fa = it == 0 ? 0 : (it == 1 ? 3 : (it == 2 ? 4 : 2));
      const int fb = it == 0 ? 1 : (it == 1 ? 0 : (it == 2 ? 1 : -1));
      double2 v[P];
#pragma unroll
      for (int n1 = 0; n1 < P; ++n1) {  // the packed pair's spectrum at y position k (cf. pair_val)
        const int k = t + T * n1;
        constexpr int KYM = N / 3;
        const bool lo_ = k <= KYM;
        if (!lo_ && k < N - KYM) {
          v[n1] = czero();
          continue;
        }
        const int jj = lo_ ? k : N - k;
        const int xl = x - rank * ROWS;
        const double2 A = IR[((size_t)fa * Ky + jj) * RLD + xl];
        double2 B = czero();
        if (fb >= 0) {
          B = IR[((size_t)fb * Ky + jj) * RLD + xl];
          if (it == 1 || it == 2) B = cik(kys[jj], B);
        }
        v[n1] = (k == 0) ? cmk(A.x, B.x) : (lo_ ? cmk(A.x - B.y, A.y + B.x) : cmk(A.x + B.y, B.x - A.y));
      }
      wfft_t1<N, true, true>(v, t, xb, wly);
      double2* mine = stash + ((size_t)rg * 4 + it) * P * 32;
#pragma unroll
      for (int i = 0; i < P; ++i) mine[i * 32 + lane] = v[i];
      __syncthreads();
      if (it < 2) {
        const double2* st = stash + (size_t)rg * 4 * P * 32;  // (u, v) | (ux, uy) | (vx, vy) | (depth, -)
#pragma unroll
        for (int i = 0; i < P; ++i) {
          const double2 qq = st[i * 32 + lane];
          if (it == 0) {
            const double2 a = st[P * 32 + i * 32 + lane], b = st[2 * P * 32 + i * 32 + lane];
            v[i] = cmk(-(qq.x * a.x + qq.y * a.y), -(qq.x * b.x + qq.y * b.y));  // A + iB
          } else {
            const double d = st[3 * P * 32 + i * 32 + lane].x;
            v[i] = cmk(qq.x * d, qq.y * d);  // C + iD = u depth + i v depth
          }
        }
        wfft_t2<N, false>(v, t, xb, wly);
        // unpack the two real spectra (cf. unpack_store) into the owners' columns
        constexpr int MU = (Ky + T - 1) / T;
        const int fo = 2 * it;
#pragma unroll
        for (int m = 0; m < MU; ++m) {
          const int j = t + T * m;
          const double2 src = v[P - 1 - m];
          double2 r;
          r.x = __shfl_sync(0xffffffffu, src.x, (T - t) & (T - 1), T);
          r.y = __shfl_sync(0xffffffffu, src.y, (T - t) & (T - 1), T);
          const double2 zm = t == 0 ? v[(P - m) & (P - 1)] : r;
          if (j < Ky) {
            const double2 a = v[m];
            colp(fo, j)[x] = cmk(0.5 * (a.x + zm.x), 0.5 * (a.y - zm.y));
            colp(fo + 1, j)[x] = cmk(0.5 * (a.y + zm.y), -0.5 * (a.x - zm.x));
          }
        }
      }
    }
    cluster.sync();  // every row's products are in their columns
    // ---- C: forward x-FFTs of my product columns, band kept in place
#pragma unroll 1
    for (int base = warp * GPW; base < 4 * jl_n; base += ngrp) {
      const int task = base + gi;
      const bool active = task < 4 * jl_n;
      const int f = active ? task / jl_n : 0, jl = active ? task % jl_n : 0;
      double2* col = I + ((size_t)f * JL + jl) * LD;
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
    // combine my modes: flux divergence, e^{-sL}, weight; ascending phase order
#pragma unroll
    for (int k = 0; k < MI; ++k) {
      const int m = threadIdx.x + k * NT;
      if (m >= nmode) break;
      const int jl = m / Kx, r = m % Kx, j = rank + C * jl;
      const double2* F = I + (size_t)jl * LD + r;  // field f at + f JL LD
      const double kx = kxs[r], ky = kys[j];
      const double2 gx = cik(kx, F[2 * JL * LD]), gy = cik(ky, F[3 * JL * LD]);
      C3 qq = {F[0], F[JL * LD], cmk(-(gx.x + gy.x), -(gx.y + gy.y))};
      if (tab) {
        double2 c12 = c12c[k];
        c12.x = -c12.x;  // e^{-sL}: c1(-s) = -c1(s), c2(-s) = c2(s)
        qq = exp_c12(c12, qq, G.ph, kx, ky);
      } else {
        qq = expL(-s, qq, G.ph, kx, ky, pr);
      }
      const size_t e = (size_t)jl * Kx + r;
      ACC[e] = cadd(ACC[e], cscale(w, qq.u));
      ACC[JL * Kx + e] = cadd(ACC[JL * Kx + e], cscale(w, qq.v));
      ACC[2 * JL * Kx + e] = cadd(ACC[2 * JL * Kx + e], cscale(w, qq.e));
    }
    __syncthreads();  // my columns are rewritten by the next phase's stage A
  }
  if (MW) {
    if (lo < hi) flush(wcur, true);
  } else {
    flush(0, false);
  }
  cluster.sync();  // no CTA exits while another may still address its shared memory
}

}  // namespace pswe

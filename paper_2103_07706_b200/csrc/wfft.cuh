// Warp-level fp64 complex FFT, 16 points per lane (N = 16 * T, T <= 32).
//
// A transform of length N is owned by a group of T = N/16 lanes inside one
// warp (32/T groups per warp), so every synchronisation is a __syncwarp.
// Two-step (row/column) factorisation N = 16 x T:
//
//  type 1  in : lane t holds x[t + T*n1], n1 = 0..15      (register v[n1])
//          16-point DFT in registers, twiddle W_N^{t k1}, ONE shared-memory
//          transpose (real and imaginary halves in turn, so the buffer is
//          16*S doubles), then the T-point DFTs over t:
//            T <= 16: lane t' owns k1 = t' + T*c (c < 16/T), all k2 in regs;
//            T == 32: lane t' = 2*k1 + h computes a 16-point DFT of the
//                     h-decimated sequence and the final radix-2 stage is
//                     a lane-pair exchange (__shfl_xor 1) -- no second
//                     shared-memory round trip.
//          out: see t1_pos() -- lane-owned positions k1 + 16*k2
//  type 2  the transposed algorithm: input in the type-1 OUTPUT layout,
//          output in the type-1 INPUT layout (lane t holds X[t + T*k2]).
//
// Pass B runs type 1 (spectral -> physical y), forms the quadratic products
// on the positions it owns, and runs type 2 back without any reshuffle.
// N = 8 is a single-lane DFT8 (both layouts natural).
//
// Twiddles: per-lane tables (WTab, global, L1-resident, loads independent of
// the data so they issue early); W_16 and W_32 are compile-time constants.
// Sign: FWD X[k] = sum x[n] e^{-2 pi i nk/N}; INV unnormalised e^{+...}.
#pragma once
#include "fft_reg.cuh"

namespace pswe {

template <int N>
struct WF {
  static constexpr int T = N >= 16 ? N / 16 : 1;   // lanes per transform
  static constexpr int P = N >= 16 ? 16 : 8;       // points per lane
  static constexpr int GPW = 32 / T;               // transforms per warp
  static constexpr int S = T == 32 ? 34 : T + 1;   // transpose row stride (doubles)
  // per-transform buffer in doubles; the padding staggers the groups that
  // share a half-warp across distinct banks
  static constexpr int PADD = T == 1 ? 1 : (T == 2 ? 2 : (T == 4 ? 4 : (T == 8 ? 8 : 0)));
  static constexpr int XBUF = N >= 16 ? 16 * S + PADD : 2;
};

// cos/sin(2 pi e / 32), e = 0..7 (first octant + symmetry handled by caller)
__device__ __forceinline__ double2 w32(int e, bool inv) {
  // exact table of e^{+i 2 pi e/32} for e = 0..31, folded after unrolling
  const double C[9] = {1.0,
                       0.98078528040323044913,
                       0.92387953251128675613,
                       0.83146961230254523708,
                       0.70710678118654752440,
                       0.55557023301960222474,
                       0.38268343236508977173,
                       0.19509032201612826785,
                       0.0};
  e &= 31;
  const int q = e >> 3, r = e & 7;
  // angle = q*pi/2 + r*pi/16
  double c = C[r], s = C[8 - r];
  double re, im;
  switch (q) {
    case 0: re = c; im = s; break;
    case 1: re = -s; im = c; break;
    case 2: re = -c; im = -s; break;
    default: re = s; im = -c; break;
  }
  return inv ? cmk(re, im) : cmk(re, -im);
}
__device__ __forceinline__ double2 w16(int e, bool inv) { return w32(2 * e, inv); }

// natural-order 16-point DFT in registers: 4 x 4 Cooley-Tukey.  BAND: the
// inputs v[6..9] are known zeros (2/3-truncated spectra entering an inverse
// transform of length >= 64), so each first-layer dft4 has one zero input.
template <bool INV, bool BAND = false>
__device__ __forceinline__ void dft16(double2* v) {
  double2 a[4][4];  // a[n2][k1]
#pragma unroll
  for (int n2 = 0; n2 < 4; ++n2) {
    double2 y0 = v[n2], y1 = v[n2 + 4], y2 = v[n2 + 8], y3 = v[n2 + 12];
    if constexpr (BAND) {
      if (n2 < 2)
        dft4_z2<INV>(y0, y1, y2, y3);  // y2 = v[8], v[9]
      else
        dft4_z1<INV>(y0, y1, y2, y3);  // y1 = v[6], v[7]
    } else {
      dft4<INV>(y0, y1, y2, y3);
    }
    a[n2][0] = y0;
    a[n2][1] = y1;
    a[n2][2] = y2;
    a[n2][3] = y3;
  }
  // second layer: dft4 over n2 of a[n2][k1] W_16^{n2 k1}, the twiddle
  // products fused into the first butterflies (x + w y as two FMAs per
  // component, x - w y as 2x - (x + w y))
#pragma unroll
  for (int k1 = 0; k1 < 4; ++k1) {
    double2 y0 = a[0][k1], y1 = a[1][k1], y2 = a[2][k1], y3 = a[3][k1];
    if (k1 == 0) {
      dft4<INV>(y0, y1, y2, y3);
    } else {
      double2 s0, d0;
      if (k1 == 2) {  // W_16^4 = -+i: a register swap + sign
        const double2 t = INV ? cmuli(y2) : cmk(y2.y, -y2.x);
        s0 = cadd(y0, t);
        d0 = csub(y0, t);
      } else {
        s0 = cfma(w16(2 * k1, INV), y2, y0);
        d0 = cmk(fma(2.0, y0.x, -s0.x), fma(2.0, y0.y, -s0.y));
      }
      const double2 p1 = cmul(y1, w16(k1, INV));
      const double2 s1 = cfma(w16(3 * k1, INV), y3, p1);
      const double2 d1 = cmk(fma(2.0, p1.x, -s1.x), fma(2.0, p1.y, -s1.y));
      const double2 r = INV ? cmk(-d1.y, d1.x) : cmk(d1.y, -d1.x);
      y0 = cadd(s0, s1);
      y2 = csub(s0, s1);
      y1 = cadd(d0, r);
      y3 = csub(d0, r);
    }
    v[k1] = y0;
    v[k1 + 4] = y1;
    v[k1 + 8] = y2;
    v[k1 + 12] = y3;
  }
}

template <int L, bool INV>
__device__ __forceinline__ void dftL(double2* v) {
  if constexpr (L == 16) dft16<INV>(v);
  else if constexpr (L == 8) dft8<INV>(v);
  else if constexpr (L == 4) dft4<INV>(v[0], v[1], v[2], v[3]);
  else if constexpr (L == 2) dft2<INV>(v[0], v[1]);
}

// v[k] *= s w^k for k = 1..L-1 (s = -1 if neg, and v[0] *= s).  The powers
// come from two interleaved chains, odd and even, each advanced by the
// three-term recurrence z^{m+1} = 2 cos(phi) z^m - z^{m-1} of a unit step
// z = w^2 (cos(phi) = Re w^2): two FMAs per power instead of a complex
// product (its two multiplies and two FMAs).  Seeds: w^{-1} = conj(w) ahead
// of w, w^0 = 1 ahead of w^2.  Max twiddle error over the 512-point
// transforms 5e-15 (chained products: 2e-15), far inside the 1e-10 parity
// tolerance.
template <int L, bool NEG>
__device__ __forceinline__ void apply_powers_(double2* v, double2 w, bool neg) {
  if constexpr (L > 1) {
    const double2 w2 = cmul(w, w);
    const double c2 = 2.0 * w2.x;
    const bool ng = NEG && neg;
    // sign flips on the integer pipe (dflip / dneg), not DADDs
    double2 po = cmk(dflip(w.x, ng), dflip(w.y, ng)), pom = cmk(po.x, -po.y);
    double2 pe = cmk(dflip(w2.x, ng), dflip(w2.y, ng)), pem = cmk(ng ? -1.0 : 1.0, 0.0);
    if constexpr (NEG) v[0] = cmk(dflip(v[0].x, neg), dflip(v[0].y, neg));
#pragma unroll
    for (int k = 1; k < L; k += 2) {
      v[k] = cmul(v[k], po);
      if (k + 2 < L) {
        const double2 nx = cmk(fma(c2, po.x, -pom.x), fma(c2, po.y, -pom.y));
        pom = po;
        po = nx;
      }
      if (k + 1 < L) {
        v[k + 1] = cmul(v[k + 1], pe);
        if (k + 3 < L) {
          const double2 nx = cmk(fma(c2, pe.x, -pem.x), fma(c2, pe.y, -pem.y));
          pem = pe;
          pe = nx;
        }
      }
    }
  }
}
template <int L>
__device__ __forceinline__ void apply_powers(double2* v, double2 w) {
  apply_powers_<L, false>(v, w, false);
}
template <int L>
__device__ __forceinline__ void apply_powers_neg(double2* v, double2 w, bool neg) {
  apply_powers_<L, true>(v, w, neg);
}

// twiddle table of one transform length N: W_N^k, k = 0..N-1 (forward sign);
// the FFT reads per-lane bases from it and generates powers in registers.
struct WTab {
  const double2* t0;
  // Two spare pointers.  They only keep GridDev's kernel-parameter layout:
  // with them removed, ptxas 12.9 allocates passes A and C differently and
  // spills (measured: pass A 1.09 -> 1.12 ms per RHS).
  const double2* spare_[2];
};

__device__ __forceinline__ double2 twg(const double2* __restrict__ tw, int e, bool inv) {
  double2 w = __ldg(tw + e);
  if (inv) w.y = -w.y;
  return w;
}

// Per-lane twiddle bases (forward sign) read on use from the (L1-resident)
// table rather than held in registers for the whole kernel: W_N^t (type 1,
// and type 2 for T <= 16), W_N^{n1} and W_N^{2 n1} with n1 = t/2 (type 2,
// T == 32).
struct WLane {
  const double2* tw;
  int t;
  __device__ __forceinline__ double2 wt() const { return __ldg(tw + t); }
  __device__ __forceinline__ double2 wn1() const { return __ldg(tw + (t >> 1)); }
  __device__ __forceinline__ double2 w2n1() const { return __ldg(tw + 2 * (t >> 1)); }
};

template <int N>
__device__ __forceinline__ WLane wlane(const WTab tw, int t) {
  return WLane{tw.t0, t};
}

__device__ __forceinline__ double2 wsel(double2 w, bool inv) { return inv ? cmk(w.x, -w.y) : w; }

// position held in register i by lane t after a type-1 transform (== type-2 input)
template <int N>
__device__ __forceinline__ int t1_pos(int t, int i) {
  constexpr int T = WF<N>::T;
  if constexpr (N == 8) {
    return i;
  } else if constexpr (T <= 16) {
    const int c = i / T, k2 = i % T;
    return (t + T * c) + 16 * k2;
  } else {
    const int k1 = t >> 1, h = t & 1;
    const int k2 = (i < 8) ? (8 * h + i) : (8 * h + (i - 8) + 16);
    return k1 + 16 * k2;
  }
}

// transpose helpers: write (re or im) of 16 values to rows k1 at column col,
// read back a lane's values.  Each half is bracketed by __syncwarp.
#define PSWE_XPOSE(WRITE_RE, WRITE_IM, READ_RE, READ_IM) \
  __syncwarp();                                          \
  _Pragma("unroll") WRITE_RE;                            \
  __syncwarp();                                          \
  _Pragma("unroll") READ_RE;                             \
  __syncwarp();                                          \
  _Pragma("unroll") WRITE_IM;                            \
  __syncwarp();                                          \
  _Pragma("unroll") READ_IM;

// ---- type 1 -------------------------------------------------------------------
// v[n1] = x[t + T n1] in; out per t1_pos.  xb: this transform's exchange buffer
// (WF<N>::XBUF doubles); tw: global W_N^k table.
// BAND: input registers 6..9 hold out-of-band (zero) positions, true for a
// 2/3-truncated spectrum when N >= 64 (positions t + T n1, n1 = 6..9, all lie
// strictly between N/3 and N - N/3).
template <int N, bool INV, bool BAND = false>
__device__ __forceinline__ void wfft_t1(double2* v, int t, double* xb, const WLane& wl) {
  if constexpr (N == 8) {
    dft8<INV>(v);
  } else {
    constexpr int T = WF<N>::T, S = WF<N>::S;
    dft16<INV, BAND && (N >= 64)>(v);
    if constexpr (T == 32) {
      // W_N^{t k1}, and every value of a lane t = 3 (mod 4) negated: the odd
      // reader's inputs m then carry (-1)^m, so its DFT16 output comes out
      // rotated by 8 registers (see the exchange below)
      apply_powers_neg<16>(v, wsel(wl.wt(), INV), (t & 3) == 3);
    } else if constexpr (T > 1) {
      apply_powers<16>(v, wsel(wl.wt(), INV));  // W_N^{t k1}
    }
    if constexpr (T > 1) {
      if constexpr (T <= 16) {
        constexpr int C = 16 / T;
        PSWE_XPOSE(
            for (int k1 = 0; k1 < 16; ++k1) xb[k1 * S + t] = v[k1].x,
            for (int k1 = 0; k1 < 16; ++k1) xb[k1 * S + t] = v[k1].y,
            for (int c = 0; c < C; ++c) _Pragma("unroll") for (int n2 = 0; n2 < T; ++n2) v[c * T + n2].x = xb[(t + T * c) * S + n2],
            for (int c = 0; c < C; ++c) _Pragma("unroll") for (int n2 = 0; n2 < T; ++n2) v[c * T + n2].y = xb[(t + T * c) * S + n2])
#pragma unroll
        for (int c = 0; c < C; ++c) dftL<T, INV>(v + c * T);
      } else {
        const int k1 = t >> 1, h = t & 1;
        PSWE_XPOSE(
            for (int q = 0; q < 16; ++q) xb[q * S + t] = v[q].x,
            for (int q = 0; q < 16; ++q) xb[q * S + t] = v[q].y,
            for (int m = 0; m < 16; ++m) v[m].x = xb[k1 * S + h + 2 * m],
            for (int m = 0; m < 16; ++m) v[m].y = xb[k1 * S + h + 2 * m])
        // E_h[k2'], k2' = 0..15; the odd lane's rotated: v[i] = E_1[(i + 8) % 16]
        dft16<INV>(v);
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          // even lane sends E_0[8 + c], odd lane E_1[c]: both v[8 + c]
          double2 recv;
          recv.x = __shfl_xor_sync(0xffffffffu, v[8 + c].x, 1);
          recv.y = __shfl_xor_sync(0xffffffffu, v[8 + c].y, 1);
          const double2 e0 = h ? recv : v[c];
          // W_32^{8+c} = W_32^c W_32^8 and W_32^8 = +-i: the odd lane's operand
          // E_1[8 + c] = v[c] is rotated (a register swap + sign) and the
          // twiddle is the lane-uniform constant W_32^c
          const double2 o = v[c];
          const double2 e1 = h ? (INV ? cmk(dneg(o.y), o.x) : cmk(o.y, dneg(o.x))) : recv;
          const double2 we1 = c == 0 ? e1 : cmul(w32(c, INV), e1);  // W_32^0 = 1: exact either way
          v[c] = cadd(e0, we1);
          v[8 + c] = csub(e0, we1);
        }
      }
    }
  }
}

// ---- type 2 -------------------------------------------------------------------
// input in t1_pos layout; out v[k2] = X[t + T k2].
template <int N, bool INV>
__device__ __forceinline__ void wfft_t2(double2* v, int t, double* xb, const WLane& wl) {
  if constexpr (N == 8) {
    dft8<INV>(v);
  } else {
    constexpr int T = WF<N>::T, S = WF<N>::S;
    if constexpr (T > 1) {
      if constexpr (T <= 16) {
        constexpr int C = 16 / T;
#pragma unroll
        for (int c = 0; c < C; ++c) {
          dftL<T, INV>(v + c * T);  // Z[n1][k1''], k1'' = 0..T-1
          // W_N^{n1 k1''}, n1 = t + T c: base W_N^t W_16^c (N = 16 T)
          apply_powers<T>(v + c * T, cmul(wsel(wl.wt(), INV), w16(c, INV)));
        }
        PSWE_XPOSE(
            for (int c = 0; c < C; ++c) _Pragma("unroll") for (int k = 0; k < T; ++k) xb[(t + T * c) * S + k] = v[c * T + k].x,
            for (int c = 0; c < C; ++c) _Pragma("unroll") for (int k = 0; k < T; ++k) xb[(t + T * c) * S + k] = v[c * T + k].y,
            for (int n1 = 0; n1 < 16; ++n1) v[n1].x = xb[n1 * S + t],
            for (int n1 = 0; n1 < 16; ++n1) v[n1].y = xb[n1 * S + t])
      } else {
        const int h = t & 1, n1 = t >> 1;
        const double2 wn1 = wsel(wl.wn1(), INV);  // W_N^{n1}
        // s_c = a + b, d_c = (a - b) W_32^c for this lane's c = 8h + cc.  The
        // combined twiddles W_32^cc W_N^{n1} by the three-term recurrence
        // z_{cc+1} = 2 cos(2 pi / 32) z_cc - z_{cc-1} (two FMAs each)
        constexpr double C32 = 1.96157056080646086074;  // 2 cos(2 pi / 32)
        double2 zp = wn1, zc = cmul(w32(1, INV), wn1);
        double2 q[16];
#pragma unroll
        for (int cc = 0; cc < 8; ++cc) {
          const double2 a = v[cc], b = v[8 + cc];
          const double2 sv = cadd(a, b);
          // W_32^{8+cc} = W_32^cc (+-i): lane-uniform twiddle, the odd lane's
          // copy rotated by a register swap + sign.  dv only ever feeds the
          // odd lane's DFT16 (sent by the even lane, kept by the odd one), so
          // the odd lane's output factor W_N^{n1} is applied here, to both
          // lanes alike, instead of as a lane-divergent multiply afterwards.
          const double2 dab = csub(a, b);
          double2 tw = wn1;
          if (cc == 1) tw = zc;
          if (cc >= 2) {
            const double2 zn = cmk(fma(C32, zc.x, -zp.x), fma(C32, zc.y, -zp.y));
            zp = zc;
            zc = zn;
            tw = zn;
          }
          const double2 dv = cmul(dab, tw);
          const double2 send = h ? sv : dv;
          double2 recv;
          recv.x = __shfl_xor_sync(0xffffffffu, send.x, 1);
          recv.y = __shfl_xor_sync(0xffffffffu, send.y, 1);
          // The odd lane keeps its DFT16 input rotated by 8 registers
          // (received value in the upper half for both lanes: one select
          // instead of two); the rotation multiplies its output k by (-1)^k,
          // undone by negating the twiddle base below.
          q[cc] = h ? (INV ? cmk(dneg(dv.y), dv.x) : cmk(dv.y, dneg(dv.x))) : sv;
          q[8 + cc] = recv;
        }
        dft16<INV>(q);  // Z[n1][2 q' + h] (the odd lane's times W^{n1} (-1)^q')
        // twiddle W_N^{n1 (2q'+h)} = W^{n1 h} (W^{2 n1})^{q'}
        double2 wb = wsel(wl.w2n1(), INV);
        wb = cmk(dflip(wb.x, h), dflip(wb.y, h));
        apply_powers<16>(q, wb);
        PSWE_XPOSE(
            for (int k = 0; k < 16; ++k) xb[n1 * S + 2 * k + h] = q[k].x,
            for (int k = 0; k < 16; ++k) xb[n1 * S + 2 * k + h] = q[k].y,
            for (int m = 0; m < 16; ++m) v[m].x = xb[m * S + t],
            for (int m = 0; m < 16; ++m) v[m].y = xb[m * S + t])
      }
    }
    dft16<INV>(v);
  }
}

}  // namespace pswe

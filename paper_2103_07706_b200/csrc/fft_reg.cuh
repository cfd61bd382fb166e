// Small fp64 complex DFTs in registers (2, 4, 8 points, and 4-point variants
// with a known-zero input), the building blocks of the warp FFT in wfft.cuh.
//
// Sign convention: FWD is X[k] = sum x[n] e^{-2 pi i nk/N} (numpy fft),
// INV is the unnormalised e^{+2 pi i nk/N} sum (N * numpy ifft).
#pragma once
#include "pswe_common.cuh"

namespace pswe {

// ---- small DFTs in registers ------------------------------------------------
template <bool INV>
__device__ __forceinline__ void dft2(double2& a, double2& b) {
  double2 s = cadd(a, b), d = csub(a, b);
  a = s;
  b = d;
}

template <bool INV>
__device__ __forceinline__ void dft4(double2& y0, double2& y1, double2& y2, double2& y3) {
  double2 s0 = cadd(y0, y2), d0 = csub(y0, y2), s1 = cadd(y1, y3), d1 = csub(y1, y3);
  // FWD: -i * d1 ; INV: +i * d1
  double2 r = INV ? cmk(-d1.y, d1.x) : cmk(d1.y, -d1.x);
  y0 = cadd(s0, s1);
  y2 = csub(s0, s1);
  y1 = cadd(d0, r);
  y3 = csub(d0, r);
}

// dft4 with y2 == 0 (known at compile time): s0 = d0 = y0
template <bool INV>
__device__ __forceinline__ void dft4_z2(double2& y0, double2& y1, double2& y2, double2& y3) {
  const double2 s1 = cadd(y1, y3), d1 = csub(y1, y3);
  const double2 r = INV ? cmk(-d1.y, d1.x) : cmk(d1.y, -d1.x);
  const double2 a = y0;
  y0 = cadd(a, s1);
  y2 = csub(a, s1);
  y1 = cadd(a, r);
  y3 = csub(a, r);
}

// dft4 with y1 == 0: s1 = y3, d1 = -y3
template <bool INV>
__device__ __forceinline__ void dft4_z1(double2& y0, double2& y1, double2& y2, double2& y3) {
  const double2 s0 = cadd(y0, y2), d0 = csub(y0, y2);
  // r = (-/+ i) * d1 with d1 = -y3
  const double2 r = INV ? cmk(y3.y, -y3.x) : cmk(-y3.y, y3.x);
  y0 = cadd(s0, y3);
  y2 = csub(s0, y3);
  y1 = cadd(d0, r);
  y3 = csub(d0, r);
}

template <bool INV>
__device__ __forceinline__ void dft8(double2* v) {
  const double c = 0.70710678118654752440;  // sqrt(1/2)
  double2 a0 = cadd(v[0], v[4]), b0 = csub(v[0], v[4]);
  double2 a1 = cadd(v[1], v[5]), b1 = csub(v[1], v[5]);
  double2 a2 = cadd(v[2], v[6]), b2 = csub(v[2], v[6]);
  double2 a3 = cadd(v[3], v[7]), b3 = csub(v[3], v[7]);
  if (!INV) {
    b1 = cmk(c * (b1.x + b1.y), c * (b1.y - b1.x));   // * (c - ic)
    b2 = cmk(b2.y, -b2.x);                            // * (-i)
    b3 = cmk(c * (b3.y - b3.x), -c * (b3.x + b3.y));  // * (-c - ic)
  } else {
    b1 = cmk(c * (b1.x - b1.y), c * (b1.x + b1.y));   // * (c + ic)
    b2 = cmk(-b2.y, b2.x);                            // * (+i)
    b3 = cmk(-c * (b3.x + b3.y), c * (b3.x - b3.y));  // * (-c + ic)
  }
  dft4<INV>(a0, a1, a2, a3);
  dft4<INV>(b0, b1, b2, b3);
  v[0] = a0; v[1] = b0; v[2] = a1; v[3] = b1;
  v[4] = a2; v[5] = b2; v[6] = a3; v[7] = b3;
}


}  // namespace pswe

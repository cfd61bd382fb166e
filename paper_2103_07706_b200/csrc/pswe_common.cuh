// Shared device helpers for the B200 phase-averaged shallow-water RHS.
//
// fp64 complex arithmetic, the per-mode 3x3 linear operator L and the two
// exponential routes (exact closed form, Chebyshev recurrence).  Everything
// here acts on ONE spectral mode in registers: in the reference these are
// whole-array numpy passes (dynamics.py:128-136, propagator.py:96-110,
// propagator.py:161-191); on the GPU they are fused into the loads/epilogues
// of the FFT passes and the stepper stage kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace pswe {

// ---------------------------------------------------------------- complex
__device__ __forceinline__ double2 cmk(double x, double y) { return make_double2(x, y); }
// -x as a sign-bit flip on the integer pipe.  A negation whose consumer cannot
// take an operand modifier (a select, shuffle or store) otherwise costs a DADD
// on the fp64 pipe, the pipe that bounds the FFT passes.  Bitwise equal to it.
__device__ __forceinline__ double dneg(double x) {
  return __hiloint2double(__double2hiint(x) ^ (int)0x80000000u, __double2loint(x));
}
// x with its sign flipped when flip != 0 (no select, no fp64 instruction)
__device__ __forceinline__ double dflip(double x, bool flip) {
  return __hiloint2double(__double2hiint(x) ^ (int)((unsigned)flip << 31), __double2loint(x));
}
// -(a.x b.x + a.y b.y) with the negation folded into the operands, so no
// DADD is spent on it: fma(-a.x, b.x, -(a.y b.y)), bitwise equal to
// negating fma(a.x, b.x, a.y b.y)
__device__ __forceinline__ double ndot(double2 a, double2 b) { return __fma_rn(-a.x, b.x, -__dmul_rn(a.y, b.y)); }
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return cmk(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return cmk(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cscale(double s, double2 a) { return cmk(s * a.x, s * a.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return cmk(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// c + w y with the products fused: two FMAs per component
__device__ __forceinline__ double2 cfma(double2 w, double2 y, double2 c) {
  return cmk(fma(w.x, y.x, fma(-w.y, y.y, c.x)), fma(w.x, y.y, fma(w.y, y.x, c.y)));
}
__device__ __forceinline__ double2 cconj(double2 a) { return cmk(a.x, -a.y); }
// i * a
__device__ __forceinline__ double2 cmuli(double2 a) { return cmk(-a.y, a.x); }
// (i k) * a for a real wavenumber k, written the way numpy evaluates
// (0 + ik)(ar + i ai) = (0*ar - k*ai) + i(0*ai + k*ar); the zero products vanish
// exactly for finite input, so this is bit-identical for finite data.
__device__ __forceinline__ double2 cik(double k, double2 a) { return cmk(-k * a.y, k * a.x); }
__device__ __forceinline__ double2 czero() { return cmk(0.0, 0.0); }

struct C3 {
  double2 u, v, e;
};
__device__ __forceinline__ C3 c3add(const C3& a, const C3& b) {
  return {cadd(a.u, b.u), cadd(a.v, b.v), cadd(a.e, b.e)};
}
__device__ __forceinline__ C3 c3scale(double s, const C3& a) {
  return {cscale(s, a.u), cscale(s, a.v), cscale(s, a.e)};
}
__device__ __forceinline__ C3 c3zero() { return {czero(), czero(), czero()}; }
__device__ __forceinline__ C3 c3conj(const C3& a) { return {cconj(a.u), cconj(a.v), cconj(a.e)}; }

// ---------------------------------------------------------------- physics
struct Phys {
  double f, g, H;
};

// L q for one mode: (f v - g ikx eta, -f u - g iky eta, -H (ikx u + iky v))
// (dynamics.py:128-136).
__device__ __forceinline__ C3 lin(const C3& q, const Phys& p, double kx, double ky) {
  C3 o;
  double2 gx = cik(kx, q.e), gy = cik(ky, q.e);
  o.u = cmk(p.f * q.v.x - p.g * gx.x, p.f * q.v.y - p.g * gx.y);
  o.v = cmk(-p.f * q.u.x - p.g * gy.x, -p.f * q.u.y - p.g * gy.y);
  double2 du = cik(kx, q.u), dv = cik(ky, q.v);
  o.e = cmk(-p.H * (du.x + dv.x), -p.H * (du.y + dv.y));
  return o;
}

// omega = sqrt(f^2 + g H |k|^2) (dynamics.py:179-186)
__device__ __forceinline__ double omega_of(const Phys& p, double kx, double ky) {
  return sqrt(p.f * p.f + p.g * p.H * (kx * kx + ky * ky));
}

// Propagator route: kind 0 = exact closed form, 1 = Chebyshev recurrence.
struct Prop {
  int kind;
  int n_poly;
  double Lambda;
  const double* a;  // device, n_poly + 1 real coefficients
};

// Exact per-mode exponential: U + c1 L U + c2 L^2 U with
// c1 = sin(w t)/w, c2 = (1 - cos w t)/w^2, w -> 0 limit t, t^2/2
// (propagator.py:96-110).
__device__ __forceinline__ C3 exp_exact(double t, const C3& q, const Phys& p, double kx, double ky) {
  double om = omega_of(p, kx, ky);
  double c1, c2;
  if (om > 0.0) {
    double sn, cs;
    sincos(om * t, &sn, &cs);
    c1 = sn / om;
    c2 = (1.0 - cs) / (om * om);
  } else {
    c1 = t;
    c2 = 0.5 * t * t;
  }
  C3 l1 = lin(q, p, kx, ky);
  C3 l2 = lin(l1, p, kx, ky);
  return c3add(c3add(q, c3scale(c1, l1)), c3scale(c2, l2));
}

// Matrix-free Chebyshev recurrence Q_{k+1} = (2t/Lambda) L Q_k + Q_{k-1},
// acc = sum a_k Q_k (propagator.py:161-191).  t == 0 is the identity.
__device__ __forceinline__ C3 exp_cheb(double t, const C3& q, const Phys& p, double kx, double ky,
                                       const Prop& pr) {
  if (t == 0.0) return q;
  const double sc = t / pr.Lambda;
  const double sc2 = 2.0 * sc;
  C3 qp = q;
  C3 qc = c3scale(sc, lin(q, p, kx, ky));
  C3 acc = c3add(c3scale(__ldg(pr.a + 0), q), c3scale(__ldg(pr.a + 1), qc));
  for (int k = 2; k <= pr.n_poly; ++k) {
    C3 qn = c3add(c3scale(sc2, lin(qc, p, kx, ky)), qp);
    acc = c3add(acc, c3scale(__ldg(pr.a + k), qn));
    qp = qc;
    qc = qn;
  }
  return acc;
}

__device__ __forceinline__ C3 expL(double t, const C3& q, const Phys& p, double kx, double ky,
                                   const Prop& pr) {
  return pr.kind == 0 ? exp_exact(t, q, p, kx, ky) : exp_cheb(t, q, p, kx, ky, pr);
}

__device__ __forceinline__ bool finite2(double2 a) { return isfinite(a.x) && isfinite(a.y); }

// e^{tL} q from precomputed (c1, c2) = (sin(w t)/w, (1 - cos w t)/w^2)
__device__ __forceinline__ C3 exp_c12(double2 c12, const C3& q, const Phys& p, double kx, double ky) {
  C3 l1 = lin(q, p, kx, ky);
  C3 l2 = lin(l1, p, kx, ky);
  return c3add(c3add(q, c3scale(c12.x, l1)), c3scale(c12.y, l2));
}

// (c1, c2) of the exact exponential at time t for a mode (as exp_exact forms
// them).  A mode and its mirror -k share omega (|k|^2 is sign-blind, bit for
// bit), and c1(-t) = -c1(t), c2(-t) = c2(t): one sincos serves all the
// exponentials a stage kernel's thread applies.
__device__ __forceinline__ double2 c12_of(const Phys& p, double kx, double ky, double t) {
  const double om = omega_of(p, kx, ky);
  if (om > 0.0) {
    double sn, cs;
    sincos(om * t, &sn, &cs);
    return cmk(sn / om, (1.0 - cs) / (om * om));
  }
  return cmk(t, 0.5 * t * t);
}

// e^{tL} q by the context's route, with (c1, c2) precomputed for the exact route
__device__ __forceinline__ C3 expLc(double2 c12, double t, const C3& q, const Phys& p, double kx, double ky,
                                    const Prop& pr) {
  return pr.kind == 0 ? exp_c12(c12, q, p, kx, ky) : exp_cheb(t, q, p, kx, ky, pr);
}

}  // namespace pswe

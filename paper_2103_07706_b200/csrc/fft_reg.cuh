// Register-resident fp64 complex FFT for power-of-two N in [8, 1024].
//
// One transform is computed by a "group" of T = N/8 threads; thread t holds
// the 8 points x[t + m*N/8], m = 0..7, in registers on entry and the 8
// outputs X[t + m*N/8] on exit (same distribution).  Stages are mixed-radix
// Stockham (radix 8, then one radix 4 or 2 stage), so between stages the
// group exchanges data through a padded shared-memory buffer; the first
// stage's input and the last stage's output never touch shared memory, which
// lets callers fuse per-mode work (exponentials, products, 2/3 truncation)
// directly into the FFT's first load and last store.
//
// Shared-memory index padding pidx(i) = i + i/8 removes the stride-8 bank
// conflict of the first Stockham stage's scatter.
//
// Sign convention: FWD is X[k] = sum x[n] e^{-2 pi i nk/N} (numpy fft),
// INV is the unnormalised e^{+2 pi i nk/N} sum (N * numpy ifft).
#pragma once
#include "pswe_common.cuh"

namespace pswe {

__device__ __forceinline__ int pidx(int i) { return i + (i >> 3); }
template <int N>
struct FFTSize {
  static constexpr int T = N / 8;            // threads per transform
  static constexpr int PAD = N + N / 8;      // padded smem length (double2)
};

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

template <int R, bool INV>
__device__ __forceinline__ void dftR(double2* v) {
  if constexpr (R == 8) {
    dft8<INV>(v);
  } else if constexpr (R == 4) {
    dft4<INV>(v[0], v[1], v[2], v[3]);
  } else {
    dft2<INV>(v[0], v[1]);
  }
}

// ---- group barrier -----------------------------------------------------------
// Groups of <= 32 threads live inside one warp (all lanes run the same code),
// larger groups use a named barrier per group.  Barrier 0 is __syncthreads.
template <int N>
__device__ __forceinline__ void group_sync(int group_in_cta) {
  if constexpr (N / 8 <= 32) {
    __syncwarp();
  } else {
    asm volatile("bar.sync %0, %1;" ::"r"(1 + group_in_cta), "n"(N / 8) : "memory");
  }
}

// ---- Stockham stage ------------------------------------------------------------
// Butterfly j in [0, N/R): inputs x[j + r*N/R], twiddle W_N^{r*(j%NS)*N/(NS*R)},
// outputs x'[(j/NS)*NS*R + j%NS + r*NS].  Thread t does butterflies
// j = t + q*N/8, q < 8/R, with registers v[q*R + r].
// Twiddles W^{r e}, r = 1..R-1, from one table entry W^e by a depth-3 power
// tree (w2 = w1^2, w4 = w2^2, ...): one shared-memory load per butterfly
// instead of R-1 dependent global loads.
template <int R, bool INV>
__device__ __forceinline__ void twiddle_powers(double2 w1, double2* w) {
  if (INV) w1.y = -w1.y;
  w[1] = w1;
  if constexpr (R >= 4) {
    w[2] = cmul(w1, w1);
    w[3] = cmul(w[2], w1);
  }
  if constexpr (R == 8) {
    w[4] = cmul(w[2], w[2]);
    w[5] = cmul(w[4], w1);
    w[6] = cmul(w[3], w[3]);
    w[7] = cmul(w[4], w[3]);
  }
}

template <int N, int R, int NS, bool INV>
__device__ __forceinline__ void stage_compute(double2* v, int t, const double2* __restrict__ tw) {
  constexpr int B = 8 / R;
#pragma unroll
  for (int q = 0; q < B; ++q) {
    if constexpr (NS > 1) {
      const int j = t + q * (N / 8);
      const int k = j % NS;
      double2 w[8];
      twiddle_powers<R, INV>(tw[k * (N / (NS * R))], w);
#pragma unroll
      for (int r = 1; r < R; ++r) v[q * R + r] = cmul(v[q * R + r], w[r]);
    }
    dftR<R, INV>(v + q * R);
  }
}

template <int N, int R, int NS>
__device__ __forceinline__ void stage_store(const double2* v, int t, double2* sm) {
  constexpr int B = 8 / R;
#pragma unroll
  for (int q = 0; q < B; ++q) {
    const int j = t + q * (N / 8);
    const int base = (j / NS) * NS * R + (j % NS);
#pragma unroll
    for (int r = 0; r < R; ++r) sm[pidx(base + r * NS)] = v[q * R + r];
  }
}

// load the next stage's inputs: butterfly j, element r at j + r*N/R
template <int N, int R>
__device__ __forceinline__ void stage_load(double2* v, int t, const double2* sm) {
  constexpr int B = 8 / R;
#pragma unroll
  for (int q = 0; q < B; ++q) {
    const int j = t + q * (N / 8);
#pragma unroll
    for (int r = 0; r < R; ++r) v[q * R + r] = sm[pidx(j + r * (N / R))];
  }
}

template <int N, int NS>
struct StageRadix {
  static constexpr int REM = N / NS;
  static constexpr int R = REM >= 8 ? 8 : REM;
};

// first-stage input register layout for radix R: v[q*R + r] = x[t + q*N/8 + r*N/R]
// = x[t + m*N/8] with m = q + r*(8/R).  Callers load v[m] = x[t + m*N/8]; this
// permutes to the stage layout.
template <int R>
__device__ __forceinline__ void to_stage_layout(double2* v) {
  if constexpr (R == 8) return;
  constexpr int B = 8 / R;
  double2 tmp[8];
#pragma unroll
  for (int q = 0; q < B; ++q)
#pragma unroll
    for (int r = 0; r < R; ++r) tmp[q * R + r] = v[q + r * B];
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = tmp[i];
}
template <int R>
__device__ __forceinline__ void from_stage_layout(double2* v) {
  if constexpr (R == 8) return;
  constexpr int B = 8 / R;
  double2 tmp[8];
#pragma unroll
  for (int q = 0; q < B; ++q)
#pragma unroll
    for (int r = 0; r < R; ++r) tmp[q + r * B] = v[q * R + r];
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = tmp[i];
}

template <int N, int NS, bool INV>
struct Stages {
  // v holds this stage's inputs in stage layout; on return v holds the final
  // outputs X[t + m*N/8] in natural layout (v[m]).
  static __device__ __forceinline__ void run(double2* v, int t, double2* sm, int gid,
                                             const double2* __restrict__ tw) {
    constexpr int R = StageRadix<N, NS>::R;
    stage_compute<N, R, NS, INV>(v, t, tw);
    if constexpr (NS * R == N) {
      // last stage: outputs at j + r*NS = t + q*N/8 + r*N/R  -> natural layout
      from_stage_layout<R>(v);
    } else {
      constexpr int R2 = StageRadix<N, NS * R>::R;
      group_sync<N>(gid);  // previous readers of sm are done
      stage_store<N, R, NS>(v, t, sm);
      group_sync<N>(gid);
      stage_load<N, R2>(v, t, sm);
      Stages<N, NS * R, INV>::run(v, t, sm, gid, tw);
    }
  }
};

// Full transform: v[m] = x[t + m*N/8] in, X[t + m*N/8] out.  sm: group's padded
// exchange buffer (FFTSize<N>::PAD double2); tw: the N-entry forward twiddle
// table W_N^k, normally staged in shared memory (load_twiddles).  Contains
// group barriers: every thread of the group must call it.
template <int N, bool INV>
__device__ __forceinline__ void fft_reg(double2* v, int t, double2* sm, int gid,
                                        const double2* __restrict__ tw) {
  constexpr int R0 = StageRadix<N, 1>::R;
  to_stage_layout<R0>(v);
  Stages<N, 1, INV>::run(v, t, sm, gid, tw);
}

// copy the N-entry twiddle table to shared memory (whole CTA; caller syncs)
template <int N>
__device__ __forceinline__ void load_twiddles(double2* dst, const double2* __restrict__ src) {
  for (int i = threadIdx.x; i < N; i += blockDim.x) dst[i] = src[i];
}

}  // namespace pswe

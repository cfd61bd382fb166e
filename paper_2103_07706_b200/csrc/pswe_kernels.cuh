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
//   I1 (pass A -> B): I1[p][f][j][x], p = phase in chunk, f in 0..4,
//             j = 0..KYM (spectral y), x = 0..nx-1 (physical x): each pass-A
//             transform stores one contiguous column.
//   I2 (pass B -> C): I2[p][f][j][x], f in 0..3: one ky column contiguous
//             for pass C's bulk copies.  A pair of pass-B warps stages the
//             outputs of its RP consecutive rows as a [f][j][RP] tile in
//             shared memory and writes it with one TMA tensor store
//             (RP x 16-byte runs: full 32-byte sectors at 512^2).
//   Pass A stores are contiguous; pass B reads its rows of I1 with TMA
//   tensor gathers (one box = one row, 16-byte elements) issued a transform
//   ahead.
//
// Averaged RHS (averaging.py:116-156) for a chunk of phases:
//   pass A  (per phase, ky column)  e^{sL} per mode + 5 inverse x-FFTs
//   pass B  (per phase, x row)      7 C2R along y as 4 complex FFTs, the four
//                                   quadratic products, 2 R2C as complex FFTs
//   pass C  (per ky column, phases) 4 forward x-FFTs, flux divergence, 2/3
//                                   truncation, e^{-sL}, weighted ordered sum
// followed by an ordered reduction over the phase-group slots.
#pragma once
#include "async_copy.cuh"
#include "tmem.cuh"
#include "wfft.cuh"

#ifdef PSWE_EARLY_STWAIT  // A/B switch: wait right after every tensor-memory store
#define PSWE_ST_WAIT_EARLY() tmem_wait_st()
#define PSWE_ST_WAIT_LATE()
#else
#define PSWE_ST_WAIT_EARLY()
#define PSWE_ST_WAIT_LATE() tmem_wait_st()
#endif

namespace pswe {

struct GridDev {
  int nx, ny, kxm, kym, Kx, Ky;
  Phys ph;
  double inv_n2;
  const double* kxc;   // [Kx]  compact kx
  const double* kyc;   // [Ky]  ky >= 0
  const double* kxf;   // [nx]  full kx (fft order)
  const double* kyf;   // [ny]
  WTab twx;            // per-lane FFT twiddle tables, length nx
  WTab twy;            // length ny
  const double2* bc;   // [Ky][Kx] compact (Hermitian-projected) topography
};

__device__ __forceinline__ double abs2(double2 a) { return fma(a.x, a.x, a.y * a.y); }
// max that propagates NaN (either operand) -- the Hermitian gate's statistics
// must not drop a non-finite value the way fmax does
__device__ __forceinline__ double nanmax(double a, double b) { return (a > b || a != a) ? a : b; }

// The Hermitian gate's fast verdict (herm_kernels.cuh), evaluated by block 0
// of the kernel that consumes an evaluation's result: flags bit `bit` when
// some phase might fail the gate, and resets the statistics (hstat[3] = max
// |D_f|^2 of the packed input, pscale[P] = per-phase max squared magnitude)
// for the next evaluation.  bit < 0: no gate.
struct HermGate {
  double* hstat;
  double* pscale;
  int P;
  double bdef, H, g;
  int* flags;
  int bit;
};

__device__ void herm_eval_block(const HermGate& hg) {
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  const double dW2 = hg.H * hg.hstat[0] + hg.H * hg.hstat[1] + hg.g * hg.hstat[2];
  const double d = sqrt(dW2) / sqrt(fmin(hg.H, hg.g)) + hg.bdef;
  int mine = 0;
  if (d != 0.0) {  // an exactly Hermitian input cannot fail
    for (int p = threadIdx.x; p < hg.P; p += blockDim.x) {
      const double sc = sqrt(hg.pscale[p]);
      // NaN anywhere makes the test false: flagged, the exact path decides
      if (!(1.01 * d < 1e-12 * (sc - 0.5 * d))) mine = 1;
    }
  }
  if (mine) bad = 1;
  __syncthreads();  // every read precedes the resets
  for (int p = threadIdx.x; p < hg.P; p += blockDim.x) hg.pscale[p] = 0.0;
  if (threadIdx.x == 0) {
    hg.hstat[0] = hg.hstat[1] = hg.hstat[2] = 0.0;
    if (bad) atomicOr(hg.flags, 1 << hg.bit);
  }
}

struct PhaseDev {
  const double* s;  // [P] live node shifts, ascending k
  const double* w;  // [P] weights
  int P;
  // window batch (window sweep): the phases of W
  // windows concatenated, win[p] = window of phase p; window w's compact
  // state is Uc + w * ustride and its slots follow the previous window's.
  // win == nullptr: one window.
  const int* win = nullptr;
  int W = 1;
  size_t ustride = 0;
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
// pass A: e^{s L} + inverse x-FFT of u, v, eta-b, ikx u, ikx v.
// One CTA = 5 warps; warp f owns output field f for the CTA's GPW tasks
// (task = one (phase, ky column)); the e^{sL} per mode is computed once per
// task by the whole CTA into a shared compact stash.
// ============================================================================
// Gather a compact kx column (Kx values, FFT order wx = 0..K, -K..-1) into
// the type-1 input layout v[n1] = x[t + T n1]; out-of-band slots are zero.
// Band membership of each register slot is resolved at compile time except
// for the slots whose position range straddles a band edge.
template <int N, int N1 = 0>
__device__ __forceinline__ void band_gather(double2* v, int t, const double2* col, bool active) {
  if constexpr (N1 < WF<N>::P) {
    constexpr int T = WF<N>::T, K = N / 3, Kx = 2 * K + 1;
    constexpr int kmin = T * N1, kmax = T * N1 + T - 1;
    const int k = t + kmin;
    if constexpr (kmax <= K) {
      v[N1] = active ? col[k] : czero();
    } else if constexpr (kmin >= N - K) {
      v[N1] = active ? col[k - N + Kx] : czero();
    } else if constexpr (kmin > K && kmax < N - K) {
      v[N1] = czero();
    } else {
      const int r = band_r(k, N, K, Kx);
      v[N1] = (active && r >= 0) ? col[r] : czero();
    }
    band_gather<N, N1 + 1>(v, t, col, active);
  }
}

// Store a type-1 output (register i holds position t1_pos(t, i)) to
// out[pos * stride] with incremental addressing.
template <int N>
__device__ __forceinline__ void store_t1_strided(const double2* v, int t, double2* out, size_t stride) {
  constexpr int T = WF<N>::T, P = WF<N>::P;
  if constexpr (N == 8 || T < 32) {
#pragma unroll
    for (int i = 0; i < P; ++i) out[(size_t)t1_pos<N>(t, i) * stride] = v[i];
  } else {
    // T == 32: positions k1 + 16 (8h + i) for i < 8, + 256 for i >= 8
    double2* p = out + (size_t)t1_pos<N>(t, 0) * stride;
    const size_t s16 = 16 * stride;
#pragma unroll
    for (int i = 0; i < 8; ++i) p[i * s16] = v[i];
    p += 256 * stride;
#pragma unroll
    for (int i = 0; i < 8; ++i) p[i * s16] = v[8 + i];
  }
}

template <int NX, bool MW = false>
struct PassAW {
  static constexpr int T = WF<NX>::T, P = WF<NX>::P, GPW = WF<NX>::GPW;
  static constexpr int WARPS = 5;
  // 3 CTAs/SM (no spills for nx >= 32); at 4 CTAs/SM (96 registers) the
  // phase-pair block spills and measured slower
  static constexpr int CTAS = 3;
  // mbarrier | buffer [SLOTS][GPW][Kx] (u, v, eta, b, (c1,c2)_p, (c1,c2)_q ->
  // u'_p, v'_p, depth_p, u'_q, v'_q, depth_q in place; window batches (MW)
  // add u, v, eta of phase q's window in slots 6..8 when it differs from p's)
  // | xbuf per group
  static constexpr int SLOTS = MW ? 9 : 6;
  // ... | the Hermitian gate's per-warp phase maxima [WARPS][2]
  // ... | kx / 2 [Kx] (the x-derivative fields, see pass A) | kx [Kx]
  static size_t bytes(int Kx) {
    return 16 + (size_t)GPW * SLOTS * Kx * sizeof(double2) + (size_t)WARPS * GPW * WF<NX>::XBUF * sizeof(double) +
           (size_t)WARPS * 2 * sizeof(double) + (size_t)2 * Kx * sizeof(double);
  }
};

// Persistent CTAs over "task blocks" (GPW consecutive ky columns of one
// phase PAIR p, q = p + 1).  Per block: the compact U columns, b and the
// phase table's (c1, c2) columns of both phases are TMA-bulk-prefetched
// (one buffer, refilled as soon as the FFT inputs are in registers), the
// whole CTA applies e^{s_p L} and e^{s_q L} per mode in place (U is read once
// for both phases), then warp f runs the inverse x-FFTs of output field f
// (u, v, eta-b, ikx u, ikx v) of both phases and stores them to I1.  Two CTA
// barriers per two transforms per warp.
template <int NX, bool MW>
__global__ void __launch_bounds__(PassAW<NX, MW>::WARPS * 32, PassAW<NX, MW>::CTAS)
    passA_kernel(GridDev G, Prop pr, PhaseDev ph, int p0, int np, const double2* __restrict__ Uc,
                 const double2* __restrict__ ctab, double2* __restrict__ I, double* __restrict__ pscale) {
  griddep_wait();
  griddep_launch();
  using W = PassAW<NX, MW>;
  constexpr int T = W::T, P = W::P, GPW = W::GPW;
  extern __shared__ __align__(128) unsigned char sbytes[];
  constexpr int Kx = 2 * (NX / 3) + 1;  // == G.Kx
  const int Ky = G.Ky;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sbytes);
  unsigned* rcnt = reinterpret_cast<unsigned*>(sbytes + 8);  // warps done with the block's buffer
  double2* buf = reinterpret_cast<double2*>(sbytes + 16);  // [SLOTS][GPW][Kx]
  double* xbuf = reinterpret_cast<double*>(buf + (size_t)GPW * W::SLOTS * Kx);
  double* gred = xbuf + (size_t)W::WARPS * GPW * WF<NX>::XBUF;  // [WARPS][2]
  // Half-scaled factors: every quadratic product pass B forms has exactly
  // one factor among (ux, vx, uy, vy, depth); pass A writes ux, vx and the
  // depth at half scale (kx / 2, and 1 / (2 nx ny)) and pass B uses ky / 2,
  // so the products come out halved -- exactly, scaling by 1/2 commutes with
  // rounding -- and pass B's real-pair unpack needs no multiply by 1/2.
  double* kxh = gred + 2 * W::WARPS;  // [Kx]
  double* kxs = kxh + Kx;              // [Kx] kx for the exponentials (shared, not L1 loads)
  for (int r = threadIdx.x; r < Kx; r += blockDim.x) {
    kxs[r] = G.kxc[r];
    kxh[r] = 0.5 * kxs[r];
  }
  const bool tab = ctab != nullptr;
  const int cols = (Ky + GPW - 1) / GPW;
  const int npair = (np + 1) / 2;
  const int nblk = npair * cols;
  const size_t KyKx = (size_t)Ky * Kx, fs = (size_t)GPW * Kx;
  const int lane = threadIdx.x & 31, f = threadIdx.x >> 5;  // warp = output field

  // block -> (phase pair pp, first column j0, ncol columns): contiguous in U, b, ctab.
  // Warp 0: lane 0 posts the byte count, lanes 0..5 each issue one bulk copy.
  // window batch: the windows of the block's two phases (MW only)
  auto wins = [&](int pp, int& wp, int& wq) {
    wp = wq = 0;
    if constexpr (MW) {
      wp = ph.win[p0 + 2 * pp];
      wq = (2 * pp + 1 < np) ? ph.win[p0 + 2 * pp + 1] : wp;
    }
  };
  auto prefetch = [&](int blk) {
    const int pp = blk / cols, j0 = (blk % cols) * GPW;
    const int ncol = min(GPW, Ky - j0);
    const int nq = (2 * pp + 1 < np) ? 2 : 1;
    int wp, wq;
    wins(pp, wp, wq);
    const uint32_t seg = (uint32_t)(ncol * Kx * sizeof(double2));
    if (lane == 0) mbar_arrive_expect_tx(bar, ((tab ? 4 + nq : 4) + (wq != wp ? 3 : 0)) * seg);
    __syncwarp();
    const double2* Up = Uc + (size_t)wp * ph.ustride;
    if (lane < 3) bulk_g2s(buf + lane * fs, Up + lane * KyKx + (size_t)j0 * Kx, seg, bar);
    if (lane == 3) bulk_g2s(buf + 3 * fs, G.bc + (size_t)j0 * Kx, seg, bar);
    if (tab && lane >= 4 && lane - 4 < nq)
      bulk_g2s(buf + lane * fs, ctab + (size_t)(p0 + 2 * pp + lane - 4) * KyKx + (size_t)j0 * Kx, seg, bar);
    if (MW && wq != wp && lane >= 6 && lane < 9)
      bulk_g2s(buf + lane * fs, Uc + (size_t)wq * ph.ustride + (lane - 6) * KyKx + (size_t)j0 * Kx, seg, bar);
  };
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    *rcnt = 0u;
    fence_mbar_init();
  }
  __syncthreads();
  if (f == 0 && (int)blockIdx.x < nblk) prefetch(blockIdx.x);

  const int tl = lane / T, t = lane % T;
  double* xb = xbuf + (size_t)(f * GPW + tl) * WF<NX>::XBUF;
  const WLane wl = wlane<NX>(G.twx, t);
  const int fi = f < 3 ? f : f - 3;  // source slot of this warp's field
#pragma unroll 1
  for (int it = 0;; ++it) {
    const int blk = (int)blockIdx.x + it * (int)gridDim.x;
    if (blk >= nblk) break;
    const int pp = blk / cols, j0 = (blk % cols) * GPW;
    const int ncol = min(GPW, Ky - j0);
    const int pa = 2 * pp;
    const bool hasq = pa + 1 < np;
    int wp, wq;
    wins(pp, wp, wq);
    const bool qown = MW && wq != wp;  // phase q's state is in slots 6..8
    mbar_wait(bar, it & 1);
    // e^{sL} per mode for both phases, in place:
    // (u, v, eta, b, c_p, c_q) -> (u', v', eta' - b)_p, (u', v', eta' - b)_q, / (nx ny)
    double kyb[GPW];
#pragma unroll
    for (int c = 0; c < GPW; ++c) kyb[c] = G.kyc[min(j0 + c, Ky - 1)];
    // Hermitian gate (pscale): max squared magnitude of u', v', eta' - b per phase
    double gmax0 = 0.0, gmax1 = 0.0;
    for (int idx = threadIdx.x; idx < ncol * Kx; idx += blockDim.x) {
      const int tt = idx / Kx, r = idx % Kx;
      double2* e = buf + idx;
      const C3 q0 = {e[0], e[fs], e[2 * fs]};
      const double2 bb = e[3 * fs];
      const double kx = kxs[r];
      double ky = kyb[0];
#pragma unroll
      for (int c = 1; c < GPW; ++c)
        if (tt == c) ky = kyb[c];
      const double2 cb = (tab && hasq) ? e[5 * fs] : czero();
      const C3 q1 = qown ? C3{e[6 * fs], e[7 * fs], e[8 * fs]} : q0;
#pragma unroll 1
      for (int sub = 0; sub < (hasq ? 2 : 1); ++sub) {
        C3 q = tab ? exp_c12(sub ? cb : e[4 * fs], sub ? q1 : q0, G.ph, kx, ky)
                   : expL(ph.s[p0 + pa + sub], sub ? q1 : q0, G.ph, kx, ky, pr);
        double2* o = e + (size_t)(3 * sub) * fs;
        const double2 dep = csub(q.e, bb);
        o[0] = cscale(G.inv_n2, q.u);
        o[fs] = cscale(G.inv_n2, q.v);
        o[2 * fs] = cscale(0.5 * G.inv_n2, dep);  // half-scaled depth (see kxh)
        if (pscale) {  // (a non-finite input is flagged through pack's statistics: fmax is enough here)
          const double m = fmax(fmax(abs2(q.u), abs2(q.v)), abs2(dep));
          if (sub) gmax1 = fmax(m, gmax1);
          else gmax0 = fmax(m, gmax0);
        }
      }
    }
    if (pscale) {
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        gmax0 = fmax(gmax0, __shfl_xor_sync(0xffffffffu, gmax0, o));
        gmax1 = fmax(gmax1, __shfl_xor_sync(0xffffffffu, gmax1, o));
      }
      if (lane == 0) {
        gred[2 * f] = gmax0;
        gred[2 * f + 1] = gmax1;
      }
    }
    fence_proxy_async();  // order these stores before the next block's TMA refill of buf
    __syncthreads();
    if (pscale && threadIdx.x == 0) {  // one atomic per phase per block
      double m0 = 0.0, m1 = 0.0;
#pragma unroll
      for (int k = 0; k < W::WARPS; ++k) {
        m0 = fmax(m0, gred[2 * k]);
        m1 = fmax(m1, gred[2 * k + 1]);
      }
      unsigned long long* ps = reinterpret_cast<unsigned long long*>(pscale + p0 + pa);
      atomicMax(ps, (unsigned long long)__double_as_longlong(m0));
      if (hasq) atomicMax(ps + 1, (unsigned long long)__double_as_longlong(m1));
    }
    const bool active = tl < ncol;
#define PSWE_A_GATHER(v, sub)                                                         \
  band_gather<NX>(v, t, buf + (size_t)(fi + 3 * (sub)) * fs + (size_t)tl * Kx, active);  \
  if (f >= 3) { /* ikx u', ikx v' */                                                 \
    _Pragma("unroll") for (int n1 = 0; n1 < P; ++n1) {                                 \
      const int r = band_r(t + T * n1, NX, NX / 3, Kx);                                \
      if (r >= 0) v[n1] = cik(kxh[r], v[n1]);                                          \
    }                                                                                  \
  }
    double2* const out0 = I + ((((size_t)pa) * 5 + f) * Ky + j0 + tl) * NX;
    double2* const out1 = out0 + (size_t)5 * Ky * NX;
    // both phases through one copy of the transform code; the buffer is
    // released (and refilled for the next block) after the last gather
    const int nsub = hasq ? 2 : 1;
#pragma unroll 1
    for (int sub = 0; sub < nsub; ++sub) {
      double2 v[P];
      PSWE_A_GATHER(v, sub)
      if (sub == nsub - 1) {
        // buffer consumed: the last warp done with it refills it for the
        // next block while the FFTs run (no CTA barrier)
        if (last_warp_arrival(rcnt, W::WARPS, lane) && blk + (int)gridDim.x < nblk) {
          fence_proxy_async();
          prefetch(blk + gridDim.x);
        }
      }
      wfft_t1<NX, true, true>(v, t, xb, wl);
      if (active) store_t1_strided<NX>(v, t, sub ? out1 : out0, 1);
    }
#undef PSWE_A_GATHER
  }
}

// ============================================================================
// pass B: per physical row x: y-C2R of the 7 fields (paired by physical
// dimension: (u,v), (ux,uy), (vx,vy), (depth,0)), quadratic products, y-R2C
// of (A,B) and (C,D), keep ky = 0..KYM.  In place on I (fields 0..3 out).
// Pairing by dimension matters: a pair's round-off is relative to the larger
// member, so (depth [m], ux [1/s]) would cost ~1e-10 relative in ux.
// One transform group (T lanes, 16 points each) per row; the products are
// formed on the y positions each lane owns between the type-1 (inverse) and
// type-2 (forward) transforms.
// ============================================================================
template <int NY>
struct PassBW {
  static constexpr int T = WF<NY>::T, P = WF<NY>::P, GPW = WF<NY>::GPW;
  static constexpr int WARPS = 4;
  static constexpr int GPC = WARPS * GPW;  // rows per CTA
  static constexpr int Ky = NY / 3 + 1;
  static constexpr int KYA = (Ky + 7) / 8 * 8;  // TMA destinations 128-byte aligned
  static constexpr int R = GPC;                 // rows per CTA (output tile width)
  // FAST (NY >= 64 and R | nx): the (u, v) stash lives in tensor memory and
  // the outputs leave through a shared [2][Ky][R] staging tile + TMA store.
  // Otherwise (small grids) the stash is in shared memory and the outputs are
  // stored directly.
  // per warp (128-byte aligned): prefetch [GPW][2][KYA] | per group: xbuf
  // [| (u, v) stash] | mbarrier;  then stage | ky [Ky] | TMEM base
  template <bool FAST>
  __host__ __device__ static constexpr size_t warp_bytes() {
    return ((size_t)GPW * 2 * KYA * sizeof(double2) + (size_t)GPW * WF<NY>::XBUF * sizeof(double) +
            (FAST ? 0 : (size_t)GPW * P * T * sizeof(double2)) + 8 + 127) /
           128 * 128;
  }
  // FAST: each warp pair owns a [2][Ky][RP] staging tile (RP = 2 GPW rows),
  // synchronised by a named barrier of its 64 threads only
  static constexpr int RP = 2 * GPW;
  static constexpr size_t PAIR_STAGE = ((size_t)2 * Ky * RP * sizeof(double2) + 1023) / 1024 * 1024;
  template <bool FAST>
  __host__ __device__ static constexpr size_t stage_bytes() {
    return FAST ? 2 * PAIR_STAGE + 1024 : 0;
  }
  template <bool FAST>
  static size_t bytes() {
    return (size_t)WARPS * warp_bytes<FAST>() + stage_bytes<FAST>() + (size_t)Ky * sizeof(double) + 16;
  }
};

// type-1 input of the packed pair A + iB at position k = t + T*N1, from the
// prefetched half-spectra A = pre[0..Ky), B = pre[Ky..2Ky).  The band tests
// are resolved at compile time except for the (at most two) register slots
// whose k range straddles a band edge.
template <int NY, int N1, bool HAS_B, bool DERIV>
__device__ __forceinline__ double2 pair_val(int t, const double2* pre, const double* kys) {
  constexpr int T = WF<NY>::T, KYM = NY / 3;
  constexpr int kmin = T * N1, kmax = T * N1 + T - 1;
  if constexpr (kmin > KYM && kmax < NY - KYM) {
    return czero();
  } else {
    const int k = t + kmin;
    bool lo;
    if constexpr (kmax <= KYM) {
      lo = true;
    } else if constexpr (kmin >= NY - KYM) {
      lo = false;
    } else {
      lo = k <= KYM;
      if (!lo && k < NY - KYM) return czero();
    }
    const int jj = lo ? k : NY - k;
    const double2 A = pre[jj];
    double2 B = czero();
    if constexpr (HAS_B) {
      B = pre[PassBW<NY>::KYA + jj];
      if constexpr (DERIV) B = cik(kys[jj], B);
    }
    if constexpr (N1 == 0) {
      if (t == 0) return cmk(A.x, B.x);  // Hermitian projection of the y-mean bin
    }
    return lo ? cmk(A.x - B.y, A.y + B.x) : cmk(A.x + B.y, B.x - A.y);
  }
}

template <int NY, bool HAS_B, bool DERIV, int N1 = 0>
__device__ __forceinline__ void build_pair_t(double2* v, int t, const double2* pre, const double* kys) {
  if constexpr (N1 < WF<NY>::P) {
    v[N1] = pair_val<NY, N1, HAS_B, DERIV>(t, pre, kys);
    build_pair_t<NY, HAS_B, DERIV, N1 + 1>(v, t, pre, kys);
  }
}

// it: 0 (u, v), 1 (ux, i ky u), 2 (vx, i ky v), 3 (depth, -)
template <int NY>
__device__ __forceinline__ void build_pair(double2* v, int t, const double2* pre, const double* kys, int it) {
  if (it == 0)
    build_pair_t<NY, true, false>(v, t, pre, kys);
  else if (it < 3)
    build_pair_t<NY, true, true>(v, t, pre, kys);
  else
    build_pair_t<NY, false, false>(v, t, pre, kys);
}

// after a type-2 forward transform (v[k2] = Z[t + T k2]): split the packed pair
// into the two real spectra X = (Z + conj Z(-j))/2, Y = (Z - conj Z(-j))/(2i)
// for j = 0..Ky-1 and store them.
// HALF: the pair's members are at full scale (multiply by 1/2); false: the
// inputs were formed at half scale (pass A/B's half-scaled factors)
template <int NY, bool HALF = true>
__device__ __forceinline__ void unpack_store(const double2* v, int t, double2* outX, double2* outY, int Ky,
                                             int stride, bool active) {
  constexpr int T = WF<NY>::T, P = WF<NY>::P;
  constexpr int MU = (NY / 3 + 1 + T - 1) / T;
#pragma unroll
  for (int m = 0; m < MU; ++m) {
    const int j = t + T * m;
    double2 zm;
    if constexpr (T == 1) {
      zm = v[(P - m) & (P - 1)];
    } else {
      const double2 src = v[P - 1 - m];
      double2 r;
      r.x = __shfl_sync(0xffffffffu, src.x, (T - t) & (T - 1), T);
      r.y = __shfl_sync(0xffffffffu, src.y, (T - t) & (T - 1), T);
      zm = t == 0 ? v[(P - m) & (P - 1)] : r;
    }
    if (active && j < Ky) {
      const double2 a = v[m];
      constexpr double h = HALF ? 0.5 : 1.0;
      outX[(size_t)j * stride] = cmk(h * (a.x + zm.x), h * (a.y - zm.y));
      outY[(size_t)j * stride] = cmk(h * (a.y + zm.y), -h * (a.x - zm.x));
    }
  }
}

// transform `it` of a row: inputs (fa, fb) of the packed pair
//   0: (u, v)   1: (ux, i ky u)   2: (vx, i ky v)   3: (depth, -)
__device__ __forceinline__ int passB_fa(int it) { return it == 0 ? 0 : (it == 1 ? 3 : (it == 2 ? 4 : 2)); }
__device__ __forceinline__ int passB_fb(int it) { return it == 0 ? 1 : (it == 1 ? 0 : (it == 2 ? 1 : -1)); }

// Queue the TMA row gathers of transform `it`'s inputs for the warp's GPW
// rows into its prefetch buffer: one box (1 x, Ky j) of I1 per field, at
// tensor coordinates (0, x, 0, f + 5 p).  Lane 0 posts the byte count, lanes
// 0..GPW-1 issue their row's gathers.
template <int NY>
__device__ __forceinline__ void passB_prefetch(int it, int lane, double2* pre, uint64_t* bar,
                                               const CUtensorMap* mI, int first_task, int ntask, int nx) {
  constexpr int GPW = WF<NY>::GPW, KYA = PassBW<NY>::KYA;
  constexpr uint32_t seg = (uint32_t)PassBW<NY>::Ky * sizeof(double2);
  const int fa = passB_fa(it), fb = passB_fb(it);
  if (lane == 0) {
    const int nrow = max(0, min(GPW, ntask - first_task));
    mbar_arrive_expect_tx(bar, (uint32_t)nrow * (fb >= 0 ? 2 * seg : seg));
  }
  __syncwarp();
  if (lane < GPW) {
    const int task = first_task + lane;
    if (task < ntask) {
      const int p = task / nx, x = task % nx;
      tma_load_4d(pre + (size_t)lane * 2 * KYA, mI, 0, x, 0, fa + 5 * p, bar);
      if (fb >= 0) tma_load_4d(pre + (size_t)lane * 2 * KYA + KYA, mI, 0, x, 0, fb + 5 * p, bar);
    }
  }
}

// (u, v) of registers i0 .. i0+3 from the stash: tensor memory (FAST, four
// loads in flight per wait) or shared memory
template <int NY, bool FAST>
__device__ __forceinline__ void uv_get4(double2 (&q)[4], const double2* uv, uint32_t taddr, int i0, int t) {
  if constexpr (FAST) {
    uint32_t r[4][4];
#pragma unroll
    for (int k = 0; k < 4; ++k) tmem_ld_x4(taddr + 4 * (i0 + k), r[k]);
    tmem_wait_ld();
#pragma unroll
    for (int k = 0; k < 4; ++k) q[k] = tmem_unpack(r[k]);
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k) q[k] = uv[(i0 + k) * WF<NY>::T + t];
  }
}

// Small grids (NY < 64 or tiles that do not divide nx): one row per task
// group, the (u, v) stash in shared memory, outputs stored directly into the
// column-major I2.  The FAST path is passB_pair_kernel.
template <int NY>
__global__ void __launch_bounds__(PassBW<NY>::WARPS * 32, 3)
    passB_kernel(GridDev Gd, int np, const __grid_constant__ CUtensorMap mI, double2* __restrict__ I2) {
  griddep_wait();
  griddep_launch();
  using W = PassBW<NY>;
  constexpr int T = W::T, P = W::P, GPW = W::GPW, KYA = W::KYA;
  extern __shared__ __align__(128) unsigned char sbytes[];
  constexpr int Ky = W::Ky;  // == Gd.Ky
  constexpr size_t WB = W::template warp_bytes<false>();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int t = lane % T, g = lane / T;
  unsigned char* wbase = sbytes + (size_t)warp * WB;
  double2* pre = reinterpret_cast<double2*>(wbase);  // [GPW][2][KYA]
  double* xb = reinterpret_cast<double*>(pre + (size_t)GPW * 2 * KYA) + (size_t)g * WF<NY>::XBUF;
  double2* uv = reinterpret_cast<double2*>(reinterpret_cast<double*>(pre + (size_t)GPW * 2 * KYA) +
                                           (size_t)GPW * WF<NY>::XBUF) +
                (size_t)g * P * T;  // [P][T]
  uint64_t* bar = reinterpret_cast<uint64_t*>(wbase + WB - 8);
  double* kys = reinterpret_cast<double*>(sbytes + (size_t)W::WARPS * WB);
  const int ntask = np * Gd.nx;
  const int first_task = (blockIdx.x * W::WARPS + warp) * GPW;
  const int task = first_task + g;
  const bool active = task < ntask;
  const int pl = active ? task / Gd.nx : 0, x = active ? task % Gd.nx : 0;
  const size_t KyNX = (size_t)Ky * Gd.nx;
  double2* out = I2 + (size_t)pl * 4 * KyNX + x;  // I2[pl][f][j][x]
  const double2* mypre = pre + (size_t)g * 2 * KYA;
  for (int i = threadIdx.x; i < Ky; i += blockDim.x) kys[i] = 0.5 * Gd.kyc[i];  // half-scaled uy, vy

  if (lane == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  passB_prefetch<NY>(0, lane, pre, bar, &mI, first_task, ntask, Gd.nx);

  double2 v[P];
  double pa[P];
  const WLane wl = wlane<NY>(Gd.twy, t);
#pragma unroll 1
  for (int it = 0; it < 4; ++it) {
    mbar_wait(bar, it & 1);
    build_pair<NY>(v, t, mypre, kys, it);
    __syncwarp();  // prefetch buffer consumed
    // queue the next transform's inputs; they land while this one computes.
    if (it < 3) passB_prefetch<NY>(it + 1, lane, pre, bar, &mI, first_task, ntask, Gd.nx);
    wfft_t1<NY, true, true>(v, t, xb, wl);
    if (it == 0) {
#pragma unroll
      for (int i = 0; i < P; ++i) uv[i * T + t] = v[i];
    } else if (it == 1) {
#pragma unroll
      for (int i = 0; i < P; ++i) {
        const double2 q = uv[i * T + t];
        pa[i] = ndot(q, v[i]);  // A = -(u ux + v uy)
      }
    } else if (it == 2) {
#pragma unroll
      for (int i = 0; i < P; ++i) {
        const double2 q = uv[i * T + t];
        v[i] = cmk(pa[i], ndot(q, v[i]));  // A + iB, B = -(u vx + v vy)
      }
    } else {
#pragma unroll
      for (int i = 0; i < P; ++i) {
        const double2 q = uv[i * T + t];
        v[i] = cmk(q.x * v[i].x, q.y * v[i].x);  // C + iD = u depth + i v depth
      }
    }
    if (it < 2) continue;
    wfft_t2<NY, false>(v, t, xb, wl);
    const int fo = it == 2 ? 0 : 2;
    unpack_store<NY, false>(v, t, out + (size_t)fo * KyNX, out + (size_t)(fo + 1) * KyNX, Ky, Gd.nx, active);
  }
}

// Latency-bound evaluations -- launchB picks this whenever the single-phase
// CTAs of all lanes would not fill the SMs: small grids with few phases, but
// also 256^2 / 512^2 with one phase (apply_nonlinear, step_reference).  The
// four inverse transforms of a row group run on four warps at once instead of in
// sequence -- warp w: 0 (u, v), 1 (ux, i ky u), 2 (vx, i ky v), 3 (depth) --
// the physical values meet in shared memory, and warps 0 and 1 run the two
// forward transforms (A + iB, C + iD) side by side: two transform latencies
// per row group instead of six.  Same inputs, outputs and arithmetic per
// value as passB_kernel.
template <int NY>
struct PassBSW {
  static constexpr int T = WF<NY>::T, P = WF<NY>::P, GPW = WF<NY>::GPW;
  static constexpr int KYA = PassBW<NY>::KYA;
  // per warp: prefetch [GPW][2][KYA] | xbuf per group | mbarrier; then the
  // physical stash [4][P][32] | ky [Ky]
  static constexpr size_t WB =
      ((size_t)GPW * 2 * KYA * sizeof(double2) + (size_t)GPW * WF<NY>::XBUF * sizeof(double) + 8 + 127) / 128 * 128;
  static size_t bytes() {
    return 4 * WB + (size_t)4 * P * 32 * sizeof(double2) + (size_t)PassBW<NY>::Ky * sizeof(double) + 16;
  }
};

template <int NY>
__global__ void __launch_bounds__(128)
    passB_split_kernel(GridDev Gd, int np, const __grid_constant__ CUtensorMap mI, double2* __restrict__ I2) {
  griddep_wait();
  griddep_launch();
  using W = PassBSW<NY>;
  constexpr int T = W::T, P = W::P, GPW = W::GPW, KYA = W::KYA;
  constexpr int Ky = PassBW<NY>::Ky;
  extern __shared__ __align__(128) unsigned char sbytes[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int t = lane % T, g = lane / T;
  unsigned char* wbase = sbytes + (size_t)warp * W::WB;
  double2* pre = reinterpret_cast<double2*>(wbase);
  double* xb = reinterpret_cast<double*>(pre + (size_t)GPW * 2 * KYA) + (size_t)g * WF<NY>::XBUF;
  uint64_t* bar = reinterpret_cast<uint64_t*>(wbase + W::WB - 8);
  double2* stash = reinterpret_cast<double2*>(sbytes + 4 * W::WB);  // [4][P][32]
  double* kys = reinterpret_cast<double*>(stash + (size_t)4 * P * 32);
  const int ntask = np * Gd.nx;
  const int first_task = blockIdx.x * GPW;  // the CTA's row group, shared by its 4 warps
  const int task = first_task + g;
  const bool active = task < ntask;
  const int pl = active ? task / Gd.nx : 0, x = active ? task % Gd.nx : 0;
  const size_t KyNX = (size_t)Ky * Gd.nx;
  double2* out = I2 + (size_t)pl * 4 * KyNX + x;
  for (int i = threadIdx.x; i < Ky; i += blockDim.x) kys[i] = 0.5 * Gd.kyc[i];  // half-scaled uy, vy
  if (lane == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  passB_prefetch<NY>(warp, lane, pre, bar, &mI, first_task, ntask, Gd.nx);
  const WLane wl = wlane<NY>(Gd.twy, t);
  double2 v[P];
  mbar_wait(bar, 0);
  build_pair<NY>(v, t, pre + (size_t)g * 2 * KYA, kys, warp);
  wfft_t1<NY, true, true>(v, t, xb, wl);
  double2* mine = stash + (size_t)warp * P * 32;
#pragma unroll
  for (int i = 0; i < P; ++i) mine[i * 32 + lane] = v[i];
  __syncthreads();
  if (warp >= 2) return;
  const double2* suv = stash;                 // (u, v)
  const double2* sux = stash + P * 32;        // (ux, uy)
  const double2* svx = stash + 2 * P * 32;    // (vx, vy)
  const double2* sd = stash + 3 * P * 32;     // (depth, -)
#pragma unroll
  for (int i = 0; i < P; ++i) {
    const double2 q = suv[i * 32 + lane];
    if (warp == 0) {
      const double2 a = sux[i * 32 + lane], b = svx[i * 32 + lane];
      v[i] = cmk(ndot(q, a), ndot(q, b));  // A + iB
    } else {
      const double d = sd[i * 32 + lane].x;
      v[i] = cmk(q.x * d, q.y * d);  // C + iD = u depth + i v depth
    }
  }
  wfft_t2<NY, false>(v, t, xb, wl);
  const int fo = warp == 0 ? 0 : 2;
  unpack_store<NY, false>(v, t, out + (size_t)fo * KyNX, out + (size_t)(fo + 1) * KyNX, Ky, Gd.nx, active);
}

// Unpack a forward pair transform (as unpack_store) into the warp pair's staging
// tile [2 fields][Ky][R] at tile row rc, in the swizzled layout of the TMA
// store map: a tile line (one field, one j: R complex = R * 16 bytes) has its
// 16-byte chunks permuted, chunk' = chunk ^ ((line >> 1) & 3) for 64-byte
// lines (R = 4, SWIZZLE_64B) and chunk ^ (line & 7) for 128-byte lines
// (R = 8, SWIZZLE_128B), so the warp's writes (consecutive j) hit distinct
// banks.  Wider tiles are unswizzled.
template <int NY, int R>
__device__ __forceinline__ int stage_slot(int line, int rc) {
  if constexpr (R == 2)  // 32-byte lines, SWIZZLE_32B: chunk ^ bit 2 of the line
    return line * 2 + (rc ^ ((line >> 2) & 1));
  else if constexpr (R == 4)
    return line * 4 + (rc ^ ((line >> 1) & 3));
  else if constexpr (R == 8)
    return line * 8 + (rc ^ (line & 7));
  else
    return line * R + rc;
}

template <int NY, int R>
__device__ __forceinline__ void unpack_stage(const double2* v, int t, double2* stage, int rc) {
  constexpr int T = WF<NY>::T, P = WF<NY>::P, Ky = NY / 3 + 1;
  constexpr int MU = (Ky + T - 1) / T;
#pragma unroll
  for (int m = 0; m < MU; ++m) {
    const int j = t + T * m;
    double2 zm;
    if constexpr (T == 1) {
      zm = v[(P - m) & (P - 1)];
    } else {
      const double2 src = v[P - 1 - m];
      double2 r;
      r.x = __shfl_sync(0xffffffffu, src.x, (T - t) & (T - 1), T);
      r.y = __shfl_sync(0xffffffffu, src.y, (T - t) & (T - 1), T);
      zm = t == 0 ? v[(P - m) & (P - 1)] : r;
    }
    if (j < Ky) {  // inputs at half scale (pass A/B's half-scaled factors): no 1/2 here
      const double2 a = v[m];
      stage[stage_slot<NY, R>(j, rc)] = cmk(a.x + zm.x, a.y - zm.y);
      stage[stage_slot<NY, R>(Ky + j, rc)] = cmk(a.y + zm.y, zm.x - a.x);
    }
  }
}

// ----------------------------------------------------------------------------
// pass B, phase-paired (FAST path): a warp processes its row for two
// consecutive phases p0, p0 + 1.  The depth fields of both phases share one
// inverse FFT (packed pair d_p0 + i d_p1, same dimension and size); the
// phase-p1 depth is parked in tensor memory until its products are formed.
// 11 row transforms per two phases instead of 12.
// ----------------------------------------------------------------------------
template <int NY>
__device__ __forceinline__ void passB_pair_prefetch(int lane, double2* pre, double2* preb, uint64_t* bar,
                                                    const CUtensorMap* mI, int first_task, int ntp, int nx,
                                                    int fa, int pa, int fb, int pb) {
  constexpr int GPW = WF<NY>::GPW, KYA = PassBW<NY>::KYA;
  constexpr uint32_t seg = (uint32_t)PassBW<NY>::Ky * sizeof(double2);
  if (lane == 0) {
    const int nrow = max(0, min(GPW, ntp - first_task));
    mbar_arrive_expect_tx(bar, (uint32_t)nrow * (fb >= 0 ? 2 * seg : seg));
  }
  __syncwarp();
  if (lane < GPW) {
    const int task = first_task + lane;
    if (task < ntp) {
      const int x = task % nx;
      tma_load_4d(pre + (size_t)lane * 2 * KYA, mI, 0, x, 0, fa + 5 * pa, bar);
      if (fb >= 0) tma_load_4d(preb + (size_t)lane * 2 * KYA, mI, 0, x, 0, fb + 5 * pb, bar);
    }
  }
}

template <int NY>
__global__ void __launch_bounds__(PassBW<NY>::WARPS * 32, 3)
    passB_pair_kernel(GridDev Gd, int np, const __grid_constant__ CUtensorMap mI, const __grid_constant__ CUtensorMap mO,
                      int qpc) {
  griddep_wait();
  griddep_launch();
  using W = PassBW<NY>;
  constexpr int T = W::T, P = W::P, GPW = W::GPW, KYA = W::KYA, R = W::R, RP = W::RP;
  static_assert(P == 16, "FAST path needs 16 points per lane");
  static_assert(W::WARPS == 4, "two warp pairs per CTA");
  extern __shared__ __align__(128) unsigned char sbytes[];
  constexpr int Ky = W::Ky;
  constexpr size_t WB = W::template warp_bytes<true>();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int t = lane % T, g = lane / T;
  unsigned char* wbase = sbytes + (size_t)warp * WB;
  double2* pre = reinterpret_cast<double2*>(wbase);  // [GPW][2][KYA]
  double2* preb = pre + KYA;
  double* xb = reinterpret_cast<double*>(pre + (size_t)GPW * 2 * KYA) + (size_t)g * WF<NY>::XBUF;
  uint64_t* bar = reinterpret_cast<uint64_t*>(wbase + WB - 8);
  // per warp pair: a [2][Ky][RP] swizzled staging tile, 1024-byte aligned
  const uint32_t stage_pad = (1024u - (smem_u32(sbytes + (size_t)W::WARPS * WB) & 1023u)) & 1023u;
  const int pr = warp >> 1, rcp = (warp & 1) * GPW + g;  // pair, row in the pair's tile
  const bool issuer = (warp & 1) == 0 && lane == 0;       // the pair's TMA-store thread
  double2* stage =
      reinterpret_cast<double2*>(sbytes + (size_t)W::WARPS * WB + stage_pad + (size_t)pr * W::PAIR_STAGE);
  double* kys = reinterpret_cast<double*>(sbytes + (size_t)W::WARPS * WB + W::template stage_bytes<true>());
  uint32_t* tslot = reinterpret_cast<uint32_t*>(kys + Ky);
  const int nx = Gd.nx;
  const int ntp = ((np + 1) / 2) * nx;  // (phase pair, row) tasks
  // the CTA's tile: rows x0 .. x0 + R - 1 of the phase pairs pq0 .. pq1 - 1
  // (qpc pairs per CTA: the prologue, the first gather's latency and the
  // last store's completion are paid once per qpc pairs)
  const int rowgroups = nx / R;
  const int pq0 = (blockIdx.x / rowgroups) * qpc, x0 = (blockIdx.x % rowgroups) * R;
  const int pq1 = min((np + 1) / 2, pq0 + qpc);
  const int rc = warp * GPW + g;
  const double2* mypre = pre + (size_t)g * 2 * KYA;
  for (int i = threadIdx.x; i < Ky; i += blockDim.x) kys[i] = 0.5 * Gd.kyc[i];  // half-scaled uy, vy
  if (lane == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(tslot, 128);
  tmem_fence_before_sync();
  __syncthreads();
  tmem_fence_after_sync();
  const uint32_t taddr = *tslot + ((uint32_t)(32 * warp) << 16);

  // inputs of transform (sub, it) of phase pair pp: fields (fa, fb) of phases (pa, pb)
  auto issue = [&](int pp, int sub, int it) {
    const int p0 = 2 * pp, ph = p0 + sub;
    const bool two = p0 + 1 < np;
    int fa, pa = ph, fb, pb = ph;
    if (it == 0) { fa = 0; fb = 1; }
    else if (it == 1) { fa = 3; fb = 0; }
    else if (it == 2) { fa = 4; fb = 1; }
    else { fa = 2; fb = two ? 2 : -1; pb = p0 + 1; }
    passB_pair_prefetch<NY>(lane, pre, preb, bar, &mI, pp * nx + x0 + warp * GPW, ntp, nx, fa, pa, fb, pb);
  };
  issue(pq0, 0, 0);

  double2 v[P];
  double pa_[P];
  const WLane wl = wlane<NY>(Gd.twy, t);
  uint32_t par = 0;
#pragma unroll 1
  for (int pp = pq0; pp < pq1; ++pp) {
  const int p0 = 2 * pp;
  const int nsub = (p0 + 1 < np) ? 2 : 1;  // CTA-uniform
#pragma unroll 1
  for (int sub = 0; sub < nsub; ++sub) {
#pragma unroll 1
    for (int it = 0; it < 4; ++it) {
      const bool in = !(sub == 1 && it == 3);
      if (in) {
        mbar_wait(bar, par);
        par ^= 1;
        if (it == 0)
          build_pair_t<NY, true, false>(v, t, mypre, kys);
        else if (it < 3)
          build_pair_t<NY, true, true>(v, t, mypre, kys);
        else if (nsub == 2)
          build_pair_t<NY, true, false>(v, t, mypre, kys);  // d_p0 + i d_p1
        else
          build_pair_t<NY, false, false>(v, t, mypre, kys);
        __syncwarp();  // prefetch buffer consumed
        // queue the next input transform: (0,0) (0,1) (0,2) (0,3) [(1,0) (1,1) (1,2)];
        // nothing after the last ((1,3) reuses the shared depth transform of (0,3))
        const bool last = nsub == 2 ? (sub == 1 && it == 2) : it == 3;
        if (!last) {
          if (it < 3) issue(pp, sub, it + 1);
          else issue(pp, sub + 1, 0);
        } else if (pp + 1 < pq1) {
          issue(pp + 1, 0, 0);  // the next pair's first input
        }
        wfft_t1<NY, true, true>(v, t, xb, wl);
      }
      // tensor-memory stores are waited for (tcgen05.wait::st) only before
      // the first load of the same columns, a transform later
      if (it == 0) {
        tmem_stash16(taddr, v);
        PSWE_ST_WAIT_EARLY();
      } else if (it == 1) {
        PSWE_ST_WAIT_LATE();  // (u, v) of it == 0
#pragma unroll
        for (int i0 = 0; i0 < P; i0 += 4) {
          double2 q[4];
          uv_get4<NY, true>(q, nullptr, taddr, i0, t);
#pragma unroll
          for (int k = 0; k < 4; ++k) pa_[i0 + k] = ndot(q[k], v[i0 + k]);
        }
        tmem_stash16d(taddr + 64, pa_);
        PSWE_ST_WAIT_EARLY();
      } else if (it == 2) {
        PSWE_ST_WAIT_LATE();  // A of it == 1
#pragma unroll
        for (int i0 = 0; i0 < P; i0 += 4) {
          double2 q[4];
          uv_get4<NY, true>(q, nullptr, taddr, i0, t);
          uint32_t r[8];
          tmem_ld_x8(taddr + 64 + 2 * i0, r);
          tmem_wait_ld();
#pragma unroll
          for (int k = 0; k < 4; ++k)  // A + iB, B = -(u vx + v vy)
            v[i0 + k] = cmk(__hiloint2double(r[2 * k + 1], r[2 * k]),
                            ndot(q[k], v[i0 + k]));
        }
      } else {
        if (sub == 0) {
          if (nsub == 2) {  // park d_p1 (imaginary part) for the second phase
            double dd[P];
#pragma unroll
            for (int i = 0; i < P; ++i) dd[i] = v[i].y;
            tmem_stash16d(taddr + 96, dd);
            PSWE_ST_WAIT_EARLY();
          }
        } else {
          PSWE_ST_WAIT_LATE();  // d_p1 of sub 0
#pragma unroll
          for (int i0 = 0; i0 < P; i0 += 4) {
            uint32_t r[8];
            tmem_ld_x8(taddr + 96 + 2 * i0, r);
            tmem_wait_ld();
#pragma unroll
            for (int k = 0; k < 4; ++k) v[i0 + k] = cmk(__hiloint2double(r[2 * k + 1], r[2 * k]), 0.0);
          }
        }
#pragma unroll
        for (int i0 = 0; i0 < P; i0 += 4) {
          double2 q[4];
          uv_get4<NY, true>(q, nullptr, taddr, i0, t);
#pragma unroll
          for (int k = 0; k < 4; ++k)  // C + iD = u depth + i v depth
            v[i0 + k] = cmk(q[k].x * v[i0 + k].x, q[k].y * v[i0 + k].x);
        }
      }
      if (it < 2) continue;
      wfft_t2<NY, false>(v, t, xb, wl);
      const int fo = it == 2 ? 0 : 2;
      if (issuer) bulk_wait_read0();
      named_bar_sync(1 + pr, 64);
      unpack_stage<NY, RP>(v, t, stage, rcp);
      fence_proxy_async();
      named_bar_sync(1 + pr, 64);
      if (issuer) {
        tma_store_3d(&mO, 2 * (x0 + pr * RP), 0, 4 * (p0 + sub) + fo, stage);
        bulk_commit();
      }
    }
  }
  }
  if (issuer) bulk_wait0();
  tmem_fence_before_sync();
  __syncthreads();
  if (warp == 0) {
    tmem_fence_after_sync();
    tmem_dealloc(*tslot, 128);
  }
}

// ============================================================================
// pass C: forward x-FFT of the 4 product spectra (warp f = field f) of the
// CTA's GPW tasks (phase, ky column), then per mode: flux divergence, 2/3
// truncation, e^{-sL}, weight, and accumulation onto the phase's slot
// (slot g = phase position in the chunk; chunks are summed in order and the
// slots reduced in order afterwards -- deterministic, no atomics).
// ============================================================================
template <int NX>
struct PassCW {
  static constexpr int T = WF<NX>::T, P = WF<NX>::P, GPW = WF<NX>::GPW;
  static constexpr int WARPS = 4;
  static constexpr int CPT = 3;  // combine modes per thread (GPW * Kx <= 3 * 128)
  static constexpr int Kx = 2 * (NX / 3) + 1;
  // a transform's exchange buffer fits in its own input column once the
  // column is in registers (NX >= 64), offset by XOFF doubles per group so
  // the groups of a warp keep XBUF's bank stagger
  static constexpr bool XB_IN_PRE = WF<NX>::XBUF + 31 <= 2 * NX;
  static constexpr int XOFF = ((WF<NX>::XBUF - 2 * NX) % 32 + 32) % 32;
  // double-buffered: prefetch [2][4][GPW][NX] (each transform's band output
  // F and exchange buffer overlay its own input column) | (c1,c2) [2][GPW][Kx]
  // | [xbuf per group] | mbarrier [2]
  static size_t bytes(int) {
    return (size_t)2 * 4 * GPW * NX * sizeof(double2) + (size_t)2 * GPW * Kx * sizeof(double2) +
           (XB_IN_PRE ? 0 : (size_t)WARPS * GPW * WF<NX>::XBUF * sizeof(double)) + 16;
  }
};

// CTA = (GPW ky columns) x (phase group g of the chunk).  Loops over the
// group's phases in ascending order with two buffers: phase pl's 4 product
// columns (contiguous in I2) and phase-table columns are TMA-bulk-copied
// while phase pl - 1 computes (a whole phase of lead).  Warp f transforms
// field f in its own column of the buffer (exchange buffer and band output
// overlay the consumed input); then every thread combines its modes (flux
// divergence, e^{-sL}, weight) into register accumulators, which are added
// to the group's slot once at the end.
template <int NX, bool MW>
__global__ void __launch_bounds__(PassCW<NX>::WARPS * 32, 3)
    passC_kernel(GridDev G, Prop pr, PhaseDev ph, int p0, int np, int Gc, const double2* __restrict__ I2,
                 const double2* __restrict__ ctab, double2* __restrict__ slots, int first_chunk) {
  griddep_wait();
  griddep_launch();
  using W = PassCW<NX>;
  constexpr int T = W::T, P = W::P, GPW = W::GPW, CPT = W::CPT;
  extern __shared__ __align__(128) unsigned char sbytes[];
  constexpr int Kx = W::Kx;  // == G.Kx
  constexpr size_t PB = (size_t)4 * GPW * NX;  // double2 per prefetch buffer
  const int Ky = G.Ky;
  double2* pre0 = reinterpret_cast<double2*>(sbytes);  // [2][4][GPW][NX]
  double2* ctb0 = pre0 + 2 * PB;                       // [2][GPW][Kx]
  double* xbuf = reinterpret_cast<double*>(ctb0 + (size_t)2 * GPW * Kx);
  uint64_t* bar = reinterpret_cast<uint64_t*>(
      xbuf + (W::XB_IN_PRE ? 0 : (size_t)W::WARPS * GPW * WF<NX>::XBUF));  // [2]
  const int cols = (Ky + GPW - 1) / GPW;
  const int cb = blockIdx.x % cols, g = blockIdx.x / cols;
  const int lo = (int)(((long long)g * np) / Gc), hi = (int)(((long long)(g + 1) * np) / Gc);
  const size_t KyKx = (size_t)Ky * Kx;
  const int j0 = cb * GPW;
  const int ncol = min(GPW, Ky - j0);  // active columns of this CTA (contiguous in I2)
  const bool tab = ctab != nullptr;
  const int lane = threadIdx.x & 31, f = threadIdx.x >> 5;

  // warp 0: lane 0 posts the byte count, lanes 0..4 each issue one bulk copy
  // (the CTA's ncol columns of field f are contiguous in I2)
  const size_t KyNX = (size_t)Ky * NX;
  auto prefetch = [&](int pl) {
    const int b = (pl - lo) & 1;
    const uint32_t seg = (uint32_t)(ncol * NX * sizeof(double2));
    const uint32_t tseg = (uint32_t)(ncol * Kx * sizeof(double2));
    if (lane == 0) mbar_arrive_expect_tx(bar + b, 4 * seg + (tab ? tseg : 0));
    __syncwarp();
    if (lane < 4)
      bulk_g2s(pre0 + b * PB + (size_t)lane * GPW * NX, I2 + ((size_t)pl * 4 + lane) * KyNX + (size_t)j0 * NX, seg,
               bar + b);
    if (lane == 4 && tab)
      bulk_g2s(ctb0 + (size_t)b * GPW * Kx, ctab + (size_t)(p0 + pl) * KyKx + (size_t)j0 * Kx, tseg, bar + b);
  };
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (f == 0) {
    if (lo < hi) prefetch(lo);
    if (lo + 1 < hi) prefetch(lo + 1);
  }

  const int tl = lane / T, t = lane % T;
  const size_t own = ((size_t)f * GPW + tl) * NX;  // this transform's column in a buffer
  const WLane wl = wlane<NX>(G.twx, t);
  C3 acc[CPT];
  // the combine's wavenumbers are fixed per thread: loaded once, not per
  // phase (their L1 latency had been exposed in the combine)
  // (one ky per CTA when it owns a single column; not at 256, where the
  // registers would spill)
  constexpr bool HOIST = NX != 256;
  constexpr int NKY = GPW == 1 ? 1 : CPT;
  double kxv[CPT], kyv[NKY];
#pragma unroll
  for (int c = 0; c < CPT; ++c) {
    acc[c] = c3zero();
    const int idx = threadIdx.x + c * W::WARPS * 32;
    const int tt = idx / Kx, r = idx % Kx;
    if (HOIST) kxv[c] = __ldg(G.kxc + r);
    if (HOIST && c < NKY) kyv[c] = G.kyc[min(j0 + (NKY == 1 ? 0 : tt), Ky - 1)];
  }
  // slot (+)= acc: this group's phases (of one window), in chunk order.  A
  // window batch (MW) zero-fills the slots first and flushes at every window
  // boundary into slot [g][window].
  auto flush = [&](int win, bool add) {
    double2* slot = slots + ((size_t)g * ph.W + win) * 3 * KyKx;
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      const int idx = threadIdx.x + c * W::WARPS * 32;
      const int tt = idx / Kx, r = idx % Kx;
      if (tt < ncol) {
        double2* sp = slot + (size_t)(j0 + tt) * Kx + r;
        C3 a = acc[c];
        if (add) a = c3add({sp[0], sp[KyKx], sp[2 * KyKx]}, a);
        sp[0] = a.u;
        sp[KyKx] = a.v;
        sp[2 * KyKx] = a.e;
      }
    }
  };
  int wcur = MW && lo < hi ? ph.win[p0 + lo] : 0;
#pragma unroll 1
  for (int pl = lo; pl < hi; ++pl) {
    if constexpr (MW) {
      const int wn = ph.win[p0 + pl];
      if (wn != wcur) {
        flush(wcur, true);
#pragma unroll
        for (int c = 0; c < CPT; ++c) acc[c] = c3zero();
        wcur = wn;
      }
    }
    const int b = (pl - lo) & 1;
    double2* pre = pre0 + b * PB;
    mbar_wait(bar + b, ((pl - lo) >> 1) & 1);
    double2 v[P];
#pragma unroll
    for (int n1 = 0; n1 < P; ++n1) v[n1] = pre[own + t + T * n1];
    __syncwarp();  // the warp's columns are in registers: reuse them
    double* xb = W::XB_IN_PRE ? reinterpret_cast<double*>(pre + own) + ((tl * W::XOFF) & 31)
                              : xbuf + (size_t)(f * GPW + tl) * WF<NX>::XBUF;
    wfft_t1<NX, false>(v, t, xb, wl);
    __syncwarp();  // the exchange buffer's last reads precede the band store
    double2* Ff = pre + own;
#pragma unroll
    for (int i = 0; i < P; ++i) {
      const int r = band_r(t1_pos<NX>(t, i), NX, NX / 3, Kx);
      if (r >= 0) Ff[r] = v[i];
    }
    __syncthreads();
    const double s = ph.s[p0 + pl], w = ph.w[p0 + pl];
    const double2* ctb = ctb0 + (size_t)b * GPW * Kx;
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      const int idx = threadIdx.x + c * W::WARPS * 32;
      const int tt = idx / Kx, r = idx % Kx;
      if (tt < ncol) {
        const double2* Ft = pre + (size_t)tt * NX;  // field f at + f GPW NX
        const double kx = HOIST ? kxv[c] : __ldg(G.kxc + r);
        const double ky = HOIST ? kyv[NKY == 1 ? 0 : c] : G.kyc[j0 + tt];
        const double2 gx = cik(kx, Ft[2 * GPW * NX + r]), gy = cik(ky, Ft[3 * GPW * NX + r]);
        C3 q = {Ft[r], Ft[GPW * NX + r], cmk(-(gx.x + gy.x), -(gx.y + gy.y))};
        if (tab) {
          double2 c12 = ctb[idx];
          c12.x = -c12.x;  // e^{-sL}: c1(-s) = -c1(s), c2(-s) = c2(s)
          q = exp_c12(c12, q, G.ph, kx, ky);
        } else {
          q = expL(-s, q, G.ph, kx, ky, pr);
        }
        acc[c] = c3add(acc[c], c3scale(w, q));
      }
    }
    __syncthreads();  // buffer b consumed
    if (f == 0 && pl + 2 < hi) prefetch(pl + 2);
  }
  if (MW) {
    if (lo < hi) flush(wcur, true);
  } else {
    flush(0, !first_chunk);
  }
}

// ordered sum of the phase-group slots -> compact tendency.  The loads of a
// batch of slots are issued before the (fixed-order) additions: a serial
// load-add chain over Gc slots was latency-bound at small sizes (64^2, M = 8:
// ~6 us for 0.7 MB).
__global__ void reduce_slots_kernel(const double2* __restrict__ slots, int Gc, size_t n,
                                    double2* __restrict__ out) {
  griddep_wait();
  griddep_launch();
  constexpr int B = 8;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    double2 a = slots[i];
    for (int g0 = 1; g0 < Gc; g0 += B) {
      double2 v[B];
#pragma unroll
      for (int k = 0; k < B; ++k) v[k] = g0 + k < Gc ? slots[(size_t)(g0 + k) * n + i] : czero();
#pragma unroll
      for (int k = 0; k < B; ++k)
        if (g0 + k < Gc) a = cadd(a, v[k]);
    }
    out[i] = a;
  }
}

// The same sum, in the same order, for a small state (small grids, whose
// whole evaluation is a latency chain): the eight warps of a block load 32
// slots of 32 consecutive entries per round (four independent coalesced
// loads per thread; the serial kernel's loads end up interleaved with its
// additions, ~3 in flight) into shared memory, and warp 0 adds them in slot
// order -- bitwise equal to reduce_slots_kernel.
__global__ void __launch_bounds__(256) reduce_slots_staged_kernel(const double2* __restrict__ slots, int Gc,
                                                                  size_t n, double2* __restrict__ out) {
  griddep_wait();
  griddep_launch();
  __shared__ double2 val[32][32];  // [slot][entry]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (size_t base = (size_t)blockIdx.x * 32; base < n; base += (size_t)gridDim.x * 32) {
    const size_t i = base + lane;
    double2 a = czero();
    for (int g0 = 0; g0 < Gc; g0 += 32) {
      double2 r[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int g = g0 + w + 8 * k;
        r[k] = (g < Gc && i < n) ? __ldg(slots + (size_t)g * n + i) : czero();
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) val[w + 8 * k][lane] = r[k];
      __syncthreads();
      if (w == 0) {
        const int ng = min(32, Gc - g0);
        for (int g = 0; g < ng; ++g) a = (g0 + g == 0) ? val[0][lane] : cadd(a, val[g][lane]);
      }
      __syncthreads();
    }
    if (w == 0 && i < n) out[i] = a;
  }
}

// The same sum for many slots (small grids, whose pass C runs many phase
// groups): the Gc slots are split into RP contiguous ranges, warp r of a
// block sums range r for 32 consecutive entries (coalesced), and warp 0 adds
// the RP range sums in order -- a fixed summation tree, so still bitwise
// deterministic, and RP times fewer dependent load batches per thread.
constexpr int RED_PARTS = 8;
__global__ void __launch_bounds__(32 * RED_PARTS) reduce_slots_split_kernel(const double2* __restrict__ slots,
                                                                          int Gc, size_t n,
                                                                          double2* __restrict__ out) {
  griddep_wait();
  griddep_launch();
  __shared__ double2 part[RED_PARTS][32];
  const int lane = threadIdx.x & 31, r = threadIdx.x >> 5;
  const int per = (Gc + RED_PARTS - 1) / RED_PARTS;
  const int g0 = r * per, g1 = min(Gc, g0 + per);
  for (size_t base = (size_t)blockIdx.x * 32; base < n; base += (size_t)gridDim.x * 32) {
    const size_t i = base + lane;
    double2 a = czero();
    if (i < n) {
      constexpr int B = 8;
      for (int g = g0; g < g1; g += B) {
        double2 v[B];
#pragma unroll
        for (int k = 0; k < B; ++k) v[k] = g + k < g1 ? slots[(size_t)(g + k) * n + i] : czero();
#pragma unroll
        for (int k = 0; k < B; ++k)
          if (g + k < g1) a = (g + k == g0) ? v[k] : cadd(a, v[k]);
      }
    }
    part[r][lane] = a;
    __syncthreads();
    if (r == 0 && i < n) {
      double2 t = part[0][lane];
      for (int q = 1; q < RED_PARTS; ++q)
        if (q * per < Gc) t = cadd(t, part[q][lane]);
      out[i] = t;
    }
    __syncthreads();
  }
}

// ============================================================================
// layout conversion full <-> compact
// ============================================================================
// pack with Hermitian projection (c(k) + conj c(-k))/2, which is what the
// reference's real(ifft2(.)) does to a field (grid.py:173-174).  With hstat,
// also the Hermitian gate's statistic: hstat[f] = max over the band of
// |c(k) - conj c(-k)|^2 per field (herm_kernels.cuh; NaN propagates).
__global__ void pack_kernel(GridDev G, const double2* __restrict__ u, const double2* __restrict__ v,
                            const double2* __restrict__ e, double2* __restrict__ Uc, double* __restrict__ hstat,
                            int W, size_t ws) {
  griddep_wait();
  griddep_launch();
  // W windows (a window batch): window w's fields at + w * ws, its compact state at + w * 3 Ky Kx
  const size_t KyKx = (size_t)G.Ky * G.Kx;
  double dmax[3] = {0.0, 0.0, 0.0};
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < (size_t)W * 3 * KyKx;
       t += (size_t)gridDim.x * blockDim.x) {
    const size_t win = t / (3 * KyKx), i = t - win * 3 * KyKx;
    const int f = (int)(i / KyKx);
    const int rem = (int)(i % KyKx);
    const int j = rem / G.Kx, r = rem % G.Kx;
    const int wx = r <= G.kxm ? r : r - G.Kx;
    const int ix = (wx + G.nx) % G.nx, jx = (G.nx - ix) % G.nx;
    const int jy = j, my = (G.ny - j) % G.ny;
    const double2* c = (f == 0 ? u : (f == 1 ? v : e)) + win * ws;
    const double2 a = c[(size_t)ix * G.ny + jy];
    const double2 b = c[(size_t)jx * G.ny + my];
    Uc[t] = cmk(0.5 * (a.x + b.x), 0.5 * (a.y - b.y));
    if (hstat) {
      const double dx = a.x - b.x, dy = a.y + b.y;
      const double d2 = fma(dx, dx, dy * dy);
      dmax[f] = nanmax(d2, dmax[f]);
    }
  }
  if (hstat) {
#pragma unroll
    for (int f = 0; f < 3; ++f) {
      double m = dmax[f];
#pragma unroll
      for (int o = 16; o; o >>= 1) m = nanmax(m, __shfl_xor_sync(0xffffffffu, m, o));
      if ((threadIdx.x & 31) == 0 && m != 0.0)
        atomicMax(reinterpret_cast<unsigned long long*>(hstat + f), (unsigned long long)__double_as_longlong(m));
    }
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
                              double2* __restrict__ v, double2* __restrict__ e, int W, size_t ws, HermGate hg) {
  griddep_wait();
  griddep_launch();
  if (hg.bit >= 0 && blockIdx.x == 0) herm_eval_block(hg);
  const size_t n = (size_t)G.nx * G.ny, cs = 3 * (size_t)G.Ky * G.Kx;
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < (size_t)W * n;
       t += (size_t)gridDim.x * blockDim.x) {
    const size_t win = t / n, i = t - win * n;
    const int ix = (int)(i / G.ny), jy = (int)(i % G.ny);
    C3 q = compact_at(G, Ac + win * cs, ix, jy);
    const size_t o = win * ws + i;
    u[o] = q.u;
    v[o] = q.v;
    e[o] = q.e;
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

// The stage kernels run over W windows (a window batch) at once: window w's
// full-layout states at + w * ws, its compact tendency at + w * 3 Ky Kx.
__device__ __forceinline__ Full3 wshift(const Full3& a, size_t o) { return {a.u + o, a.v + o, a.e + o}; }
__device__ __forceinline__ Full3w wshift(const Full3w& a, size_t o) { return {a.u + o, a.v + o, a.e + o}; }

// The next RHS's packed input, written by the stage kernel that produces it
// (the pack launch of stages 2 and 3 saved): the thread of a full mode k in
// the packed half band also evaluates its mirror -k and writes
// Uc[f][ky][kx] = (o(k) + conj o(-k)) / 2 plus the Hermitian gate's
// statistic max |o(k) - conj o(-k)|^2 per field (as pack_kernel does).
struct PackOut {
  double2* Uc;    // W compact states, or nullptr: no packing
  double* hstat;  // [3] the gate's statistic for that RHS
};

// compact index (j, r) of full mode (ix, jy) if it lies in the packed half band
__device__ __forceinline__ bool packed_mode(const GridDev& G, int ix, int jy, int& j, int& r) {
  const int wx = ix < G.nx / 2 ? ix : ix - G.nx;
  if (jy > G.kym || abs(wx) > G.kxm) return false;
  j = jy;
  r = wx >= 0 ? wx : wx + G.Kx;
  return true;
}

__device__ __forceinline__ void pack_store(const GridDev& G, const PackOut& po, size_t wo, int j, int r, const C3& o,
                                           const C3& om, double (&dmax)[3]) {
  const size_t KyKx = (size_t)G.Ky * G.Kx, i = wo + (size_t)j * G.Kx + r;
  const double2 a[3] = {o.u, o.v, o.e}, b[3] = {om.u, om.v, om.e};
#pragma unroll
  for (int f = 0; f < 3; ++f) {
    po.Uc[i + f * KyKx] = cmk(0.5 * (a[f].x + b[f].x), 0.5 * (a[f].y - b[f].y));
    const double dx = a[f].x - b[f].x, dy = a[f].y + b[f].y;
    dmax[f] = nanmax(fma(dx, dx, dy * dy), dmax[f]);
  }
}

__device__ __forceinline__ void pack_stats_flush(const PackOut& po, double (&dmax)[3]) {
#pragma unroll
  for (int f = 0; f < 3; ++f) {
    double m = dmax[f];
#pragma unroll
    for (int o = 16; o; o >>= 1) m = nanmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0 && m != 0.0)
      atomicMax(reinterpret_cast<unsigned long long*>(po.hstat + f), (unsigned long long)__double_as_longlong(m));
  }
}

__device__ __forceinline__ int mirror_ix(const GridDev& G, int ix) { return (G.nx - ix) % G.nx; }
__device__ __forceinline__ int mirror_jy(const GridDev& G, int jy) { return (G.ny - jy) % G.ny; }

// The stage kernels start under programmatic dependent launch while the
// RHS's last kernel (the slot reduction) still runs: everything that does
// not depend on that RHS -- the loads of the step's states and the
// exponentials applied to them -- is done before the wait, only the part that
// reads the tendency Ac after it (small grids, where a stage kernel is one
// latency chain per thread: ~1 us of that chain moves under the reduction).
// stage_wait: once per thread, at block-uniform points only.
__device__ __forceinline__ void stage_wait(bool& waited, const HermGate& hg) {
  if (waited) return;
  griddep_wait();
  waited = true;
  if (hg.bit >= 0 && blockIdx.x == 0) herm_eval_block(hg);
}

// stage 1 (integrator.py:96-98): e_dt = E(dt) U;  u1 = e_dt + dt * E(dt) A(U)
__global__ void stage1_kernel(GridDev G, Prop pr, double dt, Full3 U, const double2* __restrict__ Ac,
                              Full3w edt, Full3w u1, int* flags, int W, size_t ws,
                              HermGate hg, PackOut po) {
  griddep_launch();
  bool waited = false;
  const size_t n = (size_t)G.nx * G.ny, N = (size_t)W * n, cs = 3 * (size_t)G.Ky * G.Kx;
  double dmax[3] = {0.0, 0.0, 0.0};
  for (size_t i0 = blockIdx.x * (size_t)blockDim.x; i0 < N; i0 += (size_t)gridDim.x * blockDim.x) {
    const size_t t = i0 + threadIdx.x;
    C3 o = c3zero(), e = c3zero(), em = c3zero();
    size_t win = 0, i = 0;
    int ix = 0, jy = 0, j = 0, r = 0, mx = 0, my = 0;
    double kx = 0.0, ky = 0.0, kxm = 0.0, kym = 0.0;
    double2 cd = czero();
    bool pk = false;
    if (t < N) {  // before the wait: E(dt) U at this mode and, for a packed mode, at its mirror
      win = t / n, i = t - win * n;
      ix = (int)(i / G.ny), jy = (int)(i % G.ny);
      kx = G.kxf[ix], ky = G.kyf[jy];
      const Full3 Uw = wshift(U, win * ws);
      cd = pr.kind == 0 ? c12_of(G.ph, kx, ky, dt) : czero();  // this mode and its mirror
      e = expLc(cd, dt, ld3(Uw, i), G.ph, kx, ky, pr);
      pk = po.Uc && packed_mode(G, ix, jy, j, r);
      if (pk) {
        mx = mirror_ix(G, ix), my = mirror_jy(G, jy);
        kxm = G.kxf[mx], kym = G.kyf[my];
        em = expLc(cd, dt, ld3(Uw, (size_t)mx * G.ny + my), G.ph, kxm, kym, pr);
      }
    }
    stage_wait(waited, hg);
    if (t < N) {
      const C3 ea = expLc(cd, dt, compact_at(G, Ac + win * cs, ix, jy), G.ph, kx, ky, pr);
      o = c3add(e, c3scale(dt, ea));
      st3(wshift(edt, win * ws), i, e);
      st3(wshift(u1, win * ws), i, o);
      if (pk) {  // u1 at -k too: the packed input of RHS 2
        const C3 om = c3add(em, c3scale(dt, expLc(cd, dt, compact_at(G, Ac + win * cs, mx, my), G.ph, kxm, kym, pr)));
        pack_store(G, po, win * cs, j, r, o, om, dmax);
      }
    }
    flag_nonfinite(o, 1, flags);
  }
  stage_wait(waited, hg);
  if (po.Uc) pack_stats_flush(po, dmax);
}

// stage 2 (integrator.py:99-100): u2 = 3/4 E(dt/2) U + 1/4 E(-dt/2) (u1 + dt A(u1))
__global__ void stage2_kernel(GridDev G, Prop pr, double dt, Full3 U, Full3 u1, const double2* __restrict__ Ac,
                              Full3w u2, int* flags, int W, size_t ws,
                              HermGate hg, PackOut po) {
  griddep_launch();
  bool waited = false;
  const size_t n = (size_t)G.nx * G.ny, N = (size_t)W * n, cs = 3 * (size_t)G.Ky * G.Kx;
  const double h = 0.5 * dt;
  double dmax[3] = {0.0, 0.0, 0.0};
  for (size_t i0 = blockIdx.x * (size_t)blockDim.x; i0 < N; i0 += (size_t)gridDim.x * blockDim.x) {
    const size_t t = i0 + threadIdx.x;
    C3 o = c3zero(), a = c3zero(), am = c3zero(), y1 = c3zero(), y1m = c3zero();
    size_t win = 0, i = 0;
    int ix = 0, jy = 0, j = 0, r = 0, mx = 0, my = 0;
    double kx = 0.0, ky = 0.0, kxm = 0.0, kym = 0.0;
    double2 cm = czero();
    bool pk = false;
    if (t < N) {  // before the wait: E(dt/2) U and the load of u1, at this mode and its mirror
      win = t / n, i = t - win * n;
      ix = (int)(i / G.ny), jy = (int)(i % G.ny);
      kx = G.kxf[ix], ky = G.kyf[jy];
      const Full3 Uw = wshift(U, win * ws), u1w = wshift(u1, win * ws);
      const double2 ch = pr.kind == 0 ? c12_of(G.ph, kx, ky, h) : czero();
      cm = cmk(-ch.x, ch.y);  // +-dt/2
      a = expLc(ch, h, ld3(Uw, i), G.ph, kx, ky, pr);
      y1 = ld3(u1w, i);
      pk = po.Uc && packed_mode(G, ix, jy, j, r);
      if (pk) {
        mx = mirror_ix(G, ix), my = mirror_jy(G, jy);
        const size_t im = (size_t)mx * G.ny + my;
        kxm = G.kxf[mx], kym = G.kyf[my];
        am = expLc(ch, h, ld3(Uw, im), G.ph, kxm, kym, pr);
        y1m = ld3(u1w, im);
      }
    }
    stage_wait(waited, hg);
    if (t < N) {
      const C3 y = c3add(y1, c3scale(dt, compact_at(G, Ac + win * cs, ix, jy)));
      const C3 b = expLc(cm, -h, y, G.ph, kx, ky, pr);
      o = c3add(c3scale(0.75, a), c3scale(0.25, b));
      st3(wshift(u2, win * ws), i, o);
      if (pk) {  // u2 at -k too: the packed input of RHS 3
        const C3 ym = c3add(y1m, c3scale(dt, compact_at(G, Ac + win * cs, mx, my)));
        const C3 om = c3add(c3scale(0.75, am), c3scale(0.25, expLc(cm, -h, ym, G.ph, kxm, kym, pr)));
        pack_store(G, po, win * cs, j, r, o, om, dmax);
      }
    }
    flag_nonfinite(o, 2, flags);
  }
  stage_wait(waited, hg);
  if (po.Uc) pack_stats_flush(po, dmax);
}

// stage 3 (integrator.py:101-102): out = 1/3 e_dt + 2/3 E(dt/2) (u2 + dt A(u2))
__global__ void stage3_kernel(GridDev G, Prop pr, double dt, Full3 edt, Full3 u2, const double2* __restrict__ Ac,
                              Full3w out, int* flags, int W, size_t ws,
                              HermGate hg) {
  griddep_launch();
  bool waited = false;
  const size_t n = (size_t)G.nx * G.ny, N = (size_t)W * n, cs = 3 * (size_t)G.Ky * G.Kx;
  const double h = 0.5 * dt;
  for (size_t i0 = blockIdx.x * (size_t)blockDim.x; i0 < N; i0 += (size_t)gridDim.x * blockDim.x) {
    const size_t t = i0 + threadIdx.x;
    C3 o = c3zero(), y2 = c3zero(), ed = c3zero();
    size_t win = 0, i = 0;
    int ix = 0, jy = 0;
    double kx = 0.0, ky = 0.0;
    if (t < N) {  // before the wait: the loads of u2 and e_dt
      win = t / n, i = t - win * n;
      ix = (int)(i / G.ny), jy = (int)(i % G.ny);
      kx = G.kxf[ix], ky = G.kyf[jy];
      y2 = ld3(wshift(u2, win * ws), i);
      ed = ld3(wshift(edt, win * ws), i);
    }
    stage_wait(waited, hg);
    if (t < N) {
      const C3 y = c3add(y2, c3scale(dt, compact_at(G, Ac + win * cs, ix, jy)));
      const C3 b = expL(h, y, G.ph, kx, ky, pr);
      o = c3add(c3scale(1.0 / 3.0, ed), c3scale(2.0 / 3.0, b));
      st3(wshift(out, win * ws), i, o);
    }
    flag_nonfinite(o, 3, flags);
  }
  stage_wait(waited, hg);
}

// phase table (c1, c2)[p][j][r] of the exact exponential for every live phase
// and compact mode, evaluated with the reference's formula
// (propagator.py:100-103): c1 = sin(w s)/w, c2 = (1 - cos w s)/w^2.
__global__ void phase_table_kernel(GridDev G, const double* __restrict__ s, int P, double2* __restrict__ tab) {
  const size_t KyKx = (size_t)G.Ky * G.Kx, n = (size_t)P * KyKx;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int p = (int)(i / KyKx);
    const int rem = (int)(i % KyKx);
    const int j = rem / G.Kx, r = rem % G.Kx;
    const double om = omega_of(G.ph, G.kxc[r], G.kyc[j]);
    const double t = s[p];
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
    tab[i] = cmk(c1, c2);
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

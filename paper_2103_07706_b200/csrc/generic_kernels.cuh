// Any even grid size: the passes A / B / C, the snapshot C2R and their FFTs
// for lengths the warp FFT (wfft.cuh: 16 x T points, powers of two up to 512)
// does not cover -- the reference accepts every even n >= 8 (grid.py:91-93;
// its own tests use 12^2, e.g. tests/test_grid.py:49-50) and refinement 8
// means 1024^2.
//
// Same data layouts and the same pass structure as pswe_kernels.cuh (the
// host orchestration -- chunks, lanes, slots, ordered reduction, gate -- is
// shared), but every transform is one CTA-cooperative mixed-radix Stockham
// FFT in shared memory: radices 16, 8, 4, 2 as register DFTs, a direct DFT
// for the odd prime factors, twiddles read from the exact W_n^k table (twiddle_kernel).
// These kernels trade speed for generality; the power-of-two sizes keep the
// tuned kernels.
#pragma once
#include "herm_kernels.cuh"

namespace pswe {

constexpr int GEN_MAX_FACTORS = 24;
constexpr int GEN_THREADS = 256;

// radix plan of one transform length (host-built)
struct FftPlan {
  int n;
  int nf;
  int f[GEN_MAX_FACTORS];
  const double2* tw;  // W_n^k = e^{-2 pi i k / n}, k = 0..n-1
};

// W_n^e for 0 <= e < n (every caller's exponent is already reduced: the
// stage twiddle r k n / (Ns R) < n, the DFT_R twiddle ((q r) mod R) n / R < n)
__device__ __forceinline__ double2 twp(const FftPlan& pl, long long e, bool inv) {
  double2 w = __ldg(pl.tw + (int)e);
  if (inv) w.y = -w.y;
  return w;
}

// One Stockham butterfly of compile-time radix R (register DFT): inputs
// x[j + r m] twiddled by W^{r k n / (Ns R)}, outputs y[base + q Ns].
template <int R, bool INV>
__device__ __forceinline__ void gen_bfly(const double2* x, double2* y, const FftPlan& pl, int j, int m, int Ns) {
  const int n = pl.n, k = j % Ns;
  double2 v[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    double2 z = x[j + r * m];
    if (r) z = cmul(z, twp(pl, (long long)r * k * (n / (Ns * R)), INV));
    v[r] = z;
  }
  if constexpr (R == 2) {
    dft2<INV>(v[0], v[1]);
  } else if constexpr (R == 4) {
    dft4<INV>(v[0], v[1], v[2], v[3]);
  } else if constexpr (R == 8) {
    dft8<INV>(v);
  } else {
    dft16<INV>(v);
  }
  const int base = (j / Ns) * Ns * R + k;
#pragma unroll
  for (int q = 0; q < R; ++q) y[base + q * Ns] = v[q];
}

// CTA-cooperative Stockham FFT of `a` (length pl.n, shared memory) with
// scratch `b`; the result ends in the returned buffer (a or b).  All
// threads of the CTA must call it.  INV: unnormalised e^{+...}.
template <bool INV>
__device__ double2* gen_fft(double2* a, double2* b, const FftPlan& pl) {
  const int n = pl.n;
  int Ns = 1;
  double2 *x = a, *y = b;
  for (int s = 0; s < pl.nf; ++s) {
    const int R = pl.f[s];
    const int m = n / R;
    for (int j = threadIdx.x; j < m; j += blockDim.x) {
      switch (R) {
        case 16: gen_bfly<16, INV>(x, y, pl, j, m, Ns); break;
        case 8: gen_bfly<8, INV>(x, y, pl, j, m, Ns); break;
        case 4: gen_bfly<4, INV>(x, y, pl, j, m, Ns); break;
        case 2: gen_bfly<2, INV>(x, y, pl, j, m, Ns); break;
        default: {
          // odd prime radix: direct DFT_R with table twiddles W_R^{qr} = W_n^{qr n/R}
          const int k = j % Ns, base = (j / Ns) * Ns * R + k;
          for (int q = 0; q < R; ++q) {
            double2 acc = czero();
            for (int r = 0; r < R; ++r) {
              double2 z = x[j + r * m];
              if (r) z = cmul(z, twp(pl, (long long)r * k * (n / (Ns * R)), INV));
              acc = r ? cfma(twp(pl, (long long)((q * r) % R) * (n / R), INV), z, acc) : z;
            }
            y[base + q * Ns] = acc;
          }
        }
      }
    }
    __syncthreads();
    double2* t = x;
    x = y;
    y = t;
    Ns *= R;
  }
  return x;
}

// e^{sL} U of one compact mode (phase table or route), as pass A
__device__ __forceinline__ C3 gen_exp(const GridDev& G, const Prop& pr, const double2* ctab, size_t tidx, double s,
                                      const C3& q, double kx, double ky) {
  return ctab ? exp_c12(ctab[tidx], q, G.ph, kx, ky) : expL(s, q, G.ph, kx, ky, pr);
}

// ---------------------------------------------------------------- pass A
// CTA = (phase pl of the chunk, ky column j): e^{s L} per mode of the
// column, then the 5 inverse x-FFTs into I1[pl][f][j][x].
// smem: E [3][Kx] | a [nx] | b [nx]
__global__ void __launch_bounds__(GEN_THREADS)
    gen_passA_kernel(GridDev G, Prop pr, PhaseDev ph, int p0, int np, const double2* __restrict__ Uc,
                     const double2* __restrict__ ctab, double2* __restrict__ I, FftPlan plx,
                     double* __restrict__ pscale) {
  griddep_wait();
  griddep_launch();
  extern __shared__ __align__(16) unsigned char sbytes[];
  const int nx = G.nx, Kx = G.Kx, Ky = G.Ky;
  double2* E = reinterpret_cast<double2*>(sbytes);
  double2* a = E + 3 * Kx;
  double2* b = a + nx;
  __shared__ double wmax[GEN_THREADS / 32];
  const int pl = blockIdx.x / Ky, j = blockIdx.x % Ky;
  const int p = p0 + pl;
  const size_t KyKx = (size_t)Ky * Kx;
  const double2* U = Uc + (ph.win ? (size_t)ph.win[p] * ph.ustride : 0);
  const double ky = G.kyc[j];
  double gmax = 0.0;
  for (int r = threadIdx.x; r < Kx; r += blockDim.x) {
    const size_t i = (size_t)j * Kx + r;
    const C3 q0 = {U[i], U[KyKx + i], U[2 * KyKx + i]};
    const C3 q = gen_exp(G, pr, ctab, (size_t)p * KyKx + i, ph.s[p], q0, G.kxc[r], ky);
    const double2 dep = csub(q.e, G.bc[i]);
    E[r] = cscale(G.inv_n2, q.u);
    E[Kx + r] = cscale(G.inv_n2, q.v);
    E[2 * Kx + r] = cscale(G.inv_n2, dep);
    gmax = nanmax(gmax, nanmax(nanmax(abs2(q.u), abs2(q.v)), abs2(dep)));
  }
  if (pscale) {
    for (int o = 16; o; o >>= 1) gmax = nanmax(gmax, __shfl_xor_sync(0xffffffffu, gmax, o));
    if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = gmax;
  }
  __syncthreads();
  if (pscale && threadIdx.x == 0) {
    double m = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) m = nanmax(m, wmax[w]);
    atomicMax(reinterpret_cast<unsigned long long*>(pscale + p), (unsigned long long)__double_as_longlong(m));
  }
  for (int f = 0; f < 5; ++f) {
    const int fi = f < 3 ? f : f - 3;
    for (int x = threadIdx.x; x < nx; x += blockDim.x) {
      const int r = band_r(x, nx, G.kxm, Kx);
      double2 v = r >= 0 ? E[fi * Kx + r] : czero();
      if (f >= 3 && r >= 0) v = cik(G.kxc[r], v);
      a[x] = v;
    }
    __syncthreads();
    const double2* o = gen_fft<true>(a, b, plx);
    double2* dst = I + (((size_t)pl * 5 + f) * Ky + j) * nx;
    for (int x = threadIdx.x; x < nx; x += blockDim.x) dst[x] = o[x];
    __syncthreads();
  }
}

// ---------------------------------------------------------------- pass B
// CTA = (phase pl, physical row x): y-C2R of the dimension-matched pairs
// (u, v), (ux, i ky u), (vx, i ky v), (depth, -), the products, y-R2C of
// (A + iB), (C + iD); ky >= 0 half of both into I2[pl][f][j][x].
// smem: Zs [4][ny] physical pairs | a [ny] | b [ny]
__global__ void __launch_bounds__(GEN_THREADS)
    gen_passB_kernel(GridDev G, int np, const double2* __restrict__ I1, double2* __restrict__ I2, FftPlan ply) {
  griddep_wait();
  griddep_launch();
  extern __shared__ __align__(16) unsigned char sbytes[];
  const int nx = G.nx, ny = G.ny, Ky = G.Ky, kym = G.kym;
  double2* Z = reinterpret_cast<double2*>(sbytes);  // [4][ny]
  double2* a = Z + 4 * ny;
  double2* b = a + ny;
  const int pl = blockIdx.x / nx, x = blockIdx.x % nx;
  const size_t fs = (size_t)Ky * nx;  // one field of I1 / I2 for one phase
  const double2* in = I1 + (size_t)pl * 5 * fs + x;
  const int fa[4] = {0, 3, 4, 2}, fb[4] = {1, 0, 1, -1};
  for (int it = 0; it < 4; ++it) {
    for (int k = threadIdx.x; k < ny; k += blockDim.x) {
      const bool lo = k <= kym;
      if (!lo && k < ny - kym) {
        a[k] = czero();
        continue;
      }
      const int jj = lo ? k : ny - k;
      const double2 A = in[(size_t)fa[it] * fs + (size_t)jj * nx];
      double2 B = czero();
      if (fb[it] >= 0) {
        B = in[(size_t)fb[it] * fs + (size_t)jj * nx];
        if (it == 1 || it == 2) B = cik(G.kyc[jj], B);
      }
      if (k == 0)
        a[k] = cmk(A.x, B.x);  // Hermitian projection of the y-mean bin
      else
        a[k] = lo ? cmk(A.x - B.y, A.y + B.x) : cmk(A.x + B.y, B.x - A.y);
    }
    __syncthreads();
    const double2* o = gen_fft<true>(a, b, ply);
    for (int y = threadIdx.x; y < ny; y += blockDim.x) Z[(size_t)it * ny + y] = o[y];
    __syncthreads();
  }
  double2* out = I2 + (size_t)pl * 4 * fs + x;
  for (int pass = 0; pass < 2; ++pass) {
    for (int y = threadIdx.x; y < ny; y += blockDim.x) {
      const double2 q = Z[y];  // (u, v)
      if (pass == 0) {
        const double2 ux = Z[ny + y], vx = Z[2 * ny + y];
        a[y] = cmk(-(q.x * ux.x + q.y * ux.y), -(q.x * vx.x + q.y * vx.y));  // A + iB
      } else {
        const double d = Z[3 * ny + y].x;
        a[y] = cmk(q.x * d, q.y * d);  // C + iD
      }
    }
    __syncthreads();
    const double2* o = gen_fft<false>(a, b, ply);
    for (int j = threadIdx.x; j < Ky; j += blockDim.x) {
      const double2 z = o[j], zm = o[(ny - j) % ny];
      out[(size_t)(2 * pass) * fs + (size_t)j * nx] = cmk(0.5 * (z.x + zm.x), 0.5 * (z.y - zm.y));
      out[(size_t)(2 * pass + 1) * fs + (size_t)j * nx] = cmk(0.5 * (z.y + zm.y), -0.5 * (z.x - zm.x));
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- pass C
// CTA = (ky column j, phase group g of the chunk): per phase, the forward
// x-FFTs of the 4 product columns, 2/3 truncation, flux divergence, e^{-sL},
// weight, accumulated in shared memory; slot g (+)= the group's sum (window
// batches: flushed per window into zeroed slots).
// smem: F [4][Kx] | acc [3][Kx] | a [nx] | b [nx]
template <bool MW>
__global__ void __launch_bounds__(GEN_THREADS)
    gen_passC_kernel(GridDev G, Prop pr, PhaseDev ph, int p0, int np, int Gc, const double2* __restrict__ I2,
                     const double2* __restrict__ ctab, double2* __restrict__ slots, int first_chunk, FftPlan plx) {
  griddep_wait();
  griddep_launch();
  extern __shared__ __align__(16) unsigned char sbytes[];
  const int nx = G.nx, Kx = G.Kx, Ky = G.Ky;
  double2* F = reinterpret_cast<double2*>(sbytes);
  double2* acc = F + 4 * Kx;
  double2* a = acc + 3 * Kx;
  double2* b = a + nx;
  const int j = blockIdx.x % Ky, g = blockIdx.x / Ky;
  const int lo = (int)(((long long)g * np) / Gc), hi = (int)(((long long)(g + 1) * np) / Gc);
  const size_t KyKx = (size_t)Ky * Kx, fs = (size_t)Ky * nx;
  const double ky = G.kyc[j];
  auto flush = [&](int win, bool add) {
    double2* slot = slots + ((size_t)g * ph.W + win) * 3 * KyKx + (size_t)j * Kx;
    for (int r = threadIdx.x; r < Kx; r += blockDim.x)
      for (int f = 0; f < 3; ++f) {
        const double2 v = acc[f * Kx + r];
        slot[f * KyKx + r] = add ? cadd(slot[f * KyKx + r], v) : v;
      }
  };
  for (int r = threadIdx.x; r < 3 * Kx; r += blockDim.x) acc[r] = czero();
  int wcur = MW && lo < hi ? ph.win[p0 + lo] : 0;
  for (int pl = lo; pl < hi; ++pl) {
    const int p = p0 + pl;
    if (MW && ph.win[p] != wcur) {
      __syncthreads();
      flush(wcur, true);
      __syncthreads();
      for (int r = threadIdx.x; r < 3 * Kx; r += blockDim.x) acc[r] = czero();
      wcur = ph.win[p];
    }
    for (int f = 0; f < 4; ++f) {
      const double2* src = I2 + ((size_t)pl * 4 + f) * fs + (size_t)j * nx;
      for (int x = threadIdx.x; x < nx; x += blockDim.x) a[x] = src[x];
      __syncthreads();
      const double2* o = gen_fft<false>(a, b, plx);
      for (int r = threadIdx.x; r < Kx; r += blockDim.x) {
        const int w = r <= G.kxm ? r : r - Kx;
        F[f * Kx + r] = o[(w + nx) % nx];
      }
      __syncthreads();
    }
    const double s = ph.s[p], w = ph.w[p];
    for (int r = threadIdx.x; r < Kx; r += blockDim.x) {
      const double kx = G.kxc[r];
      const double2 gx = cik(kx, F[2 * Kx + r]), gy = cik(ky, F[3 * Kx + r]);
      C3 q = {F[r], F[Kx + r], cmk(-(gx.x + gy.x), -(gx.y + gy.y))};
      if (ctab) {
        double2 c12 = ctab[(size_t)p * KyKx + (size_t)j * Kx + r];
        c12.x = -c12.x;
        q = exp_c12(c12, q, G.ph, kx, ky);
      } else {
        q = expL(-s, q, G.ph, kx, ky, pr);
      }
      acc[r] = cadd(acc[r], cscale(w, q.u));
      acc[Kx + r] = cadd(acc[Kx + r], cscale(w, q.v));
      acc[2 * Kx + r] = cadd(acc[2 * Kx + r], cscale(w, q.e));
    }
    __syncthreads();
  }
  __syncthreads();
  if (MW) {
    if (lo < hi) flush(wcur, true);
  } else {
    flush(0, !first_chunk);
  }
}

// ---------------------------------------------------------------- snapshot C2R
// as diag_cols / diag_rows (diag_kernels.cuh) for any even size.
// columns: CTA = (field f, column j <= ny/2): Hermitian projection + inverse
// x-FFT, scaled -> D[f][j][x]
__global__ void __launch_bounds__(GEN_THREADS)
    gen_diag_cols_kernel(GridDev G, const double2* __restrict__ u, const double2* __restrict__ v,
                         const double2* __restrict__ e, const double2* __restrict__ bt, double2* __restrict__ D,
                         FftPlan plx) {
  extern __shared__ __align__(16) unsigned char sbytes[];
  const int nx = G.nx, ny = G.ny, nyh = ny / 2 + 1;
  double2* a = reinterpret_cast<double2*>(sbytes);
  double2* b = a + nx;
  const int f = blockIdx.x / nyh, j = blockIdx.x % nyh;
  const double2* c = f == 0 ? u : (f == 1 ? v : (f == 2 ? e : bt));
  const int jm = (ny - j) % ny;
  for (int ix = threadIdx.x; ix < nx; ix += blockDim.x) {
    const int im = (nx - ix) % nx;
    const double2 p = c[(size_t)ix * ny + j], m = c[(size_t)im * ny + jm];
    a[ix] = cmk(0.5 * (p.x + m.x), 0.5 * (p.y - m.y));
  }
  __syncthreads();
  const double2* o = gen_fft<true>(a, b, plx);
  double2* dst = D + ((size_t)f * nyh + j) * nx;
  for (int x = threadIdx.x; x < nx; x += blockDim.x) dst[x] = cscale(G.inv_n2, o[x]);
}

// rows: CTA = physical row x: y-C2R of (u, v) and (eta, b), the pointwise
// energy / depth / speed^2 and their row sums in a fixed order -> part[x][3];
// phys (optional): [3][nx][ny] physical u, v, eta
__global__ void __launch_bounds__(GEN_THREADS)
    gen_diag_rows_kernel(GridDev G, const double2* __restrict__ D, double H, double grav, double* __restrict__ part,
                         double* __restrict__ phys, FftPlan ply) {
  extern __shared__ __align__(16) unsigned char sbytes[];
  const int nx = G.nx, ny = G.ny, nyh = ny / 2 + 1;
  double2* Z = reinterpret_cast<double2*>(sbytes);  // [2][ny]
  double2* a = Z + 2 * ny;
  double2* b = a + ny;
  __shared__ double red[3][GEN_THREADS];
  const int x = blockIdx.x;
  for (int pr = 0; pr < 2; ++pr) {
    const int fa = 2 * pr, fb = 2 * pr + 1;
    for (int k = threadIdx.x; k < ny; k += blockDim.x) {
      const bool lo = k <= ny / 2;
      const int kk = lo ? k : ny - k;
      double2 A = D[((size_t)fa * nyh + kk) * nx + x], B = D[((size_t)fb * nyh + kk) * nx + x];
      if (kk == 0 || kk == ny / 2) {
        A.y = 0.0;
        B.y = 0.0;
      }
      if (!lo) {
        A.y = -A.y;
        B.y = -B.y;
      }
      a[k] = cmk(A.x - B.y, A.y + B.x);
    }
    __syncthreads();
    const double2* o = gen_fft<true>(a, b, ply);
    for (int y = threadIdx.x; y < ny; y += blockDim.x) Z[(size_t)pr * ny + y] = o[y];
    __syncthreads();
  }
  double se = 0.0, sm = 0.0, vmax = 0.0;
  for (int y = threadIdx.x; y < ny; y += blockDim.x) {
    const double uu = Z[y].x, vv = Z[y].y, eta = Z[ny + y].x, bb = Z[ny + y].y;
    if (phys) {
      const size_t nxy = (size_t)nx * ny;
      phys[(size_t)x * ny + y] = uu;
      phys[nxy + (size_t)x * ny + y] = vv;
      phys[2 * nxy + (size_t)x * ny + y] = eta;
    }
    const double depth = H + eta - bb;
    const double s2 = uu * uu + vv * vv;
    se += 0.5 * depth * s2 + 0.5 * grav * eta * (eta + 2.0 * H);
    sm += depth;
    vmax = fmax(vmax, s2);
  }
  red[0][threadIdx.x] = se;
  red[1][threadIdx.x] = sm;
  red[2][threadIdx.x] = vmax;
  __syncthreads();
  if (threadIdx.x == 0) {  // fixed order: deterministic
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    for (int i = 0; i < (int)blockDim.x; ++i) {
      a0 += red[0][i];
      a1 += red[1][i];
      a2 = fmax(a2, red[2][i]);
    }
    part[3 * (size_t)x + 0] = a0;
    part[3 * (size_t)x + 1] = a1;
    part[3 * (size_t)x + 2] = a2;
  }
}

}  // namespace pswe

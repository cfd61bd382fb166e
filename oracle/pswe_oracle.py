"""CPU oracle for the phase-averaged RHS of arXiv 2103.07706 (reference ``phaseswe``).

TEST INFRASTRUCTURE ONLY.  This module is the checker, never the product:
only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg (``--impl reference`` / ``cpu_baseline``) may import it.  The shipped
package ``paper_2103_07706_b200`` never imports anything under ``oracle/``.

What it is: an independent numpy restatement of the reference's hot path
(``/root/reference/pkg/src/phaseswe``), written on plain arrays instead of the
reference's dataclasses.  A state is one complex128 array ``U`` of shape
``(3, nx, ny)`` holding the spectral coefficients of (u, v, eta) in
unnormalised ``numpy.fft.fft2`` layout (grid.py:3-8).  Every function cites
the reference file:line it follows.

Third-party arithmetic the reference relies on (not vendored in the
reference tree): ``numpy.fft.fft2/ifft2`` (pocketfft,
numpy 2.3.5 here, ``numpy>=1.24`` in pkg/pyproject.toml:11) and
``scipy.fft.dct`` type II (scipy 1.18.1 here, ``scipy>=1.10`` in
pkg/pyproject.toml:12).  The oracle calls the same numpy FFT.

Parity pinning: ``tests/test_oracle_golden.py`` checks this oracle against
golden vectors produced by the real reference (``oracle/make_golden.py``,
fixtures in ``tests/golden/``) and against the reference's own known-answer
values.
"""

from __future__ import annotations

import math
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import scipy.fft

# --------------------------------------------------------------------------
# grid  (grid.py)
# --------------------------------------------------------------------------


def wrap(n: int) -> np.ndarray:
    """Signed FFT index order 0..n/2-1, -n/2..-1 (grid.py:76-78)."""
    return np.fft.fftfreq(n, d=1.0 / n).astype(int)


def wavenumbers(nx: int, ny: int, Lx: float, Ly: float):
    """kx, ky exactly as make_grid computes them (grid.py:98-101)."""
    kx = 2.0 * np.pi * wrap(nx) / Lx
    ky = 2.0 * np.pi * wrap(ny) / Ly
    return kx, ky


def band_mask(nx: int, ny: int) -> np.ndarray:
    """2/3-rule mask, |wrap| <= n/3 per axis in integer arithmetic (grid.py:102-103)."""
    return (3 * np.abs(wrap(nx))[:, None] <= nx) & (3 * np.abs(wrap(ny))[None, :] <= ny)


def truncate(c: np.ndarray, mask: np.ndarray) -> np.ndarray:
    """dealias: zero every mode outside the band (grid.py:183-187)."""
    return np.where(mask, c, 0.0)


def real_field(c: np.ndarray) -> np.ndarray:
    """to_physical without its validation gate: real part of ifft2 (grid.py:173-174)."""
    return np.fft.ifft2(c).real


def spectral(f: np.ndarray) -> np.ndarray:
    """to_spectral: unnormalised fft2 of a real field (grid.py:116-122)."""
    return np.fft.fft2(np.asarray(f, dtype=np.float64))


# --------------------------------------------------------------------------
# physics  (dynamics.py)
# --------------------------------------------------------------------------


class Setup:
    """Grid + physics constants bundle used by every oracle routine.

    Mirrors SpectralGrid (grid.py:34-73) and PhysicsParams (dynamics.py:34-63).
    ``b`` is the (nx, ny) spectral topography.
    """

    def __init__(self, nx, ny, Lx, Ly, f, g, H, b=None):
        self.nx, self.ny, self.Lx, self.Ly = int(nx), int(ny), float(Lx), float(Ly)
        self.f, self.g, self.H = float(f), float(g), float(H)
        self.kx, self.ky = wavenumbers(nx, ny, Lx, Ly)
        self.mask = band_mask(nx, ny)
        self.b = (np.zeros((nx, ny), complex) if b is None
                  else np.asarray(b, dtype=np.complex128))
        self.KX = self.kx[:, None]
        self.KY = self.ky[None, :]

    def omega(self) -> np.ndarray:
        """Dispersion relation per mode (dynamics.py:179-186)."""
        return np.sqrt(self.f ** 2 + self.g * self.H * (self.KX ** 2 + self.KY ** 2))

    def max_frequency(self) -> float:
        """max omega over the grid (dynamics.py:189-192)."""
        return float(np.max(self.omega()))


def linear(S: Setup, U: np.ndarray) -> np.ndarray:
    """L U per mode (dynamics.py:128-136)."""
    u, v, eta = U
    ikx, iky = 1j * S.KX, 1j * S.KY
    return np.stack([S.f * v - S.g * (ikx * eta),
                     -S.f * u - S.g * (iky * eta),
                     -S.H * (ikx * u + iky * v)])


def nonlinear(S: Setup, U: np.ndarray) -> np.ndarray:
    """N(U): pseudo-spectral advection + flux divergence, 2/3-dealiased (dynamics.py:139-176)."""
    ikx, iky = 1j * S.KX, 1j * S.KY
    cu, cv, ceta = (truncate(c, S.mask) for c in U)
    cb = truncate(S.b, S.mask)
    u, v, depth = real_field(cu), real_field(cv), real_field(ceta - cb)
    ux, uy = real_field(ikx * cu), real_field(iky * cu)
    vx, vy = real_field(ikx * cv), real_field(iky * cv)
    du = truncate(spectral(-(u * ux + v * uy)), S.mask)
    dv = truncate(spectral(-(u * vx + v * vy)), S.mask)
    fx, fy = spectral(u * depth), spectral(v * depth)
    deta = truncate(-(ikx * fx + iky * fy), S.mask)
    return np.stack([du, dv, deta])


# --------------------------------------------------------------------------
# exponentials  (propagator.py)
# --------------------------------------------------------------------------


def exact_exp(S: Setup, t: float, U: np.ndarray) -> np.ndarray:
    """e^{tL} U = U + c1 L U + c2 L^2 U per mode, omega -> 0 limit t, t^2/2 (propagator.py:96-110)."""
    om = S.omega()
    pos = om > 0.0
    safe = np.where(pos, om, 1.0)
    c1 = np.where(pos, np.sin(om * t) / safe, t)
    c2 = np.where(pos, (1.0 - np.cos(om * t)) / safe ** 2, 0.5 * t * t)
    lu = linear(S, U)
    llu = linear(S, lu)
    return U + c1 * lu + c2 * llu


def cheb_coeffs(Lambda: float, n_poly: int) -> np.ndarray:
    """Real coefficients a_k = (2 - delta_k0) J_k(Lambda) via a type-II DCT (propagator.py:113-130)."""
    npts = max(64, 2 * (n_poly + 1), int(np.ceil(Lambda)) + 64)
    theta = np.pi * (np.arange(npts) + 0.5) / npts
    h = np.exp(1j * Lambda * np.cos(theta))
    b = (scipy.fft.dct(h.real, type=2) + 1j * scipy.fft.dct(h.imag, type=2)) / npts
    b[0] *= 0.5
    a = ((-1j) ** np.arange(n_poly + 1)) * b[:n_poly + 1]
    return np.ascontiguousarray(a.real)


def choose_npoly(Lambda: float, tol: float = 1e-10) -> int:
    """Smallest degree with every dropped tail coefficient below tol (propagator.py:142-158)."""
    top = int(np.ceil(Lambda + 2.0 * Lambda ** (1.0 / 3.0))) + 60
    a = cheb_coeffs(Lambda, top)
    n = top
    while n >= 1 and abs(a[n]) < tol:
        n -= 1
    return max(n, 1)


def cheb_exp(S: Setup, t: float, U: np.ndarray, Lambda: float, n_poly: int) -> np.ndarray:
    """Chebyshev recurrence Q_{k+1} = (2t/Lambda) L Q_k + Q_{k-1} (propagator.py:161-191)."""
    if t == 0.0:
        return U
    need = abs(t) * S.max_frequency()
    if need > Lambda * (1.0 + 1e-9):
        raise ValueError(f"|t| * max_frequency = {need:.6g} exceeds Lambda = {Lambda:.6g}")
    a = cheb_coeffs(Lambda, n_poly)
    sc = t / Lambda
    q_prev, q = U, sc * linear(S, U)
    acc = a[0] * U + a[1] * q
    for k in range(2, n_poly + 1):
        q_prev, q = q, (2.0 * sc) * linear(S, q) + q_prev
        acc = acc + a[k] * q
    return acc


class Propagator:
    """kind 'exact' or 'chebyshev' (+ Lambda, n_poly), dispatch as propagator.py:194-199."""

    def __init__(self, kind="exact", Lambda=0.0, n_poly=1):
        self.kind, self.Lambda, self.n_poly = kind, float(Lambda), int(n_poly)

    def __call__(self, S: Setup, t: float, U: np.ndarray) -> np.ndarray:
        if self.kind == "exact":
            return exact_exp(S, t, U)
        return cheb_exp(S, t, U, self.Lambda, self.n_poly)


# --------------------------------------------------------------------------
# phase averaging  (averaging.py)
# --------------------------------------------------------------------------


def bump(x: np.ndarray) -> np.ndarray:
    """rho(x) = exp(-1/(1-x^2)) on |x| < 1, else 0 (averaging.py:45-51)."""
    x = np.asarray(x, dtype=np.float64)
    out = np.zeros_like(x)
    inside = np.abs(x) < 1.0
    out[inside] = np.exp(-1.0 / (1.0 - x[inside] ** 2))
    return out


def uniform(x: np.ndarray) -> np.ndarray:
    """Uniform profile on [-1, 1] (averaging.py:55-56)."""
    return np.where(np.abs(np.asarray(x)) <= 1.0, 1.0, 0.0)


def quadrature(T: float, M: int, rho=bump):
    """Nodes s_k = k T / M, k = -M..M, weights rho(s/T) normalised twice to sum 1 (averaging.py:80-106)."""
    if M == 0:
        return np.zeros(1), np.ones(1)
    k = np.arange(-M, M + 1)
    s = k * (T / M)
    r = rho(s / T)
    w = r / float(r.sum())
    return s, w / float(w.sum())


def default_node_count(T: float, lam: float) -> int:
    """max(4, ceil(T lambda_max / pi)) (averaging.py:109-113)."""
    return 0 if T <= 0.0 else max(4, int(np.ceil(T * lam / np.pi)))


def averaged_tendency(S: Setup, U: np.ndarray, s: np.ndarray, w: np.ndarray,
                      prop: Propagator | None = None, workers: int = 1,
                      nodes=None) -> np.ndarray:
    """sum_{w_k != 0} w_k e^{-s_k L} N(e^{s_k L} U), ascending reduction (averaging.py:116-156).

    ``nodes`` optionally restricts the live nodes (used for bounded CPU timing
    samples); the default is every node with nonzero weight (averaging.py:128).
    """
    prop = prop or Propagator()
    live = [i for i in range(len(s)) if w[i] != 0.0] if nodes is None else list(nodes)

    def term(i):
        si = float(s[i])
        if si == 0.0:
            return nonlinear(S, U)
        return prop(S, -si, nonlinear(S, prop(S, si, U)))

    if workers > 1:
        with ThreadPoolExecutor(max_workers=workers) as pool:
            res = list(pool.map(term, live))
    else:
        res = [term(i) for i in live]
    acc = np.zeros_like(U)
    for i, r in zip(live, res):
        acc += w[i] * r
    return acc


# --------------------------------------------------------------------------
# time stepping  (integrator.py)
# --------------------------------------------------------------------------


def ssprk3_step(S: Setup, U: np.ndarray, dt: float, s, w, prop: Propagator | None = None,
                workers: int = 1) -> np.ndarray:
    """Transformed SSPRK3 step: 3 averaged tendencies + 5 exponentials (integrator.py:83-103)."""
    prop = prop or Propagator()

    def E(t, X):
        return prop(S, t, X)

    def A(X):
        return averaged_tendency(S, X, s, w, prop, workers)

    e_dt = E(dt, U)
    u1 = e_dt + dt * E(dt, A(U))
    _finite(u1, 1)
    u2 = 0.75 * E(0.5 * dt, U) + 0.25 * E(-0.5 * dt, u1 + dt * A(u1))
    _finite(u2, 2)
    out = (1.0 / 3.0) * e_dt + (2.0 / 3.0) * E(0.5 * dt, u2 + dt * A(u2))
    _finite(out, 3)
    return out


def _finite(U, stage):
    """_require_finite: first non-finite field per stage (integrator.py:77-80)."""
    for name, c in zip(("u", "v", "eta"), U):
        if not np.all(np.isfinite(c)):
            raise RuntimeError(f"non-finite values in field {name} after stage {stage}")


def run(S: Setup, U: np.ndarray, dt: float, nsteps: int, s, w, prop=None, workers=1):
    """Step loop of integrator.run without snapshot diagnostics (integrator.py:173-179)."""
    for _ in range(nsteps):
        U = ssprk3_step(S, U, dt, s, w, prop, workers)
    return U


# --------------------------------------------------------------------------
# diagnostics used by the parity metrics  (dynamics.py, diagnostics.py)
# --------------------------------------------------------------------------


def energy_inner(S: Setup, A: np.ndarray, B: np.ndarray) -> float:
    """Energy inner product via Parseval (dynamics.py:195-207)."""
    n2 = S.nx * S.ny
    q = S.H * (np.vdot(B[0], A[0]) + np.vdot(B[1], A[1])) + S.g * np.vdot(B[2], A[2])
    return float(np.real(q) * S.Lx * S.Ly / n2 ** 2)


def energy_norm(S: Setup, A: np.ndarray) -> float:
    """sqrt(max(energy_inner(a, a), 0)) (dynamics.py:210-211)."""
    return math.sqrt(max(energy_inner(S, A, A), 0.0))


def rel_l2(got: np.ndarray, want: np.ndarray) -> float:
    """Relative L2 over the concatenated (u, v, eta) coefficients."""
    den = float(np.linalg.norm(want.ravel()))
    return float(np.linalg.norm((got - want).ravel())) / (den if den > 0 else 1.0)


def energy_mass(S: Setup, U: np.ndarray):
    """Total energy and mass from physical fields (diagnostics.py:58-78)."""
    u, v, eta = (real_field(c) for c in U)
    b = real_field(S.b)
    depth = S.H + eta - b
    area = (S.Lx / S.nx) * (S.Ly / S.ny)
    mass = float(np.sum(depth) * area)
    energy = float(np.sum(0.5 * depth * (u ** 2 + v ** 2)
                          + 0.5 * S.g * eta * (eta + 2.0 * S.H)) * area)
    return energy, mass

"""Seeded synthetic inputs for the BASELINE configs C1-C5 (host side).

The BASELINE configs are stated on the sphere (icosahedral refinement
levels, Williamson-5-like flow, an unstable jet); neither the meshes nor the
spherical data exist in the reference or in this container.  Following
SURVEY.md section 8(d), each config is restated on the reference's doubly
periodic f-plane with the same shapes, sizes and amplitudes:

  refinement r -> n = 2^(r+2) grid points per side, Lx = Ly = 2 pi a,
  f0 = 2 Omega sin 45 deg, latitude phi -> y = Ly/2 + a phi,
  longitude lambda -> x = a (lambda + pi), BASELINE window T -> half width T/2.

Fields are built in physical space, transformed, and truncated to the 2/3
band, as testcase.py:72-94 does; balanced eta solves the discrete
geostrophic relation i ky eta = -(f/g) u per mode (testcase.py:89-93).
These are input builders for tests and the benchmark, not part of the GPU
path.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .averaging import _bump, kernel_weights
from .dynamics import PhysicsParams, State
from .grid import dealias, make_grid, to_physical, to_spectral

A_EARTH = 6.371e6
OMEGA = 7.292e-5
G_EARTH = 9.81
L_DOMAIN = 2.0 * math.pi * A_EARTH
F0 = 2.0 * OMEGA * math.sin(math.pi / 4.0)
DAY = 86400.0


@dataclass
class Case:
    name: str
    grid: object
    params: PhysicsParams
    state: State
    T_half: float
    M: int
    dt: float
    nsteps: int

    @property
    def quadrature(self):
        return kernel_weights(self.T_half, self.M)

    @property
    def P(self) -> int:
        return int(np.count_nonzero(self.quadrature.w))

    @property
    def dof(self) -> int:
        return 3 * self.grid.nx * self.grid.ny


def n_of_level(r: int) -> int:
    return 2 ** (r + 2)


def y_of_lat(lat_rad: float) -> float:
    return L_DOMAIN / 2.0 + A_EARTH * lat_rad


def _spec(grid, phys):
    return dealias(grid, to_spectral(grid, np.ascontiguousarray(phys)))


def _zonal(grid, profile_y):
    c = _spec(grid, np.broadcast_to(profile_y[None, :], (grid.nx, grid.ny)))
    c[0, 0] = 0.0  # zero mean velocity (testcase.py:85-87)
    return c


def _balanced_eta(grid, cu, f, g):
    """i ky eta = -(f/g) u per mode, mean eta zero (testcase.py:89-93)."""
    ky = np.broadcast_to(grid.ky[None, :], (grid.nx, grid.ny))
    ceta = np.zeros_like(cu)
    nz = ky != 0.0
    ceta[nz] = -(f / g) * cu[nz] / (1j * ky[nz])
    return ceta


def _cone(grid, b0, r0, xc, yc):
    """Periodic cone b0 (1 - min(r, r0)/r0), dealiased (testcase.py:53-69)."""
    dx = np.abs(grid.x[:, None] - xc)
    dy = np.abs(grid.y[None, :] - yc)
    dx = np.minimum(dx, grid.Lx - dx)
    dy = np.minimum(dy, grid.Ly - dy)
    r = np.hypot(dx, dy)
    return _spec(grid, b0 * (1.0 - np.minimum(r, r0) / r0))


def _frozen(b):
    # read-only topography: the drop-in then skips re-checking it per call
    b = np.array(b, dtype=np.complex128)
    b.setflags(write=False)
    return b


def _flat(grid):
    return _frozen(np.zeros((grid.nx, grid.ny), dtype=np.complex128))


def case_c1() -> Case:
    """C1: r3 -> 32^2, H = 2.94e4/g, solid-body-like zonal flow + 1e-3 eta noise (seed 1)."""
    grid = make_grid(32, 32, L_DOMAIN, L_DOMAIN)
    H = 2.94e4 / G_EARTH
    u0 = 2.0 * math.pi * A_EARTH / (12.0 * DAY)
    cu = _zonal(grid, u0 * np.cos(2.0 * math.pi * (grid.y - grid.Ly / 2.0) / grid.Ly))
    ceta = _balanced_eta(grid, cu, F0, G_EARTH)
    amp = float(np.max(np.abs(to_physical(grid, ceta))))
    rng = np.random.default_rng(1)
    ceta = ceta + _spec(grid, 1e-3 * amp * rng.standard_normal((grid.nx, grid.ny)))
    params = PhysicsParams(f=F0, g=G_EARTH, H=H, b=_flat(grid))
    st = State(grid=grid, u=cu, v=np.zeros_like(cu), eta=ceta, t=0.0)
    return Case("C1", grid, params, st, T_half=1800.0, M=8, dt=3600.0, nsteps=0)


def case_c2() -> Case:
    """C2: r4 -> 64^2, C1 flow + 10 random Fourier modes |(p,q)| <= 8 at 1% of eta (seed 2)."""
    grid = make_grid(64, 64, L_DOMAIN, L_DOMAIN)
    H = 2.94e4 / G_EARTH
    u0 = 2.0 * math.pi * A_EARTH / (12.0 * DAY)
    cu = _zonal(grid, u0 * np.cos(2.0 * math.pi * (grid.y - grid.Ly / 2.0) / grid.Ly))
    ceta = _balanced_eta(grid, cu, F0, G_EARTH)
    amp = float(np.max(np.abs(to_physical(grid, ceta))))
    rng = np.random.default_rng(2)
    # canonical half plane: q > 0, or q == 0 and p > 0 (no conjugate duplicates)
    cands = [(p, q) for p in range(-8, 9) for q in range(0, 9)
             if p * p + q * q <= 64 and (q > 0 or p > 0)]
    pick = rng.choice(len(cands), size=10, replace=False)
    pert = np.zeros((grid.nx, grid.ny), dtype=np.complex128)
    for idx in pick:
        p, q = cands[int(idx)]
        c = rng.standard_normal() + 1j * rng.standard_normal()
        pert[p % grid.nx, q % grid.ny] += c
        pert[(-p) % grid.nx, (-q) % grid.ny] += np.conj(c)
    phys = to_physical(grid, pert)
    pert *= 0.01 * amp / float(np.max(np.abs(phys)))
    params = PhysicsParams(f=F0, g=G_EARTH, H=H, b=_flat(grid))
    st = State(grid=grid, u=cu, v=np.zeros_like(cu), eta=ceta + pert, t=0.0)
    return Case("C2", grid, params, st, T_half=3600.0, M=16, dt=3600.0, nsteps=24)


def case_c3() -> Case:
    """C3: r5 -> 128^2, 20 m/s zonal flow, H = 5960 m, cone mountain at 30N 90W (b0 2000, R = a pi/9)."""
    grid = make_grid(128, 128, L_DOMAIN, L_DOMAIN)
    H = 5960.0
    cu = _zonal(grid, 20.0 * np.cos(2.0 * math.pi * (grid.y - grid.Ly / 2.0) / grid.Ly))
    ceta = _balanced_eta(grid, cu, F0, G_EARTH)
    b = _cone(grid, 2000.0, A_EARTH * math.pi / 9.0, A_EARTH * math.pi / 2.0,
              y_of_lat(math.pi / 6.0))
    params = PhysicsParams(f=F0, g=G_EARTH, H=H, b=_frozen(b))
    st = State(grid=grid, u=cu, v=np.zeros_like(cu), eta=ceta, t=0.0)
    return Case("C3", grid, params, st, T_half=1800.0, M=32, dt=1800.0, nsteps=48)


def case_c4() -> Case:
    """C4: r6 -> 256^2, H = 1e4 m, 80 m/s bump-profile jet 25.7N-64.3N + 120 m eta bump at 45N (seed 4)."""
    grid = make_grid(256, 256, L_DOMAIN, L_DOMAIN)
    H = 1.0e4
    lo, hi = y_of_lat(math.radians(25.7)), y_of_lat(math.radians(64.3))
    mid, half = 0.5 * (lo + hi), 0.5 * (hi - lo)
    prof = 80.0 * _bump((grid.y - mid) / half) / math.exp(-1.0)
    cu = _zonal(grid, prof)
    ceta = _balanced_eta(grid, cu, F0, G_EARTH)
    rng = np.random.default_rng(4)
    xc = float(rng.uniform(0.0, grid.Lx))
    dx = np.abs(grid.x[:, None] - xc)
    dx = np.minimum(dx, grid.Lx - dx)
    yb = y_of_lat(math.radians(45.0))
    bump = (120.0 * np.exp(-((grid.y[None, :] - yb) / (A_EARTH / 3.0)) ** 2)
            * np.exp(-(dx / (A_EARTH / 15.0)) ** 2))
    ceta = ceta + _spec(grid, bump)
    params = PhysicsParams(f=F0, g=G_EARTH, H=H, b=_flat(grid))
    st = State(grid=grid, u=cu, v=np.zeros_like(cu), eta=ceta, t=0.0)
    return Case("C4", grid, params, st, T_half=2700.0, M=64, dt=1200.0, nsteps=72)


def case_c5(r: int, M: int) -> Case:
    """C5 sweep point: r in 4..7, geostrophic random state with |(p,q)| <= 16, max eta = 0.1 H (seed 5+r)."""
    n = n_of_level(r)
    grid = make_grid(n, n, L_DOMAIN, L_DOMAIN)
    H = 2.94e4 / G_EARTH
    rng = np.random.default_rng(5 + r)
    ceta = to_spectral(grid, rng.standard_normal((n, n)))
    w = np.fft.fftfreq(n, d=1.0 / n)
    keep = (w[:, None] ** 2 + w[None, :] ** 2) <= 256.0
    ceta = np.where(keep, ceta, 0.0)
    ceta[0, 0] = 0.0
    ceta *= 0.1 * H / float(np.max(np.abs(to_physical(grid, ceta))))
    kx, ky = grid.kx[:, None], grid.ky[None, :]
    cu = -(G_EARTH / F0) * (1j * ky) * ceta
    cv = (G_EARTH / F0) * (1j * kx) * ceta
    params = PhysicsParams(f=F0, g=G_EARTH, H=H, b=_flat(grid))
    st = State(grid=grid, u=cu, v=cv, eta=ceta, t=0.0)
    return Case(f"C5-r{r}-M{M}", grid, params, st, T_half=1800.0, M=M, dt=3600.0, nsteps=0)


CASES = {"C1": case_c1, "C2": case_c2, "C3": case_c3, "C4": case_c4}

"""State / physics containers and the single-operator entry points.

``State`` and ``PhysicsParams`` mirror phaseswe.dynamics (dynamics.py:34-118)
so the drop-in accepts and returns the same objects; every function here
also accepts the reference's own ``phaseswe`` objects (duck typing on
``.grid``, ``.u``, ``.v``, ``.eta``, ``.t``, ``.f``, ``.g``, ``.H``, ``.b``).

``apply_linear`` and ``apply_nonlinear`` run on the GPU through the C ABI
(``pswe_apply_linear`` / ``pswe_apply_nonlinear``).  ``energy_inner`` /
``energy_norm`` are host-side diagnostics (Parseval sums) used by parity
checks, as in the reference.
"""

from __future__ import annotations

from dataclasses import dataclass, field, replace

import numpy as np

from . import _native

__all__ = ["PhysicsParams", "State", "flat_bottom", "apply_linear", "apply_nonlinear",
           "dispersion_omega", "max_frequency", "energy_inner", "energy_norm"]


def _mirror(c: np.ndarray) -> np.ndarray:
    # c at the negated wavevector: index i -> (-i) mod n on both axes
    return np.roll(np.flip(c, axis=(0, 1)), shift=(1, 1), axis=(0, 1))


@dataclass(frozen=True)
class PhysicsParams:
    """f, g, H and spectral topography b (dynamics.py:34-63)."""

    f: float
    g: float
    H: float
    b: np.ndarray = field(repr=False)

    def __post_init__(self):
        if not self.g > 0:
            raise ValueError(f"g must be positive, got {self.g}")
        if not self.H > 0:
            raise ValueError(f"H must be positive, got {self.H}")
        b = np.asarray(self.b, dtype=np.complex128)
        object.__setattr__(self, "b", b)
        if b.ndim != 2:
            raise ValueError(f"b must be a 2D spectral field, got shape {b.shape}")
        peak = float(np.max(np.abs(b)))
        if peak > 0.0:
            if float(np.max(np.abs(b - np.conj(_mirror(b))))) > 1e-9 * peak:
                raise ValueError("topography b must be Hermitian-symmetric")
            top = float(np.fft.ifft2(b).real.max())
            if top >= self.H:
                raise ValueError(f"topography peak {top:.6g} must stay below H = {self.H:.6g}")


def flat_bottom(grid, f: float, g: float, H: float) -> PhysicsParams:
    return PhysicsParams(f=f, g=g, H=H, b=np.zeros((grid.nx, grid.ny), dtype=np.complex128))


@dataclass(frozen=True)
class State:
    """Spectral (u, v, eta) at time t; +, -, scalar * act per field (dynamics.py:72-118)."""

    grid: object
    u: np.ndarray = field(repr=False)
    v: np.ndarray = field(repr=False)
    eta: np.ndarray = field(repr=False)
    t: float = 0.0

    def __post_init__(self):
        want = (self.grid.nx, self.grid.ny)
        for name in ("u", "v", "eta"):
            a = np.asarray(getattr(self, name), dtype=np.complex128)
            if a.shape != want:
                raise ValueError(f"field {name} has shape {a.shape}, expected {want}")
            object.__setattr__(self, name, a)

    def _same_grid(self, other) -> None:
        a, b = self.grid, other.grid
        if a is not b and (a.nx, a.ny, a.Lx, a.Ly) != (b.nx, b.ny, b.Lx, b.Ly):
            raise ValueError("states live on different grids")

    def __add__(self, other):
        self._same_grid(other)
        return replace(self, u=self.u + other.u, v=self.v + other.v, eta=self.eta + other.eta)

    def __sub__(self, other):
        self._same_grid(other)
        return replace(self, u=self.u - other.u, v=self.v - other.v, eta=self.eta - other.eta)

    def __mul__(self, a: float):
        return replace(self, u=a * self.u, v=a * self.v, eta=a * self.eta)

    __rmul__ = __mul__

    def with_time(self, t: float):
        return replace(self, t=t)


# ---------------------------------------------------------------- plumbing
def context(state_or_grid, params):
    """Cached native context for this grid + physics, topography uploaded."""
    grid = getattr(state_or_grid, "grid", state_or_grid)
    b = np.asarray(params.b)
    if b.shape != (grid.nx, grid.ny):
        raise ValueError(f"topography shape {b.shape} does not match grid {(grid.nx, grid.ny)}")
    ctx = _native.context_for(grid.nx, grid.ny, grid.Lx, grid.Ly, params.f, params.g, params.H)
    ctx.set_topography(params.b)
    return ctx


def upload(ctx, state, band: bool = False):
    """State fields -> device tensors.  ``band``: only the 2/3 band is
    copied (for consumers that truncate their input to it first)."""
    fields = [getattr(state, n) for n in ("u", "v", "eta")]
    if any(not isinstance(a, np.ndarray) for a in fields):
        return [ctx.to_device(a) for a in fields]
    for a in fields:
        if a.shape != (ctx.nx, ctx.ny):
            raise ValueError(f"field shape {a.shape} does not match the grid ({ctx.nx}, {ctx.ny})")
    return _native.upload_fields(fields, ctx.device, band_ctx=ctx if band else None)


def download(tensors, band_ctx=None, hosts=None):
    """Device tensors -> numpy.  ``band_ctx``: the tensors vanish outside the
    2/3 band (a dealiased tendency), so only the band is copied back."""
    if tensors and tensors[0].is_cuda:
        return _native.download_fields(tensors, band_ctx=band_ctx, hosts=hosts)
    return [t.numpy() for t in tensors]


def rebuild(state, fields, t):
    """Same State class as the input (ours or phaseswe's) with new fields/time."""
    u, v, eta = fields
    return type(state)(grid=state.grid, u=u, v=v, eta=eta, t=t)


# ---------------------------------------------------------------- operators
def apply_linear(state, params):
    """L U per mode on the GPU (dynamics.py:128-136)."""
    ctx = context(state, params)
    return rebuild(state, download(ctx.apply_linear(upload(ctx, state))), state.t)


def apply_nonlinear(state, params):
    """N(U) on the GPU (dynamics.py:139-176): fused pseudo-spectral passes,
    2/3-dealiased; the input passes the Hermitian gate of to_physical
    (grid.py:159-172) or ValueError names its worst mode."""
    ctx = context(state, params)
    U = upload(ctx, state, band=True)
    return rebuild(state, download(ctx.apply_nonlinear(U), band_ctx=ctx), state.t)


def dispersion_omega(kappa, params) -> np.ndarray:
    """omega = sqrt(f^2 + g H |k|^2) (dynamics.py:179-186)."""
    kx, ky = kappa
    return np.sqrt(params.f ** 2 + params.g * params.H * (np.asarray(kx) ** 2 + np.asarray(ky) ** 2))


def max_frequency(grid, params) -> float:
    """Largest |eigenvalue| of L on the grid (dynamics.py:189-192)."""
    kx, ky = grid.kx[:, None], grid.ky[None, :]
    return float(np.max(dispersion_omega((kx, ky), params)))


def energy_inner(a, b, params) -> float:
    """Energy inner product via Parseval (dynamics.py:195-207); host diagnostic."""
    g = a.grid
    npts = g.nx * g.ny
    q = params.H * (np.vdot(b.u, a.u) + np.vdot(b.v, a.v)) + params.g * np.vdot(b.eta, a.eta)
    return float(np.real(q) * g.Lx * g.Ly / npts ** 2)


def energy_norm(a, params) -> float:
    return float(np.sqrt(max(energy_inner(a, a, params), 0.0)))

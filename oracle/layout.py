"""Compact band layout in numpy (TEST INFRASTRUCTURE, see oracle/pswe_oracle.py header).

Mirrors the layout of include/pswe_b200.h: U[f][j][r], j = ky index 0..ny/3,
r = compact kx index (wx = r for r <= nx/3, r - Kx after).  ``pack`` applies
the Hermitian projection (c(k) + conj c(-k))/2 that real(ifft2(.)) implies
(grid.py:173-174); ``unpack`` expands with zeros outside the 2/3 band and the
conjugate mirror for ky < 0.
"""

from __future__ import annotations

import numpy as np


def kx_order(nx: int) -> np.ndarray:
    km = nx // 3
    r = np.arange(2 * km + 1)
    return np.where(r <= km, r, r - (2 * km + 1))


def pack(U: np.ndarray) -> np.ndarray:
    U = np.asarray(U, dtype=np.complex128)
    nf, nx, ny = U.shape
    wx = kx_order(nx)
    Ky = ny // 3 + 1
    j = np.arange(Ky)
    a = U[:, (wx % nx)[None, :], j[:, None]]
    b = U[:, ((-wx) % nx)[None, :], ((-j) % ny)[:, None]]
    return 0.5 * (a + np.conj(b))


def unpack(Uc: np.ndarray, nx: int, ny: int) -> np.ndarray:
    Uc = np.asarray(Uc, dtype=np.complex128)
    nf, Ky, Kx = Uc.shape
    wx = kx_order(nx)
    out = np.zeros((nf, nx, ny), dtype=np.complex128)
    for j in range(Ky):
        out[:, wx % nx, j] = Uc[:, j, :]
        if j > 0:
            out[:, (-wx) % nx, ny - j] = np.conj(Uc[:, j, :])
    return out

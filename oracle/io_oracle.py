"""TEST INFRASTRUCTURE ONLY -- the checker for the snapshot writer.

Restates the reference's run-output format (phaseswe io.py) so the tests can
compare bytes: physical fields as little-endian float64, row-major (nx, ny),
y fastest, one ``snap_<step:07d>_<field>.f64`` per field plus a ``.meta``
text sidecar (io.py:37-70), and the diagnostics CSV (io.py:127-133).
Physical fields are real(ifft2(.)) (grid.py:173-174) via numpy.
Only tests/ may import this module.
"""

import os

import numpy as np

FIELDS = ("u", "v", "eta")


def physical(c):
    return np.fft.ifft2(np.asarray(c, dtype=np.complex128)).real


def write_snapshot(outdir, step, nx, ny, Lx, Ly, t, phys):
    """io.py:37-70 with the physical fields given."""
    prefix = f"snap_{step:07d}"
    for name, data in zip(FIELDS, phys):
        base = os.path.join(outdir, f"{prefix}_{name}")
        with open(base + ".f64", "wb") as fh:
            fh.write(np.ascontiguousarray(data, dtype="<f8").tobytes(order="C"))
        lines = [f"field = {name}", f"step = {step}", f"time_seconds = {t!r}", f"nx = {nx}", f"ny = {ny}",
                 f"Lx = {Lx!r}", f"Ly = {Ly!r}", "dtype = float64", "byte_order = little",
                 "layout = row-major, shape (nx, ny), y index fastest"]
        with open(base + ".meta", "w", encoding="utf-8") as fh:
            fh.write("\n".join(lines) + "\n")


def write_diagnostics(outdir, times, steps, energy, mass, max_speed):
    """io.py:127-133."""
    rows = ["time_seconds,step,energy,mass,max_speed"]
    rows += [f"{t!r},{s},{e!r},{m!r},{v!r}" for t, s, e, m, v in zip(times, steps, energy, mass, max_speed)]
    with open(os.path.join(outdir, "diagnostics.csv"), "w", encoding="utf-8") as fh:
        fh.write("\n".join(rows) + "\n")

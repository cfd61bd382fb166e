"""Averaging-window sweep on the GPU.

The reference runs one full trajectory per window T in sequence
(harness.py:110-147 ``cmd_sweep``, validation.py:251-271
``_check_window_sweep``) and compares each final state with a fine-step
reference run.  Here every window is an independent device-resident run
(its own native context: quadrature, phase table, intermediates) on its own
CUDA stream, all launched together from persistent host threads, so the
windows share the GPU: small windows (few phases) fill the gaps of large
ones.  The
per-window results are bitwise identical to running the windows one by one.
"""

from __future__ import annotations

import threading
from dataclasses import dataclass

import numpy as np

from . import _native
from .integrator import make_step_config, run

__all__ = ["WindowResult", "window_sweep", "l2_error_normalized"]

# Persistent worker threads: a native context is cached per (grid, physics,
# thread), so keeping the workers alive keeps each window's context (phase
# table, intermediates, captured step graph) warm across sweeps.
_POOL = None
_POOL_SIZE = 0
_TLS = threading.local()


def _pool(n):
    global _POOL, _POOL_SIZE
    if _POOL is None or _POOL_SIZE < n:
        from concurrent.futures import ThreadPoolExecutor
        _POOL = ThreadPoolExecutor(max_workers=n, thread_name_prefix="pswe-window")
        _POOL_SIZE = n
    return _POOL


def _worker_stream(torch):
    s = getattr(_TLS, "stream", None)
    if s is None:
        s = torch.cuda.Stream()
        _TLS.stream = s
    return s


@dataclass
class WindowResult:
    T: float
    M: int
    final: object
    trajectory: object
    l2_eta: float = float("nan")
    l2_u: float = float("nan")


def l2_error_normalized(test, ref):
    """Physical relative L2 errors (eta, joint velocity) of test vs ref (diagnostics.py:28-44)."""
    tu, tv, te = (np.fft.ifft2(getattr(test, n)).real for n in ("u", "v", "eta"))
    ru, rv, re = (np.fft.ifft2(getattr(ref, n)).real for n in ("u", "v", "eta"))
    eta_ref = float(np.sqrt(np.sum(re ** 2)))
    vel_ref = float(np.sqrt(np.sum(ru ** 2 + rv ** 2)))
    if eta_ref == 0.0 or vel_ref == 0.0:
        raise ValueError("reference state has a zero-norm field; normalized error is undefined")
    return (float(np.sqrt(np.sum((te - re) ** 2))) / eta_ref,
            float(np.sqrt(np.sum((tu - ru) ** 2 + (tv - rv) ** 2))) / vel_ref)


def window_sweep(initial, params, dt: float, t_end: float, windows, M=None, propagator: str = "exact",
                 reference=None, snapshot_every: float = 0.0):
    """Run ``run(initial, make_step_config(grid, params, dt, T=T, M=M), params, t_end)``
    for every window T concurrently; returns one WindowResult per window, in order.
    With ``reference`` (a State at t_end), the normalized L2 errors are filled in."""
    torch = _native._torch()
    grid = initial.grid
    cfgs = []
    for T in windows:
        m = None if M is None else (M if T > 0 else 0)
        cfgs.append(make_step_config(grid, params, dt=dt, T=float(T), M=m, propagator=propagator))
    device = torch.cuda.current_device()

    def work(i):
        torch.cuda.set_device(device)
        stream = _worker_stream(torch)
        with torch.cuda.stream(stream):  # each window on its own stream (and context)
            traj = run(initial, cfgs[i], params, t_end, snapshot_every=snapshot_every)
        stream.synchronize()
        return traj

    results = list(_pool(len(cfgs)).map(work, range(len(cfgs))))
    out = []
    for T, cfg, traj in zip(windows, cfgs, results):
        r = WindowResult(T=float(T), M=int(cfg.quadrature.M), final=traj.states[-1], trajectory=traj)
        if reference is not None:
            r.l2_eta, r.l2_u = l2_error_normalized(r.final, reference)
        out.append(r)
    return out

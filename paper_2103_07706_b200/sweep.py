"""Averaging-window sweep on the GPU.

The reference runs one full trajectory per window T in sequence
(harness.py:110-147 ``cmd_sweep``, validation.py:251-271
``_check_window_sweep``) and compares each final state with a fine-step
reference run.  Here the windows are one **window batch**
(``pswe_set_window_batch`` / ``pswe_window_batch_run``): the live phases of
all windows form one batch axis of (window, phase) pairs, pass A reads each
phase's own window state, pass C accumulates into per-window slots, and the
stage kernels advance all windows at once -- one launch sequence per stage
serves every window, captured once as a CUDA graph.

Per-window results equal the one-by-one runs up to the grouping of the
phase sums and the pass-B phase pairing (round-off, ~1e-15 relative): the
windows share chunks and pairs.  Windows whose exponential routes differ (the
Chebyshev Lambda grows with T) cannot share a launch sequence and run one
after the other; so does a batch that any window's step flags (a
non-finite stage or a non-Hermitian input), so that the failing window
raises the reference's own error.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native
from .dynamics import context, download, rebuild
from .integrator import Trajectory, _whole_steps, make_step_config, run
from .propagator import configure

__all__ = ["WindowResult", "window_sweep", "l2_error_normalized"]


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


def _sequential(initial, params, t_end, cfgs, snapshot_every):
    return [run(initial, cfg, params, t_end, snapshot_every=snapshot_every) for cfg in cfgs]


def _batched(initial, params, dt, t_end, cfgs, snapshot_every):
    """All windows as one window batch; None when a step flags (then the
    caller replays them one by one)."""
    torch = _native._torch()
    W = len(cfgs)
    n_steps = _whole_steps(t_end, dt, "t_end")
    stride = 0
    if snapshot_every != 0.0:
        stride = _whole_steps(snapshot_every, dt, "snapshot_every")
        if stride <= 0:
            raise ValueError(f"snapshot_every must be positive, got {snapshot_every}")
    trajs = [Trajectory() for _ in range(W)]
    if n_steps == 0:
        for tr in trajs:
            tr.record(0, initial, params)
        return trajs
    ctx = context(initial, params)
    configure(ctx, cfgs[0].propagator_spec)
    ctx.set_window_batch([cfg.quadrature for cfg in cfgs])
    U0 = torch.stack([ctx.to_device(np.asarray(getattr(initial, n))) for n in ("u", "v", "eta")])
    U = U0.unsqueeze(0).repeat(W, 1, 1, 1).contiguous()  # (W, 3, nx, ny)
    d0 = ctx.diagnostics(list(U0))  # the common initial record (gated like run's)
    for tr in trajs:
        tr.record_values(0, initial, *d0)
    marks = sorted({i for i in range(stride, n_steps + 1, stride)} | {n_steps}) if stride else [n_steps]
    done, t = 0, initial.t
    for mark in marks:
        if ctx.window_batch_run(dt, mark - done, U):
            return None
        for _ in range(mark - done):
            t = t + dt
        done = mark
        for w, tr in enumerate(trajs):
            fields = list(U[w])
            diag = ctx.diagnostics(fields)
            tr.record_values(done, rebuild(initial, download(fields), t), *diag)
    return trajs


def window_sweep(initial, params, dt: float, t_end: float, windows, M=None, propagator: str = "exact",
                 reference=None, snapshot_every: float = 0.0, batched: bool = True):
    """``run(initial, make_step_config(grid, params, dt, T=T, M=M), params, t_end)``
    for every window T; returns one WindowResult per window, in order.  With
    ``reference`` (a State at t_end) the normalized L2 errors are filled in.
    ``batched`` (default): one window batch on the GPU when the windows share
    the exponential route; otherwise, or when a step flags, one run per window."""
    grid = initial.grid
    cfgs = []
    for T in windows:
        m = None if M is None else (M if T > 0 else 0)
        cfgs.append(make_step_config(grid, params, dt=dt, T=float(T), M=m, propagator=propagator))
    trajs = None
    specs = {(c.propagator_spec.kind, c.propagator_spec.Lambda, c.propagator_spec.n_poly) for c in cfgs}
    if batched and cfgs and len(specs) == 1:
        trajs = _batched(initial, params, dt, t_end, cfgs, snapshot_every)
    if trajs is None:
        trajs = _sequential(initial, params, t_end, cfgs, snapshot_every)
    out = []
    for T, cfg, traj in zip(windows, cfgs, trajs):
        r = WindowResult(T=float(T), M=int(cfg.quadrature.M), final=traj.states[-1], trajectory=traj)
        if reference is not None:
            r.l2_eta, r.l2_u = l2_error_normalized(r.final, reference)
        out.append(r)
    return out

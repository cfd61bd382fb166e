"""Phase-sharded averaged tendency across ranks.

The averaged tendency is a sum of independent phase terms
(averaging.py:130-146).  ``sharded_averaged_tendency`` splits the live nodes
into contiguous, ascending slices, one per rank of a ``torch.distributed``
group; each rank evaluates its slice on its own GPU (the same batched launch
sequence as ``averaged_tendency``, with the other nodes' weights zeroed, so
node numbers in error messages stay the reference's), the compact 2/3-band
partial sums are all-gathered (NCCL over NVLink between GPUs) and summed in
rank order.  The result is deterministic for a given world size; it differs
from the one-GPU sum only by the grouping of the additions.

Error behaviour follows averaging.py:138-141 across ranks: every rank raises
the message of the first failing node in ascending order, whichever rank
owns it (the failure is agreed on before the data gather, so no rank waits
on a peer that has given up).

This is not the bench's multi-GPU mode -- ``bench.py --gpus N`` runs N
independent replicas (weak scaling) and reports this strong-
scaling path beside it as ``phase_sharded``.
"""

from __future__ import annotations

import numpy as np

__all__ = ["live_nodes", "shard_bounds", "shard_weights", "ordered_gather_sum", "device_partial",
           "sharded_averaged_tendency"]


def live_nodes(w) -> np.ndarray:
    """Indices of the nonzero-weight nodes, ascending (averaging.py:128)."""
    return np.flatnonzero(np.asarray(w) != 0.0)


def shard_bounds(n_live: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous balanced slice [lo, hi) of ``n_live`` nodes for ``rank``."""
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world of size {world}")
    return n_live * rank // world, n_live * (rank + 1) // world


def shard_weights(w, world: int, rank: int) -> np.ndarray:
    """The full weight vector with every live node outside this rank's
    slice set to zero (the library skips zero-weight nodes)."""
    w = np.asarray(w, dtype=np.float64)
    live = live_nodes(w)
    lo, hi = shard_bounds(len(live), world, rank)
    out = np.zeros_like(w)
    out[live[lo:hi]] = w[live[lo:hi]]
    return out


def _first_error(err: str | None, group, world: int, device) -> str | None:
    """Agree across ranks on the first failure in rank (= node) order."""
    import torch
    import torch.distributed as dist

    flag = torch.tensor([1 if err else 0], dtype=torch.int32, device=device)
    flags = [torch.zeros_like(flag) for _ in range(world)]
    dist.all_gather(flags, flag, group=group)
    if not any(int(f.item()) for f in flags):
        return None
    msgs = [None] * world
    dist.all_gather_object(msgs, err, group=group)
    return next(m for m in msgs if m)


def ordered_gather_sum(part, group=None):
    """All-gather one tensor per rank and sum the copies in rank order
    (a fixed order: bitwise reproducible, unlike a reduction collective)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    send = torch.view_as_real(part) if part.is_complex() else part
    bufs = [torch.empty_like(send) for _ in range(world)]
    dist.all_gather(bufs, send.contiguous(), group=group)
    acc = bufs[0].clone()
    for b in bufs[1:]:
        acc += b
    return torch.view_as_complex(acc) if part.is_complex() else acc


def device_partial(state, quadrature, w_rank, params, spec):
    """This rank's weighted partial sum, compact 2/3-band layout on its GPU,
    and the function that turns the summed compact tensor into host fields."""
    from . import dynamics
    from .propagator import configure

    ctx = dynamics.context(state, params)
    configure(ctx, spec)

    def finish(total):
        return dynamics.download(list(ctx.unpack(total)), band_ctx=ctx)

    if not np.any(w_rank != 0.0):
        return finish, ctx.empty_compact().zero_()
    ctx.set_quadrature(quadrature.s, w_rank)
    Uc = ctx.pack(dynamics.upload(ctx, state, band=True))
    return finish, ctx.averaged_tendency_compact(Uc)


def sharded_averaged_tendency(state, quadrature, params, propagator_spec, group=None, partial=None):
    """``averaged_tendency`` with the phase sum split over the ranks of
    ``group`` (default: the world).  Every rank receives the full result.

    ``partial(state, quadrature, w_rank, params, spec) -> (finish, tensor)``
    evaluates this rank's share (default ``device_partial``; tests substitute
    a CPU stand-in); ``finish(summed tensor)`` returns the three fields.
    """
    import torch
    import torch.distributed as dist

    from .averaging import node_error
    from .dynamics import rebuild

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    w_rank = shard_weights(quadrature.w, world, rank)
    err, finish, part = None, None, None
    try:
        finish, part = (partial or device_partial)(state, quadrature, w_rank, params, propagator_spec)
    except Exception as exc:  # noqa: BLE001 -- every rank must reach the agreement collective below
        exc = node_error(exc)
        if isinstance(exc, ValueError):
            err = "value:" + str(exc)
        elif isinstance(exc, RuntimeError):
            err = "runtime:" + str(exc)
        else:
            err = f"runtime:{type(exc).__name__}: {exc}"
    device = part.device if part is not None else (
        torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else torch.device("cpu"))
    first = _first_error(err, group, world, device)
    if first is not None:
        kind, msg = first.split(":", 1)
        raise ValueError(msg) if kind == "value" else RuntimeError(msg)
    return rebuild(state, finish(ordered_gather_sum(part, group)), state.t)

"""Phase-sharded averaged tendency (sharding.py): the host
logic -- node partition, failure agreement, all-gather and rank-ordered sum
-- on CPU with gloo, world size 2.  The per-rank phase sums come from the
oracle here (a CPU stand-in for the device partial); the GPU path is in
tests/test_gpu_parity.py."""

import os
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT


def test_shard_weights_partition_the_live_nodes():
    sys.path.insert(0, str(ROOT))
    from paper_2103_07706_b200 import kernel_weights
    from paper_2103_07706_b200.sharding import live_nodes, shard_weights

    q = kernel_weights(3600.0, 16)  # bump: endpoints have zero weight -> 31 live nodes
    live = live_nodes(q.w)
    assert len(live) == 31
    for world in (1, 2, 3, 4, 8, 40):
        parts = [shard_weights(q.w, world, r) for r in range(world)]
        owned = [live_nodes(p) for p in parts]
        # disjoint, contiguous, ascending in rank order, covering every live node
        assert np.array_equal(np.concatenate(owned), live)
        assert np.array_equal(np.sum(parts, axis=0), q.w)
        sizes = [len(o) for o in owned]
        assert max(sizes) - min(sizes) <= 1


def _oracle_partial(state, quadrature, w_rank, params, spec):
    from oracle import pswe_oracle as O

    g = state.grid
    S = O.Setup(g.nx, g.ny, g.Lx, g.Ly, params.f, params.g, params.H, params.b)
    U = np.stack([state.u, state.v, state.eta])
    if not np.any(w_rank != 0.0):
        part = np.zeros_like(U)
    else:
        part = O.averaged_tendency(S, U, quadrature.s, w_rank)
    return (lambda t: list(t.numpy())), torch.from_numpy(part)


def _failing_partial(state, quadrature, w_rank, params, spec):
    from paper_2103_07706_b200.sharding import live_nodes

    k = int(live_nodes(w_rank)[0]) - quadrature.M
    if k > -quadrature.M + 3:  # every rank but the first fails on its first node
        raise ValueError(f"averaging node k = {k} (s = 1 s) failed: |t| * max_frequency = 2 exceeds Lambda = 1")
    return _oracle_partial(state, quadrature, w_rank, params, spec)


def _odd_partial(state, quadrature, w_rank, params, spec):
    from paper_2103_07706_b200.sharding import live_nodes

    if int(live_nodes(w_rank)[0]) - quadrature.M > -quadrature.M + 3:  # rank 1 only
        raise KeyError("boom")  # neither ValueError nor RuntimeError
    return _oracle_partial(state, quadrature, w_rank, params, spec)


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, str(ROOT))
    from paper_2103_07706_b200 import cases
    from paper_2103_07706_b200.sharding import sharded_averaged_tendency

    dist.init_process_group("gloo", rank=rank, world_size=world)
    c = cases.case_c1()
    got = sharded_averaged_tendency(c.state, c.quadrature, c.params, None, partial=_oracle_partial)
    try:
        sharded_averaged_tendency(c.state, c.quadrature, c.params, None, partial=_failing_partial)
        msg = None
    except RuntimeError as exc:
        msg = str(exc)
    # any exception type on one rank is agreed on too (no rank left waiting)
    try:
        sharded_averaged_tendency(c.state, c.quadrature, c.params, None, partial=_odd_partial)
        odd = None
    except RuntimeError as exc:
        odd = str(exc)
    out.put((rank, np.stack([got.u, got.v, got.eta]), got.t, msg, odd))
    dist.destroy_process_group()


def test_sharded_sum_two_ranks_gloo():
    sys.path.insert(0, str(ROOT))
    from oracle import pswe_oracle as O
    from paper_2103_07706_b200 import cases
    from paper_2103_07706_b200.sharding import shard_weights

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29600 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=300) for _ in procs), key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0

    c = cases.case_c1()
    g = c.grid
    S = O.Setup(g.nx, g.ny, g.Lx, g.Ly, c.params.f, c.params.g, c.params.H, c.params.b)
    U = np.stack([c.state.u, c.state.v, c.state.eta])
    parts = [O.averaged_tendency(S, U, c.quadrature.s, shard_weights(c.quadrature.w, 2, r)) for r in range(2)]
    # every rank holds the same result: the partial sums added in rank order, bitwise
    for rank, got, t, msg, odd in res:
        assert odd == "KeyError: 'boom'"
        assert np.array_equal(got, parts[0] + parts[1])
        assert t == c.state.t
        # the failure of the first failing node (rank 1's first node) reaches both ranks
        assert msg is not None and msg.startswith("averaging node k = ")
    assert res[0][3] == res[1][3]
    # and it is the averaged tendency (grouping of the sum only)
    want = O.averaged_tendency(S, U, c.quadrature.s, c.quadrature.w)
    assert O.rel_l2(res[0][1], want) <= 1e-14

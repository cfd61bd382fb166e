"""Phase-sharded averaged tendency on the GPU (sharding.py).

One GPU only: world size 1 over NCCL (the real collective path), and two
ranks sharing cuda:0 whose device partials are gathered over gloo on the
host -- the ranks' kernels are independent (no rank waits on another's
kernel), only the gather is collective."""

import os
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT, rel_l2

pytestmark = pytest.mark.gpu


def _plain(c):
    import paper_2103_07706_b200 as pk

    out = pk.averaged_tendency(c.state, c.quadrature, c.params, pk.PropagatorSpec.exact())
    return np.stack([out.u, out.v, out.eta])


def test_world_of_one_over_nccl_is_the_plain_call_bitwise():
    import paper_2103_07706_b200 as pk
    from paper_2103_07706_b200 import cases
    from paper_2103_07706_b200.sharding import sharded_averaged_tendency

    torch.cuda.set_device(0)
    port = 29700 + os.getpid() % 1000
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        for c in (cases.case_c1(), cases.case_c5(6, 32)):
            got = sharded_averaged_tendency(c.state, c.quadrature, c.params, pk.PropagatorSpec.exact())
            assert np.array_equal(np.stack([got.u, got.v, got.eta]), _plain(c))
            assert got.t == c.state.t
    finally:
        dist.destroy_process_group()


def _host_gathered(state, quadrature, w_rank, params, spec):
    from paper_2103_07706_b200.sharding import device_partial

    finish, part = device_partial(state, quadrature, w_rank, params, spec)
    return (lambda t: finish(t.to("cuda"))), part.cpu()


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, str(ROOT))
    import paper_2103_07706_b200 as pk
    from paper_2103_07706_b200 import cases
    from paper_2103_07706_b200.sharding import sharded_averaged_tendency

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    c = cases.case_c5(7, 8)
    got = sharded_averaged_tendency(c.state, c.quadrature, c.params, pk.PropagatorSpec.exact(),
                                    partial=_host_gathered)
    out.put((rank, np.stack([got.u, got.v, got.eta])))
    dist.destroy_process_group()


def test_two_ranks_512_match_the_single_gpu_sum():
    from paper_2103_07706_b200 import cases

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29800 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=600) for _ in procs), key=lambda r: r[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert np.array_equal(res[0][1], res[1][1])
    want = _plain(cases.case_c5(7, 8))
    assert rel_l2(res[0][1], want) <= 1e-13

"""bench.py's multi-GPU replica coordination (barrier + max over ranks) on CPU with gloo, world size 2."""

import json
import os
import subprocess
import sys

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    sys.path.insert(0, str(ROOT))
    import bench
    dist.init_process_group("gloo", rank=rank, world_size=world)
    bench.barrier(world)
    got = bench.max_over_ranks(float(rank + 1) * 1.5, world, "cpu")
    ws, r, _ = bench.dist_env()
    out.put((rank, got, ws, r))
    dist.destroy_process_group()


def test_max_over_ranks_two_processes():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [r[1] for r in res] == [3.0, 3.0]
    assert [(r[2], r[3]) for r in res] == [(2, 0), (2, 1)]


def test_reference_arm_runs_on_cpu_and_prints_contract_line():
    """--impl reference (oracle port on host cores) on a small grid; rank 0 prints one JSON line."""
    env = dict(os.environ, OMP_NUM_THREADS="1")
    p = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--level", "3", "--M", "4",
                        "--steps", "2", "--warmup", "1"], capture_output=True, text=True, env=env, timeout=300)
    assert p.returncode == 0, p.stderr
    line = json.loads(p.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "cpu_baseline", "e2e", "config"):
        assert key in line
    from oracle import reference as R
    want_kind = "reference" if R.load() is not None else "port"
    assert line["impl"] == "reference" and line["cpu_baseline"]["kind"] == want_kind
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["value"] > 0


def test_cpu_baseline_leg_checks_parity():
    """bench.py's cpu_baseline leg: the whole workload on the host cores
    (the reference itself when oracle/_ref is built) and the rel-L2 parity
    of a given result against it -- here the oracle port's own result."""
    import numpy as np
    sys.path.insert(0, str(ROOT))
    import bench
    from oracle import pswe_oracle as O
    from paper_2103_07706_b200 import cases
    c = cases.case_c5(3, 4)  # 32^2, 7 phases
    g, q = c.grid, c.quadrature
    S = O.Setup(g.nx, g.ny, g.Lx, g.Ly, c.params.f, c.params.g, c.params.H)
    got = O.averaged_tendency(S, np.stack([c.state.u, c.state.v, c.state.eta]), q.s, q.w)
    out = bench.cpu_baseline(c, list(got), one_core_budget_s=0.2)
    assert out["value"] > 0 and out["cores"] >= 1
    assert out["parity"]["rel_l2"] <= 1e-13 and out["parity"]["tol"] == 1e-10
    assert "numpy" in out["host"] and "cpu_model" in out["host"]
    if out["kind"] == "reference":
        assert out["one_core"]["cores"] == 1

"""Benchmark: averaged-RHS phase x DOF/s on B200 (BASELINE.json metric).

Workload (default): the C5 throughput point at the largest mesh, refinement
7 -> 512^2 grid, M = 256 (511 live phases), exact exponentials, fp64,
seeded synthetic geostrophic state (SURVEY.md 8d planar stand-in for the
spherical C5 sweep).  One "step" = one averaged-RHS evaluation over all 511
phases.  metric = P * 3 n^2 * steps / device seconds, summed over replicas.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--level 7] [--M 256] [--no-cpu] [--no-sweep]

Multi-GPU: the path is run as independent replicas (north_star: no
multi-GPU path); under torchrun every rank times its own replica, the time is
the max over ranks and value = all ranks' units / that time ("scaling": "weak").
`--gpus N` without a launcher re-executes itself under torch.distributed.run.
--impl reference times the unmodified reference (phaseswe, installed into
oracle/_ref by oracle/build_ref.sh) on the host cores on bounded phase samples
of the same workload; the numpy port (oracle/pswe_oracle.py) stands in only
when the reference is absent.  The default run's `cpu_baseline` evaluates the
whole workload with the reference on all host cores and checks the GPU output
against it (`parity`).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import pathlib
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "averaged-RHS phase×DOF/s (1 GPU, fp64)"
UNIT = "phase*DOF/s"


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def init_dist(ws, backend):
    import torch.distributed as dist
    if ws > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group(backend=backend)
    return dist


def max_over_ranks(value: float, ws: int, device=None) -> float:
    """Max of a float over ranks (device timing rule); identity for one rank."""
    if ws == 1:
        return value
    import torch
    import torch.distributed as dist
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def alg_bytes(n: int, P: int) -> dict:
    """Algorithmic bytes for one averaged-RHS evaluation on an n^2 grid."""
    K = n // 3 + 1
    Kx = 2 * (n // 3) + 1
    field = 16 * n * K  # one intermediate field, complex128, n x (n/3+1)
    return {
        "B_phase": 352 * n * K,  # survey model: 2 * 16 * (7 + 4) * n * K
        "B_eval": P * 352 * n * K + 112 * Kx * K,
        # our passes: A writes 5 fields (+ reads U, b), B reads 5 writes 4, C reads 4
        "passA_phase": 5 * field + 4 * 16 * Kx * K,
        "passB_phase": 9 * field,
        "passC_phase": 4 * field,
    }


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (OSError, FileNotFoundError):
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.thread is not None:
            self.thread.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx.append(float(r[1]))
            except ValueError:
                continue
            for name, val in zip(names, r[3:]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def flush_l2(buf):
    buf.add_(1.0)  # 256 MiB write > 126 MB L2


def cpu_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def oracle_sample(case, nodes, threads):
    """Time the oracle port on a subset of live nodes; returns (seconds, phases)."""
    from oracle import pswe_oracle as O
    g, p = case.grid, case.params
    S = O.Setup(g.nx, g.ny, g.Lx, g.Ly, p.f, p.g, p.H, p.b)
    U = np.stack([case.state.u, case.state.v, case.state.eta])
    q = case.quadrature
    t0 = time.perf_counter()
    O.averaged_tendency(S, U, q.s, q.w, workers=threads, nodes=nodes)
    return time.perf_counter() - t0, len(nodes)


def host_info(threads):
    import platform
    import scipy
    model = platform.processor() or ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu_model": model, "threads_used": threads, "host_threads": os.cpu_count(),
            "numpy": np.__version__, "scipy": scipy.__version__,
            "blas_threads_env": {k: os.environ.get(k) for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS",
                                                               "MKL_NUM_THREADS")}}


def _ref_eval(R, prob, quad, threads):
    """The reference's public averaged_tendency (averaging.py:116-156) with a
    ThreadPoolExecutor of `threads` workers (None = its serial path)."""
    from concurrent.futures import ThreadPoolExecutor
    from phaseswe import averaging
    if threads is None:
        t0 = time.perf_counter()
        out = averaging.averaged_tendency(prob.state, quad, prob.params, prob.spec)
        return time.perf_counter() - t0, out
    with ThreadPoolExecutor(max_workers=threads) as ex:
        t0 = time.perf_counter()
        out = averaging.averaged_tendency(prob.state, quad, prob.params, prob.spec, executor=ex)
        return time.perf_counter() - t0, out


def cpu_baseline(case, gpu_fields=None, one_core_budget_s: float = 6.0) -> dict:
    """The reference on the host cores, same run (SURVEY.md 8d CPU plan).

    * C cores: the reference's averaged_tendency over ALL live phases of the
      benchmarked workload with a ThreadPoolExecutor(C) -- the unsampled
      figure -- and its result is the parity check of the GPU output
      (`parity`, rel L2 over (u, v, eta), tolerance 1e-10).
    * 1 core: the reference's serial path (executor=None) on the 2m+1
      central nodes, m sized for about `one_core_budget_s`.
    Falls back to the numpy port (oracle/pswe_oracle.py) when the reference
    is not installed (oracle/build_ref.sh)."""
    from oracle import reference as R
    threads = cpu_threads()
    prob = R.problem(case)
    info = host_info(threads)
    if prob is None:
        from oracle import pswe_oracle as O
        g, p = case.grid, case.params
        S = O.Setup(g.nx, g.ny, g.Lx, g.Ly, p.f, p.g, p.H, p.b)
        q = case.quadrature
        t0 = time.perf_counter()
        want = O.averaged_tendency(S, np.stack([case.state.u, case.state.v, case.state.eta]), q.s, q.w,
                                   workers=threads)
        used = time.perf_counter() - t0
        out = {"value": case.P * case.dof / used, "unit": UNIT, "cores": threads, "kind": "port",
               "sample": f"oracle/pswe_oracle.py averaged_tendency over all {case.P} live phases of {case.name}, "
                         f"{threads} threads, {used:.1f} s (reference not installed)", "host": info}
    else:
        used, got = _ref_eval(R, prob, prob.quadrature, threads)
        want = np.stack([got.u, got.v, got.eta])
        out = {"value": case.P * case.dof / used, "unit": UNIT, "cores": threads, "kind": "reference",
               "sample": f"phaseswe.averaging.averaged_tendency (unmodified reference, {R.where()}) over all "
                         f"{case.P} live phases of {case.name} ({case.grid.nx}^2), ThreadPoolExecutor({threads}), "
                         f"{used:.1f} s", "host": info}
        # 1 core: the serial path on a central block of nodes
        t1, _ = _ref_eval(R, prob, prob.sub_quadrature(1), None)
        m = max(1, min(case.M - 1, int(one_core_budget_s / max(t1 / 3, 1e-6) / 2)))
        q1 = prob.sub_quadrature(m)
        t1, _ = _ref_eval(R, prob, q1, None)
        ph = int(np.count_nonzero(q1.w))
        out["one_core"] = {"value": ph * case.dof / t1, "unit": UNIT, "cores": 1,
                           "sample": f"executor=None on the {ph} central nodes (renormalised sub-quadrature), "
                                     f"{t1:.1f} s"}
    if gpu_fields is not None:
        diff = np.sqrt(sum(np.sum(np.abs(a - b) ** 2) for a, b in zip(gpu_fields, want)))
        norm = np.sqrt(sum(np.sum(np.abs(b) ** 2) for b in want))
        out["parity"] = {"rel_l2": float(diff / norm), "tol": 1e-10, "against": out["kind"],
                         "what": "GPU averaged RHS of the timed workload vs the CPU evaluation above"}
    return out


def cpu_step_runs(threads=None, full_budget_s=60.0) -> list:
    """C2-C4 on the host cores: the reference's step_averaged_ssprk3
    (integrator.py:83-103) per step and its run(..., workers=C)
    (integrator.py:145-183); a full run is timed when one step times the
    step count fits `full_budget_s`, otherwise extrapolated (marked)."""
    from concurrent.futures import ThreadPoolExecutor
    from oracle import reference as R
    from paper_2103_07706_b200 import cases
    if R.load() is None:
        return []
    from phaseswe import integrator
    threads = threads or cpu_threads()
    out = []
    for name in ("C2", "C3", "C4"):
        c = cases.CASES[name]()
        prob = R.problem(c)
        cfg = integrator.StepConfig(dt=c.dt, quadrature=prob.quadrature, propagator_spec=prob.spec)
        with ThreadPoolExecutor(max_workers=threads) as ex:
            t0 = time.perf_counter()
            integrator.step_averaged_ssprk3(prob.state, cfg, prob.params, ex)
            step_s = time.perf_counter() - t0
        ent = {"config": name, "grid": c.grid.nx, "M": c.M, "P": c.P, "steps": c.nsteps, "cores": threads,
               "step_s": step_s, "phase_dof_per_s": 3 * c.P * c.dof / step_s}
        if step_s * c.nsteps <= full_budget_s:
            t0 = time.perf_counter()
            integrator.run(prob.state, cfg, prob.params, t_end=c.nsteps * c.dt, workers=threads)
            ent["run_s"] = time.perf_counter() - t0
        else:
            ent["run_s_extrapolated"] = step_s * c.nsteps
        out.append(ent)
    return out


def run_reference(args, ws, rank):
    """--impl reference: the unmodified reference (oracle/_ref phaseswe) on the
    host cores, rank 0 only; every step is the reference's public
    averaged_tendency on a bounded sample of the workload (the 2m+1 central
    nodes, ~2 per core, weights renormalised), ThreadPoolExecutor(all
    cores).  Falls back to the numpy port if the reference is absent."""
    if rank != 0:
        return
    from oracle import reference as R
    from paper_2103_07706_b200 import cases
    case = cases.case_c5(args.level, args.M)
    threads = cpu_threads()
    prob = R.problem(case)
    if prob is not None:
        # about eight phases per host thread per step (the full evaluation's
        # thread efficiency at a fraction of its 7-10 s)
        m = max(1, min(case.M - 1, 4 * threads))
        quad = prob.sub_quadrature(m)
        per_step = int(np.count_nonzero(quad.w))
        for _ in range(args.warmup):
            _ref_eval(R, prob, quad, threads)
        total = 0.0
        for _ in range(args.steps):
            total += _ref_eval(R, prob, quad, threads)[0]
        kind = "reference"
        sample = (f"phaseswe.averaging.averaged_tendency (unmodified reference, {R.where()}) on the {per_step} "
                  f"central of {case.P} live phases per step (renormalised sub-quadrature), "
                  f"ThreadPoolExecutor({threads})")
    else:
        live = [i for i in range(len(case.quadrature.w)) if case.quadrature.w[i] != 0.0]
        per_step = max(1, min(len(live), threads))
        for _ in range(args.warmup):
            oracle_sample(case, live[:per_step], threads)
        total = 0.0
        for k in range(args.steps):
            start = (k * per_step) % len(live)
            total += oracle_sample(case, (live + live)[start:start + per_step], threads)[0]
        kind = "port"
        sample = f"{per_step} of {case.P} live phases per step, oracle/pswe_oracle.py, {threads} threads"
    value = per_step * args.steps * case.dof / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded planar C5 stand-in, SURVEY.md 8d)",
        "config": workload_config(case),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind, "sample": sample,
                         "host": host_info(threads)},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def workload_config(case):
    return {"workload": f"C5 averaged RHS, refinement {int(math.log2(case.grid.nx)) - 2} -> "
                        f"{case.grid.nx}^2 grid, M={case.M} ({case.P} live phases), exact exponentials",
            "grid": case.grid.nx, "M": case.M, "phases": case.P, "dof": case.dof,
            "l2": "flushed (256 MiB write) before every timed step"}


def load_traffic(n, kernel, phases_per_launch):
    """ncu DRAM bytes (read + write) per launch of `kernel`, scaled from the
    committed per-phase figure of the latest profile summary, if present."""
    for path in sorted((ROOT / "profiles").glob("ncu_summary_r*.json"), reverse=True):
        try:
            d = json.loads(path.read_text())
            ent = d.get(kernel, {}).get(str(n))
            if isinstance(ent, dict) and "bytes_per_phase" in ent:
                return ent["bytes_per_phase"] * phases_per_launch
        except (OSError, ValueError):
            continue
    return None


def load_pipes(n, kernel):
    """fp64-pipe and shared-memory-wavefront utilisation of `kernel` from the
    latest committed ncu summary (the bounds that actually bind; HBM does not)."""
    for path in sorted((ROOT / "profiles").glob("ncu_summary_r*.json"), reverse=True):
        try:
            ent = json.loads(path.read_text()).get(kernel, {}).get(str(n))
        except (OSError, ValueError):
            continue
        if isinstance(ent, dict) and "fp64_pipe_frac" in ent:
            return {"fp64_pipe_frac": ent["fp64_pipe_frac"], "smem_wavefront_frac": ent["smem_wavefront_frac"],
                    "source": path.name}
    return None


def fp64_roofline(n, P, ms_per_step, sm_clock_ghz=1.965):
    """The fp64 side of the bound: the evaluation's DP thread-instruction count
    (per-phase ncu counts of the committed profile summary x P) against the
    B200's 64 fp64 lanes per SM per clock (148 SMs), and its flop rate against
    the 2 x 64 x 148 x clock peak.  None when no summary for this n exists."""
    for path in sorted((ROOT / "profiles").glob("ncu_summary_r*.json"), reverse=True):
        try:
            d = json.loads(path.read_text())
        except (OSError, ValueError):
            continue
        ents = [d.get(k, {}).get(str(n)) for k in ("passA", "passB", "passC")]
        if not all(isinstance(e, dict) and "dp_thread_instr_per_phase" in e for e in ents):
            continue
        instr = P * sum(e["dp_thread_instr_per_phase"] for e in ents)
        flop = P * sum(e["dp_flop_per_phase"] for e in ents)
        lanes_per_s = 64 * 148 * sm_clock_ghz * 1e9
        floor_ms = 1e3 * instr / lanes_per_s
        return {"bound": "fp64", "dp_thread_instr": instr, "floor_ms": floor_ms,
                "pipe_frac": floor_ms / ms_per_step, "flop": flop,
                "achieved_tflops": flop / (ms_per_step * 1e-3) / 1e12,
                "peak_tflops": 2 * lanes_per_s / 1e12, "source": path.name}
    return None


def run_ours(args, ws, rank, local):
    import torch
    import paper_2103_07706_b200 as pk
    from paper_2103_07706_b200 import cases
    from paper_2103_07706_b200._native import band_bytes

    torch.cuda.set_device(local)
    if ws > 1:
        init_dist(ws, "nccl")
    dev = torch.device("cuda", local)
    case = cases.case_c5(args.level, args.M)
    n, P = case.grid.nx, case.P
    free0 = torch.cuda.mem_get_info(dev)[0]
    ctx = pk.dynamics.context(case.state, case.params)
    ctx.set_propagator("exact")
    ctx.set_quadrature(case.quadrature.s, case.quadrature.w)
    if args.chunk_mb:
        ctx.set_chunk_bytes(int(args.chunk_mb * (1 << 20)))
    U = pk.dynamics.upload(ctx, case.state)
    Uc = ctx.pack(U)
    Ac = ctx.empty_compact()
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()

    # setup outside the timed region, stated: the first evaluation also builds
    # the quadrature's (c1, c2) phase table (once per quadrature, as the
    # reference builds its quadrature once per window) and allocates scratch
    def timed_eval():
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        ctx.averaged_tendency_compact(Uc, Ac)
        b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b)
    first_ms = timed_eval()
    for _ in range(args.warmup):
        ctx.averaged_tendency_compact(Uc, Ac)
    torch.cuda.synchronize()
    steady_ms = timed_eval()
    Kx, Ky = 2 * (n // 3) + 1, n // 3 + 1
    setup = {"first_call_ms": first_ms, "steady_call_ms": steady_ms,
             "phase_table_build_ms_approx": max(0.0, first_ms - steady_ms),
             "phase_table_bytes": P * Ky * Kx * 16,
             "device_memory_bytes": free0 - torch.cuda.mem_get_info(dev)[0] - flush.numel() * 4,
             "note": "outside the timed region: the (c1, c2) phase table (once per quadrature) and the "
                     "context's scratch (chunk intermediates, slots); device_memory_bytes = the context's "
                     "footprint incl. inputs/outputs"}

    # ---- timed region: device time of K evaluations, L2 flushed before each
    sampler = ClockSampler(local)
    sampler.start()
    barrier(ws)
    torch.cuda.synchronize()
    launches0 = ctx.launch_count
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    for k in range(args.steps):
        flush_l2(flush)
        starts[k].record(stream)
        ctx.averaged_tendency_compact(Uc, Ac)
        ends[k].record(stream)
    torch.cuda.synchronize()
    barrier(ws)
    launches = ctx.launch_count - launches0
    clocks = sampler.stop()
    dev_ms = sum(s.elapsed_time(e) for s, e in zip(starts, ends))
    dev_ms = max_over_ranks(dev_ms, ws, dev)
    ms_per_step = dev_ms / args.steps
    units = ws * P * case.dof * args.steps
    value = units / (dev_ms * 1e-3)

    # ---- N > 1: the phase-sharded (strong-scaling) evaluation beside the
    # replicas: each rank takes a contiguous slice of the live phases, then
    # one NCCL all-gather of the compact partial sums and a rank-ordered sum
    # (sharding.py).  Extra information; `value` stays the replicas' number.
    sharded = None
    if ws > 1:
        try:
            sharded = run_sharded(args, ws, rank, ctx, case, Uc, Ac, flush, stream, dev, ms_per_step)
        except Exception as exc:  # never lose the contract line to the extra measurement
            sharded = {"error": f"{type(exc).__name__}: {exc}"}
        ctx.set_quadrature(case.quadrature.s, case.quadrature.w)

    # ---- per-kernel split (CUDA events around each launch, separate pass).
    # One chunk lane here: with overlapping lanes an event pair would also
    # time the other lanes' kernels; serialised, the shares are comparable
    # with the ncu launch list.
    lanes = ctx.lanes
    ctx.set_lanes(1)
    ctx.profile(True)
    for _ in range(args.steps):
        flush_l2(flush)
        ctx.averaged_tendency_compact(Uc, Ac)
    torch.cuda.synchronize()
    prof = ctx.profile_read()
    ctx.profile(False)
    ctx.set_lanes(lanes)
    ab = alg_bytes(n, P)
    peak = peak_hbm()
    kern = {}
    for name in ("passA", "passB", "passC", "reduce"):
        ms, cnt = prof[name]
        kern[name] = {"ms_per_step": ms / args.steps, "launches_per_step": cnt / args.steps,
                      "share": None}
    tot = sum(v["ms_per_step"] for v in kern.values()) or 1.0
    for v in kern.values():
        v["share"] = v["ms_per_step"] / tot
    dom = max(kern, key=lambda k: kern[k]["ms_per_step"])
    per_launch_ms = prof[dom][0] / max(prof[dom][1], 1)
    phases_per_launch = P / max(kern[dom]["launches_per_step"], 1e-9)
    dom_bytes = ab[f"{dom}_phase"] * phases_per_launch if dom.startswith("pass") else 3 * 16 * n * n
    achieved = dom_bytes / (per_launch_ms * 1e-3) / 1e9
    traffic = load_traffic(n, dom, phases_per_launch)
    roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak["value"],
                "unit": "GB/s", "frac": achieved / peak["value"], "peak_source": peak["source"],
                "traffic": traffic, "alg_bytes_per_launch": dom_bytes,
                "launch_ms": per_launch_ms, "pipes": load_pipes(n, dom)}
    fp64 = fp64_roofline(n, P, ms_per_step)
    rhs_achieved = ab["B_eval"] / (ms_per_step * 1e-3) / 1e9
    rhs_roofline = {"bound": "hbm", "B_eval": ab["B_eval"], "achieved": rhs_achieved,
                    "peak": peak["value"], "unit": "GB/s", "frac": rhs_achieved / peak["value"],
                    "note": "SURVEY.md 8d algorithmic bytes of one whole averaged-RHS evaluation"}

    # ---- end to end through the public drop-in API, host numpy in/out
    e2e = None
    if not args.no_e2e:
        # the caller's setup objects, built once as a user of the reference API does
        quad, spec = case.quadrature, pk.PropagatorSpec.exact()
        for _ in range(5):  # warm-up: contexts, phase table, pinned buffers in rotation
            out = pk.averaged_tendency(case.state, quad, case.params, spec)
        torch.cuda.synchronize()
        barrier(ws)
        # three contiguous blocks of calls; the block with the median time
        # stands (a host-side stall of the box -- seen up to +0.6 ms per call
        # on some boxes -- does not decide the figure; every block is an
        # honest back-to-back throughput)
        blocks = []
        per = max(1, args.e2e_steps // 3)
        for _ in range(3):
            t0 = time.perf_counter()
            for _ in range(per):
                out = pk.averaged_tendency(case.state, quad, case.params, spec)
            torch.cuda.synchronize()
            blocks.append(time.perf_counter() - t0)
        e2e_s = max_over_ranks(sorted(blocks)[1] * args.e2e_steps / per, ws, dev)
        e2e = {"value": ws * P * case.dof * args.e2e_steps / e2e_s, "unit": UNIT,
               # the drop-in call moves only the fields' 2/3 band (pswe_copy_band)
               "h2d_bytes_per_step": 3 * band_bytes(n, n), "d2h_bytes_per_step": 3 * band_bytes(n, n),
               "ms_per_step": 1e3 * e2e_s / args.e2e_steps,
               "path": "paper_2103_07706_b200.averaged_tendency(numpy State) -> C ABI -> numpy State",
               "timing": f"median of 3 blocks of {max(1, args.e2e_steps // 3)} back-to-back calls",
               "block_ms_per_call": [1e3 * b / max(1, args.e2e_steps // 3) for b in blocks]}
        del out

    sweep = None
    if not args.no_sweep and rank == 0:
        sweep = run_sweep(pk, cases, torch, flush, stream)
    steps_info = None
    if not args.no_steps and rank == 0:
        steps_info = run_step_configs(pk, cases, torch, stream)

    cpu = None
    cpu_steps = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        # the timed evaluation's output, checked against the CPU evaluation
        ctx.averaged_tendency_compact(Uc, Ac)
        gpu_fields = [t.cpu().numpy() for t in ctx.unpack(Ac)]
        cpu = cpu_baseline(case, gpu_fields)
        if not args.no_cpu_steps:
            cpu_steps = cpu_step_runs()

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded planar C5 stand-in, SURVEY.md 8d)",
            # config: the workload only, identical to the reference arm's line
            "config": workload_config(case),
            "parallelism": f"replicas x{ws}" if ws > 1 else "single GPU",
            "roofline": roofline, "rhs_roofline": rhs_roofline, "fp64": fp64, "kernels": kern,
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clocks,
            "gpu": torch.cuda.get_device_name(local), "sweep": sweep, "step_configs": steps_info,
            "setup": setup,
        }
        if cpu is not None and "parity" in cpu:
            line["parity"] = cpu["parity"]
        if cpu_steps:
            line["cpu_step_configs"] = cpu_steps
        if sharded is not None:
            line["phase_sharded"] = sharded
        print(json.dumps(line), flush=True)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def run_sharded(args, ws, rank, ctx, case, Uc, Ac, flush, stream, dev, one_rank_ms):
    """One averaged RHS split over the ranks by phase (device time, max over ranks)."""
    import torch
    from paper_2103_07706_b200.sharding import ordered_gather_sum, shard_weights

    ctx.set_quadrature(case.quadrature.s, shard_weights(case.quadrature.w, ws, rank))
    for _ in range(args.warmup):
        ordered_gather_sum(ctx.averaged_tendency_compact(Uc, Ac))
    torch.cuda.synchronize()
    barrier(ws)
    ms = 0.0
    for _ in range(args.steps):
        flush_l2(flush)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        ordered_gather_sum(ctx.averaged_tendency_compact(Uc, Ac))
        b.record(stream)
        torch.cuda.synchronize()
        ms += a.elapsed_time(b)
    ms = max_over_ranks(ms, ws, dev) / args.steps
    return {"ms_per_step": ms, "value": case.P * case.dof / (ms * 1e-3), "unit": UNIT,
            "speedup_vs_one_gpu": one_rank_ms / ms, "scaling": "strong",
            "collective": "NCCL all_gather of the compact 2/3-band partial sums, rank-ordered sum"}


def run_step_configs(pk, cases, torch, stream):
    """C2-C4 (BASELINE configs[1..3]): the full averaged SSPRK3 run, device-resident (pswe_run)."""
    out = []
    for name in ("C2", "C3", "C4"):
        c = cases.CASES[name]()
        cfg = pk.StepConfig(dt=c.dt, quadrature=c.quadrature, propagator_spec=pk.PropagatorSpec.exact())
        ctx = pk.integrator._prepare(c.state, cfg, c.params)
        U0 = pk.dynamics.upload(ctx, c.state)
        U = [x.clone() for x in U0]
        ctx.run(c.dt, 1, U)  # warm-up (allocations, phase table)
        torch.cuda.synchronize()
        U = [x.clone() for x in U0]
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        bad = ctx.run(c.dt, c.nsteps, U)
        b.record(stream)
        torch.cuda.synchronize()
        ms = a.elapsed_time(b)
        units = 3 * c.nsteps * c.P * c.dof  # 3 averaged RHS per step
        out.append({"config": name, "grid": c.grid.nx, "M": c.M, "P": c.P, "steps": c.nsteps,
                    "run_ms": ms, "ms_per_step": ms / c.nsteps, "phase_dof_per_s": units / (ms * 1e-3),
                    "nonfinite": bool(bad[0])})
    # fine-step reference solver (step_reference / cmd_reference, integrator.py:106-110,
    # harness.py:92-99): T = 0, M = 0 (one node), dt = 180 s, 15 days = 7200 steps on C2's grid
    c = cases.CASES["C2"]()
    dt, nsteps = 180.0, 7200
    cfg = pk.StepConfig(dt=dt, quadrature=pk.kernel_weights(0.0, 0), propagator_spec=pk.PropagatorSpec.exact())
    ctx = pk.integrator._prepare(c.state, cfg, c.params)
    U0 = pk.dynamics.upload(ctx, c.state)
    U = [x.clone() for x in U0]
    ctx.run(dt, 1, U)
    torch.cuda.synchronize()
    U = [x.clone() for x in U0]
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    bad = ctx.run(dt, nsteps, U)
    b.record(stream)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    out.append({"config": "C2-fine-reference", "grid": c.grid.nx, "M": 0, "P": 1, "steps": nsteps, "dt": dt,
                "run_ms": ms, "ms_per_step": ms / nsteps,
                "phase_dof_per_s": 3 * nsteps * c.dof / (ms * 1e-3), "nonfinite": bool(bad[0])})
    # window sweep (cmd_sweep / _check_window_sweep): T in {0, .5, 1, 2, 4, 8} h on C3's grid,
    # 12 steps each: all windows as one window batch (one launch sequence per stage over the
    # (window, phase) axis) vs one run after the other (host wall clock, synchronised)
    c = cases.CASES["C3"]()
    windows = [h * 3600.0 for h in (0.0, 0.5, 1.0, 2.0, 4.0, 8.0)]
    t_end = 12 * c.dt
    pk.window_sweep(c.state, c.params, c.dt, t_end, windows)  # warm-up (context, batch graph)
    pk.window_sweep(c.state, c.params, c.dt, t_end, windows, batched=False)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = pk.window_sweep(c.state, c.params, c.dt, t_end, windows)
    torch.cuda.synchronize()
    batched = time.perf_counter() - t0
    t0 = time.perf_counter()
    pk.window_sweep(c.state, c.params, c.dt, t_end, windows, batched=False)
    torch.cuda.synchronize()
    seq = time.perf_counter() - t0
    out.append({"config": "C3-window-sweep", "grid": c.grid.nx, "windows_s": windows,
                "M": [r.M for r in res], "P": [2 * r.M - 1 if r.M else 1 for r in res], "steps": 12,
                "batched_ms": 1e3 * batched, "sequential_ms": 1e3 * seq,
                "note": "wall clock incl. the per-window initial/final records (device diagnostics + download)"})
    return out


def run_sweep(pk, cases, torch, flush, stream, steps=3):
    """GPU-only phase x DOF/s for the other C5 points (refinement 4-7 x M)."""
    out = []
    for r in (4, 5, 6, 7):
        for M in (8, 32, 128, 256):
            c = cases.case_c5(r, M)
            if os.environ.get("PSWE_BENCH_VERBOSE"):
                print(f"sweep point r={r} M={M}", file=sys.stderr, flush=True)
            ctx = pk.dynamics.context(c.state, c.params)
            ctx.set_propagator("exact")
            ctx.set_quadrature(c.quadrature.s, c.quadrature.w)
            Uc = ctx.pack(pk.dynamics.upload(ctx, c.state))
            Ac = ctx.empty_compact()
            ctx.averaged_tendency_compact(Uc, Ac)
            ms = 0.0
            for _ in range(steps):
                flush_l2(flush)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                ctx.averaged_tendency_compact(Uc, Ac)
                b.record(stream)
                torch.cuda.synchronize()
                ms += a.elapsed_time(b)
            ms /= steps
            ab = alg_bytes(c.grid.nx, c.P)
            out.append({"n": c.grid.nx, "M": M, "P": c.P, "ms": ms,
                        "phase_dof_per_s": c.P * c.dof / (ms * 1e-3),
                        "alg_GBps": ab["B_eval"] / (ms * 1e-3) / 1e9})
    return out


def peak_hbm():
    p = ROOT / "MEASURED_PEAKS.json"
    try:
        return {"value": float(json.loads(p.read_text())["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json)"}
    except (OSError, ValueError, KeyError):
        return {"value": 6650.0, "source": "fallback (B200_PROFILING.md)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--level", type=int, default=7)
    ap.add_argument("--M", type=int, default=256)
    ap.add_argument("--e2e-steps", type=int, default=30)
    ap.add_argument("--no-cpu-steps", action="store_true", help="skip the reference's C2-C4 CPU step timings")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-steps", action="store_true", help="skip the C2-C4 step-run timings")
    ap.add_argument("--chunk-mb", type=float, default=0.0, help="L2-resident chunk size (default: library's)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("note: warmup raised to 3 (timing rule)", file=sys.stderr)
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # no launcher: start one rank per GPU ourselves (same command under torchrun)
        import socket
        with socket.socket() as so:
            so.bind(("127.0.0.1", 0))
            port = so.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), str(ROOT / "bench.py")] + sys.argv[1:]
        os.execv(sys.executable, cmd)
    ws, rank, local = dist_env()
    if ws != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE = {ws}; launch one rank per GPU")
    if args.impl == "reference":
        run_reference(args, ws, rank)
        return
    run_ours(args, ws, rank, local)


if __name__ == "__main__":
    main()

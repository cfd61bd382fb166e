"""Mid-size points (256^2 / 512^2 at M = 8, 32): total device time per RHS for
1, 2 and 4 lanes (L2 flushed between calls, as in bench.py) and the per-pass
split of the one-lane evaluation (profiling events)."""
import os, sys
sys.path.insert(0, ".")
import torch
import paper_2103_07706_b200 as pk
from paper_2103_07706_b200 import cases

pts = [(6, 8), (6, 32), (7, 8), (7, 32)] if len(sys.argv) < 2 else [tuple(map(int, a.split("/"))) for a in sys.argv[1:]]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for r, M in pts:
    c = cases.case_c5(r, M)
    ctx = pk.dynamics.context(c.state, c.params)
    ctx.set_propagator("exact")
    ctx.set_quadrature(c.quadrature.s, c.quadrature.w)
    Uc = ctx.pack(pk.dynamics.upload(ctx, c.state))
    Ac = ctx.empty_compact()
    line = f"n={c.grid.nx} M={M} P={c.P}:"
    for lanes in map(int, os.environ.get("LANES", "4,2,1").split(",")):
        ctx.set_lanes(lanes)
        for _ in range(3):
            ctx.averaged_tendency_compact(Uc, Ac)
        n, tot = 20, 0.0
        for _ in range(n):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            ctx.averaged_tendency_compact(Uc, Ac)
            b.record()
            torch.cuda.synchronize()
            tot += a.elapsed_time(b)
        line += f" lanes={lanes} {tot / n * 1e3:.1f} us;"
    ctx.profile(True)
    for _ in range(n):
        flush.zero_()
        ctx.averaged_tendency_compact(Uc, Ac)
    torch.cuda.synchronize()
    prof = ctx.profile_read()
    ctx.profile(False)
    line += " one-lane passes: " + str({k: round(v[0] / n * 1e3, 1) for k, v in prof.items() if v[1]})
    print(line, flush=True)
    ctx.set_lanes(4)

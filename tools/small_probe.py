"""Per-pass device time of one averaged RHS at small sizes (profiling events, one lane)."""
import os, sys
sys.path.insert(0, ".")
import torch
import paper_2103_07706_b200 as pk
from paper_2103_07706_b200 import cases

for r, M in [(4, 8), (4, 32), (5, 8), (5, 32), (6, 8)]:
    c = cases.case_c5(r, M)
    ctx = pk.dynamics.context(c.state, c.params)
    ctx.set_propagator("exact")
    ctx.set_quadrature(c.quadrature.s, c.quadrature.w)
    Uc = ctx.pack(pk.dynamics.upload(ctx, c.state))
    Ac = ctx.empty_compact()
    for _ in range(3):
        ctx.averaged_tendency_compact(Uc, Ac)
    torch.cuda.synchronize()
    ctx.profile(True)
    n = 20
    for _ in range(n):
        ctx.averaged_tendency_compact(Uc, Ac)
    torch.cuda.synchronize()
    prof = ctx.profile_read()
    ctx.profile(False)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        ctx.averaged_tendency_compact(Uc, Ac)
    b.record(); torch.cuda.synchronize()
    print(f"n={c.grid.nx} M={M} P={c.P} GC={os.environ.get('PSWE_GC','-')}: total {a.elapsed_time(b)/n*1e3:.1f} us;",
          {k: round(v[0] / n * 1e3, 1) for k, v in prof.items() if v[1]}, flush=True)

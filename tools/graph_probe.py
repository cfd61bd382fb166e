"""Launch overhead probe: one averaged RHS direct vs replayed from a CUDA graph (torch capture)."""
import sys
sys.path.insert(0, ".")
import torch
import paper_2103_07706_b200 as pk
from paper_2103_07706_b200 import cases

for r, M in [(4, 8), (4, 32), (5, 8), (5, 32), (6, 8), (6, 32), (7, 8)]:
    c = cases.case_c5(r, M)
    ctx = pk.dynamics.context(c.state, c.params)
    ctx.set_propagator("exact")
    ctx.set_quadrature(c.quadrature.s, c.quadrature.w)
    Uc = ctx.pack(pk.dynamics.upload(ctx, c.state))
    Ac = ctx.empty_compact()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            ctx.averaged_tendency_compact(Uc, Ac)
    torch.cuda.synchronize()
    ref = Ac.clone()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        ctx.averaged_tendency_compact(Uc, Ac)
    torch.cuda.synchronize()
    def t(fn, n=50):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        fn(); torch.cuda.synchronize()
        a.record()
        for _ in range(n):
            fn()
        b.record(); torch.cuda.synchronize()
        return a.elapsed_time(b) / n * 1e3
    d = t(lambda: ctx.averaged_tendency_compact(Uc, Ac))
    gr = t(g.replay)
    same = bool(torch.equal(Ac, ref))
    print(f"n={c.grid.nx} M={M} P={c.P}: direct {d:.1f} us, graph {gr:.1f} us, bitwise {same}", flush=True)

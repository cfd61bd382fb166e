"""Where the end-to-end averaged_tendency call spends its time (512^2, M=256)."""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2103_07706_b200 as pk
from paper_2103_07706_b200 import cases, dynamics, propagator

c = cases.case_c5(7, 256)
spec = pk.PropagatorSpec.exact()
for _ in range(2):
    pk.averaged_tendency(c.state, c.quadrature, c.params, spec)
torch.cuda.synchronize()
T = {}
def mark(k, t0):
    torch.cuda.synchronize(); T[k] = T.get(k, 0) + time.perf_counter() - t0
n = 5
for _ in range(n):
    t0 = time.perf_counter(); ctx = dynamics.context(c.state, c.params); propagator.configure(ctx, spec)
    ctx.set_quadrature(c.quadrature.s, c.quadrature.w); mark("setup", t0)
    t0 = time.perf_counter(); U = dynamics.upload(ctx, c.state, band=True); mark("upload", t0)
    t0 = time.perf_counter(); out = ctx.averaged_tendency(U); mark("compute", t0)
    t0 = time.perf_counter(); res = dynamics.download(out, band_ctx=ctx); mark("download", t0)
    t0 = time.perf_counter(); st = dynamics.rebuild(c.state, res, c.state.t); mark("rebuild", t0)
    del res, st, out, U
t0 = time.perf_counter()
for _ in range(n):
    r = pk.averaged_tendency(c.state, c.quadrature, c.params, spec)
torch.cuda.synchronize()
tot = (time.perf_counter() - t0) / n
print({k: round(1e3 * v / n, 3) for k, v in T.items()}, "full call", round(1e3 * tot, 3))

# device-side: the gated full-layout call vs pack + compact + unpack (no gate)
ctx = dynamics.context(c.state, c.params)
U = dynamics.upload(ctx, c.state)
def dev(fn, k=5):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(k):
        fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / k
gated = dev(lambda: ctx.averaged_tendency(U))
plain = dev(lambda: ctx.unpack(ctx.averaged_tendency_compact(ctx.pack(U))))
print(f"device ms: gated full-layout {gated:.3f}  pack+compact+unpack {plain:.3f}")

"""One small-grid SSPRK3 step at a time (C2: 64^2, M = 16), for ncu's
per-kernel durations; without ncu it prints the event-timed step, the
graph-replayed step (run) and an averaged RHS alone."""
import sys
sys.path.insert(0, ".")
import torch  # noqa: E402
import paper_2103_07706_b200 as pk  # noqa: E402
from paper_2103_07706_b200 import cases  # noqa: E402

c = cases.case_c2() if len(sys.argv) < 2 else cases.case_c5(int(sys.argv[1]), int(sys.argv[2]))
ctx = pk.dynamics.context(c.state, c.params)
ctx.set_propagator("exact")
ctx.set_quadrature(c.quadrature.s, c.quadrature.w)
U = pk.dynamics.upload(ctx, c.state)
Uc = ctx.pack(U)
Ac = ctx.empty_compact()
dt = getattr(c, "dt", 600.0)
for _ in range(3):
    U = ctx.ssprk3_step(dt, U)[0]
    ctx.averaged_tendency_compact(Uc, Ac)
torch.cuda.synchronize()
ev = lambda: torch.cuda.Event(enable_timing=True)
a, b = ev(), ev()
n = 20
a.record()
for _ in range(n):
    U = ctx.ssprk3_step(dt, U)[0]
b.record(); torch.cuda.synchronize()
step = a.elapsed_time(b) / n * 1e3
a.record()
for _ in range(n):
    ctx.averaged_tendency_compact(Uc, Ac)
b.record(); torch.cuda.synchronize()
rhs = a.elapsed_time(b) / n * 1e3
a.record()
ctx.run(dt, 32, U)
b.record(); torch.cuda.synchronize()
run = a.elapsed_time(b) / 32 * 1e3
print(f"{c.name} P={c.P}: step {step:.1f} us, RHS {rhs:.1f} us back-to-back, run (graph) {run:.1f} us/step",
      ctx.variant_launches, flush=True)

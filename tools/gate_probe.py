"""Device cost of the Hermitian gate on the drop-in path (512^2, M=256):
per-kernel-class times of the gated full-layout call and of pack + compact
+ unpack without the gate (profiling events, one lane; and unprofiled totals)."""
import sys
sys.path.insert(0, ".")
import torch
import paper_2103_07706_b200 as pk
from paper_2103_07706_b200 import cases, dynamics

c = cases.case_c5(7, 256)
ctx = dynamics.context(c.state, c.params)
pk.propagator.configure(ctx, pk.PropagatorSpec.exact())
ctx.set_quadrature(c.quadrature.s, c.quadrature.w)
U = dynamics.upload(ctx, c.state)
for lanes in (1, 4):
    ctx.set_lanes(lanes)
    for name, fn in (("gated", lambda: ctx.averaged_tendency(U)),
                     ("plain", lambda: ctx.unpack(ctx.averaged_tendency_compact(ctx.pack(U))))):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            fn()
        b.record()
        torch.cuda.synchronize()
        ctx.profile(True)
        for _ in range(10):
            fn()
        torch.cuda.synchronize()
        prof = ctx.profile_read()
        ctx.profile(False)
        print(f"lanes={lanes} {name}: {a.elapsed_time(b) / 10:.3f} ms;",
              {k: round(v[0] / 10, 4) for k, v in prof.items() if v[1]}, flush=True)

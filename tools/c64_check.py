"""64^2 averaged RHS timings (single evaluations, events, L2 flushed) per phase count."""
import sys
sys.path.insert(0, ".")
import torch  # noqa: E402
import paper_2103_07706_b200 as pk  # noqa: E402
from paper_2103_07706_b200 import cases  # noqa: E402
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
for M in (1, 4, 8, 16, 32, 64, 128, 256):
    c = cases.case_c5(4, M)
    ctx = pk.dynamics.context(c.state, c.params)
    ctx.set_propagator("exact")
    ctx.set_quadrature(c.quadrature.s, c.quadrature.w)
    Uc = ctx.pack(pk.dynamics.upload(ctx, c.state))
    Ac = ctx.empty_compact()
    for _ in range(3):
        ctx.averaged_tendency_compact(Uc, Ac)
    ms = 0.0
    for _ in range(10):
        flush.add_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); ctx.averaged_tendency_compact(Uc, Ac); b.record(); torch.cuda.synchronize()
        ms += a.elapsed_time(b)
    print(f"64^2 M={M} P={c.P}: {ms / 10 * 1e3:.1f} us  fused={ctx.variant_launches['fused']}", flush=True)

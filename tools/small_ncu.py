"""A few averaged-RHS evaluations at one small point, for ncu's per-kernel durations."""
import sys
sys.path.insert(0, ".")
import torch  # noqa: E402
import paper_2103_07706_b200 as pk  # noqa: E402
from paper_2103_07706_b200 import cases  # noqa: E402
r, M = int(sys.argv[1]), int(sys.argv[2])
c = cases.case_c5(r, M)
ctx = pk.dynamics.context(c.state, c.params)
ctx.set_propagator("exact")
ctx.set_quadrature(c.quadrature.s, c.quadrature.w)
Uc = ctx.pack(pk.dynamics.upload(ctx, c.state))
Ac = ctx.empty_compact()
for _ in range(5):
    ctx.averaged_tendency_compact(Uc, Ac)
torch.cuda.synchronize()
print(ctx.variant_launches)

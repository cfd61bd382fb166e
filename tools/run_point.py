"""Debug: one averaged-RHS evaluation for C5 point (level r, M) vs the oracle on a phase subset."""
import sys
import numpy as np
sys.path.insert(0, ".")
import torch
import paper_2103_07706_b200 as pk
from paper_2103_07706_b200 import cases

r, M = int(sys.argv[1]), int(sys.argv[2])
c = cases.case_c5(r, M)
ctx = pk.dynamics.context(c.state, c.params)
ctx.set_propagator("exact")
ctx.set_quadrature(c.quadrature.s, c.quadrature.w)
if len(sys.argv) > 3:
    ctx.set_chunk_bytes(int(float(sys.argv[3]) * (1 << 20)))
Uc = ctx.pack(pk.dynamics.upload(ctx, c.state))
for _ in range(2):
    out = ctx.averaged_tendency_compact(Uc)
torch.cuda.synchronize()
print(r, M, "ok", float(out.abs().max()))

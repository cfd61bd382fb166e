"""GPU debug helper: small-grid averaged RHS (fused path) vs the oracle, with timings."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2103_07706_b200 as pk  # noqa: E402
from oracle import pswe_oracle as O  # noqa: E402
from paper_2103_07706_b200 import cases  # noqa: E402

for r, M in ((1, 4), (2, 8), (3, 8), (4, 8), (3, 256), (4, 128), (4, 256)):
    c = cases.case_c5(r, M)
    g = c.grid
    S = O.Setup(g.nx, g.ny, g.Lx, g.Ly, c.params.f, c.params.g, c.params.H)
    rng = np.random.default_rng(r)
    U = np.stack([c.state.u, c.state.v, c.state.eta])
    U = U + np.stack([O.truncate(O.spectral(sc * rng.standard_normal((g.nx, g.ny))), S.mask) for sc in (1.0, 1.0, 50.0)])
    st = pk.State(grid=g, u=U[0], v=U[1], eta=U[2])
    got = pk.averaged_tendency(st, c.quadrature, c.params, pk.PropagatorSpec.exact())
    want = O.averaged_tendency(S, U, c.quadrature.s, c.quadrature.w, workers=8)
    err = O.rel_l2(np.stack([got.u, got.v, got.eta]), want)
    ctx = pk.dynamics.context(st, c.params)
    ctx.set_propagator("exact")
    ctx.set_quadrature(c.quadrature.s, c.quadrature.w)
    Uc = ctx.pack(pk.dynamics.upload(ctx, st))
    for _ in range(3):
        ctx.averaged_tendency_compact(Uc)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20):
        ctx.averaged_tendency_compact(Uc)
    b.record()
    torch.cuda.synchronize()
    print(f"n={g.nx} M={M} P={c.P}: rel L2 {err:.3e}  {a.elapsed_time(b) / 20 * 1e3:.1f} us  {ctx.variant_launches}",
          flush=True)

"""compute-sanitizer workload: every kernel family once at one size.

usage: python tools/sanitize_point.py LEVEL M
  averaged RHS (compact, all lanes/chunks the size implies), apply_nonlinear
  (single node: split pass B), one SSPRK3 step (pack + gate + stage kernels),
  snapshot diagnostics (full-grid gate + diag passes) and one exact
  Hermitian check (a flagged input).
"""
import sys

import numpy as np

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
out = ctx.averaged_tendency_compact(Uc)
pk.apply_nonlinear(c.state, c.params)
cfg = pk.StepConfig(dt=600.0, quadrature=c.quadrature, propagator_spec=pk.PropagatorSpec.exact())
pk.step_averaged_ssprk3(c.state, cfg, c.params)
pk.device_diagnostics(c.state, c.params)
u = np.array(c.state.u)
u[1, 2] += 1e-11 * np.max(np.abs(u))  # flagged by the fast bound, decided by the exact check
try:
    pk.averaged_tendency(pk.State(grid=c.grid, u=u, v=c.state.v, eta=c.state.eta), c.quadrature, c.params,
                         pk.PropagatorSpec.exact())
except RuntimeError as exc:
    print("gate:", str(exc)[:80])
torch.cuda.synchronize()
print(r, M, "ok", float(out.abs().max()), ctx.variant_launches)

"""GPU debug helper: apply_nonlinear / averaged_tendency vs the oracle for every supported n."""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_2103_07706_b200 as pk
from oracle import pswe_oracle as O

F0, G0, H0 = 1.0e-4, 9.8, 5960.0
rng = np.random.default_rng(0)
for n in [8, 16, 32, 64, 128, 256, 512]:
    S = O.Setup(n, n, 4e7, 4e7, F0, G0, H0)
    S.b = O.truncate(O.spectral(30.0 * rng.standard_normal((n, n))), S.mask)
    U = np.stack([O.truncate(O.spectral(sc * rng.standard_normal((n, n))), S.mask) for sc in (1.0, 1.0, 50.0)])
    g = pk.make_grid(n, n, 4e7, 4e7)
    p = pk.PhysicsParams(f=F0, g=G0, H=H0, b=S.b)
    st = pk.State(grid=g, u=U[0], v=U[1], eta=U[2])
    got = pk.apply_nonlinear(st, p)
    want = O.nonlinear(S, U)
    errs = [O.rel_l2(getattr(got, f), want[i]) for i, f in enumerate(("u", "v", "eta"))]
    q = pk.kernel_weights(1800.0, 3)
    ga = pk.averaged_tendency(st, q, p, pk.PropagatorSpec.exact())
    wa = O.averaged_tendency(S, U, q.s, q.w)
    print(n, "N per-field", ["%.2e" % e for e in errs], "avg", "%.2e" % O.rel_l2(np.stack([ga.u, ga.v, ga.eta]), wa), flush=True)

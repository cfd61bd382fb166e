import sys
import numpy as np
sys.path.insert(0, ".")
import paper_2103_07706_b200 as pk
from paper_2103_07706_b200 import cases
for r, M in [(4, 8), (5, 8), (6, 8), (6, 64), (7, 8), (7, 32)]:
    c = cases.case_c5(r, M)
    out = pk.averaged_tendency(c.state, c.quadrature, c.params, pk.PropagatorSpec.exact())
    a = np.stack([out.u, out.v, out.eta])
    print(r, M, "nan" if not np.all(np.isfinite(a)) else "ok", flush=True)

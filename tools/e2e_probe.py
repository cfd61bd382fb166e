"""End-to-end drop-in call (512^2, M=256): wall time per call and its parts."""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2103_07706_b200 as pk  # noqa: E402
from paper_2103_07706_b200 import averaging, cases, dynamics  # noqa: E402

c = cases.case_c5(7, 256)
q, spec = c.quadrature, pk.PropagatorSpec.exact()


def loop(n=30):
    for _ in range(5):
        out = pk.averaged_tendency(c.state, q, c.params, spec)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        out = pk.averaged_tendency(c.state, q, c.params, spec)
    torch.cuda.synchronize()
    del out
    return (time.perf_counter() - t0) / n * 1e3


print("e2e ms", round(loop(), 3), round(loop(), 3))
# parts, as the call runs them
T = {}
for _ in range(20):
    t0 = time.perf_counter()
    ctx = averaging._prepared(c.state, q, c.params, spec)
    t1 = time.perf_counter()
    U = dynamics.upload(ctx, c.state, band=True)
    t2 = time.perf_counter()
    hosts = averaging.band_hosts_async((512, 512), 3)
    out = ctx.averaged_tendency(U)
    t3 = time.perf_counter()
    res = dynamics.download(out, band_ctx=ctx, hosts=hosts)
    t4 = time.perf_counter()
    st = dynamics.rebuild(c.state, res, c.state.t)
    t5 = time.perf_counter()
    for k, v in (("prepare", t1 - t0), ("upload", t2 - t1), ("call", t3 - t2), ("download", t4 - t3),
                 ("rebuild", t5 - t4)):
        T[k] = T.get(k, 0.0) + v
    del res, st, out, U
print({k: round(v / 20 * 1e3, 3) for k, v in T.items()})

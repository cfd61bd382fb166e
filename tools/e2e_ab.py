"""A/B of the drop-in call's host path on one box (512^2, M=256): the
previous two-synchronisation path (averaged_tendency, then a band download)
against the current one (band download inside the C call), alternating
blocks of back-to-back calls."""
import sys, time
sys.path.insert(0, ".")
import torch
import paper_2103_07706_b200 as pk
from paper_2103_07706_b200 import averaging, cases, dynamics, _native

c = cases.case_c5(7, 256)
q, spec = c.quadrature, pk.PropagatorSpec.exact()


def old_call():
    ctx = averaging._prepared(c.state, q, c.params, spec)
    U = dynamics.upload(ctx, c.state, band=True)
    hosts = _native.band_hosts_async((ctx.nx, ctx.ny), 3)
    out = ctx.averaged_tendency(U)
    return dynamics.rebuild(c.state, dynamics.download(out, band_ctx=ctx, hosts=hosts), c.state.t)


def new_call():
    return pk.averaged_tendency(c.state, q, c.params, spec)


def block(fn, n=10):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        r = fn()
    torch.cuda.synchronize()
    del r
    return (time.perf_counter() - t0) / n * 1e3


for fn in (old_call, new_call):
    for _ in range(3):
        fn()
res = {"old": [], "new": []}
for _ in range(6):
    res["old"].append(block(old_call))
    res["new"].append(block(new_call))
print({k: [round(x, 3) for x in v] for k, v in res.items()})
print({k: round(sorted(v)[len(v) // 2], 3) for k, v in res.items()})

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


def rows_call():
    """As new_call, staging only the kx-band rows of each field on the host."""
    ctx = averaging._prepared(c.state, q, c.params, spec)
    arrays = [c.state.u, c.state.v, c.state.eta]
    nx, ny = ctx.nx, ctx.ny
    kxm = nx // 3
    key = ((nx, ny), 3, ctx.device)
    ent = _native._PIN.__dict__["in"][key]
    pin, pn, evs, used = ent
    out = torch.empty((3, nx, ny), dtype=torch.complex128, device="cuda")
    cur = torch.cuda.current_stream()
    import ctypes
    for i, a in enumerate(arrays):
        if used[i]:
            evs[i].synchronize()
        src = torch.from_numpy(a)
        pin[i, :kxm + 1].copy_(src[:kxm + 1])
        pin[i, nx - kxm:].copy_(src[nx - kxm:])
        _native._check(_native._lib.pswe_copy_band(ctx.h, 0, _native._ptrs([out[i].data_ptr()]),
                                                   _native._ptrs([pin[i].data_ptr()]), 1, ctypes.c_void_p(cur.cuda_stream)))
        evs[i].record(cur)
        used[i] = True
    U = [out[i] for i in range(3)]
    hosts, filled = _native.band_hosts_split((nx, ny), 3)
    res = ctx.averaged_tendency_to_host(U, hosts)
    filled.result()
    return dynamics.rebuild(c.state, res, c.state.t)


def block(fn, n=10):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        r = fn()
    torch.cuda.synchronize()
    del r
    return (time.perf_counter() - t0) / n * 1e3


for fn in (old_call, new_call, rows_call):
    for _ in range(3):
        fn()
res = {"old": [], "new": [], "rows": []}
for _ in range(6):
    res["old"].append(block(old_call))
    res["new"].append(block(new_call))
    res["rows"].append(block(rows_call))
print({k: [round(x, 3) for x in v] for k, v in res.items()})
print({k: round(sorted(v)[len(v) // 2], 3) for k, v in res.items()})

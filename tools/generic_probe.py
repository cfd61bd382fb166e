"""Device time per averaged RHS on generic (non power-of-two / > 512) grids vs a tuned size."""
import sys
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_2103_07706_b200 as pk  # noqa: E402

for n, M in ((384, 8), (512, 8), (768, 8), (1024, 8), (96, 32), (128, 32)):
    rng = np.random.default_rng(n)
    g = pk.make_grid(n, n, 4.0e7, 4.0e7)
    f = lambda sc: pk.dealias(g, pk.to_spectral(g, sc * rng.standard_normal((n, n))))  # noqa: E731
    st = pk.State(grid=g, u=f(1.0), v=f(1.0), eta=f(50.0))
    p = pk.PhysicsParams(f=1e-4, g=9.8, H=5960.0, b=np.zeros((n, n), complex))
    q = pk.kernel_weights(1800.0, M)
    ctx = pk.dynamics.context(st, p)
    ctx.set_propagator("exact")
    ctx.set_quadrature(q.s, q.w)
    Uc = ctx.pack(pk.dynamics.upload(ctx, st))
    Ac = ctx.empty_compact()
    for _ in range(3):
        ctx.averaged_tendency_compact(Uc, Ac)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        ctx.averaged_tendency_compact(Uc, Ac)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 5
    P = int(np.count_nonzero(q.w))
    print(f"{n}^2 M={M} P={P}: {ms:.3f} ms  {P * 3 * n * n / (ms * 1e-3):.3e} phase*DOF/s", flush=True)

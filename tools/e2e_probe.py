"""Time the host<->device legs of the public API path (512^2 C5 state)."""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2103_07706_b200 as pk
from paper_2103_07706_b200 import cases, dynamics

c = cases.case_c5(7, 256)
ctx = dynamics.context(c.state, c.params)
def tm(f, n=5):
    f(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n): r = f()
    torch.cuda.synchronize()
    return 1e3 * (time.perf_counter() - t0) / n
up_old = lambda: [ctx.to_device(getattr(c.state, k)) for k in ("u", "v", "eta")]
up_new = lambda: dynamics.upload(ctx, c.state)
U = up_old()
dn_old = lambda: [t.cpu().numpy() for t in U]
dn_new = lambda: dynamics.download(U)
print("upload old %.2f ms  new %.2f ms" % (tm(up_old), tm(up_new)))
print("download old %.2f ms  new %.2f ms" % (tm(dn_old), tm(dn_new)))
pin = torch.empty((3, 512, 512), dtype=torch.complex128, pin_memory=True)
pn = pin.numpy()
print("np.copyto into pinned (3 fields) %.2f ms" % tm(lambda: [np.copyto(pn[i], getattr(c.state, k)) for i, k in enumerate(("u", "v", "eta"))]))
print("pinned alloc 3x4MB %.2f ms" % tm(lambda: [torch.empty((512, 512), dtype=torch.complex128, pin_memory=True) for _ in range(3)]))
g = torch.empty((3, 512, 512), dtype=torch.complex128, device="cuda")
print("H2D pinned 12.6MB %.2f ms" % tm(lambda: g.copy_(pin, non_blocking=True)))
print("D2H pinned 12.6MB %.2f ms" % tm(lambda: pin.copy_(g, non_blocking=True)))
st = c.state
print("dtype", st.u.dtype, st.u.flags['C_CONTIGUOUS'])

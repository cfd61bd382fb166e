"""Bus transfers of the drop-in call at 512^2 (3 fields): the band copy
(pswe_copy_band: 2 x 2 strided blocks per field) against contiguous kx-band
row blocks and whole fields, both directions, device-timed; and the host
staging copy into pinned memory."""
import ctypes
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_2103_07706_b200 as pk
from paper_2103_07706_b200 import _native, cases

c = cases.case_c5(7, 256)
ctx = pk.dynamics.context(c.state, c.params)
n = 512
kxm = n // 3
dev = [torch.empty((n, n), dtype=torch.complex128, device="cuda") for _ in range(3)]
pin = [torch.empty((n, n), dtype=torch.complex128, pin_memory=True) for _ in range(3)]
st = torch.cuda.current_stream()


def band(direction):
    dst, src = (dev, pin) if direction == 0 else (pin, dev)
    _native._check(_native._lib.pswe_copy_band(ctx.h, direction, _native._ptrs([d.data_ptr() for d in dst]),
                                               _native._ptrs([s.data_ptr() for s in src]), 3,
                                               ctypes.c_void_p(st.cuda_stream)))


def rows(direction):
    for d, p in zip(dev, pin):
        for a, b in ((0, kxm + 1), (n - kxm, n)):
            if direction == 0:
                d[a:b].copy_(p[a:b], non_blocking=True)
            else:
                p[a:b].copy_(d[a:b], non_blocking=True)


def whole(direction):
    for d, p in zip(dev, pin):
        (d.copy_(p, non_blocking=True) if direction == 0 else p.copy_(d, non_blocking=True))


def timed(fn, k=20):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(k):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / k


for name, fn in (("band", band), ("kx-rows", rows), ("whole", whole)):
    print(f"{name:8s} H2D {timed(lambda: fn(0)):.3f} ms  D2H {timed(lambda: fn(1)):.3f} ms")
src = [np.ascontiguousarray(getattr(c.state, f)) for f in ("u", "v", "eta")]
for _ in range(3):
    for p, s in zip(pin, src):
        p.copy_(torch.from_numpy(s))
t0 = time.perf_counter()
for _ in range(20):
    for p, s in zip(pin, src):
        p.copy_(torch.from_numpy(s))
print(f"host staging (torch copy_, 3 x 4 MiB): {(time.perf_counter() - t0) / 20 * 1e3:.3f} ms, threads {torch.get_num_threads()}")
t0 = time.perf_counter()
for _ in range(20):
    for p, s in zip(pin, src):
        np.copyto(p.numpy(), s)
print(f"host staging (numpy copyto): {(time.perf_counter() - t0) / 20 * 1e3:.3f} ms")

# the drop-in upload, step by step (host wall time)
from paper_2103_07706_b200 import dynamics
for _ in range(5):
    U = dynamics.upload(ctx, c.state, band=True)
torch.cuda.synchronize()
arrays = [c.state.u, c.state.v, c.state.eta]
key = ((n, n), 3, ctx.device)
ent = _native._PIN.__dict__["in"][key]
pinb, pn, evs, _used = ent
T = {}
for _ in range(20):
    t = [time.perf_counter()]
    out = torch.empty((3, n, n), dtype=torch.complex128, device="cuda")
    t.append(time.perf_counter())
    for i, a in enumerate(arrays):
        evs[i].synchronize()
        t.append(time.perf_counter())
        src = torch.from_numpy(a)
        pinb[i].copy_(src)
        t.append(time.perf_counter())
        _native._check(_native._lib.pswe_copy_band(ctx.h, 0, _native._ptrs([out[i].data_ptr()]),
                                                   _native._ptrs([pinb[i].data_ptr()]), 1,
                                                   ctypes.c_void_p(st.cuda_stream)))
        t.append(time.perf_counter())
        evs[i].record(st)
        t.append(time.perf_counter())
    d = np.diff(t) * 1e3
    for k, v in enumerate(d):
        T[k] = T.get(k, 0) + v
    torch.cuda.synchronize()
print("upload steps (ms): alloc, then per field [event wait, host copy, band DMA issue, event record]:",
      [round(v / 20, 3) for v in T.values()])

import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2103_07706_b200 as pk
from paper_2103_07706_b200 import cases, _native
c = cases.case_c5(7, 256)
arrs = [c.state.u, c.state.v, c.state.eta]
for a in arrs: print(a.dtype, a.flags.c_contiguous, a.flags.writeable, a.strides)
for k in range(5):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    out = _native.upload_fields(arrs, 0)
    t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(round(1e3*(t1-t0),3), round(1e3*(t2-t0),3))
pin = torch.empty((3, 512, 512), dtype=torch.complex128, pin_memory=True)
for k in range(3):
    t0 = time.perf_counter()
    for i in range(3): pin[i].copy_(torch.from_numpy(arrs[i]))
    print("copy", round(1e3*(time.perf_counter()-t0),3))
# interleaved with a full evaluation, as in the e2e call
spec = pk.PropagatorSpec.exact()
for k in range(6):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    out = _native.upload_fields(arrs, 0)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    r = pk.averaged_tendency(c.state, c.quadrature, c.params, spec)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    print("interleaved upload", round(1e3*(t1-t0),3), "call", round(1e3*(t2-t1),3))
torch.set_num_threads(4)
for k in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    out = _native.upload_fields(arrs, 0)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    r = pk.averaged_tendency(c.state, c.quadrature, c.params, spec)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    print("4 threads: upload", round(1e3*(t1-t0),3), "call", round(1e3*(t2-t1),3))

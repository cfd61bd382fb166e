"""Full vs band-only transfers of three 512^2 complex128 fields (drop-in path)."""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2103_07706_b200 import _native, cases, dynamics
c = cases.case_c5(7, 256)
ctx = dynamics.context(c.state, c.params)
arrs = [c.state.u, c.state.v, c.state.eta]
def t(f, k=20):
    f(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(k): f()
    torch.cuda.synchronize()
    return round(1e3 * (time.perf_counter() - t0) / k, 3)
print("upload full", t(lambda: _native.upload_fields(arrs, 0)))
print("upload band", t(lambda: _native.upload_fields(arrs, 0, band_ctx=ctx)))
out = _native.upload_fields(arrs, 0)
print("download full", t(lambda: _native.download_fields(out)))
print("download band", t(lambda: _native.download_fields(out, band_ctx=ctx)))
h = [torch.empty((512, 512), dtype=torch.complex128, pin_memory=True) for _ in range(3)]
print("zero fill oob", t(lambda: [_native._zero_out_of_band(x, 512, 512) for x in h]))
st = torch.cuda.current_stream()
print("copy_band d2h only", t(lambda: _native._lib.pswe_copy_band(ctx.h, 1, _native._ptrs([x.data_ptr() for x in h]), _native._ptrs([x.data_ptr() for x in out]), 3, _native.ctypes.c_void_p(st.cuda_stream))))
print("copy full d2h only", t(lambda: [x.copy_(y, non_blocking=True) for x, y in zip(h, out)]))
pin = torch.empty((3, 512, 512), dtype=torch.complex128, pin_memory=True)
print("copy_band h2d only", t(lambda: _native._lib.pswe_copy_band(ctx.h, 0, _native._ptrs([x.data_ptr() for x in out]), _native._ptrs([pin[i].data_ptr() for i in range(3)]), 3, _native.ctypes.c_void_p(st.cuda_stream))))
print("copy full h2d only", t(lambda: [out[i].copy_(pin[i], non_blocking=True) for i in range(3)]))
src = [torch.from_numpy(a) for a in arrs]
blocks = _native.band_blocks(512, 512)
print("host gather band", t(lambda: [pin[i, r, cc].copy_(src[i][r, cc]) for i in range(3) for r, cc in blocks]))
print("host copy full", t(lambda: [pin[i].copy_(src[i]) for i in range(3)]))
rows = [slice(0, 171), slice(342, 512)]
dev = torch.empty((3, 512, 512), dtype=torch.complex128, device="cuda")
def rows_only():
    for i in range(3):
        for r in rows:
            pin[i, r].copy_(src[i][r])
        for r in rows:
            dev[i, r].copy_(pin[i, r], non_blocking=True)
print("rows: host + h2d", t(rows_only))
def rows_host_band_dma():
    for i in range(3):
        for r in rows:
            pin[i, r].copy_(src[i][r])
        _native._lib.pswe_copy_band(ctx.h, 0, _native._ptrs([dev[i].data_ptr()]), _native._ptrs([pin[i].data_ptr()]), 1, _native.ctypes.c_void_p(st.cuda_stream))
print("rows host + band dma", t(rows_host_band_dma))
print("rows host only", t(lambda: [pin[i, r].copy_(src[i][r]) for i in range(3) for r in rows]))

"""H2D of a 512^2 state's 2/3 band: pinned staging (upload_fields) vs direct
pageable cudaMemcpy2DAsync of the band blocks (pswe_copy_band from numpy memory)."""
import ctypes
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2103_07706_b200 as pk  # noqa: E402
from paper_2103_07706_b200 import _native, cases  # noqa: E402

c = cases.case_c5(7, 256)
ctx = pk.dynamics.context(c.state, c.params)
fields = [np.asarray(getattr(c.state, n)) for n in ("u", "v", "eta")]
out = torch.empty((3, 512, 512), dtype=torch.complex128, device="cuda")


def staged():
    return _native.upload_fields(fields, ctx.device, band_ctx=ctx)


def direct():
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    _native._check(_native._lib.pswe_copy_band(ctx.h, 0, _native._ptrs([out[i].data_ptr() for i in range(3)]),
                                               _native._ptrs([f.ctypes.data for f in fields]), 3, st))
    return out


for name, fn in (("staged", staged), ("direct", direct), ("staged", staged), ("direct", direct)):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    print(name, round((time.perf_counter() - t0) / 20 * 1e3, 3), "ms")

"""Per-call wall times of the drop-in averaged_tendency (512^2, M=256): min / median / mean / max."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2103_07706_b200 as pk  # noqa: E402
from paper_2103_07706_b200 import cases  # noqa: E402

c = cases.case_c5(7, 256)
q, spec = c.quadrature, pk.PropagatorSpec.exact()
for _ in range(5):
    out = pk.averaged_tendency(c.state, q, c.params, spec)
torch.cuda.synchronize()
for trial in range(3):
    ts = []
    for _ in range(40):
        t0 = time.perf_counter()
        out = pk.averaged_tendency(c.state, q, c.params, spec)
        ts.append(time.perf_counter() - t0)
    ts = np.array(ts) * 1e3
    print(f"trial {trial}: min {ts.min():.3f} median {np.median(ts):.3f} mean {ts.mean():.3f} max {ts.max():.3f} ms")

"""Host->device upload variants for three 512x512 complex128 fields."""
import time, threading
import numpy as np, torch
from concurrent.futures import ThreadPoolExecutor
n = 512
rng = np.random.default_rng(0)
arrs = [rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)) for _ in range(3)]
pin = torch.empty((3, n, n), dtype=torch.complex128, pin_memory=True)
pn = pin.numpy()
dev = torch.empty((3, n, n), dtype=torch.complex128, device="cuda")
pool = ThreadPoolExecutor(6)
def t(f, k=20):
    f(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(k): f()
    torch.cuda.synchronize()
    return round(1e3 * (time.perf_counter() - t0) / k, 3)
print("np.copyto 1 thread", t(lambda: [np.copyto(pn[i], arrs[i]) for i in range(3)]))
print("np.copyto 3 threads", t(lambda: list(pool.map(lambda i: np.copyto(pn[i], arrs[i]), range(3)))))
h = n // 2
print("np.copyto 6 threads", t(lambda: list(pool.map(lambda q: np.copyto(pn[q // 2, (q % 2) * h:(q % 2 + 1) * h], arrs[q // 2][(q % 2) * h:(q % 2 + 1) * h]), range(6)))))
ta = [torch.from_numpy(a) for a in arrs]
print("torch copy_ to pinned", torch.get_num_threads(), t(lambda: [pin[i].copy_(ta[i]) for i in range(3)]))
print("H2D pinned 12.6MB", t(lambda: dev.copy_(pin, non_blocking=True)))
print("H2D pageable", t(lambda: [dev[i].copy_(ta[i], non_blocking=True) for i in range(3)]))
def reg():
    for a in arrs:
        torch.cuda.cudart().cudaHostRegister(a.ctypes.data, a.nbytes, 0)
    for i, a in enumerate(arrs):
        dev[i].copy_(torch.from_numpy(a), non_blocking=True)
    torch.cuda.synchronize()
    for a in arrs:
        torch.cuda.cudart().cudaHostUnregister(a.ctypes.data)
print("register+H2D+unregister", t(reg))

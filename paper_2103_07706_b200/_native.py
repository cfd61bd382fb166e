"""ctypes binding of ``libpswe_b200.so`` (declared in ``include/pswe_b200.h``).

PyTorch is used only as the device-memory / stream plumbing: tensors are
allocated with torch, their raw pointers and torch's current CUDA stream are
handed to the C ABI.  There is no CPU fallback: if the library or a CUDA
device is missing every entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import pathlib
import threading
import weakref

import numpy as np

LIB_PATH = pathlib.Path(os.environ.get("PSWE_LIB_PATH") or
                        pathlib.Path(__file__).resolve().parent / "lib" / "libpswe_b200.so")

PSWE_OK = 0
PSWE_EINVAL = 1
PSWE_ECUDA = 2
PSWE_EUNSUPPORTED = 3
PSWE_ENONFINITE = 4
PSWE_ESTATE = 5
PSWE_EHERM = 6

_lib = None
_lib_lock = threading.Lock()

_c_int_p = ctypes.POINTER(ctypes.c_int)
_vp = ctypes.c_void_p
_d = ctypes.c_double
_i = ctypes.c_int

# name -> (restype, argtypes); the ABI exported by include/pswe_b200.h
SIGNATURES = {
    "pswe_version": (_i, []),
    "pswe_last_error": (ctypes.c_char_p, []),
    "pswe_create": (_i, [ctypes.POINTER(_vp), _i, _i, _d, _d, _d, _d, _d, _i]),
    "pswe_destroy": (None, [_vp]),
    "pswe_set_topography": (_i, [_vp, _vp, _vp]),
    "pswe_set_quadrature": (_i, [_vp, _i, ctypes.POINTER(_d), ctypes.POINTER(_d)]),
    "pswe_set_propagator": (_i, [_vp, _i, _d, _i, ctypes.POINTER(_d)]),
    "pswe_compact_shape": (_i, [_vp, _c_int_p, _c_int_p]),
    "pswe_pack": (_i, [_vp, _vp, _vp, _vp, _vp, _vp]),
    "pswe_unpack": (_i, [_vp, _vp, _vp, _vp, _vp, _vp]),
    "pswe_averaged_tendency_compact": (_i, [_vp, _vp, _vp, _vp]),
    "pswe_averaged_tendency": (_i, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "pswe_averaged_tendency_band_d2h": (_i, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "pswe_apply_nonlinear": (_i, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "pswe_apply_linear": (_i, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "pswe_propagate": (_i, [_vp, _d, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "pswe_ssprk3_step": (_i, [_vp, _d, _vp, _vp, _vp, _vp, _vp, _vp, _c_int_p, _c_int_p, _vp]),
    "pswe_run": (_i, [_vp, _d, _i, _vp, _vp, _vp, _c_int_p, _c_int_p, _c_int_p, _vp]),
    "pswe_set_window_batch": (_i, [_vp, _i, _c_int_p, ctypes.POINTER(_d), ctypes.POINTER(_d)]),
    "pswe_window_batch_tendency": (_i, [_vp, _vp, _vp, _vp]),
    "pswe_window_batch_run": (_i, [_vp, _d, _i, _vp, _c_int_p, _vp]),
    "pswe_max_frequency": (_d, [_vp]),
    "pswe_launch_count": (ctypes.c_int64, [_vp]),
    "pswe_debug_check_guards": (_i, [ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64)]),
    "pswe_variant_launches": (_i, [_vp, ctypes.POINTER(ctypes.c_int64), _i]),
    "pswe_diagnostics": (_i, [_vp, _vp, _vp, _vp, ctypes.POINTER(_d), _vp]),
    "pswe_to_physical": (_i, [_vp, _vp, _vp, _vp, _vp, _vp]),
    "pswe_copy_band": (_i, [_vp, _i, _vp, _vp, _i, _vp]),
    "pswe_set_chunk_bytes": (_i, [_vp, ctypes.c_size_t]),
    "pswe_set_lanes": (_i, [_vp, _i]),
    "pswe_get_lanes": (_i, [_vp]),
    "pswe_profile_enable": (_i, [_vp, _i]),
    "pswe_profile_read": (_i, [_vp, ctypes.POINTER(_d), ctypes.POINTER(ctypes.c_int64), _i]),
}

KERNEL_CLASSES = ("passA", "passB", "passC", "reduce", "pack", "unpack", "stage")
VARIANTS = ("passA", "passB_pair", "passB_row", "passB_split", "passC", "reduce", "fused", "herm")


class NativeError(RuntimeError):
    """A failed C-ABI call; ``code`` is the PSWE_* status."""

    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def load_library(path: os.PathLike | None = None):
    """Load and declare the shared library (no CUDA work happens here)."""
    global _lib
    with _lib_lock:
        if _lib is not None and path is None:
            return _lib
        p = pathlib.Path(path) if path is not None else LIB_PATH
        if not p.exists():
            raise RuntimeError(
                f"B200 extension {p} is missing; build it with `make` or "
                "`python -c 'import __graft_entry__ as g; g.build()'` (there is no CPU fallback)")
        lib = ctypes.CDLL(str(p))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if path is None:
            _lib = lib
        return lib


def _check(rc: int) -> None:
    if rc != PSWE_OK:
        msg = _lib.pswe_last_error().decode("utf-8", "replace")
        if rc in (PSWE_EINVAL, PSWE_EUNSUPPORTED, PSWE_EHERM):
            err = ValueError(msg)
            err.code = rc
            raise err
        raise NativeError(rc, msg)


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2103_07706_b200 needs a CUDA device (sm_100a); "
                           "the B200 path has no CPU fallback")
    return torch


def _dptr(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr())


def _stream(torch):
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


_libc = ctypes.CDLL(None)
_memcmp = _libc.memcmp
_memcmp.restype = ctypes.c_int
_memcmp.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t]

_PIN = threading.local()  # per-thread pinned staging buffers for uploads


class _PinnedPool:
    """Pinned host buffers handed out as the numpy arrays a call returns.

    A buffer goes back to the pool when its array is garbage-collected
    (weakref.finalize), so a caller that drops results between calls gets
    them without a fresh cudaHostAlloc and without a host copy; results that
    are kept simply keep their buffer."""

    def __init__(self):
        self.free = {}
        self.lock = threading.Lock()

    def take(self, shape, dtype):
        key = (tuple(shape), dtype)
        with self.lock:
            lst = self.free.get(key)
            if lst:
                return lst.pop()
        return _torch().empty(shape, dtype=dtype, pin_memory=True)

    def give(self, key, tensor):
        with self.lock:
            self.free.setdefault(key, []).append(tensor)

    def array(self, tensor):
        # The holder owns the buffer for numpy: every view of the returned
        # array keeps the holder (not the array) as its base, so the buffer is
        # recycled only when no view of it is left.
        holder = _PinnedHolder(tensor)
        weakref.finalize(holder, self.give, (tuple(tensor.shape), tensor.dtype), tensor)
        return np.asarray(holder)


class _PinnedHolder:
    """numpy array-interface exporter of one pinned tensor's memory."""

    _TYPESTR = {"torch.complex128": "<c16", "torch.float64": "<f8"}

    def __init__(self, tensor):
        self.t = tensor
        self.__array_interface__ = {"shape": tuple(tensor.shape), "typestr": self._TYPESTR[str(tensor.dtype)],
                                    "data": (tensor.data_ptr(), False), "version": 3}


_POOL_OUT = _PinnedPool()


def band_blocks(nx: int, ny: int):
    """(row slice, column slice) blocks of the 2/3 band of a full (nx, ny)
    field: |kx| <= nx/3, |ky| <= ny/3 (grid.py:102-103)."""
    kxm, kym = nx // 3, ny // 3
    rows = (slice(0, kxm + 1), slice(nx - kxm, nx))
    cols = (slice(0, kym + 1), slice(ny - kym, ny))
    return [(r, c) for r in rows for c in cols]


def band_bytes(nx: int, ny: int) -> int:
    """Bytes of one complex128 field's 2/3 band (what a band copy moves)."""
    return (2 * (nx // 3) + 1) * (2 * (ny // 3) + 1) * 16


def _ptrs(xs):
    return (ctypes.c_void_p * len(xs))(*xs)


def _zero_out_of_band(h, nx, ny):
    kxm, kym = nx // 3, ny // 3
    h[kxm + 1:nx - kxm].zero_()
    h[:kxm + 1, kym + 1:ny - kym].zero_()
    h[nx - kxm:, kym + 1:ny - kym].zero_()


_FILL = None
_FILL_LOCK = threading.Lock()


def _filler():
    global _FILL
    with _FILL_LOCK:
        if _FILL is None:
            from concurrent.futures import ThreadPoolExecutor
            _FILL = ThreadPoolExecutor(max_workers=1, thread_name_prefix="pswe-fill")
        return _FILL


def band_hosts_async(shape, count: int):
    """Pinned host buffers for a band download, their out-of-band part
    zero-filled on a helper thread -- meant to run while a synchronous C-ABI
    call (which releases the GIL) waits for the device."""
    def make():
        hs = [_POOL_OUT.take(shape, _torch().complex128) for _ in range(count)]
        for h in hs:
            _zero_out_of_band(h, shape[0], shape[1])
        return hs
    return _filler().submit(make)


def band_hosts_split(shape, count: int):
    """Pinned host buffers for a band download, taken now, and a future
    that zero-fills their out-of-band part on a helper thread -- disjoint
    from the band the device copies into them, so both may run at once."""
    hs = [_POOL_OUT.take(shape, _torch().complex128) for _ in range(count)]

    def fill():
        for h in hs:
            _zero_out_of_band(h, shape[0], shape[1])

    return hs, _filler().submit(fill)


def download_fields(tensors, band_ctx=None, hosts=None):
    """CUDA tensors -> numpy arrays backed by pooled pinned host memory (one
    stream sync, no host copy).  With ``band_ctx`` (a Context) the tensors are
    known to vanish outside the 2/3 band: only the band crosses the bus and
    the host zero-fills the rest (``hosts``: a band_hosts_async future whose
    buffers are already zero-filled)."""
    torch = _torch()
    if hosts is not None:
        hosts = hosts.result()
    elif band_ctx is not None:
        hosts = [_POOL_OUT.take(t.shape, t.dtype) for t in tensors]
        nx, ny = tensors[0].shape
        for h in hosts:
            _zero_out_of_band(h, nx, ny)
    else:
        hosts = [_POOL_OUT.take(t.shape, t.dtype) for t in tensors]
    if band_ctx is not None and tensors:
        _check(_lib.pswe_copy_band(band_ctx.h, 1, _ptrs([h.data_ptr() for h in hosts]),
                                   _ptrs([t.data_ptr() for t in tensors]), len(tensors), _stream(torch)))
    else:
        for h, t in zip(hosts, tensors):
            h.copy_(t, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    return [_POOL_OUT.array(h) for h in hosts]


def upload_fields(arrays, device: int, band_ctx=None):
    """Host fields -> CUDA tensors through a reused pinned staging buffer:
    field i is copied into its slot by torch's multi-threaded host copy, then
    its H2D copy is queued on the caller's stream, so field i's DMA overlaps
    field i+1's host copy.  A slot is rewritten only after its previous DMA
    completed.  With ``band_ctx`` (a Context) only the 2/3 band is staged and
    copied -- for consumers that read nothing else (pack, i.e. the averaged
    tendency, which truncates its input to the band first, dynamics.py:
    153-156); the device tensors are undefined outside the band."""
    torch = _torch()
    arrays = [np.asarray(a) for a in arrays]
    shape = arrays[0].shape
    key = (shape, len(arrays), device)
    cache = _PIN.__dict__.setdefault("in", {})
    ent = cache.get(key)
    if ent is None:
        pin = torch.empty((len(arrays),) + shape, dtype=torch.complex128, pin_memory=True)
        # per slot: its last DMA's event (created once, re-recorded per call)
        ent = [pin, pin.numpy(), [torch.cuda.Event() for _ in arrays], [False] * len(arrays)]
        cache[key] = ent
    pin, pn, evs, used = ent
    dev = torch.device("cuda", device)
    out = torch.empty((len(arrays),) + shape, dtype=torch.complex128, device=dev)
    cur = torch.cuda.current_stream(dev)
    # staged on the host: whole fields (one threaded copy per field costs
    # less than several copies of the band's blocks -- the copies are
    # dispatch-bound); on the bus: the band only
    for i, a in enumerate(arrays):
        if used[i]:
            evs[i].synchronize()
        if a.dtype == np.complex128 and a.flags.writeable and all(st >= 0 for st in a.strides):
            pin[i].copy_(torch.from_numpy(a))
        else:  # read-only / negative strides / other dtypes: numpy's copy
            np.copyto(pn[i], a, casting="same_kind")
        if band_ctx is not None:
            _check(_lib.pswe_copy_band(band_ctx.h, 0, _ptrs([out[i].data_ptr()]), _ptrs([pin[i].data_ptr()]), 1,
                                       ctypes.c_void_p(cur.cuda_stream)))
        else:
            out[i].copy_(pin[i], non_blocking=True)
        evs[i].record(cur)
        used[i] = True
    return [out[i] for i in range(len(arrays))]


class Context:
    """One grid + physics on one CUDA device (``pswe_ctx``).

    Holds the last quadrature / propagator / topography pushed to the
    library so repeated calls with the same objects cost nothing.
    """

    def __init__(self, nx: int, ny: int, Lx: float, Ly: float, f: float, g: float, H: float,
                 device: int | None = None):
        torch = _torch()
        load_library()
        self.torch = torch
        self.device = torch.cuda.current_device() if device is None else int(device)
        self.nx, self.ny = int(nx), int(ny)
        h = ctypes.c_void_p()
        _check(_lib.pswe_create(ctypes.byref(h), self.nx, self.ny, float(Lx), float(Ly),
                                float(f), float(g), float(H), self.device))
        self.h = h
        ky, kx = ctypes.c_int(), ctypes.c_int()
        _check(_lib.pswe_compact_shape(h, ctypes.byref(ky), ctypes.byref(kx)))
        self.Ky, self.Kx = ky.value, kx.value
        self._quad_key = None
        self._prop_key = None
        self._b_copy = None
        self._b_obj = None
        self._quad_src = None  # the (s, w) array objects last pushed
        self._spec_obj = None  # the PropagatorSpec last configured (propagator.configure)

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and _lib is not None:
            _lib.pswe_destroy(h)
            self.h = None

    # ---- configuration -------------------------------------------------
    @property
    def max_frequency(self) -> float:
        return float(_lib.pswe_max_frequency(self.h))

    @property
    def launch_count(self) -> int:
        return int(_lib.pswe_launch_count(self.h))

    @property
    def variant_launches(self) -> dict:
        """{kernel variant: launches so far} (which code paths ran)."""
        cnt = (ctypes.c_int64 * len(VARIANTS))()
        _check(_lib.pswe_variant_launches(self.h, cnt, len(VARIANTS)))
        return {k: int(cnt[i]) for i, k in enumerate(VARIANTS)}

    def profile(self, enable: bool) -> None:
        _check(_lib.pswe_profile_enable(self.h, 1 if enable else 0))

    def profile_read(self) -> dict:
        """{class: (milliseconds, launches)} since the last read."""
        n = len(KERNEL_CLASSES)
        ms = (ctypes.c_double * n)()
        cnt = (ctypes.c_int64 * n)()
        _check(_lib.pswe_profile_read(self.h, ms, cnt, n))
        return {k: (ms[i], cnt[i]) for i, k in enumerate(KERNEL_CLASSES)}

    def set_chunk_bytes(self, nbytes: int) -> None:
        _check(_lib.pswe_set_chunk_bytes(self.h, int(nbytes)))

    @property
    def lanes(self) -> int:
        return int(_lib.pswe_get_lanes(self.h))

    def set_lanes(self, lanes: int) -> None:
        _check(_lib.pswe_set_lanes(self.h, int(lanes)))

    def set_quadrature(self, s: np.ndarray, w: np.ndarray) -> None:
        self._quad_src = (s, w)
        s = np.ascontiguousarray(s, dtype=np.float64)
        w = np.ascontiguousarray(w, dtype=np.float64)
        key = (s.tobytes(), w.tobytes())
        if key == self._quad_key:
            return
        dp = ctypes.POINTER(ctypes.c_double)
        _check(_lib.pswe_set_quadrature(self.h, len(s), s.ctypes.data_as(dp), w.ctypes.data_as(dp)))
        self._quad_key = key

    def set_propagator(self, kind: str, Lambda: float = 0.0, n_poly: int = 1,
                       a: np.ndarray | None = None) -> None:
        self._spec_obj = None  # propagator.configure records the spec object after this
        key = (kind, float(Lambda), int(n_poly))
        if key == self._prop_key:
            return
        if kind == "exact":
            _check(_lib.pswe_set_propagator(self.h, 0, 0.0, 1, None))
        elif kind == "chebyshev":
            a = np.ascontiguousarray(a, dtype=np.float64)
            _check(_lib.pswe_set_propagator(self.h, 1, float(Lambda), int(n_poly),
                                            a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))))
        else:
            raise ValueError(f"unknown propagator kind {kind!r}")
        self._prop_key = key

    def set_topography(self, b) -> None:
        """Upload b (full spectral layout) unless this exact content is already
        on the device.  The content is compared on every call (memcmp against
        the copy taken at the last upload), so a b changed in place between
        calls is picked up, as the reference reads params.b on every call."""
        if b is self._b_obj and isinstance(b, np.ndarray) and not b.flags.writeable and b.base is None:
            return  # the same read-only array that owns its data: cannot have changed
        arr = np.ascontiguousarray(b, dtype=np.complex128)
        if (self._b_copy is not None and self._b_copy.shape == arr.shape
                and _memcmp(self._b_copy.ctypes.data, arr.ctypes.data, arr.nbytes) == 0):
            self._b_obj = b
            return
        bt = self.to_device(arr)
        _check(_lib.pswe_set_topography(self.h, _dptr(bt), _stream(self.torch)))
        self.torch.cuda.current_stream().synchronize()
        self._b_copy = arr.copy()
        self._b_obj = b

    # ---- tensors ---------------------------------------------------------
    def to_device(self, arr):
        """numpy (nx, ny) complex128 -> contiguous CUDA tensor."""
        torch = self.torch
        if isinstance(arr, torch.Tensor):
            return arr.to(device=f"cuda:{self.device}", dtype=torch.complex128).contiguous()
        a = np.ascontiguousarray(arr, dtype=np.complex128)
        if not a.flags.writeable:  # torch.from_numpy wants a writable buffer (it is only read here)
            a = a.copy()
        return torch.from_numpy(a).to(device=f"cuda:{self.device}", non_blocking=False)

    def empty_full(self):
        return self.torch.empty((self.nx, self.ny), dtype=self.torch.complex128,
                                device=f"cuda:{self.device}")

    def empty_compact(self):
        return self.torch.empty((3, self.Ky, self.Kx), dtype=self.torch.complex128,
                                device=f"cuda:{self.device}")

    # ---- operators (device tensors in/out) ---------------------------------
    def _call3(self, fn, U, *extra):
        out = [self.empty_full() for _ in range(3)]
        _check(fn(self.h, *extra, *(_dptr(x) for x in U), *(_dptr(x) for x in out),
                  _stream(self.torch)))
        return out

    def averaged_tendency(self, U):
        return self._call3(_lib.pswe_averaged_tendency, U)

    def averaged_tendency_to_host(self, U, hosts):
        """The averaged tendency of device fields U, its 2/3 band copied
        into the pinned host tensors `hosts` within the call's single
        synchronisation; returns numpy views of `hosts`."""
        out = [self.empty_full() for _ in range(3)]
        _check(_lib.pswe_averaged_tendency_band_d2h(self.h, *(_dptr(x) for x in U), *(_dptr(x) for x in out),
                                                    _ptrs([h.data_ptr() for h in hosts]), _stream(self.torch)))
        return [_POOL_OUT.array(h) for h in hosts]

    def averaged_tendency_compact(self, Uc, out=None):
        out = self.empty_compact() if out is None else out
        _check(_lib.pswe_averaged_tendency_compact(self.h, _dptr(Uc), _dptr(out), _stream(self.torch)))
        return out

    def pack(self, U, out=None):
        out = self.empty_compact() if out is None else out
        _check(_lib.pswe_pack(self.h, *(_dptr(x) for x in U), _dptr(out), _stream(self.torch)))
        return out

    def unpack(self, Uc):
        out = [self.empty_full() for _ in range(3)]
        _check(_lib.pswe_unpack(self.h, _dptr(Uc), *(_dptr(x) for x in out), _stream(self.torch)))
        return out

    def apply_nonlinear(self, U):
        return self._call3(_lib.pswe_apply_nonlinear, U)

    def apply_linear(self, U):
        return self._call3(_lib.pswe_apply_linear, U)

    def propagate(self, t: float, U):
        return self._call3(_lib.pswe_propagate, U, ctypes.c_double(float(t)))

    def ssprk3_step(self, dt: float, U):
        """Returns (out, (stage, field)); stage 0 means all stages finite."""
        out = [self.empty_full() for _ in range(3)]
        st, fl = ctypes.c_int(0), ctypes.c_int(-1)
        rc = _lib.pswe_ssprk3_step(self.h, float(dt), *(_dptr(x) for x in U),
                                   *(_dptr(x) for x in out), ctypes.byref(st), ctypes.byref(fl),
                                   _stream(self.torch))
        if rc == PSWE_ENONFINITE:
            return out, (st.value, fl.value)
        _check(rc)
        return out, (0, -1)

    # ---- window batch ----------------------------------------------------
    def set_window_batch(self, quads) -> None:
        """W quadratures (objects with .s, .w) as one window batch."""
        n = np.array([len(q.s) for q in quads], dtype=np.int32)
        s = np.ascontiguousarray(np.concatenate([np.asarray(q.s, dtype=np.float64) for q in quads]))
        w = np.ascontiguousarray(np.concatenate([np.asarray(q.w, dtype=np.float64) for q in quads]))
        dp = ctypes.POINTER(ctypes.c_double)
        _check(_lib.pswe_set_window_batch(self.h, len(quads), n.ctypes.data_as(_c_int_p), s.ctypes.data_as(dp),
                                          w.ctypes.data_as(dp)))
        self.batch_windows = len(quads)

    def window_batch_tendency(self, Uc, out=None):
        """(W, 3, Ky, Kx) compact states -> their averaged tendencies."""
        out = self.torch.empty_like(Uc) if out is None else out
        _check(_lib.pswe_window_batch_tendency(self.h, _dptr(Uc), _dptr(out), _stream(self.torch)))
        return out

    def window_batch_run(self, dt: float, nsteps: int, U) -> int:
        """In place on U = (W, 3, nx, ny) complex128; returns 0 or the first
        flagged step (all windows then stand at its start)."""
        bs = ctypes.c_int(0)
        rc = _lib.pswe_window_batch_run(self.h, float(dt), int(nsteps), _dptr(U), ctypes.byref(bs),
                                        _stream(self.torch))
        if rc == PSWE_ENONFINITE:
            return bs.value
        _check(rc)
        return 0

    def diagnostics(self, U) -> tuple[float, float, float]:
        """(energy, mass, max speed) of a full-layout state on the device."""
        out = (ctypes.c_double * 3)()
        _check(_lib.pswe_diagnostics(self.h, *(_dptr(x) for x in U), out, _stream(self.torch)))
        return float(out[0]), float(out[1]), float(out[2])

    def to_physical(self, U):
        """(3, nx, ny) float64 CUDA tensor of the physical u, v, eta."""
        out = self.torch.empty((3, self.nx, self.ny), dtype=self.torch.float64, device=f"cuda:{self.device}")
        _check(_lib.pswe_to_physical(self.h, *(_dptr(x) for x in U), _dptr(out), _stream(self.torch)))
        return out

    def run(self, dt: float, nsteps: int, U):
        """In-place nsteps on U (list of 3 tensors). Returns (bad_step, stage, field)
        for a non-finite stage; a step whose input fails the Hermitian gate
        raises ValueError with ``bad_step`` set (1-based)."""
        bs, st, fl = ctypes.c_int(0), ctypes.c_int(0), ctypes.c_int(-1)
        rc = _lib.pswe_run(self.h, float(dt), int(nsteps), *(_dptr(x) for x in U),
                           ctypes.byref(bs), ctypes.byref(st), ctypes.byref(fl), _stream(self.torch))
        if rc == PSWE_ENONFINITE:
            return bs.value, st.value, fl.value
        try:
            _check(rc)
        except ValueError as exc:
            exc.bad_step = bs.value
            raise
        return 0, 0, -1


_ctx_cache: dict = {}
_ctx_lock = threading.Lock()


def debug_check_guards() -> tuple[int, int]:
    """(guarded buffers, damaged guard bands) under PSWE_DEBUG_GUARD
    (pswe_debug_check_guards; synchronises the device); (0, 0) otherwise."""
    g, d = ctypes.c_int64(), ctypes.c_int64()
    _check(load_library().pswe_debug_check_guards(ctypes.byref(g), ctypes.byref(d)))
    return int(g.value), int(d.value)


def release_thread_contexts() -> None:
    """Drop the calling thread's cached contexts (frees their device scratch)."""
    me = threading.get_ident()
    with _ctx_lock:
        for key in [k for k in _ctx_cache if k[-1] == me]:
            del _ctx_cache[key]


def context_for(nx, ny, Lx, Ly, f, g, H) -> Context:
    """Cached context per (grid, physics constants, device)."""
    torch = _torch()
    key = (int(nx), int(ny), float(Lx), float(Ly), float(f), float(g), float(H),
           torch.cuda.current_device(), threading.get_ident())
    with _ctx_lock:
        ctx = _ctx_cache.get(key)
        if ctx is None:
            ctx = Context(nx, ny, Lx, Ly, f, g, H)
            _ctx_cache[key] = ctx
        return ctx

"""The C-ABI library loads and exports exactly what include/pswe_b200.h declares (CPU only)."""

import ctypes
import re

import pytest

from conftest import ROOT
from paper_2103_07706_b200 import _native

HEADER = ROOT / "include" / "pswe_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(pswe_[a-z_0-9]+)\s*\(", text)))


def test_header_declares_the_abi():
    syms = declared_symbols()
    assert "pswe_averaged_tendency" in syms and "pswe_ssprk3_step" in syms
    assert set(syms) == set(_native.SIGNATURES), "ctypes table and header disagree"


def test_library_exports_every_declared_symbol():
    lib = _native.load_library()
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, f"missing exports: {missing}"
    assert lib.pswe_version() == 100


def test_library_is_built_for_sm100a():
    so = _native.LIB_PATH.read_bytes()
    assert b"sm_100a" in so or b"sm_100" in so


def test_invalid_arguments_fail_without_a_gpu():
    lib = _native.load_library()
    h = ctypes.c_void_p()
    # argument validation happens before any CUDA call
    assert lib.pswe_create(ctypes.byref(h), 6, 8, 1.0, 1.0, 1e-4, 9.8, 1.0, 0) == _native.PSWE_EINVAL
    assert b"nx must be even and >= 8" in lib.pswe_last_error()
    assert lib.pswe_create(ctypes.byref(h), 8192, 48, 1.0, 1.0, 1e-4, 9.8, 1.0, 0) == _native.PSWE_EUNSUPPORTED
    assert lib.pswe_create(ctypes.byref(h), 32, 32, 1.0, 1.0, 1e-4, -9.8, 1.0, 0) == _native.PSWE_EINVAL
    assert b"g must be positive" in lib.pswe_last_error()


def test_ops_fail_loudly_without_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    from paper_2103_07706_b200 import cases, averaged_tendency, PropagatorSpec
    c = cases.case_c1()
    with pytest.raises(RuntimeError, match="CUDA device"):
        averaged_tendency(c.state, c.quadrature, c.params, PropagatorSpec.exact())

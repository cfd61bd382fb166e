"""Shared test setup.

Markers: ``gpu`` tests need a CUDA device (run on the B200 box with
``pytest -m gpu``); everything else runs on CPU.  Parity fixtures live in
tests/golden/ (generated from the real reference by oracle/make_golden.py).
"""

import pathlib
import sys

import numpy as np
import pytest

ROOT = pathlib.Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def load_golden(name):
    path = GOLDEN / f"{name}.npz"
    if not path.exists():
        pytest.fail(f"missing golden fixture {path}; regenerate with oracle/make_golden.py")
    with np.load(path) as z:
        return {k: z[k] for k in z.files}


def rel_l2(got, want):
    got = np.asarray(got)
    want = np.asarray(want)
    den = float(np.linalg.norm(want.ravel()))
    return float(np.linalg.norm((got - want).ravel())) / (den if den > 0 else 1.0)


@pytest.fixture(scope="session")
def unit_golden():
    return load_golden("unit")

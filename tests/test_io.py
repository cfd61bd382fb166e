"""Snapshot / CSV output in the reference's format.

CPU: the host writer is byte-identical to the oracle restatement of io.py
for the same physical fields, and the readers round-trip.  GPU: the device
physical fields match real(ifft2) to 1e-14 relative and the sidecars are
byte-identical.
"""

import os

import numpy as np
import pytest

import paper_2103_07706_b200 as pk
from oracle import io_oracle as IO


def _files(d):
    return sorted(os.listdir(d))


def _bytes(d, f):
    with open(os.path.join(d, f), "rb") as fh:
        return fh.read()


def test_host_writer_is_byte_identical(tmp_path):
    rng = np.random.default_rng(3)
    g = pk.make_grid(16, 8, 4.0e7, 2.0e7)
    phys = rng.standard_normal((3, 16, 8))
    a, b = tmp_path / "ours", tmp_path / "ref"
    a.mkdir()
    b.mkdir()
    pk.io.write_fields(str(a), 42, 3600.5, g, phys)
    IO.write_snapshot(str(b), 42, 16, 8, g.Lx, g.Ly, 3600.5, phys)
    assert _files(a) == _files(b)
    for f in _files(a):
        assert _bytes(a, f) == _bytes(b, f), f
    pk.io.write_diagnostics(str(a), [0.0, 3600.0], [0, 1], [1.5, 1.25], [2.0, 2.0], [10.0, 11.0])
    IO.write_diagnostics(str(b), [0.0, 3600.0], [0, 1], [1.5, 1.25], [2.0, 2.0], [10.0, 11.0])
    assert _bytes(a, "diagnostics.csv") == _bytes(b, "diagnostics.csv")


def test_readers_round_trip(tmp_path):
    rng = np.random.default_rng(4)
    g = pk.make_grid(8, 8, 1.0e6, 1.0e6)
    phys = rng.standard_normal((3, 8, 8))
    pk.io.write_fields(str(tmp_path), 7, 12.0, g, phys)
    pk.io.write_fields(str(tmp_path), 3, 6.0, g, phys)
    assert pk.io.list_snapshot_steps(str(tmp_path)) == [3, 7]
    arr, meta = pk.io.read_snapshot_field(str(tmp_path), 7, "v")
    assert np.array_equal(arr, phys[1]) and meta["time_seconds"] == "12.0"
    st = pk.io.read_snapshot_state(str(tmp_path))
    assert st.t == 12.0
    assert np.allclose(np.fft.ifft2(st.eta).real, phys[2], rtol=0, atol=1e-12)


@pytest.mark.gpu
def test_device_snapshot_matches_reference_writer(tmp_path):
    rng = np.random.default_rng(5)
    for nx, ny in ((512, 512), (64, 32)):
        g = pk.make_grid(nx, ny, 4.0e7, 4.0e7)
        U = [np.fft.fft2(s * rng.standard_normal((nx, ny))) for s in (20.0, 10.0, 80.0)]
        st = pk.State(grid=g, u=U[0], v=U[1], eta=U[2], t=1800.0)
        a, b = tmp_path / f"ours{nx}", tmp_path / f"ref{nx}"
        a.mkdir()
        b.mkdir()
        pk.io.write_snapshot(str(a), 5, st)
        IO.write_snapshot(str(b), 5, nx, ny, g.Lx, g.Ly, st.t, [IO.physical(c) for c in U])
        assert _files(a) == _files(b)
        for f in _files(a):
            if f.endswith(".meta"):
                assert _bytes(a, f) == _bytes(b, f)
            else:
                x = np.frombuffer(_bytes(a, f), "<f8")
                y = np.frombuffer(_bytes(b, f), "<f8")
                assert np.max(np.abs(x - y)) <= 1e-14 * np.max(np.abs(y)), f

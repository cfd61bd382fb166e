"""Band-only host<->device transfers of the drop-in averaged-tendency path.

averaged_tendency truncates its input to the 2/3 band first
(dynamics.py:153-156, apply_nonlinear) and dealiases its output, so the
drop-in call moves only the band: pswe_copy_band.  The result must be
bitwise the one obtained with full-field transfers, for inputs carrying
energy outside the band, on square and rectangular grids; the device copy
must touch only the band and the host copy must zero everything else.
"""

import numpy as np
import pytest
import torch

import paper_2103_07706_b200 as pk
from paper_2103_07706_b200 import _native, cases, dynamics

pytestmark = pytest.mark.gpu


def full_spectrum_state(nx, ny, seed):
    rng = np.random.default_rng(seed)
    g = pk.make_grid(nx, ny, 4.0e7, 4.0e7 * ny / nx)
    f = [np.fft.fft2(s * rng.standard_normal((nx, ny))) for s in (20.0, 15.0, 50.0)]
    return pk.State(grid=g, u=f[0], v=f[1], eta=f[2])


@pytest.mark.parametrize("nx,ny", [(64, 64), (128, 64), (32, 128)])
def test_band_upload_download_bitwise(nx, ny):
    st = full_spectrum_state(nx, ny, 3)
    params = pk.PhysicsParams(f=1.0e-4, g=9.80616, H=5960.0, b=np.zeros((nx, ny), dtype=np.complex128))
    ctx = dynamics.context(st, params)
    full = dynamics.upload(ctx, st)
    band = dynamics.upload(ctx, st, band=True)
    Uc_full = ctx.pack(full)
    Uc_band = ctx.pack(band)
    torch.cuda.synchronize()
    assert torch.equal(Uc_full, Uc_band)
    # device -> host: unpack writes zeros outside the band
    out = ctx.unpack(Uc_full)
    a = dynamics.download(out)
    # poison the pinned pool buffers the band download will reuse
    for _ in range(2):
        junk = dynamics.download([t.fill_(7.0 + 7.0j) for t in [x.clone() for x in out]])
        del junk
    b = dynamics.download(out, band_ctx=ctx)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def test_drop_in_call_matches_full_transfer():
    """The public call (band transfers) equals the compact path fed by a
    full-field upload, bitwise."""
    c = cases.case_c5(3, 4)  # 32^2, 9 phases
    st = c.state
    rng = np.random.default_rng(5)
    noisy = type(st)(grid=st.grid, u=st.u + 1e-3 * np.fft.fft2(rng.standard_normal(st.u.shape)),
                     v=st.v, eta=st.eta, t=st.t)
    got = pk.averaged_tendency(noisy, c.quadrature, c.params, pk.PropagatorSpec.exact())
    ctx = dynamics.context(noisy, c.params)
    ctx.set_propagator("exact")
    ctx.set_quadrature(c.quadrature.s, c.quadrature.w)
    ref = dynamics.download(ctx.averaged_tendency(dynamics.upload(ctx, noisy)))
    for x, y in zip((got.u, got.v, got.eta), ref):
        assert np.array_equal(x, y)


def test_drop_in_call_odd_host_arrays():
    """Read-only, Fortran-ordered and negative-stride host fields give the
    same result as plain C-contiguous ones (the staging copy handles them)."""
    c = cases.case_c5(3, 4)
    st = c.state
    spec = pk.PropagatorSpec.exact()
    ref = pk.averaged_tendency(st, c.quadrature, c.params, spec)
    ro = [np.array(a) for a in (st.u, st.v, st.eta)]
    for a in ro:
        a.setflags(write=False)
    fortran = [np.asfortranarray(a) for a in (st.u, st.v, st.eta)]
    flipped = [np.flipud(np.flipud(a).copy()) for a in (st.u, st.v, st.eta)]  # negative strides
    assert flipped[0].strides[0] < 0
    for fields in (ro, fortran, flipped):
        s2 = type(st)(grid=st.grid, u=fields[0], v=fields[1], eta=fields[2], t=st.t)
        got = pk.averaged_tendency(s2, c.quadrature, c.params, spec)
        for x, y in zip((got.u, got.v, got.eta), (ref.u, ref.v, ref.eta)):
            assert np.array_equal(x, y)

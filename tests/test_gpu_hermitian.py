"""The Hermitian-symmetry gate of to_physical (grid.py:140-180) on the GPU
paths: a non-Hermitian input fails exactly where, and with exactly the
message, the reference fails -- inside averaged_tendency as the first
node's error (averaging.py:138-141), from apply_nonlinear as ValueError
(dynamics.py:162-164), from a step (integrator.py:93-95) and from run's
snapshot record (integrator.py:124-135, diagnostics.py:21-25); a
round-off-sized asymmetry passes, also when the fast bound flags it and the
exact check has to decide.  The expected messages come from the unmodified
reference (oracle/_ref) when it is installed, else from its documented
format."""

import re

import numpy as np
import pytest

import paper_2103_07706_b200 as pk
from oracle import reference as R
from paper_2103_07706_b200 import cases

pytestmark = pytest.mark.gpu

MSG = re.compile(r"non-Hermitian spectral field: mode \(kx index -?\d+, ky index -?\d+\) has asymmetry "
                 r"\S+ \(relative \S+\)")


def perturbed(c, field, i, j, rel):
    """c.state with one mode of `field` moved off Hermitian symmetry (its
    mirror untouched) by rel times the largest u coefficient (v may be 0)."""
    a = {n: np.array(getattr(c.state, n)) for n in ("u", "v", "eta")}
    a[field][i, j] += rel * np.max(np.abs(a["u"])) * (1.0 + 0.5j)
    return pk.State(grid=c.grid, u=a["u"], v=a["v"], eta=a["eta"], t=c.state.t)


def ref_error(fn):
    """(type, message) the reference raises for fn(phaseswe), or None if it is not installed."""
    ref = R.load()
    if ref is None:
        return None
    try:
        fn(ref)
    except Exception as exc:  # noqa: BLE001
        return type(exc), str(exc)
    return "no error"


def ref_objects(ref, c, st):
    from phaseswe import averaging, dynamics, grid, propagator
    g = grid.make_grid(c.grid.nx, c.grid.ny, c.grid.Lx, c.grid.Ly)
    p = dynamics.PhysicsParams(f=c.params.f, g=c.params.g, H=c.params.H, b=np.array(c.params.b))
    s = dynamics.State(grid=g, u=st.u, v=st.v, eta=st.eta, t=st.t)
    return g, p, s, averaging.kernel_weights(c.T_half, c.M), propagator.PropagatorSpec.exact()


def check_against_reference(exc_info, want_type, fn):
    got = str(exc_info.value)
    assert exc_info.type is want_type
    assert MSG.search(got), got
    ref = ref_error(fn)
    if ref is not None:
        assert ref != "no error"
        assert ref[0] is want_type
        assert got == ref[1], (got, ref[1])


@pytest.mark.parametrize("field,i,j", [("u", 3, 5), ("eta", 30, 2), ("v", 0, 7)])
def test_averaged_tendency_reports_the_first_node(field, i, j):
    c = cases.case_c1()
    st = perturbed(c, field, i, j, 1e-6)
    with pytest.raises(RuntimeError) as ei:
        pk.averaged_tendency(st, c.quadrature, c.params, pk.PropagatorSpec.exact())
    assert str(ei.value).startswith("averaging node k = -7 (s = ")

    def ref(m):
        from phaseswe import averaging
        _, p, s, q, spec = ref_objects(m, c, st)
        averaging.averaged_tendency(s, q, p, spec)
    check_against_reference(ei, RuntimeError, ref)


def test_apply_nonlinear_raises_value_error():
    c = cases.case_c3()  # with topography
    st = perturbed(c, "u", 5, 9, 1e-8)
    with pytest.raises(ValueError) as ei:
        pk.apply_nonlinear(st, c.params)

    def ref(m):
        from phaseswe import dynamics
        _, p, s, _, _ = ref_objects(m, c, st)
        dynamics.apply_nonlinear(s, p)
    check_against_reference(ei, ValueError, ref)


def test_step_raises_the_node_error():
    c = cases.case_c2()
    st = perturbed(c, "eta", 7, 3, 1e-7)
    cfg = pk.StepConfig(dt=c.dt, quadrature=c.quadrature, propagator_spec=pk.PropagatorSpec.exact())
    with pytest.raises(RuntimeError) as ei:
        pk.step_averaged_ssprk3(st, cfg, c.params)

    def ref(m):
        from phaseswe import integrator
        _, p, s, q, spec = ref_objects(m, c, st)
        integrator.step_averaged_ssprk3(s, integrator.StepConfig(dt=c.dt, quadrature=q, propagator_spec=spec), p)
    check_against_reference(ei, RuntimeError, ref)


def test_run_fails_at_the_initial_record():
    """run records the initial state first (integrator.py:166): the
    snapshot diagnostics' full-grid gate raises before any step."""
    c = cases.case_c2()
    st = perturbed(c, "v", 10, 20, 1e-9)  # out of the 2/3 band: only the full-grid gate sees it
    cfg = pk.StepConfig(dt=c.dt, quadrature=c.quadrature, propagator_spec=pk.PropagatorSpec.exact())
    with pytest.raises(ValueError) as ei:
        pk.run(st, cfg, c.params, t_end=2 * c.dt)

    def ref(m):
        from phaseswe import integrator
        _, p, s, q, spec = ref_objects(m, c, st)
        integrator.run(s, integrator.StepConfig(dt=c.dt, quadrature=q, propagator_spec=spec), p, t_end=2 * c.dt)
    check_against_reference(ei, ValueError, ref)


def test_roundoff_asymmetry_passes_and_is_projected():
    """numpy's fft2 leaves ~1e-16 relative asymmetry: no error, and the result
    is exactly the Hermitian part's (what real(ifft2) computes)."""
    c = cases.case_c1()
    st = perturbed(c, "u", 3, 5, 1e-15)
    got = pk.averaged_tendency(st, c.quadrature, c.params, pk.PropagatorSpec.exact())

    def herm(a):
        return 0.5 * (a + np.conj(np.roll(a[::-1, ::-1], 1, axis=(0, 1))))
    hp = pk.State(grid=c.grid, u=herm(st.u), v=herm(st.v), eta=herm(st.eta), t=st.t)
    want = pk.averaged_tendency(hp, c.quadrature, c.params, pk.PropagatorSpec.exact())
    for f in ("u", "v", "eta"):
        assert np.array_equal(getattr(got, f), getattr(want, f))


def test_flagged_but_passing_input_goes_through_the_exact_check():
    """An asymmetry the fast bound cannot clear (a u defect may reach eta'
    amplified by up to sqrt(H/g) ~ 17 under e^{sL}) but that stays under the
    reference's threshold at every node (the reference passes it; it fails
    from about 5e-11): the exact check (herm_node_kernel) decides, and the
    call succeeds."""
    c = cases.case_c1()
    st = perturbed(c, "u", 3, 5, 1e-11)
    ctx = pk.dynamics.context(st, c.params)
    before = ctx.variant_launches["herm"]
    pk.averaged_tendency(st, c.quadrature, c.params, pk.PropagatorSpec.exact())
    assert ctx.variant_launches["herm"] > before

    def ref(m):
        from phaseswe import averaging
        _, p, s, q, spec = ref_objects(m, c, st)
        averaging.averaged_tendency(s, q, p, spec)
    got = ref_error(ref)
    if got is not None:
        assert got == "no error"


def test_stage_inputs_pass_for_band_limited_states():
    """Exactly Hermitian inputs never reach the exact check (the fast bound
    clears d = 0), across a multi-step device-resident run."""
    c = cases.case_c2()
    cfg = pk.StepConfig(dt=c.dt, quadrature=c.quadrature, propagator_spec=pk.PropagatorSpec.exact())
    ctx = pk.dynamics.context(c.state, c.params)
    before = ctx.variant_launches["herm"]
    pk.run(c.state, cfg, c.params, t_end=3 * c.dt)
    # the snapshot gate runs its full-grid kernel at the records; no node check ran
    v = ctx.variant_launches
    assert v["herm"] - before == 2


def test_snapshot_writer_gates_its_fields(tmp_path):
    c = cases.case_c1()
    st = perturbed(c, "eta", 2, 1, 1e-6)
    with pytest.raises(ValueError, match="non-Hermitian spectral field"):
        pk.io.write_snapshot(str(tmp_path), 0, st)

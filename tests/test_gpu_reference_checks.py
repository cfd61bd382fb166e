"""The reference's own hot-path checks, run through the drop-in on the GPU.

Each test restates one of the reference's tests (cited) against
``paper_2103_07706_b200`` -- including the ``nonlinear=`` operator hook the
reference's tests drive with ``zero_tendency``, ``explode`` and ``broken``
(averaging.py:116-119, integrator.py:83-84), which on this path wraps GPU
exponentials around the user's Python operator.  Inputs are built locally
with the reference's recipes (conftest.py band_limited_state, a balanced
zonal jet over a cone mountain like testcase.py); tolerances are the
reference's.
"""

import math
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import paper_2103_07706_b200 as pk
from paper_2103_07706_b200 import cases

pytestmark = pytest.mark.gpu

F0, G0, H0 = 1.0e-4, 9.8, 5960.0


def grid(n):
    return pk.make_grid(n, n, 4.0e7, 4.0e7)


def flat(g):
    return pk.PhysicsParams(f=F0, g=G0, H=H0, b=np.zeros((g.nx, g.ny), dtype=complex))


def band_limited_state(g, rng, vel=1.0, eta=50.0):
    """Random Hermitian state on the 2/3 band (reference conftest.py)."""
    def field(scale):
        return pk.dealias(g, pk.to_spectral(g, scale * rng.standard_normal((g.nx, g.ny))))
    return pk.State(grid=g, u=field(vel), v=field(vel), eta=field(eta))


def jet_problem(n=32, mountain=True):
    """Balanced zonal jet (u = 20 cos(2 pi (y - L/2) / L), geostrophic eta),
    optionally over a 2000 m cone mountain: testcase.py's construction."""
    g = grid(n)
    cu = cases._zonal(g, 20.0 * np.cos(2.0 * math.pi * (g.y - g.Ly / 2.0) / g.Ly))
    ceta = cases._balanced_eta(g, cu, F0, G0)
    b = (cases._cone(g, 2000.0, g.Lx / 18.0, g.Lx / 4.0, 0.6 * g.Ly) if mountain
         else np.zeros((n, n), dtype=complex))
    params = pk.PhysicsParams(f=F0, g=G0, H=H0, b=b)
    return g, params, pk.State(grid=g, u=cu, v=np.zeros_like(cu), eta=ceta)


def zero_tendency(state, params):
    z = np.zeros_like(state.u)
    return pk.State(grid=state.grid, u=z, v=z.copy(), eta=z.copy(), t=state.t)


def l2_eta(test, ref):
    """Physical-space relative L2 of eta (diagnostics.py:28-44)."""
    a, b = np.fft.ifft2(test.eta).real, np.fft.ifft2(ref.eta).real
    return float(np.sqrt(np.sum((a - b) ** 2)) / np.sqrt(np.sum(b ** 2)))


# ------------------------------------------------------------------ stepper
def test_step_reproduces_stage_formula():
    """test_integrator.py:38-57: the fused GPU step equals the stage formula
    composed from the drop-in's own exponentials and averaged tendencies."""
    g, params, state = jet_problem()
    dt, quad, spec = 600.0, pk.kernel_weights(1200.0, 2), pk.PropagatorSpec.exact()
    got = pk.step_averaged_ssprk3(state, pk.StepConfig(dt=dt, quadrature=quad, propagator_spec=spec), params)

    def E(t, s):
        return pk.exact_exp(t, s, params)

    def A(s):
        return pk.averaged_tendency(s, quad, params, spec)

    u1 = E(dt, state) + dt * E(dt, A(state))
    u2 = 0.75 * E(0.5 * dt, state) + 0.25 * E(-0.5 * dt, u1 + dt * A(u1))
    want = (1.0 / 3.0) * E(dt, state) + (2.0 / 3.0) * E(0.5 * dt, u2 + dt * A(u2))
    assert pk.energy_norm(got - want, params) <= 1e-14 * pk.energy_norm(state, params)
    assert got.t == state.t + dt


def test_pure_linear_step_equals_exponential_through_the_hook():
    """test_integrator.py:82-96: nonlinear=zero_tendency (the operator hook)
    leaves the exact exponential; Chebyshev route to 1e-9."""
    g = grid(32)
    params = flat(g)
    state = band_limited_state(g, np.random.default_rng(20260823))
    dt = 3600.0
    want = pk.exact_exp(dt, state, params)
    norm = pk.energy_norm(state, params)
    cfg = pk.make_step_config(g, params, dt=dt, T=dt)
    got = pk.step_averaged_ssprk3(state, cfg, params, nonlinear=zero_tendency)
    assert pk.energy_norm(got - want, params) <= 1e-12 * norm
    cheb = pk.make_step_config(g, params, dt=dt, T=dt, propagator="chebyshev", tol=1e-10)
    got = pk.step_averaged_ssprk3(state, cheb, params, nonlinear=zero_tendency)
    assert pk.energy_norm(got - want, params) <= 1e-9 * norm


def test_hooked_builtin_equals_fused_path():
    """A user operator that is numerically the built-in N (wrapped, so the hook
    path runs) gives the fused path's averaged tendency and step."""
    g, params, state = jet_problem()
    quad, spec = pk.kernel_weights(1800.0, 3), pk.PropagatorSpec.exact()

    def my_n(s, p):
        return pk.apply_nonlinear(s, p)

    fused = pk.averaged_tendency(state, quad, params, spec)
    hooked = pk.averaged_tendency(state, quad, params, spec, nonlinear=my_n)
    scale = pk.energy_norm(fused, params)
    assert pk.energy_norm(fused - hooked, params) <= 1e-13 * scale
    cfg = pk.StepConfig(dt=600.0, quadrature=quad, propagator_spec=spec)
    a = pk.step_averaged_ssprk3(state, cfg, params)
    b = pk.step_averaged_ssprk3(state, cfg, params, nonlinear=my_n)
    assert pk.energy_norm(a - b, params) <= 1e-13 * pk.energy_norm(state, params)


@pytest.mark.filterwarnings("ignore:invalid value encountered")
def test_nonfinite_hook_aborts_with_stage_index():
    """test_integrator.py:182-190: nonlinear=explode -> 'stage 1'."""
    g, params, state = jet_problem()
    cfg = pk.make_step_config(g, params, dt=600.0)

    def explode(s, p):
        return np.inf * s

    with pytest.raises(RuntimeError, match="stage 1"):
        pk.step_averaged_ssprk3(state, cfg, params, nonlinear=explode)


def test_node_failure_reports_node_index():
    """test_averaging.py:160-174: a failing operator is reported as the first
    failing node, serially and with an executor."""
    g = grid(32)
    params = flat(g)
    state = band_limited_state(g, np.random.default_rng(20260823))
    quad = pk.kernel_weights(1800.0, 3)

    def broken(s, p):
        raise ValueError("boom")

    with pytest.raises(RuntimeError, match=r"averaging node k = -2 .*boom"):
        pk.averaged_tendency(state, quad, params, pk.PropagatorSpec.exact(), nonlinear=broken)
    with ThreadPoolExecutor(max_workers=4) as pool:
        with pytest.raises(RuntimeError, match="averaging node"):
            pk.averaged_tendency(state, quad, params, pk.PropagatorSpec.exact(), executor=pool, nonlinear=broken)


def test_worker_count_does_not_change_bits():
    """test_averaging.py:143-157: bitwise independent of the executor."""
    g, params, state = jet_problem()
    quad, spec = pk.kernel_weights(1800.0, 4), pk.PropagatorSpec.exact()
    serial = pk.averaged_tendency(state, quad, params, spec)
    for workers in (1, 2, 8):
        with ThreadPoolExecutor(max_workers=workers) as pool:
            par = pk.averaged_tendency(state, quad, params, spec, executor=pool)
        for f in ("u", "v", "eta"):
            assert np.array_equal(getattr(par, f), getattr(serial, f))


def test_third_order_convergence_short_horizon():
    """test_integrator.py:99-110: observed order >= 2.5 against a dt = 30 s run."""
    g, params, state = jet_problem()
    t_end = 3600.0
    ref = pk.run(state, pk.make_step_config(g, params, dt=30.0), params, t_end).states[-1]
    errs = []
    for dt in (900.0, 450.0, 225.0):
        final = pk.run(state, pk.make_step_config(g, params, dt=dt), params, t_end).states[-1]
        errs.append(l2_eta(final, ref))
    orders = [math.log2(errs[i] / errs[i + 1]) for i in range(2)]
    assert min(orders) >= 2.5, f"errors {errs}, orders {orders}"


# ------------------------------------------------------------------ propagator
def test_exact_exp_identity_group_inverse_isometry():
    """test_propagator.py:48-65 on the GPU exponential."""
    g = grid(32)
    params = flat(g)
    state = band_limited_state(g, np.random.default_rng(20260823))
    norm = pk.energy_norm(state, params)
    assert pk.energy_norm(pk.exact_exp(0.0, state, params) - state, params) <= 1e-13 * norm
    t1, t2 = 1800.0, 2700.0
    combined = pk.exact_exp(t1 + t2, state, params)
    chained = pk.exact_exp(t2, pk.exact_exp(t1, state, params), params)
    assert pk.energy_norm(combined - chained, params) <= 1e-12 * norm
    back = pk.exact_exp(-t1, pk.exact_exp(t1, state, params), params)
    assert pk.energy_norm(back - state, params) <= 1e-12 * norm
    moved = pk.exact_exp(12345.0, state, params)
    assert abs(pk.energy_norm(moved, params) - norm) <= 1e-12 * norm


def test_cheb_matches_exact_on_default_grid():
    """test_propagator.py:117-126: Chebyshev (tol 1e-12) vs exact <= 1e-10."""
    g = grid(64)
    params = flat(g)
    lam = pk.max_frequency(g, params)
    spec = pk.PropagatorSpec.chebyshev(lam * 3600.0, tol=1e-12)
    state = band_limited_state(g, np.random.default_rng(20260823))
    norm = pk.energy_norm(state, params)
    for t in (3600.0, -1800.0):
        want = pk.exact_exp(t, state, params)
        got = pk.cheb_exp(t, state, params, spec)
        assert pk.energy_norm(got - want, params) <= 1e-10 * norm


# ------------------------------------------------------------------ dynamics
def test_balanced_jet_is_discrete_steady_state():
    """test_dynamics.py:70-81: L and N of the balanced jet vanish to 1e-12;
    the mountain breaks the balance."""
    g, params, jet = jet_problem(64, mountain=False)
    scale = F0 * pk.energy_norm(jet, params)
    assert pk.energy_norm(pk.apply_linear(jet, params), params) <= 1e-12 * scale
    assert pk.energy_norm(pk.apply_nonlinear(jet, params), params) <= 1e-12 * scale
    _, rough, _ = jet_problem(64, mountain=True)
    assert pk.energy_norm(pk.apply_nonlinear(jet, rough), rough) > 1e-6 * scale


def test_nonlinear_mean_eta_tendency_is_exactly_zero():
    """test_dynamics.py:64-67."""
    g = grid(32)
    out = pk.apply_nonlinear(band_limited_state(g, np.random.default_rng(20260823)), flat(g))
    assert out.eta[0, 0] == 0.0

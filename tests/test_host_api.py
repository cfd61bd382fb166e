"""Host-side logic of the drop-in API (CPU only): validation, setup objects, cases."""

import math

import numpy as np
import pytest
import scipy.special

import paper_2103_07706_b200 as pk
from conftest import load_golden
from paper_2103_07706_b200 import cases


def test_make_grid_matches_reference_conventions():
    g = pk.make_grid(8, 8, 2 * np.pi, 2 * np.pi)
    assert np.allclose(g.kx, [0, 1, 2, 3, -4, -3, -2, -1])
    assert int(g.dealias_mask.sum()) == 25
    assert int(pk.make_grid(12, 12, 1.0, 1.0).dealias_mask.sum()) == 81
    for bad in ((7, 8), (8, 6), (4, 8)):
        with pytest.raises(ValueError, match="even and >= 8"):
            pk.make_grid(bad[0], bad[1], 1.0, 1.0)
    with pytest.raises(ValueError, match="positive"):
        pk.make_grid(8, 8, 0.0, 1.0)


def test_quadrature_matches_reference_goldens(unit_golden):
    for T, M in ((3600.0, 5), (7200.0, 8), (1800.0, 8), (3600.0, 16), (1800.0, 32), (2700.0, 64), (1800.0, 256)):
        q = pk.kernel_weights(T, M)
        assert np.array_equal(q.s, unit_golden[f"quad_{int(T)}_{M}_s"])
        assert np.array_equal(q.w, unit_golden[f"quad_{int(T)}_{M}_w"])
    assert np.array_equal(pk.kernel_weights(100.0, 3, pk.UNIFORM_KERNEL).w, unit_golden["quad_uniform_100_3_w"])
    q = pk.kernel_weights(7200.0, 8)
    assert q.w[0] == 0.0 and q.w[-1] == 0.0 and int(np.count_nonzero(q.w)) == 15


def test_quadrature_and_window_validation():
    with pytest.raises(ValueError, match="T = 0"):
        pk.kernel_weights(0.0, 2)
    with pytest.raises(ValueError, match="nonnegative"):
        pk.kernel_weights(-1.0, 2)
    with pytest.raises(ValueError, match="nodes and weights"):
        pk.Quadrature(T=1.0, M=2, s=np.zeros(3), w=np.full(3, 1.0 / 3.0))
    with pytest.raises(ValueError, match="sum"):
        pk.Quadrature(T=1.0, M=1, s=np.array([-1.0, 0.0, 1.0]), w=np.array([0.2, 0.2, 0.2]))
    assert pk.default_node_count(14400.0, 1.720899454284647e-3) == 8


def test_propagator_spec_and_chebyshev_coefficients(unit_golden):
    k = np.arange(31)
    want = np.where(k == 0, 1.0, 2.0) * scipy.special.jv(k, 5.0)
    assert np.max(np.abs(pk.cheb_coeffs(5.0, 30).a - want)) <= 1e-12
    assert np.max(np.abs(pk.cheb_coeffs(6.2, 24).a - unit_golden["cheb_6.2_24"])) <= 1e-15
    assert pk.choose_npoly(10.0, 1e-10) == 28
    for lam, n in unit_golden["npoly"]:
        assert pk.choose_npoly(float(lam), 1e-10) == int(n)
    with pytest.raises(ValueError, match="kind"):
        pk.PropagatorSpec(kind="taylor")
    with pytest.raises(ValueError, match="n_poly"):
        pk.PropagatorSpec(kind="chebyshev", Lambda=1.0, n_poly=0)
    spec = pk.PropagatorSpec.chebyshev(6.2)
    assert spec.n_poly == pk.choose_npoly(6.2, 1e-10)


def test_make_step_config_resolution():
    g = pk.make_grid(64, 64, 4.0e7, 4.0e7)
    p = pk.flat_bottom(g, 1.0e-4, 9.8, 5960.0)
    assert pk.max_frequency(g, p) == pytest.approx(1.720899454284647e-3, rel=1e-12)
    assert pk.make_step_config(g, p, dt=3600.0, T=3600.0).quadrature.M == 4
    cheb = pk.make_step_config(g, p, dt=3600.0, T=7200.0, propagator="chebyshev")
    assert cheb.propagator_spec.Lambda == pytest.approx(pk.max_frequency(g, p) * 10800.0, rel=1e-15)
    with pytest.raises(ValueError, match="propagator"):
        pk.make_step_config(g, p, dt=3600.0, propagator="magic")
    with pytest.raises(ValueError, match="dt"):
        pk.StepConfig(dt=0.0, quadrature=pk.kernel_weights(0.0, 0), propagator_spec=pk.PropagatorSpec.exact())


def test_run_validates_before_touching_the_gpu():
    c = cases.case_c1()
    cfg = pk.make_step_config(c.grid, c.params, dt=600.0)
    with pytest.raises(ValueError, match="t_end"):
        pk.run(c.state, cfg, c.params, t_end=1000.0)
    with pytest.raises(ValueError, match="snapshot_every"):
        pk.run(c.state, cfg, c.params, t_end=1200.0, snapshot_every=700.0)
    with pytest.raises(ValueError, match="workers"):
        pk.run(c.state, cfg, c.params, t_end=1200.0, workers=0)
    traj = pk.run(c.state, cfg, c.params, t_end=0.0)  # records the initial state only
    assert traj.steps == [0] and traj.times == [0.0]


def test_state_arithmetic_and_physics_validation():
    g = pk.make_grid(8, 8, 1.0, 1.0)
    a = pk.State(grid=g, u=np.ones((8, 8)), v=np.zeros((8, 8)), eta=np.zeros((8, 8)), t=1.0)
    b = 2.0 * a + a
    assert np.all(b.u == 3.0) and b.t == 1.0
    with pytest.raises(ValueError, match="shape"):
        pk.State(grid=g, u=np.ones((4, 8)), v=np.zeros((8, 8)), eta=np.zeros((8, 8)))
    with pytest.raises(ValueError, match="H must be positive"):
        pk.PhysicsParams(f=1e-4, g=9.8, H=-1.0, b=np.zeros((8, 8)))
    tall = np.zeros((8, 8), complex)
    tall[0, 0] = 64 * 7000.0
    with pytest.raises(ValueError, match="below H"):
        pk.PhysicsParams(f=1e-4, g=9.8, H=5960.0, b=tall)


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4"])
def test_cases_reproduce_the_golden_inputs(name):
    """cases.py builds the same inputs the goldens were generated from (after Hermitian projection)."""
    from oracle import layout
    c = cases.CASES[name]()
    z = load_golden(name)
    U = np.stack([c.state.u, c.state.v, c.state.eta])
    assert np.max(np.abs(layout.pack(U) - z["U"])) <= 1e-12 * np.max(np.abs(z["U"]))
    assert (c.grid.nx, c.M, c.T_half, c.dt, c.nsteps) == (int(z["nx"]), int(z["M"]), float(z["T_half"]),
                                                         float(z["dt"]), int(z["nsteps"]))


def test_case_c5_is_geostrophically_balanced():
    from oracle import pswe_oracle as O
    for r in (4, 5):
        c = cases.case_c5(r, 8)
        g, p = c.grid, c.params
        S = O.Setup(g.nx, g.ny, g.Lx, g.Ly, p.f, p.g, p.H)
        U = np.stack([c.state.u, c.state.v, c.state.eta])
        assert O.energy_norm(S, O.linear(S, U)) <= 1e-12 * p.f * O.energy_norm(S, U)
        assert c.P == 15 and math.isclose(float(np.max(np.abs(O.real_field(U[2])))), 0.1 * p.H, rel_tol=1e-12)


def test_host_to_physical_gate_matches_reference():
    """The host to_physical carries the reference's symmetry gate
    (grid.py:159-172): same exception and message, same pass/fail edge."""
    import numpy as np
    from oracle import reference as R
    from paper_2103_07706_b200 import grid as G

    rng = np.random.default_rng(3)
    g = G.make_grid(12, 16, 3.0e6, 4.0e6)
    c = np.fft.fft2(rng.standard_normal((12, 16)))
    G.to_physical(g, c)  # round-off asymmetry passes
    ref = R.load()
    for i, j, rel in ((2, 3, 1e-6), (0, 5, 1e-9), (7, 0, 2e-12), (6, 8, 1e-3)):
        bad = c.copy()
        bad[i, j] += rel * np.max(np.abs(c))
        try:
            G.to_physical(g, bad, scale=None)
            ours = None
        except ValueError as exc:
            ours = str(exc)
        assert ours is None or ours.startswith("non-Hermitian spectral field: mode (kx index ")
        if ref is not None:
            from phaseswe import grid as RG
            rg = RG.make_grid(12, 16, 3.0e6, 4.0e6)
            try:
                RG.to_physical(rg, bad)
                want = None
            except ValueError as exc:
                want = str(exc)
            assert ours == want, (ours, want)

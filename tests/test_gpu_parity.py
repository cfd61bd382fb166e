"""GPU parity: the CUDA path against the reference's golden vectors and the oracle.

Tolerances (north_star): relative L2 <= 1e-10 per averaged-RHS evaluation,
<= 1e-8 after the named number of steps; unit operators are held to the
reference's own test tolerances (1e-12 .. 1e-15).  Every call goes through
the C ABI (libpswe_b200.so) via the drop-in Python API.
"""

import numpy as np
import pytest

import paper_2103_07706_b200 as pk
from conftest import load_golden, rel_l2
from oracle import layout
from oracle import pswe_oracle as O
from paper_2103_07706_b200 import _native, cases

pytestmark = pytest.mark.gpu

F0, G0, H0 = 1.0e-4, 9.8, 5960.0
RHS_TOL = 1e-10
STEP_TOL = 1e-8


def state_from(U, grid, t=0.0):
    return pk.State(grid=grid, u=U[0], v=U[1], eta=U[2], t=t)


def arr(st):
    return np.stack([st.u, st.v, st.eta])


def flat(grid):
    return pk.PhysicsParams(f=F0, g=G0, H=H0, b=np.zeros((grid.nx, grid.ny), complex))


def golden_problem(z):
    nx, ny = int(z["nx"]), int(z["ny"])
    grid = pk.make_grid(nx, ny, float(z["Lx"]), float(z["Ly"]))
    b = layout.unpack(np.stack([z["b"]] * 3), nx, ny)[0]
    params = pk.PhysicsParams(f=float(z["f"]), g=float(z["g"]), H=float(z["H"]), b=b)
    state = state_from(layout.unpack(z["U"], nx, ny), grid)
    quad = pk.kernel_weights(float(z["T_half"]), int(z["M"]))
    return grid, params, state, quad


# ---------------------------------------------------------------- unit operators
def test_exact_exp_and_linear_match_reference_8x8(unit_golden):
    g8 = pk.make_grid(8, 8, 1.0e6, 1.0e6)
    st = state_from(unit_golden["exp8_U"], g8)
    p = flat(g8)
    for t, key in ((500.0, "exp8_p500"), (-250.0, "exp8_m250")):
        out = pk.exact_exp(t, st, p)
        want = unit_golden[key]
        assert np.max(np.abs(arr(out) - want)) <= 1e-12 * np.max(np.abs(want))
        assert out.t == t
    lin = pk.apply_linear(st, p)
    assert np.max(np.abs(arr(lin) - unit_golden["lin8"])) <= 1e-13 * np.max(np.abs(unit_golden["lin8"]))


def test_nonlinear_matches_reference_8x8_with_topography(unit_golden):
    g8 = pk.make_grid(8, 8, 1.0e6, 1.0e6)
    p = pk.PhysicsParams(f=F0, g=G0, H=H0, b=unit_golden["nl8_b"])
    out = pk.apply_nonlinear(state_from(unit_golden["nl8_U"], g8), p)
    want = unit_golden["nl8_N"]
    for f in range(3):
        assert np.max(np.abs(arr(out)[f] - want[f])) <= 1e-12 * np.max(np.abs(want[f]))


def test_averaged_tendency_32_exact_and_chebyshev(unit_golden):
    g = pk.make_grid(32, 32, 4.0e7, 4.0e7)
    st = state_from(layout.unpack(unit_golden["avg32_U"], 32, 32), g)
    q = pk.kernel_weights(1800.0, 3)
    got = pk.averaged_tendency(st, q, flat(g), pk.PropagatorSpec.exact())
    assert rel_l2(layout.pack(arr(got)), unit_golden["avg32_exact"]) <= 1e-13
    spec = pk.PropagatorSpec.chebyshev(float(unit_golden["avg32_cheb_Lambda"]))
    assert spec.n_poly == int(unit_golden["avg32_cheb_npoly"])
    got = pk.averaged_tendency(st, q, flat(g), spec)
    assert rel_l2(layout.pack(arr(got)), unit_golden["avg32_cheb"]) <= 1e-13


# ---------------------------------------------------------------- BASELINE configs
@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4"])
def test_config_rhs_matches_reference(name):
    z = load_golden(name)
    grid, params, state, quad = golden_problem(z)
    got = pk.averaged_tendency(state, quad, params, pk.PropagatorSpec.exact())
    err = rel_l2(layout.pack(arr(got)), z["rhs"])
    print(f"{name} RHS rel L2 {err:.3e}")
    assert err <= RHS_TOL
    assert got.t == state.t


@pytest.mark.parametrize("name", ["C2", "C3", "C4"])
def test_config_steps_match_reference(name):
    z = load_golden(name)
    grid, params, state, quad = golden_problem(z)
    cfg = pk.StepConfig(dt=float(z["dt"]), quadrature=quad, propagator_spec=pk.PropagatorSpec.exact())
    one = pk.step_averaged_ssprk3(state, cfg, params)
    err1 = rel_l2(layout.pack(arr(one)), z["step1"])
    assert err1 <= STEP_TOL
    assert one.t == float(z["dt"])
    if "final" in z:
        traj = pk.run(state, cfg, params, t_end=float(z["dt"]) * int(z["nsteps"]))
        fin = traj.states[-1]
        err = rel_l2(layout.pack(arr(fin)), z["final"])
        print(f"{name}: step1 {err1:.3e}, after {int(z['nsteps'])} steps {err:.3e}")
        assert err <= STEP_TOL
        assert fin.t == float(z["t_final"])


def test_fine_step_reference_matches_oracle():
    """step_reference (integrator.py:106-110): T = 0, M = 0, dt = 180 s -- the
    fine-step solver of cmd_reference, same kernels with one node."""
    z = load_golden("C2")
    grid, params, state, _ = golden_problem(z)
    dt, n = 180.0, 20
    one = pk.step_reference(state, dt, params)
    cfg = pk.StepConfig(dt=dt, quadrature=pk.kernel_weights(0.0, 0), propagator_spec=pk.PropagatorSpec.exact())
    traj = pk.run(state, cfg, params, t_end=n * dt)
    S = O.Setup(grid.nx, grid.ny, grid.Lx, grid.Ly, params.f, params.g, params.H, params.b)
    want1 = O.ssprk3_step(S, arr(state), dt, [0.0], [1.0])
    wantn = O.run(S, arr(state), dt, n, [0.0], [1.0])
    assert rel_l2(arr(one), want1) <= STEP_TOL
    assert rel_l2(arr(traj.states[-1]), wantn) <= STEP_TOL
    assert traj.states[-1].t == pytest.approx(n * dt)


# ---------------------------------------------------------------- full sizes vs oracle
def test_c5_512_rhs_matches_oracle():
    c = cases.case_c5(7, 8)  # 512^2, 15 phases
    got = pk.averaged_tendency(c.state, c.quadrature, c.params, pk.PropagatorSpec.exact())
    g = c.grid
    S = O.Setup(g.nx, g.ny, g.Lx, g.Ly, c.params.f, c.params.g, c.params.H)
    q = c.quadrature
    want = O.averaged_tendency(S, arr(c.state), q.s, q.w, workers=8)
    err = O.rel_l2(arr(got), want)
    print(f"C5 512^2 M=8 rel L2 vs oracle {err:.3e}")
    assert err <= RHS_TOL


def _oracle_rhs(c, U=None, workers=16):
    g, q = c.grid, c.quadrature
    S = O.Setup(g.nx, g.ny, g.Lx, g.Ly, c.params.f, c.params.g, c.params.H, c.params.b)
    return O.averaged_tendency(S, arr(c.state) if U is None else U, q.s, q.w, workers=workers)


@pytest.mark.parametrize("level,M", [(7, 256), (6, 256)])
def test_c5_benchmarked_rhs_matches_oracle(level, M):
    """The benchmarked configuration itself: all 2M - 1 live phases (511 at
    M = 256) through 4 lanes x several chunks, the phase-paired pass B and
    the multi-slot reduction, against the oracle's full node sum
    (averaging.py:128-156)."""
    c = cases.case_c5(level, M)
    got = pk.averaged_tendency(c.state, c.quadrature, c.params, pk.PropagatorSpec.exact())
    err = O.rel_l2(arr(got), _oracle_rhs(c))
    print(f"C5 {c.grid.nx}^2 M={M} rel L2 vs oracle {err:.3e}")
    assert err <= RHS_TOL


@pytest.mark.parametrize("M", [8, 32, 128, 256])
@pytest.mark.parametrize("level", [4, 5, 6, 7])
def test_c5_sweep_point_unbalanced_matches_oracle(level, M):
    """Every point of the C5 throughput sweep (refinements 4-7 x M in {8, 32,
    128, 256}: all 16 entries of bench.py's `sweep`), all 2M - 1 live phases
    against the oracle's node sum.  C5 states are balanced (e^{sL} U = U),
    which would hide a wrong phase shift in pass A; here an unbalanced,
    band-limited perturbation of O(1) relative size is added, so every
    phase's forward and backward exponential matters.  The points cover the
    cluster kernel (64^2, M <= 32), one-chunk chains, and several chunks per
    lane on every lane with phase pairs and several pass-C slots."""
    c = cases.case_c5(level, M)
    g = c.grid
    rng = np.random.default_rng(100 + level + 1000 * (M != 128) * M)
    S = O.Setup(g.nx, g.ny, g.Lx, g.Ly, c.params.f, c.params.g, c.params.H)
    U = arr(c.state)
    pert = np.stack([O.truncate(O.spectral(rng.standard_normal((g.nx, g.ny))), S.mask) for _ in range(3)])
    for f in range(3):
        pert[f] *= 0.5 * np.max(np.abs(U[f])) / np.max(np.abs(pert[f]))
    U = U + pert
    got = pk.averaged_tendency(state_from(U, g), c.quadrature, c.params, pk.PropagatorSpec.exact())
    err = O.rel_l2(arr(got), _oracle_rhs(c, U))
    print(f"C5 {g.nx}^2 M={M} unbalanced rel L2 vs oracle {err:.3e}")
    assert err <= RHS_TOL


def test_linearity_in_weights_at_512_m256():
    """Full-size property: A(w_even + w_odd) = A(w_even) + A(w_odd) over all 511 phases."""
    c = cases.case_c5(7, 256)
    g, q = c.grid, c.quadrature
    ctx = pk.dynamics.context(c.state, c.params)
    ctx.set_propagator("exact")
    U = pk.dynamics.upload(ctx, c.state)
    Uc = ctx.pack(U)
    w = np.array(q.w)
    idx = np.arange(len(w))
    parts = []
    for sel in (idx % 2 == 0, idx % 2 == 1, np.ones_like(idx, bool)):
        ctx.set_quadrature(q.s, np.where(sel, w, 0.0))
        parts.append(ctx.averaged_tendency_compact(Uc).cpu().numpy())
    assert rel_l2(parts[0] + parts[1], parts[2]) <= 1e-13
    # run-to-run bitwise determinism of the full 511-phase evaluation
    again = ctx.averaged_tendency_compact(Uc).cpu().numpy()
    assert np.array_equal(again, parts[2])


@pytest.mark.parametrize("level,M", [(6, 64), (7, 32)])
def test_repeated_evaluations_are_bitwise_identical(level, M):
    """Run-to-run determinism over many evaluations (guards the TMA-prefetch/in-place buffer protocol)."""
    c = cases.case_c5(level, M)
    ctx = pk.dynamics.context(c.state, c.params)
    ctx.set_propagator("exact")
    ctx.set_quadrature(c.quadrature.s, c.quadrature.w)
    Uc = ctx.pack(pk.dynamics.upload(ctx, c.state))
    first = ctx.averaged_tendency_compact(Uc).cpu().numpy()
    for _ in range(6):
        assert np.array_equal(ctx.averaged_tendency_compact(Uc).cpu().numpy(), first)


@pytest.mark.parametrize("level", [5, 7])
def test_chunking_and_lanes_do_not_change_results(level):
    """Chunk size and lane count only regroup the phase sum (and the pass-B
    phase pairing): results agree to round-off, and each configuration is
    itself bitwise reproducible."""
    c = cases.case_c5(level, 32)  # 63 phases
    ctx = pk.dynamics.context(c.state, c.params)
    ctx.set_propagator("exact")
    ctx.set_quadrature(c.quadrature.s, c.quadrature.w)
    Uc = ctx.pack(pk.dynamics.upload(ctx, c.state))
    base = ctx.averaged_tendency_compact(Uc).cpu().numpy()
    lanes0 = ctx.lanes
    per_phase = 9 * 16 * (c.grid.ny // 3 + 1) * c.grid.nx
    try:
        for chunk, lanes in ((1, 1), (1, 4), (7 * per_phase, 2), (16 * per_phase, 3), (1536 << 20, 1)):
            ctx.set_chunk_bytes(chunk)
            ctx.set_lanes(lanes)
            a = ctx.averaged_tendency_compact(Uc).cpu().numpy()
            b = ctx.averaged_tendency_compact(Uc).cpu().numpy()
            assert np.array_equal(a, b), (chunk, lanes)
            assert rel_l2(a, base) <= 1e-14, (chunk, lanes)
    finally:
        ctx.set_chunk_bytes(1536 << 20)
        ctx.set_lanes(lanes0)


def test_rectangular_grid_matches_oracle():
    rng = np.random.default_rng(5)
    g = pk.make_grid(64, 32, 4.0e7, 2.0e7)
    S = O.Setup(64, 32, 4.0e7, 2.0e7, F0, G0, H0)
    S.b = O.truncate(O.spectral(30.0 * rng.standard_normal((64, 32))), S.mask)
    U = np.stack([O.truncate(O.spectral(sc * rng.standard_normal((64, 32))), S.mask) for sc in (1.0, 1.0, 50.0)])
    p = pk.PhysicsParams(f=F0, g=G0, H=H0, b=S.b)
    q = pk.kernel_weights(3600.0, 4)
    got = pk.averaged_tendency(state_from(U, g), q, p, pk.PropagatorSpec.exact())
    want = O.averaged_tendency(S, U, q.s, q.w)
    assert O.rel_l2(arr(got), want) <= 1e-12


# ---------------------------------------------------------------- edge cases
def test_zero_window_equals_plain_nonlinearity_bitwise():
    c = cases.case_c1()
    got = pk.averaged_tendency(c.state, pk.kernel_weights(0.0, 0), c.params, pk.PropagatorSpec.exact())
    want = pk.apply_nonlinear(c.state, c.params)
    assert np.array_equal(arr(got), arr(want))


def test_uniform_kernel_includes_endpoints():
    c = cases.case_c1()
    q = pk.kernel_weights(1800.0, 3, pk.UNIFORM_KERNEL)
    got = pk.averaged_tendency(c.state, q, c.params, pk.PropagatorSpec.exact())
    g = c.grid
    S = O.Setup(g.nx, g.ny, g.Lx, g.Ly, c.params.f, c.params.g, c.params.H)
    assert O.rel_l2(arr(got), O.averaged_tendency(S, arr(c.state), q.s, q.w)) <= 1e-12


def test_mean_eta_tendency_is_exactly_zero():
    z = load_golden("C3")
    grid, params, state, quad = golden_problem(z)
    assert pk.apply_nonlinear(state, params).eta[0, 0] == 0.0
    assert pk.averaged_tendency(state, quad, params, pk.PropagatorSpec.exact()).eta[0, 0] == 0.0


def test_output_is_band_limited_and_hermitian():
    c = cases.case_c1()
    got = arr(pk.averaged_tendency(c.state, c.quadrature, c.params, pk.PropagatorSpec.exact()))
    mask = c.grid.dealias_mask
    assert np.all(got[:, ~mask] == 0.0)
    refl = np.roll(np.flip(got, axis=(1, 2)), shift=(1, 1), axis=(1, 2))
    assert np.max(np.abs(got - np.conj(refl))) <= 1e-13 * np.max(np.abs(got))


@pytest.mark.parametrize("nx,ny,M", [(12, 12, 3), (48, 48, 8), (96, 96, 16), (48, 96, 4), (30, 18, 2), (1024, 1024, 2)])
def test_any_even_grid_matches_oracle(nx, ny, M):
    """Every even n >= 8 the reference accepts (grid.py:91-93): the generic
    mixed-radix kernels (3 * 2^k, other primes, n > 512) vs the oracle, for
    N alone and the averaged tendency, with topography."""
    rng = np.random.default_rng(nx + ny)
    g = pk.make_grid(nx, ny, 4.0e7, 4.0e7 * ny / nx)
    S = O.Setup(nx, ny, g.Lx, g.Ly, F0, G0, H0)
    S.b = O.truncate(O.spectral(30.0 * rng.standard_normal((nx, ny))), S.mask)
    U = np.stack([O.truncate(O.spectral(sc * rng.standard_normal((nx, ny))), S.mask) for sc in (1.0, 1.0, 50.0)])
    p = pk.PhysicsParams(f=F0, g=G0, H=H0, b=S.b)
    st = state_from(U, g)
    assert O.rel_l2(arr(pk.apply_nonlinear(st, p)), O.nonlinear(S, U)) <= 1e-12
    q = pk.kernel_weights(3600.0, M)
    got = pk.averaged_tendency(st, q, p, pk.PropagatorSpec.exact())
    assert O.rel_l2(arr(got), O.averaged_tendency(S, U, q.s, q.w, workers=8)) <= RHS_TOL


def test_any_even_grid_steps_run_and_diagnostics():
    """48^2 (3 * 2^4): a 3-step run vs the oracle, its snapshot diagnostics vs
    the oracle's, and the 12^2 grid of the reference's own tests through a step."""
    for n, steps in ((48, 3), (12, 2)):
        rng = np.random.default_rng(n)
        g = pk.make_grid(n, n, 4.0e7, 4.0e7)
        S = O.Setup(n, n, g.Lx, g.Ly, F0, G0, H0)
        U = np.stack([O.truncate(O.spectral(sc * rng.standard_normal((n, n))), S.mask) for sc in (1.0, 1.0, 50.0)])
        p = flat(g)
        st = state_from(U, g)
        q = pk.kernel_weights(1800.0, 4)
        cfg = pk.StepConfig(dt=900.0, quadrature=q, propagator_spec=pk.PropagatorSpec.exact())
        traj = pk.run(st, cfg, p, t_end=steps * 900.0)
        want = O.run(S, U, 900.0, steps, q.s, q.w)
        assert O.rel_l2(arr(traj.states[-1]), want) <= STEP_TOL
        en, ms = O.energy_mass(S, want)
        assert abs(traj.energy[-1] - en) <= 1e-12 * abs(en)
        assert abs(traj.mass[-1] - ms) <= 1e-12 * abs(ms)


def test_oversized_grid_is_refused():
    g = pk.make_grid(8192, 8, 4.0e7, 4.0e7)
    st = pk.State(grid=g, u=np.zeros((8192, 8)), v=np.zeros((8192, 8)), eta=np.zeros((8192, 8)))
    with pytest.raises(ValueError, match="not supported by the B200 path"):
        pk.apply_nonlinear(st, flat(g))


def test_chebyshev_window_violation_names_the_node():
    c = cases.case_c1()
    spec = pk.PropagatorSpec.chebyshev(pk.max_frequency(c.grid, c.params) * 100.0)
    with pytest.raises(RuntimeError, match=r"averaging node k = -7 .*exceeds Lambda"):
        pk.averaged_tendency(c.state, c.quadrature, c.params, spec)


def test_nonfinite_state_aborts_with_stage_and_field():
    c = cases.case_c1()
    u = c.state.u.copy()
    u[40 % 32, 3] = np.inf
    bad = pk.State(grid=c.grid, u=u, v=c.state.v, eta=c.state.eta)
    cfg = pk.make_step_config(c.grid, c.params, dt=600.0)
    with pytest.raises(RuntimeError, match="non-finite values in field u after stage 1"):
        pk.step_averaged_ssprk3(bad, cfg, c.params)


def test_native_code_is_what_ran():
    c = cases.case_c1()
    ctx = pk.dynamics.context(c.state, c.params)
    before = ctx.launch_count
    pk.averaged_tendency(c.state, c.quadrature, c.params, pk.PropagatorSpec.exact())
    assert ctx.launch_count > before
    assert _native._lib is not None


def test_run_reports_failing_step_and_keeps_its_start_state():
    """pswe_run (graph-batched) finds the exact failing step, like run()'s step loop (integrator.py:173-177)."""
    c = cases.case_c1()
    cfg = pk.StepConfig(dt=3600.0, quadrature=c.quadrature, propagator_spec=pk.PropagatorSpec.exact())
    ctx = pk.integrator._prepare(c.state, cfg, c.params)
    U = pk.dynamics.upload(ctx, c.state)
    assert ctx.run(3600.0, 20, U) == (0, 0, -1)
    # a huge state blows up after a few steps; the graph batch is replayed to locate the step
    big = pk.State(grid=c.grid, u=c.state.u * 1e7, v=c.state.v, eta=c.state.eta * 1e7)
    U = pk.dynamics.upload(ctx, big)
    bad_step, stage, fld = ctx.run(3600.0, 40, U)
    assert bad_step > 1 and stage in (1, 2, 3) and fld in (0, 1, 2)
    # the returned state is the (finite) state at the start of the failing step
    assert all(bool(t.isfinite().all()) for t in U)
    U2 = pk.dynamics.upload(ctx, big)
    assert ctx.run(3600.0, bad_step - 1, U2) == (0, 0, -1)
    assert all(bool((a == b).all()) for a, b in zip(U, U2))


def test_graph_batched_run_matches_single_steps_bitwise():
    c = cases.case_c2()
    cfg = pk.StepConfig(dt=c.dt, quadrature=c.quadrature, propagator_spec=pk.PropagatorSpec.exact())
    ctx = pk.integrator._prepare(c.state, cfg, c.params)
    U = pk.dynamics.upload(ctx, c.state)
    ctx.run(c.dt, 20, U)
    V = pk.dynamics.upload(ctx, c.state)
    for _ in range(20):
        V, (st, fl) = ctx.ssprk3_step(c.dt, V)
        assert st == 0
    assert all(bool((a == b).all()) for a, b in zip(U, V))


def test_window_sweep_batch_matches_individual_runs():
    """8f item 2: all windows advance as one window batch (one launch
    sequence per stage over the (window, phase) axis).  Each window equals
    its own one-by-one run to round-off (the batch regroups the phase sums
    and pairs phases of neighbouring windows in pass B), the batch really
    ran (variant counts), and errors vs a fine reference are filled in."""
    c = cases.CASES["C2"]()
    dt, t_end = c.dt, 2 * c.dt
    windows = (0.0, 1800.0, 3600.0, 7200.0)
    ref = pk.run(c.state, pk.StepConfig(dt=180.0, quadrature=pk.kernel_weights(0.0, 0),
                                        propagator_spec=pk.PropagatorSpec.exact()), c.params, t_end).states[-1]
    ctx = pk.dynamics.context(c.state, c.params)
    before = ctx.launch_count
    res = pk.window_sweep(c.state, c.params, dt, t_end, windows, M=8, reference=ref)
    assert ctx.launch_count > before
    assert [r.T for r in res] == list(windows)
    for r in res:
        cfg = pk.make_step_config(c.grid, c.params, dt=dt, T=r.T, M=8 if r.T > 0 else 0)
        solo = pk.run(c.state, cfg, c.params, t_end)
        assert rel_l2(arr(r.final), arr(solo.states[-1])) <= 1e-13
        assert r.final.t == solo.states[-1].t
        assert r.trajectory.steps == solo.steps
        assert np.allclose(r.trajectory.energy, solo.energy, rtol=1e-12, atol=0)
        assert np.isfinite(r.l2_eta) and np.isfinite(r.l2_u)
    seq = pk.window_sweep(c.state, c.params, dt, t_end, windows, M=8, batched=False)
    for a, b in zip(res, seq):
        assert rel_l2(arr(a.final), arr(b.final)) <= 1e-13


def test_window_batch_matches_oracle():
    """Two windows of different length (7 and 15 live phases) over two steps
    with a mountain (C3's grid): each window vs the oracle's own run, and the
    batched averaged tendencies vs the oracle per window."""
    z = load_golden("C3")
    grid, params, state, _ = golden_problem(z)
    dt = float(z["dt"])
    quads = [pk.kernel_weights(900.0, 4), pk.kernel_weights(1800.0, 8)]
    S = O.Setup(grid.nx, grid.ny, grid.Lx, grid.Ly, params.f, params.g, params.H, params.b)
    ctx = pk.dynamics.context(state, params)
    ctx.set_propagator("exact")
    ctx.set_window_batch(quads)
    U = arr(state)
    # tendencies: window w sees its own state (here two different states)
    U2 = np.stack([U, 1.01 * U])
    Uc = torch_compact(ctx, U2)
    got = ctx.window_batch_tendency(Uc)
    for w, q in enumerate(quads):
        want = O.averaged_tendency(S, U2[w], q.s, q.w)
        full = np.stack([t.cpu().numpy() for t in ctx.unpack(got[w])])
        assert O.rel_l2(full, want) <= RHS_TOL
    # two steps of both windows at once
    res = pk.window_sweep(state, params, dt, 2 * dt, [900.0, 1800.0], M=None)
    for r in res:
        q = pk.make_step_config(grid, params, dt=dt, T=r.T).quadrature
        want = O.run(S, U, dt, 2, q.s, q.w)
        assert O.rel_l2(arr(r.final), want) <= STEP_TOL


def torch_compact(ctx, U2):
    import torch
    out = []
    for Uw in U2:
        out.append(ctx.pack([ctx.to_device(x) for x in Uw]))
    return torch.stack(out).contiguous()


def test_chebyshev_route_step_and_run_match_oracle():
    """The Chebyshev exponential route (propagator.py:161-191) through the
    whole stepper: 3 averaged RHS + 5 stage exponentials per step, vs the
    oracle with the same Lambda / n_poly, over a 3-step run on C2's problem."""
    z = load_golden("C2")
    grid, params, state, _ = golden_problem(z)
    cfg = pk.make_step_config(grid, params, dt=float(z["dt"]), T=float(z["T_half"]), M=8,
                              propagator="chebyshev")
    spec = cfg.propagator_spec
    S = O.Setup(grid.nx, grid.ny, grid.Lx, grid.Ly, params.f, params.g, params.H, params.b)
    prop = O.Propagator("chebyshev", spec.Lambda, spec.n_poly)
    q = cfg.quadrature
    want = O.run(S, arr(state), cfg.dt, 3, q.s, q.w, prop)
    got = pk.run(state, cfg, params, t_end=3 * cfg.dt).states[-1]
    err = rel_l2(arr(got), want)
    print(f"chebyshev 3-step run rel L2 vs oracle {err:.3e}")
    assert err <= STEP_TOL


def test_latency_paths_are_bitwise_identical(tmp_path):
    """The latency-bound paths (split pass B, programmatic dependent launch)
    change scheduling only: a run with both switched off (fresh process, the
    switches are read once) gives the same bits for a 128^2 (M = 4) RHS and step, and
    for a single-node 512^2 nonlinearity (split pass B at NY = 512).  The
    baseline run must really have taken the split path (variant counts)."""
    import os
    import subprocess
    import sys

    from conftest import ROOT

    code = (
        "import sys, json, numpy as np; sys.path.insert(0, %r)\n"
        "import paper_2103_07706_b200 as pk\n"
        "from paper_2103_07706_b200 import cases\n"
        "c = cases.case_c5(5, 4)\n"
        "a = pk.averaged_tendency(c.state, c.quadrature, c.params, pk.PropagatorSpec.exact())\n"
        "cfg = pk.StepConfig(dt=600.0, quadrature=c.quadrature, propagator_spec=pk.PropagatorSpec.exact())\n"
        "s = pk.step_averaged_ssprk3(c.state, cfg, c.params)\n"
        "v = pk.dynamics.context(c.state, c.params).variant_launches\n"
        "d = cases.case_c5(7, 8)\n"
        "n = pk.apply_nonlinear(d.state, d.params)\n"
        "v2 = pk.dynamics.context(d.state, d.params).variant_launches\n"
        "np.save(sys.argv[1], np.stack([a.u, a.v, a.eta, s.u, s.v, s.eta]))\n"
        "np.save(sys.argv[1] + '.512.npy', np.stack([n.u, n.v, n.eta]))\n"
        "print(json.dumps([v, v2]))\n" % str(ROOT))
    base = {k: v for k, v in os.environ.items() if not k.startswith("PSWE_")}
    outs, variants = [], []
    for i, env in enumerate(({}, {"PSWE_NO_SPLIT": "1", "PSWE_NO_PDL": "1"})):
        f = tmp_path / f"r{i}.npy"
        p = subprocess.run([sys.executable, "-c", code, str(f)], env={**base, **env},
                           capture_output=True, text=True, timeout=300)
        assert p.returncode == 0, p.stderr
        import json
        variants.append(json.loads(p.stdout.strip().splitlines()[-1]))
        outs.append((np.load(f), np.load(str(f) + ".512.npy")))
    assert variants[0][0]["passB_split"] > 0 and variants[1][0]["passB_split"] == 0
    assert variants[0][1]["passB_split"] > 0 and variants[1][1]["passB_split"] == 0
    assert np.array_equal(outs[0][0], outs[1][0])
    assert np.array_equal(outs[0][1], outs[1][1])


def test_prewait_work_of_the_step_chain_is_race_free(tmp_path):
    """Under programmatic dependent launch the one-launch small-grid kernels
    and the stage kernels do their chain-independent work before the
    dependency wait ("Dependent-launch prologues").  That is only
    legal while no kernel starts before everything two kernels back has
    completed; the shortest chains test it: a single-node (T = 0) run, where a
    stage kernel directly follows the one-launch kernel (no slot reduction in
    between), at 64^2 and 32^2, a C2 run, and a 700-step single-node run
    (eight steps per graph, no copies between them).  With dependent launch
    and the eight-step graphs switched off (fresh process) the bits must be
    the same."""
    import os
    import subprocess
    import sys

    from conftest import ROOT

    code = (
        "import sys, numpy as np; sys.path.insert(0, %r)\n"
        "import paper_2103_07706_b200 as pk\n"
        "from paper_2103_07706_b200 import cases\n"
        "res = []\n"
        "for c, dt, n, quad in ((cases.case_c2(), 180.0, 96, pk.kernel_weights(0.0, 0)),\n"
        "                       (cases.case_c1(), 180.0, 96, pk.kernel_weights(0.0, 0)),\n"
        "                       (cases.case_c2(), None, 12, None)):\n"
        "    cfg = pk.StepConfig(dt=dt or c.dt, quadrature=quad or c.quadrature,\n"
        "                        propagator_spec=pk.PropagatorSpec.exact())\n"
        "    s = pk.run(c.state, cfg, c.params, t_end=n * cfg.dt).states[-1]\n"
        "    res += [s.u.ravel(), s.v.ravel(), s.eta.ravel()]\n"
        "c = cases.case_c2()  # long enough for the eight-step graphs (pswe_run)\n"
        "cfg = pk.StepConfig(dt=180.0, quadrature=pk.kernel_weights(0.0, 0), propagator_spec=pk.PropagatorSpec.exact())\n"
        "s = pk.run(c.state, cfg, c.params, t_end=700 * cfg.dt).states[-1]\n"
        "res += [s.u.ravel(), s.v.ravel(), s.eta.ravel()]\n"
        "np.save(sys.argv[1], np.concatenate(res))\n" % str(ROOT))
    base = {k: v for k, v in os.environ.items() if not k.startswith("PSWE_")}
    outs = []
    for i, env in enumerate(({}, {"PSWE_NO_PDL": "1", "PSWE_NO_MULTISTEP_GRAPH": "1"})):
        f = tmp_path / f"r{i}.npy"
        p = subprocess.run([sys.executable, "-c", code, str(f)], env={**base, **env},
                           capture_output=True, text=True, timeout=300)
        assert p.returncode == 0, p.stderr
        outs.append(np.load(f))
    assert np.all(np.isfinite(outs[0]))
    assert np.array_equal(outs[0], outs[1])


def test_staged_slot_reduction_gives_the_same_bits(tmp_path):
    """The staged slot reduction (32 slots per load round through shared
    memory) and the stage kernels' 64-thread blocks on small grids change
    scheduling only: with both switched off (PSWE_NO_STAGED: the serial
    batches; PSWE_STAGE_TB256) a fresh process gives the same bits for 64^2
    evaluations with 15, 63 (two rounds of the cluster kernel's slots) and
    255 phases, a 32^2 M = 64 evaluation (127 slots: four rounds), a 256^2
    M = 8 evaluation (three-pass path, staged) and a C2 step."""
    import os
    import subprocess
    import sys

    from conftest import ROOT

    code = (
        "import sys, numpy as np; sys.path.insert(0, %r)\n"
        "import paper_2103_07706_b200 as pk\n"
        "from paper_2103_07706_b200 import cases\n"
        "outs = []\n"
        "for r, M in ((4, 8), (4, 32), (4, 128), (3, 64), (6, 8)):\n"
        "    c = cases.case_c5(r, M)\n"
        "    a = pk.averaged_tendency(c.state, c.quadrature, c.params, pk.PropagatorSpec.exact())\n"
        "    outs.append(np.concatenate([a.u.ravel(), a.v.ravel(), a.eta.ravel()]))\n"
        "c = cases.case_c2()\n"
        "cfg = pk.StepConfig(dt=c.dt, quadrature=c.quadrature, propagator_spec=pk.PropagatorSpec.exact())\n"
        "s = pk.step_averaged_ssprk3(c.state, cfg, c.params)\n"
        "outs.append(np.concatenate([s.u.ravel(), s.v.ravel(), s.eta.ravel()]))\n"
        "np.save(sys.argv[1], np.concatenate(outs))\n" % str(ROOT))
    base = {k: v for k, v in os.environ.items() if not k.startswith("PSWE_")}
    outs = []
    for i, env in enumerate(({}, {"PSWE_NO_STAGED": "1", "PSWE_STAGE_TB256": "1"})):
        f = tmp_path / f"r{i}.npy"
        p = subprocess.run([sys.executable, "-c", code, str(f)], env={**base, **env},
                           capture_output=True, text=True, timeout=300)
        assert p.returncode == 0, p.stderr
        outs.append(np.load(f))
    assert np.all(np.isfinite(outs[0]))
    assert np.array_equal(outs[0], outs[1])


def test_pairs_per_cta_give_the_same_bits(tmp_path):
    """Pass B's CTAs may take two phase pairs each (chosen for grids of many
    waves); scheduling only: one and two pairs per CTA give the same bits at
    256^2 for M = 32 (an odd phase count: the last pair holds one phase) and
    M = 5 (an odd pair count: the last CTA row holds one pair)."""
    import os
    import subprocess
    import sys

    from conftest import ROOT

    code = (
        "import sys, numpy as np; sys.path.insert(0, %r)\n"
        "import paper_2103_07706_b200 as pk\n"
        "from paper_2103_07706_b200 import cases\n"
        "outs = []\n"
        "for M in (32, 5):\n"
        "    c = cases.case_c5(6, 32)\n"
        "    q = pk.kernel_weights(c.quadrature.T, M)\n"
        "    a = pk.averaged_tendency(c.state, q, c.params, pk.PropagatorSpec.exact())\n"
        "    outs.append(np.stack([a.u, a.v, a.eta]))\n"
        "np.save(sys.argv[1], np.stack(outs))\n" % str(ROOT))
    base = {k: v for k, v in os.environ.items() if not k.startswith("PSWE_")}
    outs = []
    for q in ("1", "2"):
        f = tmp_path / f"q{q}.npy"
        p = subprocess.run([sys.executable, "-c", code, str(f)], env={**base, "PSWE_QPC": q},
                           capture_output=True, text=True, timeout=300)
        assert p.returncode == 0, p.stderr
        outs.append(np.load(f))
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.parametrize("level", [6, 7])
def test_single_node_large_grid_matches_oracle(level):
    """One node on 256^2 / 512^2 (apply_nonlinear and the fine-step
    reference's step): the split pass B at NY = 256 / 512 against the oracle."""
    c = cases.case_c5(level, 8)
    g = c.grid
    rng = np.random.default_rng(level)
    S = O.Setup(g.nx, g.ny, g.Lx, g.Ly, c.params.f, c.params.g, c.params.H)
    U = arr(c.state) + np.stack([O.truncate(O.spectral(sc * rng.standard_normal((g.nx, g.ny))), S.mask)
                                 for sc in (1.0, 1.0, 50.0)])
    st = state_from(U, g)
    got = pk.apply_nonlinear(st, c.params)
    assert O.rel_l2(arr(got), O.nonlinear(S, U)) <= 1e-12
    one = pk.step_reference(st, 180.0, c.params)
    assert O.rel_l2(arr(one), O.ssprk3_step(S, U, 180.0, [0.0], [1.0])) <= STEP_TOL
    v = pk.dynamics.context(st, c.params).variant_launches
    assert v["passB_split"] > 0


_VARIANT_WORKLOAD = (
    "import sys, json, numpy as np; sys.path.insert(0, %r)\n"
    "import paper_2103_07706_b200 as pk\n"
    "from paper_2103_07706_b200 import cases, _native\n"
    "outs, var = [], {}\n"
    "for r, M in ((3, 256), (4, 8), (5, 4), (5, 32), (6, 128), (7, 8), (7, 64)):\n"
    "    c = cases.case_c5(r, M)\n"
    "    ctx = pk.dynamics.context(c.state, c.params)\n"
    "    ctx.set_propagator('exact')\n"
    "    ctx.set_quadrature(c.quadrature.s, c.quadrature.w)\n"
    "    Uc = ctx.pack(pk.dynamics.upload(ctx, c.state))\n"
    "    for _ in range(3):\n"
    "        outs.append(ctx.averaged_tendency_compact(Uc).cpu().numpy())\n"
    "    for k, v in ctx.variant_launches.items(): var[k] = var.get(k, 0) + v\n"
    "c = cases.case_c2()\n"
    "cfg = pk.StepConfig(dt=c.dt, quadrature=c.quadrature, propagator_spec=pk.PropagatorSpec.exact())\n"
    "tr = pk.run(c.state, cfg, c.params, t_end=4 * c.dt)\n"
    "s = tr.states[-1]\n"
    "outs.append(np.stack([s.u, s.v, s.eta]))\n"
    "outs.append(np.array(pk.device_diagnostics(s, c.params)))\n"
    "g = pk.make_grid(64, 32, 4.0e7, 2.0e7)\n"
    "rng = np.random.default_rng(9)\n"
    "f = lambda sc: pk.dealias(g, pk.to_spectral(g, sc * rng.standard_normal((64, 32))))\n"
    "st = pk.State(grid=g, u=f(1.0), v=f(1.0), eta=f(50.0))\n"
    "p = pk.PhysicsParams(f=1e-4, g=9.8, H=5960.0, b=np.zeros((64, 32), complex))\n"
    "ctx = pk.dynamics.context(st, p)\n"
    "for _ in range(2):\n"
    "    a = pk.averaged_tendency(st, pk.kernel_weights(3600.0, 256), p, pk.PropagatorSpec.exact())\n"
    "    outs.append(np.stack([a.u, a.v, a.eta]))\n"
    "for k, v in ctx.variant_launches.items(): var[k] = var.get(k, 0) + v\n"
    "g = pk.make_grid(48, 48, 4.0e7, 4.0e7)\n"
    "f = lambda sc: pk.dealias(g, pk.to_spectral(g, sc * rng.standard_normal((48, 48))))\n"
    "st = pk.State(grid=g, u=f(1.0), v=f(1.0), eta=f(50.0))\n"
    "p = pk.PhysicsParams(f=1e-4, g=9.8, H=5960.0, b=np.zeros((48, 48), complex))\n"
    "a = pk.averaged_tendency(st, pk.kernel_weights(3600.0, 16), p, pk.PropagatorSpec.exact())\n"
    "outs.append(np.stack([a.u, a.v, a.eta]))\n"
    "c = cases.case_c3()\n"
    "ws = pk.window_sweep(c.state, c.params, c.dt, 2 * c.dt, [0.0, 1800.0, 3600.0], M=4)\n"
    "for w in ws: outs.append(np.stack([w.final.u, w.final.v, w.final.eta]))\n"
    "np.savez(sys.argv[1], *outs)\n"
    "gd, dm = _native.debug_check_guards()\n"
    "print(json.dumps({'var': var, 'guards': [gd, dm]}))\n")


def _variant_runs(tmp_path, envs):
    """Run the variant workload in fresh processes, one per environment;
    returns [(outputs, launches per variant, (guarded buffers, damaged guards))]."""
    import json
    import os
    import subprocess
    import sys

    from conftest import ROOT

    code = _VARIANT_WORKLOAD % str(ROOT)
    base = {k: v for k, v in os.environ.items() if not k.startswith("PSWE_")}
    res = []
    for i, env in enumerate(envs):
        f = tmp_path / f"p{i}.npz"
        p = subprocess.run([sys.executable, "-c", code, str(f)], env={**base, **env},
                           capture_output=True, text=True, timeout=600)
        assert p.returncode == 0, p.stderr
        info = json.loads(p.stdout.strip().splitlines()[-1])
        with np.load(f) as z:
            res.append(([z[k] for k in z.files], info["var"], tuple(info["guards"])))
    return res


def test_poisoned_scratch_gives_the_same_bits(tmp_path):
    """Stand-in for compute-sanitizer's initcheck/racecheck (closed on the
    GPU pool): with every intermediate, slot and the output NaN-filled before
    each evaluation (PSWE_DEBUG_POISON), every kernel variant -- split,
    row and paired pass B, one and four lanes, one and many chunks and pass-C
    groups -- must produce the same bits as without, so no entry is read
    before it is written and no read races its producer."""
    res = _variant_runs(tmp_path, ({}, {"PSWE_DEBUG_POISON": "1"}))
    var = res[1][1]
    for name in ("passB_split", "passB_row", "passB_pair", "reduce", "fused"):
        assert var[name] > 0, (name, var)
    for a, b in zip(res[0][0], res[1][0]):
        assert np.all(np.isfinite(b))
        assert np.array_equal(a, b)


def test_guard_bands_stay_intact(tmp_path):
    """Stand-in for compute-sanitizer's memcheck (closed on the GPU pool,
    profiles/sanitizer_closed_r02.log): with PSWE_DEBUG_GUARD every context
    buffer (tables, intermediates, slots, stepper and diagnostics scratch)
    sits between 64 KiB NaN guard bands.  Over every kernel family -- the
    three passes in all their variants, fused and cluster small-grid kernels,
    generic mixed-radix sizes, the stepper and graph replay, diagnostics, the
    window batch -- no guard may change (no write past a buffer's ends) and
    the results must keep their bits (no read past them: it would bring in
    NaNs)."""
    res = _variant_runs(tmp_path, ({}, {"PSWE_DEBUG_GUARD": "1"}))
    assert res[0][2] == (0, 0)
    guarded, damaged = res[1][2]
    assert guarded >= 20, guarded
    assert damaged == 0
    for a, b in zip(res[0][0], res[1][0]):
        assert np.all(np.isfinite(b))
        assert np.array_equal(a, b)


def test_fused_small_grid_kernel_matches_three_pass_path(tmp_path):
    """n <= 64: the one-CTA-per-phase-group kernel (fused_kernels.cuh, n <= 32)
    and the 4-CTA cluster kernel (cluster_kernels.cuh, 64^2, few phases) vs
    the three-pass pipeline (PSWE_NO_FUSED) -- same transforms and formulas,
    so equal to round-off -- and vs the oracle, at every small size, one and
    many phases per CTA, a window batch and the stepper (C1, C2)."""
    import json
    import os
    import subprocess
    import sys

    from conftest import ROOT

    code = (
        "import sys, json, numpy as np; sys.path.insert(0, %r)\n"
        "import paper_2103_07706_b200 as pk\n"
        "from paper_2103_07706_b200 import cases\n"
        "outs = []\n"
        "for r, M in ((1, 4), (2, 8), (3, 8), (3, 64), (3, 256), (4, 8), (4, 16)):\n"
        "    c = cases.case_c5(r, M)\n"
        "    a = pk.averaged_tendency(c.state, c.quadrature, c.params, pk.PropagatorSpec.exact())\n"
        "    outs.append(np.stack([a.u, a.v, a.eta]))\n"
        "for c in (cases.case_c1(), cases.case_c2()):\n"
        "    cfg = pk.StepConfig(dt=c.dt, quadrature=c.quadrature, propagator_spec=pk.PropagatorSpec.exact())\n"
        "    s = pk.run(c.state, cfg, c.params, t_end=3 * c.dt).states[-1]\n"
        "    outs.append(np.stack([s.u, s.v, s.eta]))\n"
        "res = pk.window_sweep(c.state, c.params, c.dt, 2 * c.dt, [0.0, 1800.0, 3600.0], M=8)\n"
        "outs += [np.stack([r.final.u, r.final.v, r.final.eta]) for r in res]\n"
        "np.savez(sys.argv[1], *outs)\n"
        "print(json.dumps(pk.dynamics.context(c.state, c.params).variant_launches))\n" % str(ROOT))
    base = {k: v for k, v in os.environ.items() if not k.startswith("PSWE_")}
    res, var = [], []
    for i, env in enumerate(({}, {"PSWE_NO_FUSED": "1"})):
        f = tmp_path / f"f{i}.npz"
        p = subprocess.run([sys.executable, "-c", code, str(f)], env={**base, **env},
                           capture_output=True, text=True, timeout=600)
        assert p.returncode == 0, p.stderr
        var.append(json.loads(p.stdout.strip().splitlines()[-1]))
        with np.load(f) as z:
            res.append([z[k] for k in z.files])
    assert var[0]["fused"] > 0 and var[1]["fused"] == 0
    for a, b in zip(res[0], res[1]):
        assert rel_l2(a, b) <= 1e-13
    # and the fused results against the oracle at 32^2 / M = 128 (unbalanced state)
    c = cases.case_c5(3, 128)
    g = c.grid
    rng = np.random.default_rng(11)
    S = O.Setup(g.nx, g.ny, g.Lx, g.Ly, c.params.f, c.params.g, c.params.H)
    U = arr(c.state) + np.stack([O.truncate(O.spectral(sc * rng.standard_normal((32, 32))), S.mask)
                                 for sc in (1.0, 1.0, 50.0)])
    got = pk.averaged_tendency(state_from(U, g), c.quadrature, c.params, pk.PropagatorSpec.exact())
    assert O.rel_l2(arr(got), O.averaged_tendency(S, U, c.quadrature.s, c.quadrature.w, workers=8)) <= RHS_TOL


def test_generic_sizes_chebyshev_window_batch_and_gate():
    """The generic kernels (48^2 = 3 * 2^4) under the other routes: the
    Chebyshev exponential vs the oracle, a two-window batch vs one-by-one
    runs, and a non-Hermitian input failing with the reference's message."""
    n = 48
    rng = np.random.default_rng(48)
    g = pk.make_grid(n, n, 4.0e7, 4.0e7)
    S = O.Setup(n, n, g.Lx, g.Ly, F0, G0, H0)
    U = np.stack([O.truncate(O.spectral(sc * rng.standard_normal((n, n))), S.mask) for sc in (1.0, 1.0, 50.0)])
    p = flat(g)
    st = state_from(U, g)
    lam = pk.max_frequency(g, p)
    spec = pk.PropagatorSpec.chebyshev(lam * 3600.0)
    q = pk.kernel_weights(1800.0, 4)
    got = pk.averaged_tendency(st, q, p, spec)
    want = O.averaged_tendency(S, U, q.s, q.w, O.Propagator("chebyshev", spec.Lambda, spec.n_poly))
    assert O.rel_l2(arr(got), want) <= RHS_TOL
    res = pk.window_sweep(st, p, 900.0, 1800.0, [0.0, 1800.0], M=4)
    for r in res:
        solo = pk.run(st, pk.make_step_config(g, p, dt=900.0, T=r.T, M=4 if r.T > 0 else 0), p, 1800.0)
        assert rel_l2(arr(r.final), arr(solo.states[-1])) <= 1e-13
    bad = U.copy()
    bad[0, 3, 5] += 1e-6 * np.max(np.abs(U[0]))
    with pytest.raises(RuntimeError, match=r"averaging node k = -3 .*non-Hermitian spectral field: mode"):
        pk.averaged_tendency(state_from(bad, g), q, p, pk.PropagatorSpec.exact())

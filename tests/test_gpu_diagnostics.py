"""GPU snapshot diagnostics against the oracle.

energy and mass (diagnostics.py:58-78) and the maximum speed of
Trajectory.record (integrator.py:124-135) computed on the device by a full
2-D C2R must match the numpy restatement to 1e-12 relative, for band-limited
and non-band-limited states, with and without topography, square and
rectangular grids; run() records them at every snapshot.
"""

import numpy as np
import pytest

import paper_2103_07706_b200 as pk
from conftest import load_golden
from oracle import layout
from oracle import pswe_oracle as O
from paper_2103_07706_b200 import integrator

pytestmark = pytest.mark.gpu

TOL = 1e-12


def oracle_diag(state, params):
    S = O.Setup(state.grid.nx, state.grid.ny, state.grid.Lx, state.grid.Ly, params.f, params.g, params.H,
                np.asarray(params.b))
    U = np.stack([state.u, state.v, state.eta])
    en, ms = O.energy_mass(S, U)
    speed = np.hypot(O.real_field(state.u), O.real_field(state.v)).max()
    return en, ms, float(speed)


def random_state(nx, ny, seed, asym=0.0):
    """Full-spectrum (not band-limited) real fields; `asym` adds a
    non-Hermitian perturbation of that relative size."""
    rng = np.random.default_rng(seed)
    g = pk.make_grid(nx, ny, 4.0e7, 4.0e7 * ny / nx)
    fields = []
    for scale in (20.0, 15.0, 50.0):
        c = np.fft.fft2(scale * rng.standard_normal((nx, ny)))
        c = c + asym * scale * (rng.standard_normal((nx, ny)) + 1j * rng.standard_normal((nx, ny)))
        fields.append(c)
    return pk.State(grid=g, u=fields[0], v=fields[1], eta=fields[2], t=0.0)


def check(state, params):
    got = integrator.device_diagnostics(state, params)
    want = oracle_diag(state, params)
    for g, w in zip(got, want):
        assert abs(g - w) <= TOL * abs(w), (got, want)


def test_diagnostics_gate_non_hermitian_input():
    """The snapshot path's to_physical gate (diagnostics.py:21-25): a
    non-Hermitian u fails with the host gate's (= the reference's) message;
    a round-off-sized asymmetry (1e-15) passes."""
    st = random_state(64, 32, seed=3, asym=1e-3)
    params = pk.PhysicsParams(f=1.0e-4, g=9.81, H=5000.0, b=np.zeros((64, 32), complex))
    vel = max(float(np.max(np.abs(st.u))), float(np.max(np.abs(st.v))))
    with pytest.raises(ValueError) as want:
        pk.to_physical(st.grid, st.u, vel)
    with pytest.raises(ValueError) as got:
        integrator.device_diagnostics(st, params)
    assert str(got.value) == str(want.value)
    check(random_state(64, 32, seed=3, asym=1e-15), params)


@pytest.mark.parametrize("nx,ny", [(64, 64), (512, 512), (64, 32), (8, 16)])
def test_diagnostics_random_full_spectrum(nx, ny):
    st = random_state(nx, ny, seed=nx + ny)
    rng = np.random.default_rng(7)
    bphys = 100.0 * rng.random((nx, ny))
    params = pk.PhysicsParams(f=1.0e-4, g=9.81, H=5000.0, b=np.fft.fft2(bphys))
    check(st, params)


@pytest.mark.parametrize("name", ["C1", "C3"])
def test_diagnostics_golden_states(name):
    z = load_golden(name)
    nx, ny = int(z["nx"]), int(z["ny"])
    grid = pk.make_grid(nx, ny, float(z["Lx"]), float(z["Ly"]))
    b = layout.unpack(np.stack([z["b"]] * 3), nx, ny)[0]
    params = pk.PhysicsParams(f=float(z["f"]), g=float(z["g"]), H=float(z["H"]), b=b)
    U = layout.unpack(z["U"], nx, ny)
    check(pk.State(grid=grid, u=U[0], v=U[1], eta=U[2], t=0.0), params)


def test_run_records_device_diagnostics_at_snapshots():
    z = load_golden("C2")
    nx, ny = int(z["nx"]), int(z["ny"])
    grid = pk.make_grid(nx, ny, float(z["Lx"]), float(z["Ly"]))
    b = layout.unpack(np.stack([z["b"]] * 3), nx, ny)[0]
    params = pk.PhysicsParams(f=float(z["f"]), g=float(z["g"]), H=float(z["H"]), b=b)
    U = layout.unpack(z["U"], nx, ny)
    st = pk.State(grid=grid, u=U[0], v=U[1], eta=U[2], t=0.0)
    cfg = pk.make_step_config(grid, params, dt=float(z["dt"]), T=float(z["T_half"]), M=int(z["M"]))
    traj = pk.run(st, cfg, params, t_end=4 * cfg.dt, snapshot_every=2 * cfg.dt)
    assert traj.steps == [0, 2, 4]
    for s, en, ms, sp in zip(traj.states, traj.energy, traj.mass, traj.max_speed):
        w = oracle_diag(s, params)
        assert abs(en - w[0]) <= TOL * abs(w[0])
        assert abs(ms - w[1]) <= TOL * abs(w[1])
        assert abs(sp - w[2]) <= TOL * abs(w[2])

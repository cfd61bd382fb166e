"""The reference's acceptance gate (tests/test_acceptance.py), through the drop-in on the GPU.

Each test restates one guarantee of the reference's acceptance suite and
checks it end to end with ``paper_2103_07706_b200``:

* the balanced jet stays steady over 100 averaged steps (:164-182);
* the mean elevation is constant per averaged step (:239-253);
* the averaging-window experiment (the paper's Fig. 3; :192-205 and the
  ``sweep_trees`` fixture :52-69): a 15-day run of the jet over the mountain
  for T in {0, 0.5, 1, 2, 4, 8} h against an unaveraged dt = 180 s reference
  has an interior optimum in both error curves -- here the six windows run as
  one window batch and the 7200-step reference as one device-resident run;
  repeating the sweep gives the same bits (the reference's determinism
  guarantee across worker counts, :208-236);
* the small-grid oracle equivalences (:256-298): N against the direct
  truncated-convolution sum, L against the dense per-mode matrix.

The case is the reference's default (testcase.py:44-50, 53-95: two opposing
20 m/s Gaussian jets in discrete geostrophic balance, a 2000 m cone of
radius Ly/9 centred on the eastward jet, f = 1e-4, g = 9.8, H = 5960 m on a
4e7 m square), built with the same numpy operations.
"""

import math
import time

import numpy as np
import pytest

import paper_2103_07706_b200 as pk
from paper_2103_07706_b200 import cases
from paper_2103_07706_b200.sweep import l2_error_normalized

pytestmark = pytest.mark.gpu

F0, G0, H0, U0, B0 = 1.0e-4, 9.8, 5960.0, 20.0, 2000.0
TLIST = [0.0, 1800.0, 3600.0, 7200.0, 14400.0, 28800.0]


def default_problem(n=64, mountain=True):
    g = pk.make_grid(n, n, 4.0e7, 4.0e7)
    w = g.Ly / 16.0
    prof = U0 * (np.exp(-(((g.y - 0.25 * g.Ly) / w) ** 2)) - np.exp(-(((g.y - 0.75 * g.Ly) / w) ** 2)))
    cu = cases._zonal(g, prof)
    ceta = cases._balanced_eta(g, cu, F0, G0)
    b = cases._cone(g, B0, g.Ly / 9.0, 0.5 * g.Lx, 0.25 * g.Ly) if mountain else np.zeros((n, n), complex)
    return g, pk.PhysicsParams(f=F0, g=G0, H=H0, b=b), pk.State(grid=g, u=cu, v=np.zeros_like(cu), eta=ceta)


def test_balanced_jet_is_preserved():
    g, flat, jet = default_problem(mountain=False)
    started = time.perf_counter()
    eta0 = np.fft.ifft2(jet.eta).real
    drifts = []
    for T in (0.0, 3600.0):
        cfg = pk.make_step_config(g, flat, dt=3600.0, T=T)
        final = pk.run(jet, cfg, flat, t_end=100 * 3600.0).states[-1]
        diff = np.fft.ifft2(final.eta).real - eta0
        drifts.append(float(np.sqrt(np.sum(diff ** 2) / np.sum(eta0 ** 2))))
    elapsed = time.perf_counter() - started
    print(f"eta drift {drifts[0]:.3e} (T = 0), {drifts[1]:.3e} (T = 1 h), {elapsed:.2f} s")
    assert max(drifts) <= 1e-10 and elapsed < 60.0


def test_mean_elevation_is_conserved_per_step():
    g, rough, jet = default_problem()
    scale = float(np.sqrt(np.mean(np.fft.ifft2(jet.eta).real ** 2)))
    cfg = pk.make_step_config(g, rough, dt=3600.0, T=3600.0)
    npts = g.nx * g.ny
    state, means = jet, [float(np.real(jet.eta[0, 0])) / npts]
    for _ in range(24):
        state = pk.step_averaged_ssprk3(state, cfg, rough)
        means.append(float(np.real(state.eta[0, 0])) / npts)
    per_step = max(abs(means[i + 1] - means[i]) for i in range(24)) / scale
    print(f"max per-step change {per_step:.3e} of eta rms over 1 day")
    assert per_step <= 1e-13


def test_averaging_window_has_interior_optimum_and_is_deterministic():
    g, rough, jet = default_problem()
    t_end = 15 * 86400.0
    started = time.perf_counter()
    ref = pk.run(jet, pk.make_step_config(g, rough, dt=180.0, T=0.0), rough, t_end).states[-1]
    res = pk.window_sweep(jet, rough, 3600.0, t_end, TLIST, reference=ref)
    elapsed = time.perf_counter() - started
    ctx = pk.dynamics.context(jet, rough)
    for name, errs in (("eta", [r.l2_eta for r in res]), ("velocity", [r.l2_u for r in res])):
        imin = int(np.argmin(errs))
        print(f"{name}: errors {['%.4f' % e for e in errs]}, min at T = {TLIST[imin] / 3600:g} h")
        assert 0 < imin < len(errs) - 1
        assert errs[imin] < errs[0] and errs[imin] < errs[-1]
    print(f"reference (7200 steps) + 6-window sweep (360 steps each): {elapsed:.2f} s")
    # the same sweep again: the same bits (the reference guarantees this across worker counts)
    again = pk.window_sweep(jet, rough, 3600.0, t_end, TLIST, reference=ref)
    for a, b in zip(res, again):
        for f in ("u", "v", "eta"):
            assert np.array_equal(getattr(a.final, f), getattr(b.final, f))
        assert a.trajectory.energy == b.trajectory.energy
    assert ctx.launch_count > 0


def test_window_sweep_matches_the_reference_run():
    """The same 15-day experiment against the unmodified reference's own
    result (tests/golden/acceptance_sweep.npz, written by
    oracle/make_acceptance_golden.py from phaseswe: 360 averaged steps per
    window and the 7200-step reference): final states to the north_star
    run tolerance (rel L2 <= 1e-8) and the normalized errors."""
    from conftest import load_golden, rel_l2
    z = load_golden("acceptance_sweep")
    g, rough, jet = default_problem()
    t_end = 15 * 86400.0
    ref = pk.run(jet, pk.make_step_config(g, rough, dt=180.0, T=0.0), rough, t_end).states[-1]
    assert rel_l2(np.stack([ref.u, ref.v, ref.eta]), z["reference"]) <= 1e-8
    res = pk.window_sweep(jet, rough, 3600.0, t_end, list(z["T"]), reference=ref)
    for k, r in enumerate(res):
        assert r.M == int(z["M"][k])
        err = rel_l2(np.stack([r.final.u, r.final.v, r.final.eta]), z["finals"][k])
        print(f"T = {r.T:g} s: final state rel L2 vs the reference {err:.2e}; "
              f"l2_eta {r.l2_eta:.6g} (reference {z['l2_eta'][k]:.6g})")
        assert err <= 1e-8
        assert abs(r.l2_eta - z["l2_eta"][k]) <= 1e-6 * z["l2_eta"][k]
        assert abs(r.l2_u - z["l2_u"][k]) <= 1e-6 * z["l2_u"][k]


def truncated_convolution(grid, ca, cb):
    """Direct O(n^4) truncated-convolution sum (the reference's conftest.py oracle, restated)."""
    nx, ny = grid.nx, grid.ny
    wx = np.fft.fftfreq(nx, d=1.0 / nx).astype(int)
    wy = np.fft.fftfreq(ny, d=1.0 / ny).astype(int)
    keep_x = [i for i in range(nx) if 3 * abs(wx[i]) <= nx]
    keep_y = [j for j in range(ny) if 3 * abs(wy[j]) <= ny]
    ix = {int(wx[i]): i for i in range(nx)}
    iy = {int(wy[j]): j for j in range(ny)}
    out = np.zeros((nx, ny), dtype=np.complex128)
    for i in keep_x:
        for j in keep_y:
            for p in keep_x:
                for q in keep_y:
                    rx, ry = int(wx[i]) - int(wx[p]), int(wy[j]) - int(wy[q])
                    if rx in ix and ry in iy and 3 * abs(rx) <= nx and 3 * abs(ry) <= ny:
                        out[i, j] += ca[p, q] * cb[ix[rx], iy[ry]]
    return out / (nx * ny)


def test_small_grid_oracle_equivalences():
    g = pk.make_grid(8, 8, 1.0e6, 1.0e6)
    rng = np.random.default_rng(17)
    b = pk.dealias(g, pk.to_spectral(g, 30.0 * rng.standard_normal((8, 8))))
    params = pk.PhysicsParams(f=F0, g=G0, H=H0, b=b)

    def field(sc):
        return pk.dealias(g, pk.to_spectral(g, sc * rng.standard_normal((8, 8))))
    st = pk.State(grid=g, u=field(2.0), v=field(2.0), eta=field(20.0))
    out = pk.apply_nonlinear(st, params)
    kx2, ky2 = g.kx[:, None], g.ky[None, :]

    def conv(a, c):
        return truncated_convolution(g, a, c)
    cu, cv, depth = st.u, st.v, st.eta - b
    want = (-(conv(cu, 1j * kx2 * cu) + conv(cv, 1j * ky2 * cu)),
            -(conv(cu, 1j * kx2 * cv) + conv(cv, 1j * ky2 * cv)),
            -(1j * kx2 * conv(cu, depth) + 1j * ky2 * conv(cv, depth)))
    err_n = max(float(np.max(np.abs(a - w))) / float(np.max(np.abs(w)))
                for a, w in zip((out.u, out.v, out.eta), want))
    lin = pk.apply_linear(st, params)
    scale = max(float(np.max(np.abs(c))) for c in (lin.u, lin.v, lin.eta))
    worst = 0.0
    for i in range(8):
        for j in range(8):
            kx, ky = g.kx[i], g.ky[j]
            mat = np.array([[0.0, F0, -1j * G0 * kx], [-F0, 0.0, -1j * G0 * ky], [-1j * H0 * kx, -1j * H0 * ky, 0.0]])
            w = mat @ np.array([st.u[i, j], st.v[i, j], st.eta[i, j]])
            worst = max(worst, float(np.max(np.abs(np.array([lin.u[i, j], lin.v[i, j], lin.eta[i, j]]) - w))))
    print(f"nonlinear vs convolution {err_n:.2e}, linear vs 3x3 {worst / scale:.2e}")
    assert err_n <= 1e-12 and worst / scale <= 1e-13
    assert math.isfinite(err_n)

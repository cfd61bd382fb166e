"""Pin the CPU oracle (oracle/pswe_oracle.py) against the real reference.

Golden vectors in tests/golden/ were produced by the reference package itself
(oracle/make_golden.py); the known-answer values below are the reference's
own test constants.  CPU only.
"""

import math

import numpy as np
import pytest
import scipy.special

from conftest import load_golden, rel_l2
from oracle import layout
from oracle import pswe_oracle as O

F0, G0, H0 = 1.0e-4, 9.8, 5960.0


def setup_from(z, b=None):
    return O.Setup(int(z["nx"]), int(z["ny"]), float(z["Lx"]), float(z["Ly"]), float(z["f"]),
                   float(z["g"]), float(z["H"]), b)


# ------------------------------------------------------------ known answers
def test_known_answers():
    S = O.Setup(64, 64, 4.0e7, 4.0e7, F0, G0, H0)
    lam = S.max_frequency()
    assert lam == pytest.approx(1.720899454284647e-3, rel=1e-12)       # test_dynamics.py:91-96
    assert O.choose_npoly(10.0, 1e-10) == 28                            # test_propagator.py:107
    assert O.choose_npoly(0.0) == 1
    for T, want in ((0.0, 0), (1.0, 4), (3600.0, 4), (7200.0, 4), (14400.0, 8), (28800.0, 16)):
        assert O.default_node_count(T, 1.720899454284647e-3) == want    # test_averaging.py:75-82
    rho = O.bump(np.array([-1.5, -1.0, 0.0, 0.5, 1.0, 2.0]))
    assert rho[0] == 0.0 and rho[2] == np.exp(-1.0) and rho[4] == 0.0   # test_averaging.py:177-182
    assert rho[3] == pytest.approx(np.exp(-1.0 / 0.75), rel=1e-15)
    assert int(O.band_mask(8, 8).sum()) == 25                           # test_grid.py:39-51
    assert int(O.band_mask(12, 12).sum()) == 81
    assert list(O.wrap(8)) == [0, 1, 2, 3, -4, -3, -2, -1]              # test_dynamics.py:182-183


def test_cheb_coeffs_match_bessel_and_reference(unit_golden):
    k = np.arange(31)
    want = np.where(k == 0, 1.0, 2.0) * scipy.special.jv(k, 5.0)
    assert np.max(np.abs(O.cheb_coeffs(5.0, 30) - want)) <= 1e-12
    assert np.max(np.abs(O.cheb_coeffs(5.0, 30) - unit_golden["cheb_5_30"])) <= 1e-15
    assert np.max(np.abs(O.cheb_coeffs(6.2, 24) - unit_golden["cheb_6.2_24"])) <= 1e-15
    for lam, n in unit_golden["npoly"]:
        assert O.choose_npoly(float(lam), 1e-10) == int(n)


def test_quadrature_matches_reference(unit_golden):
    for key in unit_golden:
        if key.startswith("quad_") and key.endswith("_s") and "uniform" not in key:
            _, T, M, _ = key.split("_")
            s, w = O.quadrature(float(T), int(M))
            assert np.array_equal(s, unit_golden[key])
            assert np.array_equal(w, unit_golden[key[:-2] + "_w"])
    _, w = O.quadrature(100.0, 3, O.uniform)
    assert np.array_equal(w, unit_golden["quad_uniform_100_3_w"])
    # bump endpoints carry zero weight, so 2M - 1 live phases
    _, w = O.quadrature(1800.0, 8)
    assert int(np.count_nonzero(w)) == 15


# ------------------------------------------------------------ unit operators
def test_exact_exp_and_linear_8x8(unit_golden):
    S = O.Setup(8, 8, 1.0e6, 1.0e6, F0, G0, H0)
    U = unit_golden["exp8_U"]
    assert rel_l2(O.exact_exp(S, 500.0, U), unit_golden["exp8_p500"]) <= 1e-15
    assert rel_l2(O.exact_exp(S, -250.0, U), unit_golden["exp8_m250"]) <= 1e-15
    assert rel_l2(O.linear(S, U), unit_golden["lin8"]) <= 1e-15


def test_nonlinear_8x8_with_topography(unit_golden):
    S = O.Setup(8, 8, 1.0e6, 1.0e6, F0, G0, H0, unit_golden["nl8_b"])
    assert rel_l2(O.nonlinear(S, unit_golden["nl8_U"]), unit_golden["nl8_N"]) <= 1e-14


def test_averaged_tendency_32_exact_and_chebyshev(unit_golden):
    S = O.Setup(32, 32, 4.0e7, 4.0e7, F0, G0, H0)
    U = layout.unpack(unit_golden["avg32_U"], 32, 32)
    s, w = O.quadrature(1800.0, 3)
    got = layout.pack(O.averaged_tendency(S, U, s, w))
    assert rel_l2(got, unit_golden["avg32_exact"]) <= 1e-14
    prop = O.Propagator("chebyshev", float(unit_golden["avg32_cheb_Lambda"]), int(unit_golden["avg32_cheb_npoly"]))
    got = layout.pack(O.averaged_tendency(S, U, s, w, prop))
    assert rel_l2(got, unit_golden["avg32_cheb"]) <= 1e-14


def test_layout_roundtrip():
    rng = np.random.default_rng(3)
    for nx, ny in ((8, 8), (32, 16), (64, 64)):
        S = O.Setup(nx, ny, 1.0, 2.0, F0, G0, H0)
        U = np.stack([O.truncate(O.spectral(rng.standard_normal((nx, ny))), S.mask) for _ in range(3)])
        Uc = layout.pack(U)
        assert Uc.shape == (3, ny // 3 + 1, 2 * (nx // 3) + 1)
        assert np.max(np.abs(layout.unpack(Uc, nx, ny) - U)) <= 1e-12 * np.max(np.abs(U))
        assert np.array_equal(layout.pack(layout.unpack(Uc, nx, ny)), Uc)


# ------------------------------------------------------------ BASELINE configs
@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4"])
def test_config_rhs_matches_reference(name):
    z = load_golden(name)
    nx, ny = int(z["nx"]), int(z["ny"])
    S = setup_from(z, layout.unpack(np.stack([z["b"]] * 3), nx, ny)[0])
    U = layout.unpack(z["U"], nx, ny)
    s, w = O.quadrature(float(z["T_half"]), int(z["M"]))
    got = layout.pack(O.averaged_tendency(S, U, s, w, workers=8))
    assert rel_l2(got, z["rhs"]) <= 1e-13


@pytest.mark.parametrize("name", ["C2", "C3", "C4"])
def test_config_first_step_matches_reference(name):
    z = load_golden(name)
    nx, ny = int(z["nx"]), int(z["ny"])
    S = setup_from(z, layout.unpack(np.stack([z["b"]] * 3), nx, ny)[0])
    U = layout.unpack(z["U"], nx, ny)
    s, w = O.quadrature(float(z["T_half"]), int(z["M"]))
    got = layout.pack(O.ssprk3_step(S, U, float(z["dt"]), s, w, workers=8))
    assert rel_l2(got, z["step1"]) <= 1e-13


def test_c2_full_run_matches_reference():
    z = load_golden("C2")
    nx, ny = int(z["nx"]), int(z["ny"])
    S = setup_from(z)
    U = layout.unpack(z["U"], nx, ny)
    s, w = O.quadrature(float(z["T_half"]), int(z["M"]))
    got = layout.pack(O.run(S, U, float(z["dt"]), int(z["nsteps"]), s, w, workers=8))
    assert rel_l2(got, z["final"]) <= 1e-12
    assert float(z["t_final"]) == math.fsum([float(z["dt"])] * int(z["nsteps"]))

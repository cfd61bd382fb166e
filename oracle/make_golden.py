"""Generate golden vectors from the REAL reference (``phaseswe``) for tests/golden/.

TEST INFRASTRUCTURE.  Runs only in the build container, where the reference is
mounted read-only at /root/reference; the fixtures it writes are committed so
the GPU box (which has no /root/reference) can check against them.

    PYTHONPATH=/root/reference/pkg/src python oracle/make_golden.py [--only NAME ...] [--workers 8]

Fixture format (npz, complex128 arrays in the COMPACT band layout
[field][ky 0..ny/3][kx compact], see include/pswe_b200.h): every input is first
projected onto its Hermitian part and expanded back to the full fft2 layout,
so the reference runs on exactly the state the tests later rebuild from the
fixture.
"""

from __future__ import annotations

import argparse
import pathlib
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")

import phaseswe as ref  # noqa: E402  (the reference itself)
from phaseswe import averaging as ref_avg  # noqa: E402
from phaseswe import integrator as ref_int  # noqa: E402

from oracle import layout  # noqa: E402
from paper_2103_07706_b200 import cases  # noqa: E402

OUT = ROOT / "tests" / "golden"


def ref_objects(case):
    """The case rebuilt as reference objects on an exactly Hermitian state."""
    g = case.grid
    grid = ref.make_grid(g.nx, g.ny, g.Lx, g.Ly)
    U = np.stack([case.state.u, case.state.v, case.state.eta])
    Uc = layout.pack(U)
    Uf = layout.unpack(Uc, g.nx, g.ny)
    b = layout.unpack(layout.pack(np.stack([case.params.b] * 3)), g.nx, g.ny)[0]
    params = ref.PhysicsParams(f=case.params.f, g=case.params.g, H=case.params.H, b=b)
    state = ref.State(grid=grid, u=Uf[0], v=Uf[1], eta=Uf[2], t=0.0)
    return grid, params, state, Uc, layout.pack(np.stack([b] * 3))[0]


def as_compact(st):
    return layout.pack(np.stack([st.u, st.v, st.eta]))


def config_golden(name, workers):
    case = cases.CASES[name]()
    grid, params, state, Uc, bc = ref_objects(case)
    quad = ref.kernel_weights(case.T_half, case.M)
    spec = ref.PropagatorSpec.exact()
    pool = ThreadPoolExecutor(workers) if workers > 1 else None
    t0 = time.time()
    rhs = ref_avg.averaged_tendency(state, quad, params, spec, executor=pool)
    out = dict(U=Uc, b=bc, rhs=as_compact(rhs), nx=grid.nx, ny=grid.ny, Lx=grid.Lx, Ly=grid.Ly,
               f=params.f, g=params.g, H=params.H, T_half=case.T_half, M=case.M, dt=case.dt,
               nsteps=case.nsteps)
    print(f"{name}: rhs {time.time() - t0:.1f}s", flush=True)
    if case.nsteps:
        cfg = ref_int.StepConfig(dt=case.dt, quadrature=quad, propagator_spec=spec)
        st = ref_int.step_averaged_ssprk3(state, cfg, params, pool)
        out["step1"] = as_compact(st)
        for i in range(1, case.nsteps):
            st = ref_int.step_averaged_ssprk3(st, cfg, params, pool)
            if (i + 1) % 8 == 0:
                print(f"{name}: step {i + 1}/{case.nsteps} {time.time() - t0:.1f}s", flush=True)
        out["final"] = as_compact(st)
        out["t_final"] = st.t
    if pool is not None:
        pool.shutdown()
    np.savez_compressed(OUT / f"{name}.npz", **out)
    print(f"{name}: done {time.time() - t0:.1f}s", flush=True)


def unit_golden():
    """Small known-answer cases mirroring the reference's own unit tests."""
    out = {}
    rng = np.random.default_rng(20260823)  # conftest.py:16-18 seed
    F0, G0, H0 = 1.0e-4, 9.8, 5960.0

    def blstate(grid, vel=1.0, eta=50.0):
        def fld(sc):
            return ref.dealias(grid, ref.to_spectral(grid, sc * rng.standard_normal((grid.nx, grid.ny))))
        return ref.State(grid=grid, u=fld(vel), v=fld(vel), eta=fld(eta), t=0.0)

    def herm(st, grid):
        U = layout.unpack(layout.pack(np.stack([st.u, st.v, st.eta])), grid.nx, grid.ny)
        return ref.State(grid=grid, u=U[0], v=U[1], eta=U[2], t=st.t)

    # exact_exp on 8x8 (test_propagator.py:36-45), arbitrary t
    g8 = ref.make_grid(8, 8, 1.0e6, 1.0e6)
    flat8 = ref.PhysicsParams(f=F0, g=G0, H=H0, b=np.zeros((8, 8), complex))
    s8 = herm(blstate(g8), g8)
    out["exp8_U"] = np.stack([s8.u, s8.v, s8.eta])
    out["exp8_p500"] = np.stack([getattr(ref.exact_exp(500.0, s8, flat8), n) for n in ("u", "v", "eta")])
    out["exp8_m250"] = np.stack([getattr(ref.exact_exp(-250.0, s8, flat8), n) for n in ("u", "v", "eta")])
    out["lin8"] = np.stack([getattr(ref.apply_linear(s8, flat8), n) for n in ("u", "v", "eta")])
    # apply_nonlinear with topography on 8x8 (test_dynamics.py:44-61)
    sN = herm(blstate(g8, 2.0, 20.0), g8)
    bN = ref.dealias(g8, ref.to_spectral(g8, 30.0 * rng.standard_normal((8, 8))))
    bN = layout.unpack(layout.pack(np.stack([bN] * 3)), 8, 8)[0]
    pN = ref.PhysicsParams(f=F0, g=G0, H=H0, b=bN)
    out["nl8_U"] = np.stack([sN.u, sN.v, sN.eta])
    out["nl8_b"] = bN
    out["nl8_N"] = np.stack([getattr(ref.apply_nonlinear(sN, pN), n) for n in ("u", "v", "eta")])
    # averaged tendency on 32x32 (test_averaging.py:85-110), exact and Chebyshev
    g32 = ref.make_grid(32, 32, 4.0e7, 4.0e7)
    flat32 = ref.PhysicsParams(f=F0, g=G0, H=H0, b=np.zeros((32, 32), complex))
    s32 = herm(blstate(g32), g32)
    q = ref.kernel_weights(1800.0, 3)
    out["avg32_U"] = layout.pack(np.stack([s32.u, s32.v, s32.eta]))
    out["avg32_exact"] = as_compact(ref.averaged_tendency(s32, q, flat32, ref.PropagatorSpec.exact()))
    lam = ref.max_frequency(g32, flat32) * 1800.0
    cspec = ref.PropagatorSpec.chebyshev(lam)
    out["avg32_cheb"] = as_compact(ref.averaged_tendency(s32, q, flat32, cspec))
    out["avg32_cheb_Lambda"] = cspec.Lambda
    out["avg32_cheb_npoly"] = cspec.n_poly
    # quadrature / coefficient KATs
    for T, M in ((3600.0, 5), (7200.0, 8), (1800.0, 8), (3600.0, 16), (1800.0, 32), (2700.0, 64), (1800.0, 256)):
        qq = ref.kernel_weights(T, M)
        out[f"quad_{int(T)}_{M}_s"] = qq.s
        out[f"quad_{int(T)}_{M}_w"] = qq.w
    out["quad_uniform_100_3_w"] = ref.kernel_weights(100.0, 3, ref.UNIFORM_KERNEL).w
    out["cheb_5_30"] = ref.cheb_coeffs(5.0, 30).a
    out["cheb_6.2_24"] = ref.cheb_coeffs(6.2, 24).a
    out["npoly"] = np.array([[lam_, ref.choose_npoly(lam_, 1e-10)] for lam_ in (0.0, 1.0, 6.2, 10.0, 20.0, 100.0)])
    np.savez_compressed(OUT / "unit.npz", **out)
    print("unit: done", flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", nargs="*", default=None)
    ap.add_argument("--workers", type=int, default=8)
    a = ap.parse_args()
    OUT.mkdir(parents=True, exist_ok=True)
    names = a.only or ["unit", "C1", "C2", "C3", "C4"]
    for n in names:
        if n == "unit":
            unit_golden()
        else:
            config_golden(n, a.workers)


if __name__ == "__main__":
    main()

"""Golden fixture of the reference's window-sweep acceptance experiment.

TEST INFRASTRUCTURE (like make_golden.py): imports the unmodified reference
(/root/reference/pkg/src or oracle/_ref) in this container and writes
tests/golden/acceptance_sweep.npz -- the final states and normalized errors
of the 15-day default-case runs for T in {0, 0.5, 1, 2, 4, 8} h (dt = 1 h,
M auto) and of the unaveraged dt = 180 s reference run, exactly as the
reference's tests/test_acceptance.py builds them (sweep_trees fixture,
:52-69, via harness._execute's run; errors by diagnostics.l2_error_normalized).
Takes a few minutes of CPU.

usage: python oracle/make_acceptance_golden.py [workers]
"""
import pathlib
import sys
import time

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
from oracle import reference as R  # noqa: E402

ref = R.load()
assert ref is not None, "the reference is not available"
from phaseswe.diagnostics import l2_error_normalized  # noqa: E402
from phaseswe.grid import make_grid  # noqa: E402
from phaseswe.integrator import make_step_config, run  # noqa: E402
from phaseswe.testcase import balanced_jet, default_case, physics_params  # noqa: E402

workers = int(sys.argv[1]) if len(sys.argv) > 1 else 8
TLIST = [0.0, 1800.0, 3600.0, 7200.0, 14400.0, 28800.0]
t_end = 15 * 86400.0
grid = make_grid(64, 64, 4.0e7, 4.0e7)
case = default_case(4.0e7, 4.0e7)
params = physics_params(case, grid, with_mountain=True)
jet = balanced_jet(case, grid)
t0 = time.perf_counter()
fine = run(jet, make_step_config(grid, params, dt=180.0, T=0.0), params, t_end, workers=1).states[-1]
print(f"reference run: {time.perf_counter() - t0:.1f} s", flush=True)
finals, eta, vel, Ms = [], [], [], []
for T in TLIST:
    t0 = time.perf_counter()
    cfg = make_step_config(grid, params, dt=3600.0, T=T)
    final = run(jet, cfg, params, t_end, workers=workers).states[-1]
    e, u = l2_error_normalized(final, fine)
    finals.append(np.stack([final.u, final.v, final.eta]))
    eta.append(e)
    vel.append(u)
    Ms.append(cfg.quadrature.M)
    print(f"T = {T:g} s (M = {cfg.quadrature.M}): l2_eta {e:.6g} l2_u {u:.6g}, {time.perf_counter() - t0:.1f} s",
          flush=True)
out = HERE.parent / "tests" / "golden" / "acceptance_sweep.npz"
np.savez_compressed(out, T=np.array(TLIST), M=np.array(Ms), l2_eta=np.array(eta), l2_u=np.array(vel),
                    finals=np.stack(finals), reference=np.stack([fine.u, fine.v, fine.eta]))
print("wrote", out)

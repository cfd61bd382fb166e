"""Outputs of a set of evaluations (averaged RHS over the kernel variants,
N at 512^2, a stepper step) saved to OUT.npz, for bit-for-bit comparisons
of two builds (PSWE_LIB_PATH).  usage: python tools/bits_check.py OUT.npz"""
import sys
sys.path.insert(0, ".")
import numpy as np
import paper_2103_07706_b200 as pk
from paper_2103_07706_b200 import cases

res = {}
for r, M in [(4, 8), (5, 4), (5, 32), (6, 8), (6, 32), (7, 8), (7, 256)]:
    c = cases.case_c5(r, M)
    a = pk.averaged_tendency(c.state, c.quadrature, c.params, pk.PropagatorSpec.exact())
    res[f"rhs_{r}_{M}"] = np.stack([a.u, a.v, a.eta])
d = cases.case_c5(7, 8)
n = pk.apply_nonlinear(d.state, d.params)
res["N512"] = np.stack([n.u, n.v, n.eta])
c = cases.case_c3()
cfg = pk.StepConfig(dt=1800.0, quadrature=c.quadrature, propagator_spec=pk.PropagatorSpec.exact())
s = pk.step_averaged_ssprk3(c.state, cfg, c.params)
res["C3step"] = np.stack([s.u, s.v, s.eta])
c = cases.case_c2()
cfg = pk.StepConfig(dt=c.dt, quadrature=c.quadrature, propagator_spec=pk.PropagatorSpec.exact())
s = pk.run(c.state, cfg, c.params, t_end=4 * c.dt).states[-1]
res["C2run"] = np.stack([s.u, s.v, s.eta])
c = cases.case_c3()
for w in pk.window_sweep(c.state, c.params, c.dt, 2 * c.dt, [0.0, 1800.0, 3600.0], M=4):
    res[f"win{w.T:g}"] = np.stack([w.final.u, w.final.v, w.final.eta])
np.savez(sys.argv[1], **res)
if len(sys.argv) > 2:
    ref = np.load(sys.argv[2])
    for k in res:
        same = np.array_equal(res[k], ref[k])
        err = float(np.linalg.norm(res[k] - ref[k]) / np.linalg.norm(ref[k]))
        print(k, "bitwise" if same else f"differs rel {err:.2e}")

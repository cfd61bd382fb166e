"""Debug: C4 RHS and first-step errors vs the reference goldens."""
import sys
import numpy as np
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2103_07706_b200 as pk
from conftest import load_golden, rel_l2
from oracle import layout
for name in sys.argv[1:] or ["C4"]:
    z = load_golden(name)
    nx, ny = int(z["nx"]), int(z["ny"])
    grid = pk.make_grid(nx, ny, float(z["Lx"]), float(z["Ly"]))
    b = layout.unpack(np.stack([z["b"]] * 3), nx, ny)[0]
    params = pk.PhysicsParams(f=float(z["f"]), g=float(z["g"]), H=float(z["H"]), b=b)
    U = layout.unpack(z["U"], nx, ny)
    st = pk.State(grid=grid, u=U[0], v=U[1], eta=U[2])
    quad = pk.kernel_weights(float(z["T_half"]), int(z["M"]))
    rhs = pk.averaged_tendency(st, quad, params, pk.PropagatorSpec.exact())
    e0 = rel_l2(layout.pack(np.stack([rhs.u, rhs.v, rhs.eta])), z["rhs"])
    cfg = pk.StepConfig(dt=float(z["dt"]), quadrature=quad, propagator_spec=pk.PropagatorSpec.exact())
    one = pk.step_averaged_ssprk3(st, cfg, params)
    e1 = rel_l2(layout.pack(np.stack([one.u, one.v, one.eta])), z["step1"])
    rhs2 = pk.averaged_tendency(st, quad, params, pk.PropagatorSpec.exact())
    e2 = rel_l2(layout.pack(np.stack([rhs2.u, rhs2.v, rhs2.eta])), z["rhs"])
    print(name, "rhs", e0, "step1", e1, "rhs again", e2, flush=True)

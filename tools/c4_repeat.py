import sys
import numpy as np
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import paper_2103_07706_b200 as pk
from conftest import load_golden, rel_l2
from oracle import layout
z = load_golden("C4")
nx, ny = int(z["nx"]), int(z["ny"])
grid = pk.make_grid(nx, ny, float(z["Lx"]), float(z["Ly"]))
b = layout.unpack(np.stack([z["b"]] * 3), nx, ny)[0]
params = pk.PhysicsParams(f=float(z["f"]), g=float(z["g"]), H=float(z["H"]), b=b)
U = layout.unpack(z["U"], nx, ny)
st = pk.State(grid=grid, u=U[0], v=U[1], eta=U[2])
quad = pk.kernel_weights(float(z["T_half"]), int(z["M"]))
errs = []
for _ in range(8):
    rhs = pk.averaged_tendency(st, quad, params, pk.PropagatorSpec.exact())
    errs.append(rel_l2(layout.pack(np.stack([rhs.u, rhs.v, rhs.eta])), z["rhs"]))
print(sys.argv[1] if len(sys.argv) > 1 else "cur", "max err over 8 calls %.2e" % max(errs), flush=True)

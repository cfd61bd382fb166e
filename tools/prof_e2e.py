import sys, time, cProfile, pstats
sys.path.insert(0, ".")
import torch
import paper_2103_07706_b200 as pk
from paper_2103_07706_b200 import cases
c = cases.case_c5(7, 256)
spec = pk.PropagatorSpec.exact()
for _ in range(3):
    pk.averaged_tendency(c.state, c.quadrature, c.params, spec)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(10):
    pk.averaged_tendency(c.state, c.quadrature, c.params, spec)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)

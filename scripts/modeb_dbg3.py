import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1901_02090_b200 as B
import paper_1901_02090_b200.solver as SV
orig = SV._pcg
def cap(setup, W, config, cb, r_floor=0.0):
    print("r0", float(W.r.norm()), "floor", r_floor)
    return orig(setup, W, config, cb, r_floor)
SV._pcg = cap
g = B.build_grid(2, (12, 20), (1.0, 1.0))
sy = B.assemble_system(g, B.Permeability(np.ones((240, 2))), B.PressureDrop(1, 1.0, 0.0))
dec = B.regular_partition(g, (1, 4))
cfg = B.SolveConfig(tau=float("inf"), scaling="multiplicity", constraints="initial", tol=1e-10)
r = B.solve(sy, dec, cfg)
print(r.it)

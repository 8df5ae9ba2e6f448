"""Host-side timing of the public solve() on config 3 (dev tool)."""
import cProfile, math, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1901_02090_b200 as B
from paper_1901_02090_b200 import fields
c = fields.CONFIGS[3]
k = fields.config_field(3)
g = B.build_grid(c["dim"], c["counts"], c["sizes"])
dec = B.regular_partition(g, c["splits"])
system = B.assemble_system(g, B.Permeability(k), B.Wells(0, g.n_cells - 1))
cfg = B.SolveConfig(tau=c["tau"], scaling=c["scaling"], constraints="adaptive", tol=c["tol"])
st = B.BddcSetup(system, dec, cfg)
for _ in range(3):
    rep = B.solve(system, dec, cfg, setup=st)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(5):
    rep = B.solve(system, dec, cfg, setup=st)
print("e2e ms/solve", (time.perf_counter() - t) / 5 * 1000, "it", rep.it)
pr = cProfile.Profile()
pr.enable()
for _ in range(3):
    rep = B.solve(system, dec, cfg, setup=st)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)

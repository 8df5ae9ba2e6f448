"""cProfile of BddcSetup (host overhead hunt; dev tool)."""
import cProfile, pstats, math, os, sys, io
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1901_02090_b200 as B
from paper_1901_02090_b200 import fields
c = fields.CONFIGS[3]; k = fields.config_field(3)
g = B.build_grid(c["dim"], c["counts"], c["sizes"]); dec = B.regular_partition(g, c["splits"])
system = B.assemble_system(g, B.Permeability(k), B.Wells(0, g.n_cells - 1))
cfg = B.SolveConfig(tau=c["tau"], scaling=c["scaling"], constraints="adaptive", tol=c["tol"])
st = B.BddcSetup(system, dec, cfg); torch.cuda.synchronize(); del st
pr = cProfile.Profile(); pr.enable()
st = B.BddcSetup(system, dec, cfg); torch.cuda.synchronize()
pr.disable()
s = io.StringIO(); pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(25); print(s.getvalue()[:5000])

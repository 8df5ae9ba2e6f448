"""Wall time of setup + FIRST solve (what a one-shot user pays) on config 3 (dev tool)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1901_02090_b200 as B
from paper_1901_02090_b200 import fields
c = fields.CONFIGS[3]
k = fields.config_field(3)
g = B.build_grid(c["dim"], c["counts"], c["sizes"])
t = time.perf_counter(); dec = B.regular_partition(g, c["splits"]); tp = time.perf_counter() - t
system = B.assemble_system(g, B.Permeability(k), B.Wells(0, g.n_cells - 1))
cfg = B.SolveConfig(tau=c["tau"], scaling=c["scaling"], constraints="adaptive", tol=c["tol"])
torch.zeros(1, device="cuda"); torch.cuda.synchronize()
for rep in range(2):
    t0 = time.perf_counter()
    st = B.BddcSetup(system, dec, cfg)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    w = st.work(); torch.cuda.synchronize(); t2 = time.perf_counter()
    r = B.solve(system, dec, cfg, setup=st); t3 = time.perf_counter()
    r = B.solve(system, dec, cfg, setup=st); t4 = time.perf_counter()
    print(f"rep {rep}: partition {tp:.3f}s setup {t1-t0:.3f}s work-alloc {t2-t1:.3f}s first solve {t3-t2:.3f}s "
          f"second solve {t4-t3:.3f}s it={r.it}")
    del st, w, r

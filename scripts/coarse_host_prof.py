"""Host time of the coarse ND symbolic analysis vs the device factorisation inside one setup."""
import math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1901_02090_b200 as B
from paper_1901_02090_b200 import fields, coarse_nd, solver as SV
cid = int(sys.argv[1]) if len(sys.argv) > 1 else 3
c = fields.CONFIGS[cid]
k = fields.config_field(cid)
g = B.build_grid(c["dim"], c["counts"], c["sizes"])
dec = B.regular_partition(g, c["splits"])
system = B.assemble_system(g, B.Permeability(k), B.Wells(0, g.n_cells - 1))
cfg = B.SolveConfig(tau=c["tau"], scaling=c["scaling"], constraints="adaptive", tol=c["tol"])
T = {}
orig_init, orig_factor = coarse_nd.CoarseND.__init__, coarse_nd.CoarseND.factor
def init(self, *a, **kw):
    t = time.perf_counter(); orig_init(self, *a, **kw); T["init"] = time.perf_counter() - t
def factor(self, *a, **kw):
    torch.cuda.synchronize(); t = time.perf_counter(); orig_factor(self, *a, **kw); torch.cuda.synchronize()
    T["factor"] = time.perf_counter() - t
coarse_nd.CoarseND.__init__, coarse_nd.CoarseND.factor = init, factor
for r in range(3):
    tm = {}
    torch.cuda.synchronize(); t = time.perf_counter()
    st = B.BddcSetup(system, dec, cfg, timings=tm)
    torch.cuda.synchronize()
    print(f"setup {time.perf_counter() - t:.3f}s  ND init(host) {T['init']*1e3:.1f} ms  factor(dev, synced) {T['factor']*1e3:.1f} ms",
          {k2: round(v, 1) for k2, v in tm.items()})
    del st

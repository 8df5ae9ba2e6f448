"""Which device allocations inside BddcSetup block the host (allocator syncs)."""
import math, os, sys, time, traceback
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1901_02090_b200 as B
from paper_1901_02090_b200 import fields
c = fields.CONFIGS[3]; k = fields.config_field(3)
g = B.build_grid(c["dim"], c["counts"], c["sizes"]); dec = B.regular_partition(g, c["splits"])
system = B.assemble_system(g, B.Permeability(k), B.Wells(0, g.n_cells - 1))
cfg = B.SolveConfig(tau=c["tau"], scaling=c["scaling"], constraints="adaptive", tol=c["tol"])
st = B.BddcSetup(system, dec, cfg); torch.cuda.synchronize(); del st
orig = torch.empty
log = []
def empty(*a, **kw):
    t = time.perf_counter(); r = orig(*a, **kw); dt = time.perf_counter() - t
    if dt > 1e-3:
        fr = traceback.extract_stack(limit=3)[0]
        log.append((dt * 1e3, r.numel() * r.element_size() / 1e6, f"{os.path.basename(fr.filename)}:{fr.lineno}"))
    return r
torch.empty = empty
torch.cuda.synchronize(); t = time.perf_counter()
st = B.BddcSetup(system, dec, cfg); torch.cuda.synchronize()
print("setup wall", round((time.perf_counter() - t) * 1e3, 1), "ms; reserved GB", torch.cuda.memory_reserved() / 1e9)
for dt, mb, where in log:
    print(f"  {dt:7.1f} ms  {mb:9.1f} MB  {where}")

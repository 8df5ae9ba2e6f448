"""Setup time with a fresh Decomposition (no cached topology / ND geometry) vs a reused one."""
import math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1901_02090_b200 as B
from paper_1901_02090_b200 import fields
cid = int(sys.argv[1]) if len(sys.argv) > 1 else 3
c = fields.CONFIGS[cid]
k = fields.config_field(cid)
g = B.build_grid(c["dim"], c["counts"], c["sizes"])
system = B.assemble_system(g, B.Permeability(k), B.Wells(0, g.n_cells - 1))
cfg = B.SolveConfig(tau=c["tau"], scaling=c["scaling"], constraints="adaptive" if math.isfinite(c["tau"]) else "initial", tol=c["tol"])
dec = B.regular_partition(g, c["splits"])
st = B.BddcSetup(system, dec, cfg); del st
for label in ("reused dec", "fresh dec", "reused dec", "fresh dec"):
    if label == "fresh dec":
        t = time.time(); dec = B.regular_partition(g, c["splits"]); tdec = time.time() - t
    else:
        tdec = 0.0
    torch.cuda.synchronize(); t = time.time()
    tm = {}
    st = B.BddcSetup(system, dec, cfg, timings=tm)
    torch.cuda.synchronize(); ts = time.time() - t
    print(f"{label}: partition {tdec:.3f}s setup {ts:.3f}s", {k2: round(v, 1) for k2, v in tm.items()}, flush=True)
    del st

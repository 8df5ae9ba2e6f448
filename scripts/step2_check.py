"""Step 2 as one two-rhs local-solve pass vs two passes: equality and solve time (C3)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1901_02090_b200 as B
from paper_1901_02090_b200 import fields, solver as S
cid = int(sys.argv[1]) if len(sys.argv) > 1 else 3
c = fields.CONFIGS[cid]
g = B.build_grid(c["dim"], c["counts"], c["sizes"])
dec = B.regular_partition(g, c["splits"])
system = B.assemble_system(g, B.Permeability(fields.config_field(cid)), B.Wells(0, g.n_cells - 1))
cfg = B.SolveConfig(tau=c["tau"], scaling=c["scaling"], constraints=c["constraints"], tol=c["tol"])
st = B.BddcSetup(system, dec, cfg)
f_dev = torch.as_tensor(system.f, dtype=torch.float64, device="cuda")
out = {}
for fused in (False, True):
    st.step2_fused = fused
    r = B.solve(system, dec, cfg, setup=st)
    out[fused] = r
    for _ in range(3):
        S.solve(system, dec, cfg, setup=st, f_device=f_dev, return_device=True)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        S.solve(system, dec, cfg, setup=st, f_device=f_dev, return_device=True)
    b.record(); b.synchronize()
    print(f"fused={fused}: {a.elapsed_time(b) / 10:.3f} ms per solve, it={r.it}", flush=True)
rel = lambda x, y: np.linalg.norm(x - y) / np.linalg.norm(y)
print("u0", rel(out[True].u0, out[False].u0), "u*", rel(out[True].u_star, out[False].u_star),
      "u", rel(out[True].u, out[False].u), "p", rel(out[True].p, out[False].p))

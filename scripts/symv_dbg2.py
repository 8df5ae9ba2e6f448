import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1901_02090_b200 as B
from paper_1901_02090_b200 import fields
cid = int(sys.argv[1])
c = fields.CONFIGS[cid]
g = B.build_grid(c["dim"], c["counts"], c["sizes"])
dec = B.regular_partition(g, c["splits"])
system = B.assemble_system(g, B.Permeability(fields.config_field(cid)), B.Wells(0, g.n_cells - 1))
cfg = B.SolveConfig(tau=c["tau"], scaling=c["scaling"], constraints=c["constraints"], tol=c["tol"])
st = B.BddcSetup(system, dec, cfg)
torch.cuda.synchronize()
print("setup ok", flush=True)
x = np.random.default_rng(0).standard_normal(dec.n_gamma)
for k in range(3):
    print("a", np.linalg.norm(st.schur_matvec(x)), st._sched.cpu().numpy(), flush=True)

"""The bench's stencil roofline (A u, B u, B^T p over operand sets larger than L2)
on config argv[1] (default 3), without the rest of the bench."""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_1901_02090_b200 as B
from paper_1901_02090_b200 import fields, _native as nat

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 3
c = fields.CONFIGS[cid]
g = B.build_grid(c["dim"], c["counts"], c["sizes"])
dec = B.regular_partition(g, c["splits"])
system = B.assemble_system(g, B.Permeability(fields.config_field(cid)), B.Wells(0, g.n_cells - 1))
cfg = B.SolveConfig(tau=c["tau"], scaling=c["scaling"], constraints=c["constraints"], tol=c["tol"])
st = B.BddcSetup(system, dec, cfg)
peak = bench._peaks()[0]
print(json.dumps(bench._stencil_roofline(st, g, nat, peak, torch.device("cuda")), indent=1))

"""One interface-Schur GEMV (gather_symv_kernel) between cudaProfilerStart/Stop on
config 3, for `ncu --set full --profile-from-start off` (roofline traffic)."""
import os, sys
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
st.time_kernel("S", 2)
torch.cuda.synchronize()
torch.cuda.profiler.start()
st.time_kernel("S", 1)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok")

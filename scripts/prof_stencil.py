"""RT0 stencil kernels (A u, B u, B^T p) on config argv[1] (default 3) between
cudaProfilerStart/Stop for ncu; operands fresh (not L2-resident)."""
import ctypes as C, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1901_02090_b200 as B
from paper_1901_02090_b200 import fields, _native as nat

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 3
c = fields.CONFIGS[cid]
g = B.build_grid(c["dim"], c["counts"], c["sizes"])
dec = B.regular_partition(g, c["splits"])
system = B.assemble_system(g, B.Permeability(fields.config_field(cid)), B.Wells(0, g.n_cells - 1))
cfg = B.SolveConfig(tau=c["tau"], scaling=c["scaling"], constraints=c["constraints"], tol=c["tol"])
st = B.BddcSetup(system, dec, cfg)
gp = C.byref(st.geom)
s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
nf, nc = st.geom.n_flux, g.n_cells
u = torch.randn(nf, dtype=torch.float64, device="cuda")
y = torch.empty(nf, dtype=torch.float64, device="cuda")
pc = torch.randn(nc, dtype=torch.float64, device="cuda")
oc = torch.empty(nc, dtype=torch.float64, device="cuda")
flush = torch.ones(64 << 20, dtype=torch.float64, device="cuda")
ops = [lambda: nat.call("bddc_flux_A", gp, nat.ptr(st.d_coef), nat.ptr(u), 1.0, 0.0, nat.ptr(y), s),
       lambda: nat.call("bddc_cell_div", gp, nat.ptr(u), None, 0.0, 1.0, None, None, nat.ptr(oc), s),
       lambda: nat.call("bddc_grad", gp, nat.ptr(pc), 1.0, 0.0, nat.ptr(y), s)]
for f in ops:
    f()
torch.cuda.synchronize()
torch.cuda.profiler.start()
for f in ops:
    flush.sum()
    f()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok")

"""C3 (or argv[1]) PCG pieces between cudaProfilerStart/Stop for ncu: the bulk T GEMV
at the concurrent grid and at one CTA per SM, the LDG GEMV on the full grid, the
restriction and one ND solve (each piece once, after a warm run)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1901_02090_b200 as B
from paper_1901_02090_b200 import fields, _native as nat
from paper_1901_02090_b200.solver import _p, _stream

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 3
c = fields.CONFIGS[cid]
g = B.build_grid(3, c["counts"], c["sizes"])
dec = B.regular_partition(g, c["splits"])
system = B.assemble_system(g, B.Permeability(fields.config_field(cid)), B.Wells(0, g.n_cells - 1))
cfg = B.SolveConfig(tau=c["tau"], scaling=c["scaling"], constraints=c["constraints"], tol=c["tol"])
st = B.BddcSetup(system, dec, cfg)
B.solve(system, dec, cfg, setup=st)
r = torch.randn(st.n_gamma, dtype=torch.float64, device="cuda")


def restrict():
    nat.call("bddc_gather_gemv_t", st.N, st.maxG, st.maxC, _p(st.d_nG), _p(st.d_nC), _p(st.d_gpos),
             _p(st.d_Psi), _p(r), _p(st.d_delta), _p(st.w_v), _stream())


pieces = [
    lambda: st._symv(st.d_Tp, r, st.d_delta, st.w_yb, st.t_grid_bulk, 1, _stream()),
    lambda: st._symv(st.d_Tp, r, st.d_delta, st.w_yb, 0, 1, _stream()),
    lambda: nat.call("bddc_gather_symv", st.N, st.maxG, _p(st.d_nG), _p(st.d_gpos), _p(st.d_Tp), _p(r),
                     _p(st.d_delta), _p(st.w_yb), 0, _stream()),
    restrict,
    st._coarse_solve,
]
for f in pieces:
    f()
torch.cuda.synchronize()
torch.cuda.profiler.start()
for f in pieces:
    f()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok")

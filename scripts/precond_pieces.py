"""C3 preconditioner pieces with the bulk T GEMV: T alone per grid, the coarse
chain alone, and the whole preconditioner (T beside the chain) per grid."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1901_02090_b200 as B
from paper_1901_02090_b200 import fields, _native as nat
from paper_1901_02090_b200.solver import _p, _stream
c = fields.CONFIGS[3]
g = B.build_grid(3, c["counts"], c["sizes"])
dec = B.regular_partition(g, c["splits"])
system = B.assemble_system(g, B.Permeability(fields.config_field(3)), B.Wells(0, g.n_cells - 1))
cfg = B.SolveConfig(tau=c["tau"], scaling=c["scaling"], constraints=c["constraints"], tol=c["tol"])
st = B.BddcSetup(system, dec, cfg)
B.solve(system, dec, cfg, setup=st)
W = st.work()
r = torch.randn(st.n_gamma, dtype=torch.float64, device="cuda")


def timeit(fn, reps=30):
    fn(); torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record(); b.synchronize()
    return a.elapsed_time(b) / reps * 1000.0


def chain():
    ss = _stream()
    nat.call("bddc_gather_gemv_t", st.N, st.maxG, st.maxC, _p(st.d_nG), _p(st.d_nC), _p(st.d_gpos),
             _p(st.d_Psi), _p(r), _p(st.d_delta), _p(st.w_v), ss)
    nat.call("bddc_coarse_restrict", st.nfc, _p(st.d_cown), _p(st.w_v), _p(st.w_rc), ss)
    nat.call("bddc_fill", st.N, 0.0, _p(st.w_rc[st.nfc:]), ss)
    st._coarse_solve()


print(f"chain alone {timeit(chain):.1f} us", flush=True)
print(f"nd solve alone {timeit(st._coarse_solve):.1f} us", flush=True)
for grid in (148, 120, 100, 84, 72, 60, 48):
    tT = timeit(lambda: st._symv(st.d_Tp, r, st.d_delta, st.w_yb, grid, 1, _stream()))
    st.t_grid_bulk = grid
    tP = timeit(lambda: st._precond(r, W.zv))
    print(f"grid {grid}: T alone {tT:.1f} us ({1.245e9 / tT / 1e3:.0f} GB/s), precond {tP:.1f} us", flush=True)

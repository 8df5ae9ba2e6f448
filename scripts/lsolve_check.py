"""Determinism of the batched local solve outputs (u, p, rg) over repeated calls,
for the argument combinations the solver uses and one with every input set."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1901_02090_b200 as B
from paper_1901_02090_b200 import solver as S, _native as nat
from paper_1901_02090_b200.solver import _p
counts, splits = ((16, 16), (2, 2)) if len(sys.argv) < 2 else ((30, 30, 15), (3, 3, 3))
rng = np.random.default_rng(0)
g = B.build_grid(len(counts), counts, (1.0,) * len(counts))
k = 10 ** rng.uniform(-2, 2, (g.n_cells, len(counts)))
system = B.assemble_system(g, B.Permeability(k), B.Wells(0, g.n_cells - 1))
dec = B.regular_partition(g, splits)
st = B.BddcSetup(system, dec, B.SolveConfig())
dev = st.dev
x = torch.randn(st.n_gamma, dtype=torch.float64, device=dev)
gc = torch.randn(g.n_cells, dtype=torch.float64, device=dev)
ff = torch.randn(st.geom.n_flux, dtype=torch.float64, device=dev)
for combo in ("x,g,rg", "f,g,rg", "x,u", "x,g,u", "f,g,x,u", "g,rg", "f,rg"):
    outs = []
    for rep in range(4):
        u = torch.zeros(st.geom.n_flux, dtype=torch.float64, device=dev)
        pc = torch.zeros(g.n_cells, dtype=torch.float64, device=dev)
        rg = torch.zeros(st.N * st.maxG, dtype=torch.float64, device=dev)
        a = nat.LocalSolveArgs()
        if "x" in combo:
            a.x_gamma, a.x_scale = _p(x).value, 1.0
        if "g" in combo:
            a.g_cell, a.g_scale = _p(gc).value, 1.0
        if "f" in combo:
            a.f_flux, a.f_scale = _p(ff).value, 1.0
        if "u" in combo:
            a.u_out, a.u_mode = _p(u).value, 0
        a.p_out = _p(pc).value
        if "rg" in combo:
            a.rg_broken = _p(rg).value
        nat.call("bddc_local_solve", C.byref(st.geom), _p(st.d_coef), _p(st.d_gcode), _p(st.d_gpos),
                 _p(st.d_fslot), _p(st.d_Qp), _p(st.d_Dsub), C.byref(a), S._stream())
        torch.cuda.synchronize()
        outs.append((u.clone(), pc.clone(), rg.clone()))
    d = [max(float((outs[0][j] - o[j]).abs().max()) for o in outs[1:]) for j in range(3)]
    print(f"{combo:10s} max diff over repeats: u {d[0]:.1e} p {d[1]:.1e} rg {d[2]:.1e}")

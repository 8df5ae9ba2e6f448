import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, scipy.sparse as sp
import paper_1901_02090_b200 as B
counts, splits = (12, 20), tuple(int(v) for v in sys.argv[1:3]) if len(sys.argv) > 2 else (1, 4)
g = B.build_grid(2, counts, (1.0, 1.0))
k = np.ones((g.n_cells, 2))
sy = B.assemble_system(g, B.Permeability(k), B.PressureDrop(1, 1.0, 0.0))
dec = B.regular_partition(g, splits)
cfg = B.SolveConfig(tau=float("inf"), scaling="multiplicity", constraints="initial", tol=1e-12)
st = B.BddcSetup(sy, dec, cfg)
A = sy.A.tocsr(); Bm = sy.B.tocsr()
nf = sy.n_flux
# flux dofs of subdomain i: faces of its cells
cells_of = [np.nonzero(dec.cell_sub == i)[0] for i in range(dec.n_subdomains)]
for i in range(dec.n_subdomains):
    cs = cells_of[i]
    dofs = np.unique(Bm[cs].indices)
    gam = dec.gamma[dec.gpos[i][:dec.nG[i]]] if False else None
    # gamma dofs of i in local slot order
    gp = dec.gpos[i, :dec.nG[i]]
    gd = dec.gamma[gp]
    idof = np.setdiff1d(dofs, gd)
    # local A: element assembly restricted to cells of i
    rows, cols, vals = [], [], []
    Al = sp.lil_matrix((nf, nf))
    for a in range(2):
        lo, hi = g.cell_faces(a, 1)
        c = 1.0 / 6.0 / k[cs, a]
        for d, o in ((lo[cs], hi[cs]), (hi[cs], lo[cs])):
            for dd, oo, cc in zip(d, o, c):
                if dd >= 0:
                    Al[dd, dd] += 2 * cc
                    if oo >= 0: Al[dd, oo] += cc
    Al = Al.tocsr()
    Bl = Bm[cs]
    floating = st.floating[i]
    AII = Al[idof][:, idof].toarray(); AIG = Al[idof][:, gd].toarray(); AGG = Al[gd][:, gd].toarray()
    BI = Bl[:, idof].toarray(); BG = Bl[:, gd].toarray()
    nI, nc = len(idof), len(cs)
    K = np.block([[AII, BI.T], [BI, np.zeros((nc, nc))]])
    R = np.vstack([AIG, BG])
    if floating:
        V = np.concatenate([np.zeros(nI), np.ones(nc)])
        K = np.block([[K, V[:, None]], [V[None, :], np.zeros((1, 1))]])
        R = np.vstack([R, np.zeros((1, len(gd)))])
    S = AGG - R.T @ np.linalg.solve(K, R)
    Sg = st.schur_dense(i)
    print(i, "floating", floating, "nG", len(gd), "S err", np.abs(S - Sg).max() / np.abs(S).max(), "eigmin", np.linalg.eigvalsh(Sg).min())
ng = dec.n_gamma
E = np.eye(ng)
Sm = np.array([st.schur_matvec(E[:, j]) for j in range(ng)]).T
Mm = np.array([st.precondition(E[:, j]) for j in range(ng)]).T
Pm = np.array([st.project_balanced(E[:, j]) for j in range(ng)]).T
print("S sym", np.abs(Sm - Sm.T).max(), "M sym", np.abs(Mm - Mm.T).max(), "P sym", np.abs(Pm - Pm.T).max(), "P idem", np.abs(Pm @ Pm - Pm).max())
ev = np.linalg.eigvalsh(0.5 * (Pm @ Mm @ Pm + (Pm @ Mm @ Pm).T))
print("PMP eig", ev[:6], ev[-3:])
evs = np.linalg.eigvalsh(Pm @ Sm @ Pm)
print("PSP eig", evs[:6], evs[-3:])
for eager in (True, False):
    st.force_eager = eager
    try:
        r = B.solve(sy, dec, cfg, setup=st)
        print("eager", eager, "it", r.it, "res", r.residuals[:5], r.residuals[-3:])
    except Exception as e:
        print("eager", eager, "EXC", e, getattr(e, "report", None) and e.report.residuals[:8])
# project the rhs and solve densely
import torch
import paper_1901_02090_b200.solver as SV
orig = SV._pcg
def cap(setup, W, config, cb):
    setup.cap_r = W.r.cpu().numpy().copy()
    return orig(setup, W, config, cb)
SV._pcg = cap
try:
    B.solve(sy, dec, cfg, setup=st)
except Exception as e:
    pass
r = st.cap_r
print("|r|", np.linalg.norm(r), "|Pr-r|", np.linalg.norm(Pm @ r - r))
x = np.zeros_like(r); res = r.copy(); z = Pm @ Mm @ res; p = z.copy(); rz = res @ z
for it in range(60):
    Ap = Pm @ Sm @ p; al = rz / (p @ Ap); x += al * p; res -= al * Ap
    if it % 10 == 0: print(it, np.linalg.norm(res) / np.linalg.norm(r))
    z = Pm @ Mm @ res; rz2 = res @ z; p = z + rz2 / rz * p; rz = rz2
phi = st.net_flux_matrix().toarray() if hasattr(st.net_flux_matrix(), "toarray") else st.net_flux_matrix()
print("Phi r", phi @ r)

import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, scipy.linalg as sla, torch
import paper_1901_02090_b200 as B
from paper_1901_02090_b200 import solver as S
g = B.build_grid(2, (12, 12), (1.0, 1.0))
rng = np.random.default_rng(3)
k = 10.0 ** rng.uniform(-2, 2, g.n_cells)
system = B.assemble_system(g, B.Permeability.isotropic(g, k), B.Wells(0, g.n_cells - 1))
dec = B.regular_partition(g, (3, 3))
st = B.BddcSetup(system, dec, B.SolveConfig(tau=3.0, constraints="adaptive"))
n = dec.n_gamma
E = np.eye(n)
Sm = np.stack([st.schur_matvec(E[:, c]) for c in range(n)], axis=1)
Mm = np.stack([st.precondition(E[:, c]) for c in range(n)], axis=1)
print("n", n, "N", st.N, "S sym", np.abs(Sm - Sm.T).max(), "M sym", np.abs(Mm - Mm.T).max())
Z = sla.null_space(st.net_flux_matrix().toarray())
Sb = Z.T @ Sm @ Z; Mb = Z.T @ Mm @ Z
w, V = sla.eigh(0.5 * (Mb + Mb.T))
W = (V * np.sqrt(np.maximum(w, 0))) @ V.T
lam = np.sort(sla.eigh(W @ (0.5 * (Sb + Sb.T)) @ W, eigvals_only=True))
print("dense", lam[:4], lam[-4:], len(lam))
# instrumented Lanczos
orig = S._dot
log = []
def dot(setup, x, y, nn, op, hist=None):
    orig(setup, x, y, nn, op, hist)
S._dot = dot
lg = S.preconditioned_spectrum(st)
print("gpu", lg[:4], lg[-4:], len(lg))
dbg = {}
lg = S.preconditioned_spectrum(st, _debug=dbg)
print("alphas", np.array(dbg["alphas"][:8]))
print("betas", np.array(dbg["betas"][:8]))
a, b = np.array(dbg["alphas"]), np.array(dbg["betas"])
T = np.diag(a) + np.diag(b[:len(a) - 1], 1) + np.diag(b[:len(a) - 1], -1)
print("numpy eig of T", np.sort(np.linalg.eigvalsh(T))[:4], np.sort(np.linalg.eigvalsh(T))[-4:])
np.set_printoptions(linewidth=200, precision=3)
print("all alphas", a)
print("all betas", b)
Qh, SQh = dbg["Q"], dbg["SQ"]
P = Z @ Z.T
G = Qh @ Sm @ Qh.T
print("Q^T S Q - I (first 15):", np.abs(G[:15, :15] - np.eye(15)).max(), "full:", np.abs(G - np.eye(len(G))).max())
print("SQ vs P S Q:", np.abs(SQh - (P @ Sm @ Qh.T).T).max(axis=1)[:20])
print("Q in range P:", np.abs(Qh - (P @ Qh.T).T).max(axis=1)[:20])

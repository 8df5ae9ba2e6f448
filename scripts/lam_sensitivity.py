"""Eigenvalue sensitivity of the reference pair problems (build container only).

Captures the reference's dense pair problems during setup of a golden case and
measures how far the top eigenvalues move under (a) a symmetric relative
perturbation of S at the 1e-15 level (summation-order noise) and (b) a
Rayleigh-quotient re-evaluation in extended precision.  Used to decide what
eigenvalue agreement is attainable between two f64 implementations.
"""
import sys, numpy as np
sys.path.insert(0, "/root/reference/pkg/src"); sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/oracle")
import make_golden as MG
from bddcflow import adaptive as A
name = sys.argv[1] if len(sys.argv) > 1 else "g3d_c3block"
cap = []
orig = A.pair_eig
def spy(problem, *a, **k):
    r = orig(problem, *a, **k)
    cap.append((problem, r))
    return r
A.pair_eig = spy
import bddcflow.solver as S
counts, sizes, splits, scaling, tau, tol, kmaker = MG.CASES[name]
from bddcflow import grid as G, decomposition as D
k = np.asarray(kmaker(), float)
g = G.build_grid(len(counts), counts, sizes)
sysm = G.assemble_system(g, G.Permeability(k), G.Wells(0, g.n_cells - 1))
dec = D.regular_partition(g, splits)
cfg = S.SolveConfig(tau=tau, scaling=scaling, constraints="adaptive", tol=tol)
S.BddcSetup(sysm, dec, cfg)
rng = np.random.default_rng(0)
worst = 0
for prob, rep in cap:
    lam = rep.eigenvalues[rep.eigenvalues > tau]
    if not len(lam):
        continue
    spread = np.zeros(len(lam))
    for t in range(3):
        E = rng.standard_normal(prob.S.shape); E = (E + E.T) / 2
        Sp = prob.S + 1e-15 * np.abs(prob.S) * E
        P2 = prob._replace(S=Sp) if hasattr(prob, "_replace") else None
        if P2 is None:
            import copy; P2 = copy.copy(prob); P2.S = Sp
        l2 = orig(P2).eigenvalues[:len(lam)]
        spread = np.maximum(spread, np.abs(l2 - lam) / lam)
    # extended-precision Rayleigh quotient on the reference eigenvectors
    W = rep.eigenvectors[:, :len(lam)].astype(np.longdouble)
    L = rep.jump_form if False else None
    IE = np.eye(prob.size) - prob.E
    Lm = (prob.Pi @ IE.T @ prob.S @ IE @ prob.Pi).astype(np.longdouble)
    Rm = (prob.Pi @ prob.S @ prob.Pi).astype(np.longdouble)
    rq = np.array([(W[:, j] @ Lm @ W[:, j]) / (W[:, j] @ Rm @ W[:, j]) for j in range(len(lam))], dtype=float)
    print(f"pair ({prob.i},{prob.j}) lam {np.array2string(lam[:4], precision=10)} "
          f"noise1e-15 spread {spread.max():.2e}  rq-vs-lam {np.max(np.abs(rq-lam)/lam):.2e}")
    worst = max(worst, spread.max())
print("worst spread", worst)

# reduced m x m pencil (the formulation csrc/adaptive.cu solves) with LAPACK S^-1
import scipy.linalg as sla
for prob, rep in cap:
    lam = rep.eigenvalues[rep.eigenvalues > tau]
    if not len(lam) or lam[0] < 1e4:
        continue
    ni = len(prob.dofs_i)
    Si, Sj = prob.S[:ni, :ni], prob.S[ni:, ni:]
    pi, pj = np.asarray(prob.pos_i), np.asarray(prob.pos_j) - ni
    di = prob.E[pi, pi]; dj = prob.E[pi, pj + ni]
    A = dj[:, None] * Si[np.ix_(pi, pi)] * dj[None, :] + di[:, None] * Sj[np.ix_(pj, pj)] * di[None, :]
    res = []
    for how in ("cho", "inv", "cho_noise"):
        if how == "cho":
            Xi = sla.cho_solve(sla.cho_factor(Si), np.eye(ni)); Xj = sla.cho_solve(sla.cho_factor(Sj), np.eye(len(Sj)))
        elif how == "inv":
            Xi = np.linalg.inv(Si); Xj = np.linalg.inv(Sj)
        else:
            E1 = rng.standard_normal(Si.shape); E1 = (E1 + E1.T) / 2
            Xi = sla.cho_solve(sla.cho_factor(Si + 1e-15 * np.abs(Si) * E1), np.eye(ni)); Xj = sla.cho_solve(sla.cho_factor(Sj), np.eye(len(Sj)))
        M = Xi[np.ix_(pi, pi)] + Xj[np.ix_(pj, pj)]
        M = (M + M.T) / 2
        R = np.linalg.cholesky(M)
        Bh = R.T @ A @ R
        q = R.T @ np.ones(len(pi)); q /= np.linalg.norm(q)
        Pq = np.eye(len(q)) - np.outer(q, q)
        ev = np.sort(np.linalg.eigvalsh(Pq @ Bh @ Pq))[::-1][:len(lam)]
        res.append(f"{how}: {np.max(np.abs(ev - lam) / lam):.2e}")
    wS = np.linalg.eigvalsh(Si)
    print(f"reduced pair ({prob.i},{prob.j}) m={len(pi)} cond(Si)={wS[-1]/wS[0]:.2e}", *res)

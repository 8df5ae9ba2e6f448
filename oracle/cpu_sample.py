"""Bounded CPU-baseline sample of the reference algorithm at a large config.

TEST/BENCH INFRASTRUCTURE ONLY (used by bench.py's `cpu_baseline` leg and
`--impl reference`).  A full reference run at BASELINE config 3 takes
hours, so this times the oracle's per-unit costs on a
sample of the same workload and scales them by the unit counts:

* per subdomain: SuperLU factorisation of the interior KKT and of the
  constrained KKT (substructure.py:66, coarse.py:159), one Schur apply
  (substructure.py:85-88) and one Delta solve (coarse.py:237-245);
* the dense coarse LU solve (coarse.py:208-215) timed at a reduced order and
  scaled by (n/n_s)^2;
* the dense balanced projection Q(Q^T x) (solver.py:175-179) timed on a
  row block of Q and scaled by the row count.

time_to_solve ~= 4 N t_kkt + it * (N (t_schur + t_delta) + t_coarse + 2 t_proj)
The result is labelled "extrapolated" by the caller.
"""

from __future__ import annotations

import os
import time

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp

from . import bddc_oracle as O


def _timeit(fn, reps):
    fn()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    return (time.perf_counter() - t) / reps


def sample_solve(counts, sizes, k, splits, it, n_coarse, rows_per_sub,
                 n_sub_sample=3, seed=0):
    """Estimate the reference time-to-solve (prebuilt setup) for one config."""
    rng = np.random.default_rng(seed)
    t_all = time.perf_counter()
    dim = len(counts)
    n3 = tuple(counts) + (1,) * (3 - dim)
    s3 = tuple(splits) + (1,) * (3 - dim)
    w3 = [O.near_equal(n3[a], s3[a]) for a in range(3)]
    N = int(np.prod(s3))
    kk = k.reshape(n3[2], n3[1], n3[0], dim)
    t_fac, t_schur, t_delta, t_cfac, t_kkt = [], [], [], [], []
    # interior subdomains sampled along the diagonal of the subdomain grid;
    # each is timed inside a 3x3(x3) block of subdomains cropped from the
    # field (identical local structure, independent of the global size)
    for q in range(n_sub_sample):
        frac = (q + 1) / (n_sub_sample + 1)
        sc = [min(max(int(frac * s3[a]), 1), s3[a] - 2) if s3[a] >= 3 else 0
              for a in range(3)]
        lo3 = [sc[a] - 1 if s3[a] >= 3 else 0 for a in range(3)]
        nb = [3 if s3[a] >= 3 else s3[a] for a in range(3)]
        c0 = [int(np.sum(w3[a][:lo3[a]])) for a in range(3)]
        c1 = [c0[a] + int(np.sum(w3[a][lo3[a]:lo3[a] + nb[a]])) for a in range(3)]
        kb = kk[c0[2]:c1[2], c0[1]:c1[1], c0[0]:c1[0]].reshape(-1, dim)
        bc = tuple(c1[a] - c0[a] for a in range(dim))
        mesh = O.Mesh(bc, sizes)
        P = O.BoxPartition(mesh, tuple(nb[:dim]))
        B = O.divergence(mesh)
        centre = (1 if nb[0] == 3 else 0) + nb[0] * ((1 if nb[1] == 3 else 0)
                                                     + nb[1] * (1 if nb[2] == 3 else 0))
        t0 = time.perf_counter()
        lo = O.LocalOp(mesh, kb, P, B, int(centre))
        t_fac.append(time.perf_counter() - t0)
        x = rng.standard_normal(lo.nG)
        t_schur.append(_timeit(lambda: lo.schur_apply(x), 3))
        t_kkt.append(_timeit(lambda: lo.trace_solve(x, np.zeros(lo.nP)), 3))
        # constrained KKT with the measured average number of rows
        nc = max(int(round(rows_per_sub)), 1)
        C = np.zeros((nc, lo.nI + lo.nG))
        C[:, lo.nI:] = rng.standard_normal((nc, lo.nG))
        K = sp.bmat([[lo.A_loc, lo.B_loc.T, sp.csr_matrix(C.T), None],
                     [lo.B_loc, None, None, lo.V.T],
                     [sp.csr_matrix(C), None, None, None],
                     [None, lo.V, None, None]], format="csc")
        t0 = time.perf_counter()
        from scipy.sparse.linalg import splu
        lu = splu(K)
        t_cfac.append(time.perf_counter() - t0)
        rhs = np.zeros(K.shape[0])
        rhs[lo.nI:lo.nI + lo.nG] = x
        t_delta.append(_timeit(lambda: lu.solve(rhs), 3))
    n_g_total = 0
    for a in range(dim):
        e = list(n3)
        e[a] = s3[a] - 1
        n_g_total += int(np.prod(e[:3]))
    # dense coarse LU solve, scaled by n^2
    n_s = min(n_coarse, 3000)
    M = rng.standard_normal((n_s, n_s)) + n_s * np.eye(n_s)
    lu0 = sla.lu_factor(M)
    b = rng.standard_normal(n_s)
    t_coarse = _timeit(lambda: sla.lu_solve(lu0, b), 5) * (n_coarse / n_s) ** 2
    # balanced projection Q(Q^T x) with Q: n_gamma x (N-1), scaled by rows
    n_g = n_g_total
    rows = min(n_g, 40000)
    Qb = rng.standard_normal((rows, max(N - 1, 1)))
    xb = rng.standard_normal(rows)
    t_proj = _timeit(lambda: Qb @ (Qb.T @ xb), 3) * (n_g / rows)
    ts, td, tk = float(np.mean(t_schur)), float(np.mean(t_delta)), float(np.mean(t_kkt))
    t_iter = N * (ts + td) + t_coarse + 2 * t_proj
    t_solve = 4 * N * tk + it * t_iter
    return dict(
        time_to_solve_s=t_solve, t_iter_s=t_iter, it=it,
        it_per_s=it / t_solve,
        per_sub=dict(schur_apply_s=ts, delta_solve_s=td, kkt_solve_s=tk,
                     interior_splu_s=float(np.mean(t_fac)),
                     constrained_splu_s=float(np.mean(t_cfac))),
        coarse_solve_s=t_coarse, projection_s=t_proj,
        setup_local_factor_s_est=N * (float(np.mean(t_fac)) + float(np.mean(t_cfac))),
        sample=(f"{n_sub_sample} interior subdomains x (interior splu + constrained splu "
                f"+ schur_apply + delta_solve), coarse lu_solve at n={n_s} scaled to "
                f"n={n_coarse}, projection on {rows} of {n_g} rows; scaled to N={N}, it={it}"),
        cores=os.cpu_count(),
        wall_s=time.perf_counter() - t_all,
    )

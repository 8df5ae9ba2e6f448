"""Generate golden fixtures from the UNMODIFIED reference (run in the build container).

Imports `bddcflow` read-only from /root/reference/pkg/src (it is not on the
GPU box) and writes small `.npz` files under tests/golden/.  Each fixture
holds the inputs (grid, permeability, partition, config) and the
reference's outputs: u, p, it, kappa, omega_tilde, n_c, residual history,
per-pair eigenvalues and selected counts, one subdomain Schur complement,
and one application of schur_matvec / precondition / project_balanced to a
seeded vector.  Mode A (wells at cells 0 and n-1, no-flow) only: the
reference cannot express BASELINE's pressure-drop boundary conditions.

Usage:  python oracle/make_golden.py [name ...]
"""

from __future__ import annotations

import math
import os
import sys
import time
import warnings

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)
warnings.filterwarnings("ignore", message="coefficient jumps")

from bddcflow import solver as R_solver          # noqa: E402
from bddcflow import grid as R_grid              # noqa: E402
from bddcflow import decomposition as R_dec      # noqa: E402

from paper_1901_02090_b200 import fields         # noqa: E402


def _random_k(counts, seed, orders=6.0):
    rng = np.random.default_rng(seed)
    n = int(np.prod(counts))
    return 10.0 ** rng.uniform(-orders / 2, orders / 2, (n, len(counts)))


def _c3_block(z0, nz=15, ny=30, nx=30, y0=40, x0=10):
    """Cells cropped from the config-3 field (default 30x30x15, C3's 10x10x5 subdomains)."""
    k = fields.config_field(3).reshape(85, 220, 60, 3)
    return np.ascontiguousarray(k[z0:z0 + nz, y0:y0 + ny, x0:x0 + nx].reshape(-1, 3))


CASES = {
    # name: (counts, sizes, splits, scaling, tau, tol, k-maker)
    "g2d_small": ((8, 8), (1.0, 1.0), (2, 2), "multiplicity", math.inf,
                  1e-10, lambda: _random_k((8, 8), 1)),
    "g2d_adapt": ((12, 12), (1.0, 1.0), (3, 3), "stiffness", 3.0, 1e-10,
                  lambda: _random_k((12, 12), 2)),
    "g2d_aniso": ((9, 21), (2.0, 0.5), (3, 3), "multiplicity", 5.0, 1e-10,
                  lambda: _random_k((9, 21), 7)),
    "g3d_adapt": ((6, 6, 6), (1.0, 1.0, 1.0), (2, 2, 2), "multiplicity",
                  5.0, 1e-10, lambda: _random_k((6, 6, 6), 3)),
    "g3d_thin": ((5, 5, 5), (1.0, 2.0, 0.5), (3, 3, 3), "stiffness", 5.0,
                 1e-10, lambda: _random_k((5, 5, 5), 4)),
    "g3d_box": ((8, 6, 4), (20.0, 10.0, 2.0), (2, 2, 2), "stiffness", 10.0,
                1e-10, lambda: _random_k((8, 6, 4), 9)),
    "g3d_c3block": ((30, 30, 15), (20.0, 10.0, 2.0), (3, 3, 3), "multiplicity", 10.0,
                    1e-8, lambda: _c3_block(28)),
    "g3d_uneven": ((12, 10, 8), (1.0, 2.0, 0.5), ((3, 5, 4), (2, 4, 4), (5, 3)), "multiplicity",
                   5.0, 1e-10, lambda: _random_k((12, 10, 8), 11)),
    # C4-shaped subdomains (5x5x5 cells): 4x4x2 of them, across the z = 35 field seam
    "g3d_c4block": ((20, 20, 10), (20.0, 10.0, 2.0), (4, 4, 2), "multiplicity", 10.0,
                    1e-8, lambda: _c3_block(30, nz=10, ny=20, nx=20)),
    # C3-shaped subdomains (10x10x5 cells), 4x4x4 = 64 of them (interior subdomains
    # with all six faces shared), across the seam
    "g3d_c3_64": ((40, 40, 20), (20.0, 10.0, 2.0), (4, 4, 4), "multiplicity", 10.0,
                  1e-8, lambda: _c3_block(25, nz=20, ny=40, nx=40, y0=90, x0=10)),
    "g2d_ms": ((12, 12), (1.0, 1.0), (3, 3), "multiplicity", math.inf, 1e-10,
               lambda: _random_k((12, 12), 21)),
    "g3d_ms": ((8, 6, 6), (20.0, 10.0, 2.0), (2, 3, 2), "stiffness", math.inf, 1e-10,
               lambda: _random_k((8, 6, 6), 22)),
    "c0": (fields.CONFIGS[0]["counts"], fields.CONFIGS[0]["sizes"],
           fields.CONFIGS[0]["splits"], "stiffness", math.inf, 1e-8,
           lambda: fields.config_field(0)),
    "c1": (fields.CONFIGS[1]["counts"], fields.CONFIGS[1]["sizes"],
           fields.CONFIGS[1]["splits"], "multiplicity", 10.0, 1e-8,
           lambda: fields.config_field(1)),
    "c1_rho": (fields.CONFIGS[1]["counts"], fields.CONFIGS[1]["sizes"],
               fields.CONFIGS[1]["splits"], "stiffness", 10.0, 1e-8,
               lambda: fields.config_field(1)),
    "c2_tau10": (fields.CONFIGS[2]["counts"], fields.CONFIGS[2]["sizes"],
                 fields.CONFIGS[2]["splits"], "multiplicity", 10.0, 1e-8,
                 lambda: fields.config_field(2)),
    "c2_tau2": (fields.CONFIGS[2]["counts"], fields.CONFIGS[2]["sizes"],
                fields.CONFIGS[2]["splits"], "multiplicity", 2.0, 1e-8,
                lambda: fields.config_field(2)),
    "c2_tau100": (fields.CONFIGS[2]["counts"], fields.CONFIGS[2]["sizes"],
                  fields.CONFIGS[2]["splits"], "multiplicity", 100.0, 1e-8,
                  lambda: fields.config_field(2)),
    # tau = inf: face averages only, pairs still solved for omega~ (solver.py:85-88)
    "c2_tauinf": (fields.CONFIGS[2]["counts"], fields.CONFIGS[2]["sizes"],
                  fields.CONFIGS[2]["splits"], "multiplicity", math.inf, 1e-8,
                  lambda: fields.config_field(2)),
}
ADAPTIVE_AT_INF = {"c2_tauinf"}
# lumped RT0 mass matrices (grid.py:204-227, assemble_system(lumped=True))
CASES["g2d_lumped"] = ((12, 12), (1.0, 1.0), (3, 3), "stiffness", 3.0, 1e-10,
                       lambda: _random_k((12, 12), 31))
CASES["g3d_lumped"] = ((8, 6, 6), (20.0, 10.0, 2.0), (2, 3, 2), "multiplicity", 5.0, 1e-10,
                       lambda: _random_k((8, 6, 6), 32))
LUMPED = {"g2d_lumped", "g3d_lumped"}


def make(name):
    counts, sizes, splits, scaling, tau, tol, kmaker = CASES[name]
    k = np.asarray(kmaker(), dtype=np.float64)
    dim = len(counts)
    g = R_grid.build_grid(dim, counts, sizes)
    perm = R_grid.Permeability(k)
    system = R_grid.assemble_system(g, perm, R_grid.Wells(0, g.n_cells - 1),
                                    lumped=name in LUMPED)
    if any(np.ndim(sp) > 0 for sp in splits):
        # uneven strips: the reference's Decomposition(grid, part) with a box part
        part = np.zeros(g.n_cells, dtype=np.int64)
        stride = 1
        for a in range(dim):
            bounds = np.cumsum(splits[a])
            strip = np.searchsorted(bounds, np.arange(counts[a]), side="right")
            part += stride * strip[g.cell_coords[:, a]]
            stride *= len(splits[a])
        dec = R_dec.Decomposition(g, part)
    else:
        dec = R_dec.regular_partition(g, splits)
    mode = "adaptive" if math.isfinite(tau) or name in ADAPTIVE_AT_INF else "initial"
    if name.endswith("_ms"):
        mode = "multiscale"   # MsMFEM baseline (adaptive.py:207-269)
    cfg = R_solver.SolveConfig(tau=tau, scaling=scaling, constraints=mode,
                               tol=tol)
    t0 = time.time()
    setup = R_solver.BddcSetup(system, dec, cfg)
    t1 = time.time()
    rep = R_solver.solve(system, dec, cfg, setup=setup)
    t2 = time.time()

    rng = np.random.default_rng(1234)
    x = rng.standard_normal(len(dec.gamma))
    out = dict(
        constraints=mode, lumped=name in LUMPED,
        counts=np.array(counts), sizes=np.array(sizes, dtype=np.float64),
        splits=np.array([len(sp) if np.ndim(sp) > 0 else sp for sp in splits]),
        scaling=scaling, tau=tau, tol=tol, k=k,
        u=rep.u, p=rep.p, it=rep.it, kappa=rep.kappa,
        omega_tilde=rep.omega_tilde, n_c=rep.n_c, residuals=rep.residuals,
        u0=rep.u0, u_star=rep.u_star,
        conservation_defect=rep.conservation_defect,
        gamma=dec.gamma, x=x,
        Sx=setup.schur_matvec(x), Mx=setup.precondition(x),
        Px=setup.project_balanced(x),
        S_sub0=setup.subs[0].schur_dense(),
        S_sublast=setup.subs[-1].schur_dense(),
        D=setup.system.D,
        setup_s=t1 - t0, solve_s=t2 - t1,
    )
    # per-face selected counts and the leading eigenvalues of every pair
    pairs = sorted(dec.faces.keys())
    out["pairs"] = np.array(pairs, dtype=np.int64).reshape(-1, 2)
    out["face_rows"] = np.array(
        [len(setup.cset.rows_for_face(i, j)) // 2 for (i, j) in pairs])
    if setup.pair_reports:
        top = 24
        lam = np.full((len(pairs), top), np.nan)
        sel = np.zeros(len(pairs), dtype=np.int64)
        for q, key in enumerate(pairs):
            ev = setup.pair_reports[key].eigenvalues[:top]
            lam[q, :len(ev)] = ev
            sel[q] = setup.pair_reports[key].selected
        out["pair_lam"] = lam
        out["pair_selected"] = sel
    if any(np.ndim(sp) > 0 for sp in splits):
        wmax = max(len(sp) for sp in splits)
        out["widths"] = np.array([list(sp) + [-1] * (wmax - len(sp)) for sp in splits])
    path = os.path.join(REPO, "tests", "golden", f"{name}.npz")
    np.savez_compressed(path, **out)
    print(f"{name}: it={rep.it} kappa={rep.kappa:.6g} n_c={rep.n_c} "
          f"omega={rep.omega_tilde:.6g} setup={t1 - t0:.2f}s "
          f"solve={t2 - t1:.2f}s -> {os.path.getsize(path) / 1e3:.0f} KB")


if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for n in names:
        make(n)

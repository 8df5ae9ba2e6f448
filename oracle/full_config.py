"""Full-size oracle runs of BASELINE configs 3 and 4 -> compact committed fixtures.

TEST INFRASTRUCTURE ONLY.  Runs the CPU restatement (`oracle/bddc_oracle.py`)
at the north-star configuration (C3: 60x220x85 cells, 6x22x17 subdomains,
adaptive tau = 10) and at C4 (12x44x17 subdomains), mode A (wells at cells 0
and n-1, the reference-native boundary condition), with the harness
substitutions the unmodified reference cannot do without at this size
(SURVEY 8c): box topology in closed form, sparse LU of the pinned coarse
saddle instead of the dense `lu_factor` (coarse.py:196), the balanced
projection in Laplacian form instead of the dense QR of Phi^T
(solver.py:166-179), the pressure Neumann problem by DCT instead of SuperLU
(solver.py:254-274), and forked workers over the S_i and pair loops.  Every
substitution is pinned against the literal form on the golden cases
(tests/test_oracle_golden.py::test_oracle_substitutions).

The fixture (tests/golden/full_c{3,4}.npz) is compact: scalars, per-face
selected counts / rows / leading eigenvalues, residual history, and for
every long vector (u, p, u0, u*, S x, M x, P x for a seeded x) its norm, a
seeded sample of entries and a CountSketch (oracle/sketch.py), from which
tests estimate the relative L2 distance of the GPU vector.

Usage:  python oracle/full_config.py 3 [--workers 8]
"""

from __future__ import annotations

import argparse
import os
import sys
import time
import warnings

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
sys.path.insert(0, REPO)

from oracle import bddc_oracle as O            # noqa: E402
from oracle.sketch import count_sketch, sample_idx   # noqa: E402
from paper_1901_02090_b200 import fields        # noqa: E402

X_SEED = 1234
O.PERMC = "MMD_AT_PLUS_A"   # less fill than COLAMD on these KKTs (memory at 2244 subdomains)


def fingerprint(out, name, v):
    v = np.asarray(v, dtype=np.float64)
    out[name + "_norm"] = float(np.linalg.norm(v))
    out[name + "_sketch"] = count_sketch(v)
    idx = sample_idx(len(v))
    out[name + "_idx"] = idx
    out[name + "_sample"] = v[idx]


def compact_pair_lam(out, lams, sel):
    """Per face the selected eigenvalues (> tau) and the next one (omega), flattened:
    face q owns pair_lam_flat[pair_lam_ptr[q]:pair_lam_ptr[q + 1]]."""
    parts = [np.asarray(l, dtype=np.float64)[:int(k) + 1] for l, k in zip(lams, sel)]
    out["pair_lam_ptr"] = np.concatenate([[0], np.cumsum([len(p) for p in parts])]).astype(np.int64)
    out["pair_lam_flat"] = np.concatenate(parts) if parts else np.zeros(0)


def run(cfg_id, workers):
    spec = fields.CONFIGS[cfg_id]
    t0 = time.time()
    log = lambda m: print(f"[{time.time() - t0:8.1f}s] {m}", flush=True)
    k = fields.config_field(cfg_id)
    log("field")
    cfg = O.Config(tau=spec["tau"], scaling=spec["scaling"], constraints=spec["constraints"],
                   tol=spec["tol"], coarse="sparse", project="laplacian", pressure="dct",
                   workers=workers, log=log)
    mesh = O.Mesh(spec["counts"], spec["sizes"])
    f = O.well_rhs(mesh, 0, mesh.n_cells - 1)
    st = O.Setup(mesh, k, f, spec["splits"], cfg)
    t_setup = time.time() - t0
    log("setup done")
    its = []
    rep = O.solve(st, callback=lambda x, r: (its.append(1), log(f"pcg it {len(its)}")))
    t_solve = time.time() - t0 - t_setup
    log(f"solve: it={rep.it} kappa={rep.kappa:.6g} n_c={rep.n_c} omega={rep.omega_tilde:.6g}")
    P = st.P
    out = dict(config=cfg_id, counts=np.array(spec["counts"]),
               sizes=np.array(spec["sizes"], dtype=np.float64),
               splits=np.array(spec["splits"]), scaling=spec["scaling"], tau=spec["tau"],
               tol=spec["tol"], constraints=spec["constraints"],
               it=rep.it, kappa=rep.kappa, n_c=rep.n_c, omega_tilde=rep.omega_tilde,
               residuals=rep.residuals, conservation_defect=rep.conservation_defect,
               pressure_warning=rep.pressure_warning, n_gamma=len(P.gamma),
               setup_s=t_setup, solve_s=t_solve, workers=workers, x_seed=X_SEED)
    for name, v in (("u", rep.u), ("p", rep.p), ("u0", rep.u0), ("u_star", rep.u_star)):
        fingerprint(out, name, v)
    x = np.random.default_rng(X_SEED).standard_normal(len(P.gamma))
    fingerprint(out, "Sx", st.schur_matvec(x))
    fingerprint(out, "Mx", st.precondition(x))
    fingerprint(out, "Px", st.project(x))
    log("operator fingerprints")
    pairs = list(P.pairs)
    out["pairs"] = np.array(pairs, dtype=np.int64).reshape(-1, 2)
    out["face_rows"] = np.array([len(r) for r in st.cons.face_rows])
    sel = np.array([st.pairs[key].selected for key in pairs])
    out["pair_selected"] = sel
    compact_pair_lam(out, [st.pairs[key].lam for key in pairs], sel)
    out["pair_omega"] = np.array([st.pairs[key].omega(spec["tau"]) for key in pairs])
    path = os.path.join(REPO, "tests", "golden", f"full_c{cfg_id}.npz")
    np.savez_compressed(path, **out)
    log(f"wrote {path} ({os.path.getsize(path) / 1e3:.0f} KB)")


if __name__ == "__main__":
    warnings.filterwarnings("ignore")
    ap = argparse.ArgumentParser()
    ap.add_argument("config", type=int, choices=(3, 4))
    ap.add_argument("--workers", type=int, default=os.cpu_count() or 1)
    a = ap.parse_args()
    run(a.config, a.workers)

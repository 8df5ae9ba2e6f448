"""Print the GPU path's distance to every golden fixture (calibrates the test bars)."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from _golden import load, names, rel   # noqa: E402

import paper_1901_02090_b200 as B      # noqa: E402

out = {}
for name in (sys.argv[1:] or names()):
    d = load(name)
    g = B.build_grid(len(d["counts"]), d["counts"], d["sizes"])
    system = B.assemble_system(g, B.Permeability(d["k"]), B.Wells(0, g.n_cells - 1))
    dec = B.regular_partition(g, d["splits"])
    cfg = B.SolveConfig(tau=d["tau"], scaling=d["scaling"], constraints=d["mode"], tol=d["tol"])
    st = B.BddcSetup(system, dec, cfg)
    rep = B.solve(system, dec, cfg, setup=st)
    r = dict(it=rep.it, it_ref=int(d["it"]), kappa=rep.kappa, kappa_ref=float(d["kappa"]),
             n_c=rep.n_c, n_c_ref=int(d["n_c"]),
             du=rel(rep.u, d["u"]), dp=rel(rep.p, d["p"]), du0=rel(rep.u0, d["u0"]),
             dus=rel(rep.u_star, d["u_star"]),
             cd=rep.conservation_defect, cd_ref=float(d["conservation_defect"]),
             Sx=rel(st.schur_matvec(d["x"]), d["Sx"]), Mx=rel(st.precondition(d["x"]), d["Mx"]),
             Px=rel(st.project_balanced(d["x"]), d["Px"]),
             S0=rel(st.schur_dense(0), d["S_sub0"]),
             Sl=rel(st.schur_dense(dec.n_subdomains - 1), d["S_sublast"]))
    if st.omega_tilde is not None and np.isfinite(float(d["omega_tilde"])):
        r["domega"] = abs(st.omega_tilde - float(d["omega_tilde"])) / float(d["omega_tilde"])
    out[name] = r
    print(name, json.dumps({k: (float(f"{v:.3g}") if isinstance(v, float) else v) for k, v in r.items()}),
          flush=True)

"""Pair-eigensolver phase time (device) for CTA sizes of the large-face launch (C3)."""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1901_02090_b200 as B
from paper_1901_02090_b200 import fields, _native as nat
c = fields.CONFIGS[3]; k = fields.config_field(3)
g = B.build_grid(c["dim"], c["counts"], c["sizes"]); dec = B.regular_partition(g, c["splits"])
system = B.assemble_system(g, B.Permeability(k), B.Wells(0, g.n_cells - 1))
cfg = B.SolveConfig(tau=c["tau"], scaling=c["scaling"], constraints="adaptive", tol=c["tol"])
lib = nat.load()
ref = None
for t in (256, 512):
    lib.bddc_set_pair_threads(t)
    tm = {}
    st = B.BddcSetup(system, dec, cfg); del st
    st = B.BddcSetup(system, dec, cfg, timings=tm)
    lam = st.pair_lambda.cpu().numpy()
    if ref is None:
        ref = lam
    m = ~(lam != lam)
    print(t, "pairs ms", round(tm["pairs"], 2), "setup ms", round(tm["total"], 1), "max lam diff",
          float(abs(lam[m] - ref[m]).max()), flush=True)
    del st

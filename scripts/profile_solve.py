"""Build a config's setup, then run ONE solve between cudaProfilerStart/Stop
(for `ncu --profile-from-start off`).  --what setup profiles the setup instead."""
import argparse, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1901_02090_b200 as B
from paper_1901_02090_b200 import fields

ap = argparse.ArgumentParser()
ap.add_argument("cfg", type=int)
ap.add_argument("--what", default="solve")
ap.add_argument("--eager", action="store_true", help="host-driven PCG loop (ncu sees every kernel)")
a = ap.parse_args()
c = fields.CONFIGS[a.cfg]
k = fields.config_field(a.cfg)
g = B.build_grid(c["dim"], c["counts"], c["sizes"])
dec = B.regular_partition(g, c["splits"])
system = B.assemble_system(g, B.Permeability(k), B.Wells(0, g.n_cells - 1))
cfg = B.SolveConfig(tau=c["tau"], scaling=c["scaling"],
                    constraints="adaptive" if math.isfinite(c["tau"]) else "initial", tol=c["tol"])
if a.what == "setup":
    torch.cuda.synchronize(); torch.cuda.profiler.start()
    st = B.BddcSetup(system, dec, cfg)
    torch.cuda.synchronize(); torch.cuda.profiler.stop()
else:
    st = B.BddcSetup(system, dec, cfg)
    st.force_eager = a.eager
    r = B.solve(system, dec, cfg, setup=st)      # warm
    torch.cuda.synchronize(); torch.cuda.profiler.start()
    r = B.solve(system, dec, cfg, setup=st)
    torch.cuda.synchronize(); torch.cuda.profiler.stop()
    print("it", r.it, "kappa", r.kappa)

"""Device time of every native call in one BddcSetup, with its leading args (dev tool)."""
import os, sys, time, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1901_02090_b200 as B
from paper_1901_02090_b200 import fields, _native as nat
cfgi = int(sys.argv[1]) if len(sys.argv) > 1 else 3
c = fields.CONFIGS[cfgi]
k = fields.config_field(cfgi)
g = B.build_grid(c["dim"], c["counts"], c["sizes"])
dec = B.regular_partition(g, c["splits"])
system = B.assemble_system(g, B.Permeability(k), B.Wells(0, g.n_cells - 1))
cfg = B.SolveConfig(tau=c["tau"], scaling=c["scaling"], constraints="adaptive", tol=c["tol"])
st = B.BddcSetup(system, dec, cfg)
del st
torch.cuda.synchronize()
orig = nat.call
log = []


def timed(name, *args):
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    r = orig(name, *args)
    b.record()
    log.append((name, args[:7], a, b))
    return r


nat.call = timed
import paper_1901_02090_b200.solver as S
import paper_1901_02090_b200.coarse_nd as ND
S.nat.call = timed
ND.nat.call = timed
st = B.BddcSetup(system, dec, cfg)
torch.cuda.synchronize()
tot = collections.Counter()
rows = []
for name, args, a, b in log:
    t = a.elapsed_time(b)
    tot[name] += t
    if t > 0.5:
        short = [x if isinstance(x, (int, float)) else "." for x in args]
        rows.append((t, name, short))
for t, name, short in sorted(rows, key=lambda r: -r[0])[:25]:
    print(f"{t:8.2f} ms  {name:28s} {short}")
print("totals:", {k: round(v, 1) for k, v in tot.most_common(10)})

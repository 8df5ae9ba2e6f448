"""Per-level shape and warm device time of the coarse ND solve (C3 by default)."""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1901_02090_b200 as B
from paper_1901_02090_b200 import fields, _native as nat
from paper_1901_02090_b200.solver import _p, _stream
cid = int(sys.argv[1]) if len(sys.argv) > 1 else 3
if len(sys.argv) > 2:   # merge schedule, e.g. 3,3,3,4
    from paper_1901_02090_b200 import coarse_nd
    coarse_nd.ND_MERGE = [int(v) for v in sys.argv[2].split(",")]
c = fields.CONFIGS[cid]
k = fields.config_field(cid)
g = B.build_grid(c["dim"], c["counts"], c["sizes"])
dec = B.regular_partition(g, c["splits"])
system = B.assemble_system(g, B.Permeability(k), B.Wells(0, g.n_cells - 1))
cfg = B.SolveConfig(tau=c["tau"], scaling=c["scaling"], constraints="adaptive", tol=c["tol"])
st = B.BddcSetup(system, dec, cfg)
tm = {}
st = B.BddcSetup(system, dec, cfg, timings=tm)
nd = st.nd
r = torch.randn(st.nfc + st.N, dtype=torch.float64, device="cuda")
x = torch.zeros_like(r)
ys, cb = nd._bufs()
for _ in range(3):
    nd.solve(r, x)
torch.cuda.synchronize()
R = 50
def timeit(fn):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn(); a.record()
    for _ in range(R):
        fn()
    b.record(); b.synchronize()
    return a.elapsed_time(b) * 1000 / R
print(sys.argv[2:], "levels", len(nd.levels), "whole solve", round(timeit(lambda: nd.solve(r, x)), 1), "us",
      "setup coarse ms", round(tm.get("coarse", 0), 1))
tot_bytes = 0
for li, L in enumerate(nd.levels):
    fwd = lambda L=L, li=li: nat.call("bddc_nd_fwd", L.ysize, L.n_ft, L.smax, _p(L.ftasks), _p(L.info), _p(L.data_off),
                                      _p(L.sep_flat), _p(L.lptr), _p(L.lsrc), _p(L.Fc), _p(r), None, None, 0, _p(nd._rs), _p(ys[li]),
                                      _p(cb), None, _stream())
    bwd = lambda L=L, li=li: nat.call("bddc_nd_bwd", L.n_bt, L.bmax, L.wpr, _p(L.btasks), _p(L.info), _p(L.data_off),
                                      _p(L.sep_flat), _p(L.bnd_flat), _p(L.Fc), _p(ys[li]), _p(x), _stream())
    tf, tb = timeit(fwd), timeit(bwd)
    tot_bytes += 8 * L.csize
    print(f"level {li}: nodes {L.m} sep max {L.smax} bnd max {L.bmax} factor {8 * L.csize / 1e6:.1f} MB "
          f"fwd tasks {L.n_ft} bwd tasks {L.n_bt} wpr {L.wpr}: fwd {tf:.1f} us  bwd {tb:.1f} us")
print(f"factor bytes total {tot_bytes / 1e6:.1f} MB")

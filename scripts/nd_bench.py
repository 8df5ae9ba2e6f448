"""Time the ND coarse solve (whole solve and per level, CUDA-graph replay) on a config (dev tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1901_02090_b200 as B
from paper_1901_02090_b200 import fields, _native as nat
from paper_1901_02090_b200.coarse_nd import _p, _stream
cfgi = int(sys.argv[1]) if len(sys.argv) > 1 else 3
c = fields.CONFIGS[cfgi]
k = fields.config_field(cfgi)
g = B.build_grid(c["dim"], c["counts"], c["sizes"])
dec = B.regular_partition(g, c["splits"])
system = B.assemble_system(g, B.Permeability(k), B.Wells(0, g.n_cells - 1))
cfg = B.SolveConfig(tau=c["tau"], scaling=c["scaling"], constraints="adaptive", tol=c["tol"])
st = B.BddcSetup(system, dec, cfg)
nd = st.nd
r = torch.randn(st.nfc + st.N, dtype=torch.float64, device="cuda")
x = torch.zeros_like(r)


def gtime(fn, reps=50):
    gr = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn()
        torch.cuda.synchronize()
        with torch.cuda.graph(gr, stream=s):
            fn()
    torch.cuda.synchronize()
    for _ in range(3):
        gr.replay()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        gr.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1000


print(f"nd solve (graph) {gtime(lambda: nd.solve(r, x)):.1f} us, factor MB {nd.bytes / 1e6:.1f}")
ys, cb = nd._bufs()
for li, L in enumerate(nd.levels):
    f = lambda: nat.call("bddc_nd_fwd", L.ysize, L.n_ft, L.smax, _p(L.ftasks), _p(L.info), _p(L.data_off),
                         _p(L.sep_flat), _p(L.lptr), _p(L.lsrc), _p(L.Fc), _p(r), None, None, 0, _p(nd._rs), _p(ys[li]), _p(cb), None, _stream())
    b = lambda: nat.call("bddc_nd_bwd", L.n_bt, L.bmax, L.wpr, _p(L.btasks), _p(L.info), _p(L.data_off),
                         _p(L.sep_flat), _p(L.bnd_flat), _p(L.Fc), _p(ys[li]), _p(x), _stream())
    tf = gtime(lambda: [f() for _ in range(10)]) / 10
    tb = gtime(lambda: [b() for _ in range(10)]) / 10
    mb = L.csize * 8 / 1e6
    print(f"level {li:2d} m={L.m:4d} s={L.smax:4d} b={L.bmax:5d} MB={mb:6.2f}: fwd {tf:6.1f} us  bwd {tb:6.1f} us")

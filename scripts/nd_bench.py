"""Time the ND coarse solve (per-level launches vs one persistent kernel) on a config (dev tool)."""
import math, os, sys, time
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
nd = st.nd
r = torch.randn(st.nfc + st.N, dtype=torch.float64, device="cuda")
xs = {}
lib = nat.load()
for mode in ("levels_nopdl", False, True):
    lib.bddc_set_pdl(0 if mode == "levels_nopdl" else 1)
    nd.persistent = mode is True
    x = torch.zeros_like(r)
    nd.solve(r, x, st.d_Pcinv, st.npc)
    torch.cuda.synchronize()
    xs[mode] = x
    gr = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        nd.solve(r, x, st.d_Pcinv, st.npc)
        torch.cuda.synchronize()
        with torch.cuda.graph(gr, stream=s):
            nd.solve(r, x, st.d_Pcinv, st.npc)
    torch.cuda.synchronize()
    for _ in range(3):
        gr.replay()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        gr.replay()
    e1.record()
    torch.cuda.synchronize()
    print(f"persistent={mode}: nd solve graph mean {e0.elapsed_time(e1) / 50 * 1000:.1f} us")
d = (xs[True] - xs[False]).norm() / xs[False].norm()
print("rel diff pdl vs no-pdl", float((xs["levels_nopdl"] - xs[False]).norm() / xs[False].norm()))
print("rel diff persistent vs levels", float(d), "items", nd.p_nitems, "nodes", nd.p_nn, "smem", nd.p_smem,
      "factor MB", nd.bytes / 1e6)


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


from paper_1901_02090_b200.coarse_nd import _p, _stream
tiny = torch.zeros(4, dtype=torch.float64, device="cuda")
print("41 tiny kernels in a graph: %.1f us" % gtime(lambda: [nat.call("bddc_fill", 1, 0.0, _p(tiny), _stream()) for _ in range(41)]))
nd.persistent = False
ys, cb = nd._bufs()
x = torch.zeros_like(r)
for li, L in enumerate(nd.levels):
    f = lambda: nat.call("bddc_nd_fwd", L.ysize, L.n_ft, L.smax, _p(L.ftasks), _p(L.info), _p(L.data_off),
                         _p(L.sep_flat), _p(L.lptr), _p(L.lsrc), _p(L.Fc), _p(r), _p(nd._rs), _p(ys[li]), _p(cb), _stream())
    b = lambda: nat.call("bddc_nd_bwd", L.n_bt, L.bmax, L.wpr, _p(L.btasks), _p(L.info), _p(L.data_off),
                         _p(L.sep_flat), _p(L.bnd_flat), _p(L.Fc), _p(ys[li]), _p(x), _stream())
    f10 = lambda: [f() for _ in range(10)]
    b10 = lambda: [b() for _ in range(10)]
    tf, tb = gtime(f10) / 10, gtime(b10) / 10
    mb = L.csize * 8 / 1e6
    print(f"level {li:2d} m={L.m:4d} s={L.smax:4d} b={L.bmax:5d} MB={mb:6.2f}: fwd(gather+gemv) {tf:6.1f} us  bwd {tb:6.1f} us"
          f"  ({mb * 1e6 / 1e3 / (tf + tb):.0f} GB/s)")

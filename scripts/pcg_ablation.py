"""Attribute the C3 PCG iteration time: capture pieces of the loop body as CUDA
graphs (torch.cuda.graph) and time K replays of each, warm, with CUDA events."""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1901_02090_b200 as B
from paper_1901_02090_b200 import fields, solver as S, _native as nat
from paper_1901_02090_b200.solver import _p, _stream

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 3
c = fields.CONFIGS[cid]
k = fields.config_field(cid)
g = B.build_grid(c["dim"], c["counts"], c["sizes"])
dec = B.regular_partition(g, c["splits"])
system = B.assemble_system(g, B.Permeability(k), B.Wells(0, g.n_cells - 1))
cfg = B.SolveConfig(tau=c["tau"], scaling=c["scaling"], constraints="adaptive" if math.isfinite(c["tau"]) else "initial",
                    tol=c["tol"])
st = B.BddcSetup(system, dec, cfg)
B.solve(system, dec, cfg, setup=st)
W = st.work()
Bf = st._pcg_bufs(cfg.maxit)
ng, N = st.n_gamma, st.N


def chain():
    ss = _stream()
    nat.call("bddc_gather_gemv_t", N, st.maxG, st.maxC, _p(st.d_nG), _p(st.d_nC), _p(st.d_gpos), _p(st.d_Psi),
             _p(W.r), _p(st.d_delta), _p(st.w_v), ss)
    st.nd.solve(None, st.w_xc, restricted=(st.w_v, st.d_cown))


def tgemv():
    st._symv(st.d_Tp, W.r, st.d_delta, st.w_yb, st.t_grid_bulk, 1, _stream())


def tgemv_full():
    st._symv(st.d_Tp, W.r, st.d_delta, st.w_yb, 0, 1, _stream())


def sgemv():
    st._symv(st.d_Sp, W.p, None, st.w_yb, 0, 0, _stream())


def prolong():
    nat.call("bddc_prolong", N, st.maxG, st.maxC, _p(st.d_nG), _p(st.d_nC), _p(st.d_sub_rows), _p(st.d_Psi),
             _p(st.w_xc), _p(st.w_yb), _p(st.d_delta), _p(st.w_yb2), _stream())


def scatter():
    nat.call("bddc_scatter", ng, _p(st.d_gown), _p(st.w_yb2), _p(W.zv), _stream())


def restrict():
    nat.call("bddc_gather_gemv_t", N, st.maxG, st.maxC, _p(st.d_nG), _p(st.d_nC), _p(st.d_gpos), _p(st.d_Psi),
             _p(W.r), _p(st.d_delta), _p(st.w_v), _stream())


pieces = {
    "body": lambda: S._pcg_body(st, W, Bf),
    "schur(S gemv+scatter)": lambda: st._schur(W.p, W.Ap),
    "S gemv": sgemv,
    "project": lambda: st._project(W.Ap),
    "project+dot": lambda: st._project(W.Ap, dot=(W.p, 100 + 15, None)),
    "project+dot (from slots)": lambda: st._project(W.Ap, dot=(W.p, 100 + 15, None), yb=st.w_yb),
    "precond": lambda: st._precond(W.r, W.zv),
    "T gemv (t_grid_bulk)": tgemv,
    "T gemv (all SMs)": tgemv_full,
    "coarse chain": chain,
    "restriction": restrict,
    "nd.solve": st._coarse_solve,
    "prolong": prolong,
    "scatter": scatter,
    "cg_update_dot": lambda: nat.call("bddc_cg_update_dot", ng, _p(W.x), _p(W.p), _p(W.r), _p(W.Ap),
                                      _p(st.w_dot), _p(st.w_scal), 100 + 15, None, _stream()),
    "p_update": lambda: nat.call("bddc_p_update", ng, _p(st.w_scal), _p(W.zv), _p(W.p), _stream()),
}
only = sys.argv[2].split(",") if len(sys.argv) > 2 else None
if only:
    pieces = {k2: v for k2, v in pieces.items() if any(o in k2 for o in only)}
K = 34
flush = torch.empty(32 << 20, dtype=torch.float64, device="cuda")
for name, fn in pieces.items():
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(2):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        for _ in range(K):
            fn()
    gr.replay()
    torch.cuda.synchronize()
    ts = []
    for rep in range(3):
        flush.fill_(rep)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        gr.replay()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1000.0 / K)
    print(f"{name:24s} {min(ts):8.1f} us per call", flush=True)

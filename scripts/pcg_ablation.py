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
    nat.call("bddc_coarse_restrict", st.nfc, _p(st.d_cown), _p(st.w_v), _p(st.w_rc), ss)
    nat.call("bddc_fill", N, 0.0, _p(st.w_rc[st.nfc:]), ss)
    st._coarse_solve()


def tgemv():
    nat.call("bddc_gather_symv", N, st.maxG, _p(st.d_nG), _p(st.d_gpos), _p(st.d_Tp), _p(W.r), _p(st.d_delta),
             _p(st.w_yb), st.t_grid, _stream())


def tgemv_full():
    nat.call("bddc_gather_symv", N, st.maxG, _p(st.d_nG), _p(st.d_gpos), _p(st.d_Tp), _p(W.r), _p(st.d_delta),
             _p(st.w_yb), 0, _stream())


def prolong():
    nat.call("bddc_prolong", N, st.maxG, st.maxC, _p(st.d_nG), _p(st.d_nC), _p(st.d_sub_rows), _p(st.d_Psi),
             _p(st.w_xc), _p(st.w_yb), _p(st.d_delta), _p(st.w_yb2), _stream())


def scatter():
    nat.call("bddc_scatter", ng, _p(st.d_gown), _p(st.w_yb2), _p(W.zv), _stream())


def phi():
    nat.call("bddc_phi", N, st.maxG, _p(st.d_nG), _p(st.d_gpos), _p(st.d_gcode), _p(W.zv), _p(st.w_phi), _stream())


def gemv():
    nat.call("bddc_gemv", N, N, N, _p(st.d_Lp), _p(st.w_phi), _p(st.w_z), _stream())


def proj_apply():
    nat.call("bddc_proj_apply", ng, st.maxG, _p(st.d_gown), _p(st.w_z), _p(W.zv), _stream())


def dots_updates():
    S._dot(st, W.p, W.Ap, ng, 1, Bf.alphas)
    nat.call("bddc_cg_update", ng, _p(st.w_scal), _p(W.x), _p(W.p), _p(W.r), _p(W.Ap), _stream())
    S._dot(st, W.r, W.r, ng, 2, Bf.res)
    S._dot(st, W.r, W.zv, ng, 3, Bf.betas)
    nat.call("bddc_p_update", ng, _p(st.w_scal), _p(W.zv), _p(W.p), _stream())


def one_dot():
    S._dot(st, W.r, W.r, ng, 100 + 12)


pieces = {
    "body": lambda: S._pcg_body(st, W, Bf),
    "schur(S gemv+scatter)": lambda: st._schur(W.p, W.Ap),
    "project": lambda: st._project(W.Ap),
    "precond": lambda: st._precond(W.r, W.zv),
    "T gemv (t_grid)": tgemv,
    "T gemv (grid N)": tgemv_full,
    "coarse chain": chain,
    "nd.solve": st._coarse_solve,
    "prolong": prolong,
    "scatter": scatter,
    "phi": phi,
    "gemv Lp": gemv,
    "proj_apply": proj_apply,
    "dots+updates": dots_updates,
    "one dot": one_dot,
}
def with_tgrid(tg):
    def f():
        old = st.t_grid
        st.t_grid = tg
        st._precond(W.r, W.zv)
        st.t_grid = old
    return f


def prolong_staged():
    nat.load().bddc_set_prolong_direct(0)
    prolong()
    nat.load().bddc_set_prolong_direct(1)


pieces["prolong staged"] = prolong_staged
only = sys.argv[2].split(",") if len(sys.argv) > 2 else None
def body_tgrid(tg):
    def f():
        old = st.t_grid
        st.t_grid = tg
        S._pcg_body(st, W, Bf)
        st.t_grid = old
    return f


for tg in (0, 148, 296, 444, 592):
    pieces[f"precond t_grid={tg}"] = with_tgrid(tg)
    pieces[f"body t_grid={tg}"] = body_tgrid(tg)
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

"""Graph-replay timing of the preconditioner pieces on config 3 (dev tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1901_02090_b200 as B
from paper_1901_02090_b200 import fields, _native as nat
from paper_1901_02090_b200.solver import _p, _stream
CFG = int(os.environ.get("CFG", "3"))
c = fields.CONFIGS[CFG]
k = fields.config_field(CFG)
g = B.build_grid(c["dim"], c["counts"], c["sizes"])
dec = B.regular_partition(g, c["splits"])
system = B.assemble_system(g, B.Permeability(k), B.Wells(0, g.n_cells - 1))
cfg = B.SolveConfig(tau=c["tau"], scaling=c["scaling"], constraints="adaptive", tol=c["tol"])
st = B.BddcSetup(system, dec, cfg)
st.nd._bufs()
r = torch.randn(st.n_gamma, dtype=torch.float64, device="cuda")
out = torch.empty_like(r)


def T_only():
    nat.call("bddc_gather_symv", st.N, st.maxG, _p(st.d_nG), _p(st.d_gpos), _p(st.d_Tp), _p(r),
             _p(st.d_delta), _p(st.w_yb), 0, _stream())


def coarse_only():
    s = _stream()
    nat.call("bddc_gather_gemv_t", st.N, st.maxG, st.maxC, _p(st.d_nG), _p(st.d_nC), _p(st.d_gpos),
             _p(st.d_Psi), _p(r), _p(st.d_delta), _p(st.w_v), s)
    nat.call("bddc_coarse_restrict", st.nfc, _p(st.d_cown), _p(st.w_v), _p(st.w_rc), s)
    nat.call("bddc_fill", st.N, 0.0, _p(st.w_rc[st.nfc:]), s)
    st._coarse_solve()


def nd_only():
    st._coarse_solve()


def full():
    st._precond(r, out)


def schur():
    st._schur(r, out)


def project():
    st._project(out)


def gemv_t():
    nat.call("bddc_gather_gemv_t", st.N, st.maxG, st.maxC, _p(st.d_nG), _p(st.d_nC), _p(st.d_gpos),
             _p(st.d_Psi), _p(r), _p(st.d_delta), _p(st.w_v), _stream())


def prolong():
    nat.call("bddc_prolong", st.N, st.maxG, st.maxC, _p(st.d_nG), _p(st.d_nC), _p(st.d_sub_rows),
             _p(st.d_Psi), _p(st.w_xc), _p(st.w_yb), _p(st.d_delta), _p(st.w_yb2), _stream())


def lap():
    S3 = dec.S3
    nat.call("bddc_lap_solve", S3[0], S3[1], S3[2], _p(st.d_eig_u), None, _p(st.w_phi), _p(st.w_z), _stream())


import numpy as np
nC = st.nC if hasattr(st, "nC") else None
psi_bytes = float(np.sum(np.asarray(st.nC, dtype=np.float64) * dec.nG)) * 8
print(f"PsiT live bytes {psi_bytes/1e6:.1f} MB (maxC={st.maxC}, mean nC={np.mean(st.nC):.1f})")
for name, fn in [("gemv_t", gemv_t), ("prolong", prolong), ("lap_solve", lap), ("T_symv", T_only), ("coarse_chain", coarse_only), ("nd_solve", nd_only),
                 ("precond", full), ("schur", schur), ("project", project)]:
    s = torch.cuda.Stream()
    gr = torch.cuda.CUDAGraph()
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
    for _ in range(50):
        gr.replay()
    e1.record()
    torch.cuda.synchronize()
    print(f"{name:14s} {e0.elapsed_time(e1) / 50 * 1000:8.1f} us")


for mult in (1, 2, 3, 0):
    st.t_grid = st.n_sm * mult
    s = torch.cuda.Stream()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        full()
        torch.cuda.synchronize()
        with torch.cuda.graph(gr, stream=s):
            full()
    torch.cuda.synchronize()
    for _ in range(3):
        gr.replay()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        gr.replay()
    e1.record()
    torch.cuda.synchronize()
    print(f"T grid {st.t_grid:5d}: precond {e0.elapsed_time(e1) / 50 * 1000:7.1f} us")


def gt(fn, reps=50):
    s = torch.cuda.Stream()
    gr = torch.cuda.CUDAGraph()
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


def forked(first_side=True, tgrid=0):
    def fn():
        main = torch.cuda.current_stream()
        side = st.side_stream
        f = torch.cuda.Event()
        f.record(main)
        side.wait_event(f)
        def do_side():
            with torch.cuda.stream(side):
                nd_only()
                j = torch.cuda.Event()
                j.record(side)
            return j
        if first_side:
            j = do_side()
        nat.call("bddc_gather_symv", st.N, st.maxG, _p(st.d_nG), _p(st.d_gpos), _p(st.d_Tp), _p(r),
                 _p(st.d_delta), _p(st.w_yb), tgrid, _stream())
        if not first_side:
            j = do_side()
        main.wait_event(j)
    return fn


print("T only %.1f, nd only %.1f, T then nd %.1f" % (gt(T_only), gt(nd_only), gt(lambda: (T_only(), nd_only()))))
for fs in (True, False):
    for tg in (148, 296, 0):
        print(f"forked side_first={fs} tgrid={tg}: {gt(forked(fs, tg)):.1f} us")

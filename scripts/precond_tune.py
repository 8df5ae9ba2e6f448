"""Preconditioner apply time (warm CUDA-graph replays) over the concurrency knobs:
the Psi^T restriction before the fork or beside T, and the T_i GEMV grid.
argv[1] = config (3, 4)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1901_02090_b200 as B
from paper_1901_02090_b200 import fields

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 3
if os.environ.get("SYMV_GROUPS"):   # subdomains per CTA of the grid-stride LDG GEMV
    from paper_1901_02090_b200 import _native as _nat
    _nat.load().bddc_set_symv_groups(int(os.environ["SYMV_GROUPS"]))
c = fields.CONFIGS[cid]
g = B.build_grid(3, c["counts"], c["sizes"])
dec = B.regular_partition(g, c["splits"])
system = B.assemble_system(g, B.Permeability(fields.config_field(cid)), B.Wells(0, g.n_cells - 1))
cfg = B.SolveConfig(tau=c["tau"], scaling=c["scaling"], constraints=c["constraints"], tol=c["tol"])
st = B.BddcSetup(system, dec, cfg)
B.solve(system, dec, cfg, setup=st)
W = st.work()
r = torch.randn(st.n_gamma, dtype=torch.float64, device="cuda")
K = 20


def timeit(fn):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        for _ in range(K):
            fn()
    gr.replay()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        gr.replay()
        b.record()
        b.synchronize()
        best = min(best, a.elapsed_time(b) * 1000.0 / K)
    return best


grids = [0, 444, 296, 148, 120, 100, 84]
if os.environ.get("T_GRIDS"):   # e.g. T_GRIDS=88,92,96,100,104,108 for a fine scan
    grids = [int(v) for v in os.environ["T_GRIDS"].split(",")]
print(f"config {cid}: symv_bulk {st.symv_bulk}", flush=True)
for rf in ((False,) if os.environ.get("T_GRIDS") else (False, True)):
    st.restrict_first = rf
    for tg in grids:
        st.t_grid_bulk = tg
        st.t_grid = tg
        t = timeit(lambda: st._precond(r, W.zv))
        print(f"restrict_first {rf:d} T grid {tg:3d}: precond {t:7.1f} us",
              flush=True)

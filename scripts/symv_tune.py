"""Bulk-streamed vs LDG symmetric GEMV at C3: equality, single-launch time, and
PCG-only it/s of whole solves over the T-GEMV grid (the coarse chain runs beside it)."""
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1901_02090_b200 as B                      # noqa: E402
from paper_1901_02090_b200 import fields               # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 3
c = fields.CONFIGS[cid]
g = B.build_grid(c["dim"], c["counts"], c["sizes"])
dec = B.regular_partition(g, c["splits"])
system = B.assemble_system(g, B.Permeability(fields.config_field(cid)), B.Wells(0, g.n_cells - 1))
cfg = B.SolveConfig(tau=c["tau"], scaling=c["scaling"], constraints=c["constraints"], tol=c["tol"])
st = B.BddcSetup(system, dec, cfg)
x = np.random.default_rng(0).standard_normal(dec.n_gamma)
st.symv_bulk = False
y0 = st.schur_matvec(x)
m0 = st.precondition(x)
st.symv_bulk = True
y1 = st.schur_matvec(x)
m1 = st.precondition(x)
print("S x bulk vs ldg rel", np.linalg.norm(y1 - y0) / np.linalg.norm(y0),
      "M x rel", np.linalg.norm(m1 - m0) / np.linalg.norm(m0), flush=True)
y2 = st.schur_matvec(x)
print("bulk repeat bitwise", np.array_equal(y1, y2))
alg = 8.0 * sum(int(n) * (int(n) + 1) / 2 for n in dec.nG)
for mode in (False, True):
    st.symv_bulk = mode
    t = st.time_kernel("S", reps=50)
    print(f"S gemv bulk={mode}: {t * 1e6:.1f} us  {alg / t / 1e9:.0f} GB/s (algorithmic)", flush=True)


def pcg_rate(reps=6):
    st._drop_graphs()
    B.solve(system, dec, cfg, setup=st)
    st.pcg_timer = []
    its = 0
    for _ in range(reps):
        its += B.solve(system, dec, cfg, setup=st).it
    torch.cuda.synchronize()
    s = sum(a.elapsed_time(b) for a, b in st.pcg_timer) / 1000.0
    st.pcg_timer = None
    return its / s


for rf in (False, True):
    st.restrict_first = rf
    for tg in (148, 136, 124, 112, 100, 92, 84, 76):
        st.t_grid_bulk = tg
        print(f"restrict_first={rf} t_grid={tg}: PCG {pcg_rate():.0f} it/s", flush=True)

"""local_solve_kernel alone at a BASELINE config: one-rhs and two-rhs passes over the
packed Q, mean launch time and GB/s (A/B builds through BDDC_LIB)."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1901_02090_b200 as B
from paper_1901_02090_b200 import _native as nat, fields

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 3
c = fields.CONFIGS[cid]
g = B.build_grid(c["dim"], c["counts"], c["sizes"])
dec = B.regular_partition(g, c["splits"])
system = B.assemble_system(g, B.Permeability(fields.config_field(cid)), B.Wells(0, g.n_cells - 1))
cfg = B.SolveConfig(tau=float("inf"), scaling=c["scaling"], constraints="initial", tol=c["tol"])
st = B.BddcSetup(system, dec, cfg)
W = st.work()
p = nat.ptr
gp = C.byref(st.geom)
stream = C.c_void_p(torch.cuda.current_stream().cuda_stream)
x = torch.randn(st.n_gamma, dtype=torch.float64, device="cuda")
fc = torch.randn(st.geom.n_cells, dtype=torch.float64, device="cuda")
nt = st.maxP // 32
qbytes = st.N * (nt * (nt + 1) // 2) * 8192
for two in (False, True):
    a = nat.LocalSolveArgs()
    a.x_gamma, a.x_scale = p(x).value, 1.0
    a.u_out, a.u_mode = p(W.u0).value, 0
    if two:
        a.g_cell2, a.g_scale2 = p(fc).value, 1.0
        a.u_out2 = p(W.us).value
    def run():
        nat.call("bddc_local_solve", gp, p(st.d_coef), p(st.d_gcode), p(st.d_gpos), p(st.d_fslot),
                 p(st.d_Qp), p(st.d_Dsub), C.byref(a), stream)
    for _ in range(3):
        run()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        run()
    e1.record()
    e1.synchronize()
    us = e0.elapsed_time(e1) * 1000 / 20
    print(f"{os.environ.get('BDDC_LIB', 'default')}: two={two} {us:.1f} us  Q {qbytes / us / 1e3:.0f} GB/s", flush=True)
    lib = nat.load()
    if hasattr(lib, "bddc_ls_timing_read"):   # -DLS_TIMING build: mean cycles per CTA and phase
        buf = (C.c_ulonglong * 8)()
        lib.bddc_ls_timing_read(buf, 1)
        n = 23 * st.N
        print("  phase cycles per CTA [prologue, lines1, rhs, symv, lines2, epilogue]:",
              [round(buf[k] / n) for k in range(5)], flush=True)

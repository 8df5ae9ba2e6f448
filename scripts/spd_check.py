"""Check the batched SPD inverse on the matrices a real setup produces (debug tool)."""
import ctypes as C, os, sys, math
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import paper_1901_02090_b200 as B
from paper_1901_02090_b200 import _native as nat, solver as SV
import _golden as GD
lib = nat.load()
name = sys.argv[1] if len(sys.argv) > 1 else "c2_tau10"
d = GD.load(name)
g = B.build_grid(len(d["counts"]), d["counts"], d["sizes"])
system = B.assemble_system(g, B.Permeability(d["k"]), B.Wells(0, g.n_cells - 1))
dec = B.regular_partition(g, d["splits"])
G = SV._geom(dec); gp = C.byref(G)
dev = torch.device("cuda"); st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
t = lambda a, dt=torch.int32: torch.as_tensor(np.ascontiguousarray(a), dtype=dt, device=dev)
N, mg, mp = dec.n_subdomains, dec.maxG, dec.maxP
k = torch.as_tensor(d["k"], device=dev); coef = torch.empty(G.n_cells * 3, dtype=torch.float64, device=dev)
nat.call("bddc_cell_coeffs", gp, nat.ptr(k), nat.ptr(coef), st)
fslot = t(dec.fslot); gcode = t(dec.gcode)
P = torch.empty(N * mp * mp, dtype=torch.float64, device=dev)
Gc = torch.empty(N * mg * dec.maxL, dtype=torch.float64, device=dev)
SAd = torch.empty(N * mg, dtype=torch.float64, device=dev); SApart = torch.empty(N * mg, dtype=torch.int32, device=dev)
SAoff = torch.empty(N * mg, dtype=torch.float64, device=dev); alpha = torch.empty(N, dtype=torch.float64, device=dev)
nat.call("bddc_local_build", gp, nat.ptr(coef), nat.ptr(fslot), nat.ptr(P), nat.ptr(Gc), nat.ptr(SAd), nat.ptr(SApart), nat.ptr(SAoff), nat.ptr(alpha), st)
P0 = P.clone().view(N, mp, mp)
for b in (64, 32):
    Pm = P0.clone()
    ws = torch.empty(lib.bddc_spd_inverse_workspace(mp, N, b) // 8 + 2, dtype=torch.float64, device=dev)
    info = torch.zeros(1, dtype=torch.int32, device=dev)
    nat.call("bddc_spd_inverse_batched", nat.ptr(Pm), mp, mp, mp * mp, N, b, nat.ptr(ws), nat.ptr(info), st)
    ref = torch.linalg.inv(P0)
    err = ((Pm - ref).abs().amax(dim=(1, 2)) / ref.abs().amax(dim=(1, 2)))
    print(name, "P", mp, "b", b, "info", int(info.item()), "max rel err", float(err.max()), "argmax", int(err.argmax()),
          "sym err", float((P0 - P0.transpose(1, 2)).abs().max()), "nan", bool(torch.isnan(Pm).any()))

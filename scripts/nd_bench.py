"""Time the ND coarse solve levels standalone (dev tool)."""
import math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1901_02090_b200 as B
from paper_1901_02090_b200 import fields, _native as nat
c = fields.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 3]
k = fields.config_field(3 if len(sys.argv) < 2 else int(sys.argv[1]))
g = B.build_grid(c["dim"], c["counts"], c["sizes"])
dec = B.regular_partition(g, c["splits"])
system = B.assemble_system(g, B.Permeability(k), B.Wells(0, g.n_cells - 1))
cfg = B.SolveConfig(tau=c["tau"], scaling=c["scaling"], constraints="adaptive", tol=c["tol"])
st = B.BddcSetup(system, dec, cfg)
nd = st.nd
r = torch.randn(st.nfc + st.N, dtype=torch.float64, device="cuda")
x = torch.empty_like(r)
nd.solve(r, x, st.d_Pcinv, st.npc)
torch.cuda.synchronize()
for L in nd.levels:
    print(f"level m={L.m:5d} smax={L.smax:5d} bmax={L.bmax:5d} compact MB={L.csize*8/1e6:8.2f} tasks={L.n_ft}/{L.n_bt} lsrc={L.lsrc.numel()}")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(50):
    nd.solve(r, x, st.d_Pcinv, st.npc)
e1.record(); torch.cuda.synchronize()
print("nd solve mean ms", e0.elapsed_time(e1) / 50, "factor MB", nd.bytes / 1e6)
nat.profile_start()
nd.solve(r, x, st.d_Pcinv, st.npc)
prof = nat.profile_stop()
for n, (cnt, t) in prof.items():
    print(n, cnt, round(t, 3), "ms")
# device time inside a CUDA graph (no host launch overhead)
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    nd.solve(r, x, st.d_Pcinv, st.npc)
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        nd.solve(r, x, st.d_Pcinv, st.npc)
torch.cuda.synchronize()
e0.record()
for _ in range(50):
    g.replay()
e1.record(); torch.cuda.synchronize()
print("nd solve graph mean ms", e0.elapsed_time(e1) / 50)

"""Every batched SPD inverse of one real setup, timed in place (bddc_spd_log_*), plus
the setup's device time; argv[1] = config (default 3)."""
import ctypes as C, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1901_02090_b200 as B
from paper_1901_02090_b200 import fields, _native as nat

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 3
c = fields.CONFIGS[cid]
g = B.build_grid(c["dim"], c["counts"], c["sizes"])
dec = B.regular_partition(g, c["splits"])
system = B.assemble_system(g, B.Permeability(fields.config_field(cid)), B.Wells(0, g.n_cells - 1))
cfg = B.SolveConfig(tau=c["tau"], scaling=c["scaling"], constraints=c["constraints"], tol=c["tol"])
lib = nat.load()
B.BddcSetup(system, dec, cfg)
for rep in range(2):
    tm = {}
    lib.bddc_spd_log_enable(1)
    st = B.BddcSetup(system, dec, cfg, timings=tm)
    torch.cuda.synchronize()
    buf = np.zeros(1024)
    n = lib.bddc_spd_log_read(buf.ctypes.data_as(C.c_void_p), 256)
    lib.bddc_spd_log_enable(0)
    print(f"setup {tm.get('total', 0):.1f} ms; phases", {k: round(v, 1) for k, v in tm.items()})
    for nn, bt, fl, ms in buf[:4 * n].reshape(-1, 4):
        print(f"  {int(bt):5d} x {int(nn):5d} flags {int(fl)}: {ms:8.3f} ms  {bt * nn ** 3 / ms / 1e9:6.2f} TF/s")
nC = np.asarray(st.nC)
print("nC: max", nC.max(), "mean", nC.mean(), "count > 64:", int((nC > 64).sum()), "> 32:", int((nC > 32).sum()))

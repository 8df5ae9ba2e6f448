"""Run one BASELINE config end to end on the GPU and print timings (dev tool)."""
import argparse, math, sys, time, os
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1901_02090_b200 as B
from paper_1901_02090_b200 import fields

ap = argparse.ArgumentParser()
ap.add_argument("cfg", type=int)
ap.add_argument("--scaling", default=None)
ap.add_argument("--tau", type=float, default=None)
ap.add_argument("--tol", type=float, default=None)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--bc", default="A", choices=["A", "B"])
a = ap.parse_args()
c = dict(fields.CONFIGS[a.cfg])
t = time.time(); k = fields.config_field(a.cfg); tk = time.time() - t
g = B.build_grid(c["dim"], c["counts"], c["sizes"])
t = time.time(); dec = B.regular_partition(g, c["splits"]); td = time.time() - t
system = B.assemble_system(g, B.Permeability(k), B.Wells(0, g.n_cells - 1) if a.bc == "A"
                           else B.PressureDrop(1, 1.0, 0.0))
tau = a.tau if a.tau is not None else c["tau"]
cfg = B.SolveConfig(tau=tau, scaling=a.scaling or c["scaling"],
                    constraints="adaptive" if math.isfinite(tau) else c["constraints"],
                    tol=a.tol or c["tol"], maxit=5000)
print(f"cfg {a.cfg}: field {tk:.2f}s topo {td:.2f}s N={dec.n_subdomains} n_gamma={dec.n_gamma} maxG={dec.maxG} maxP={dec.maxP}", flush=True)
for rep in range(a.reps):
    tm = {}
    torch.cuda.synchronize(); t = time.time()
    st = B.BddcSetup(system, dec, cfg, timings=tm)
    torch.cuda.synchronize(); ts = time.time() - t
    print(f"setup {ts:.3f}s  phases(ms): " + " ".join(f"{k}={v:.1f}" for k, v in tm.items()), flush=True)
    print(f"  n_c={st.n_c} nfc={st.nfc} maxC={st.maxC} omega={st.omega_tilde} mem={torch.cuda.max_memory_allocated()/1e9:.1f}GB", flush=True)
    for rr in range(3):
        t = time.time()
        r = B.solve(system, dec, cfg, setup=st)
        torch.cuda.synchronize(); tsol = time.time() - t
        print(f"  solve[{rr}] {tsol:.3f}s it={r.it} kappa={r.kappa:.4f} it/s={r.it/tsol:.1f} cons={r.conservation_defect:.2e} pw={r.pressure_warning}", flush=True)
    del st
    torch.cuda.empty_cache()
if a.bc == "B":
    res = system.A @ r.u + system.B.T @ r.p - system.g
    print(f"mode B residuals: momentum {np.linalg.norm(res) / np.linalg.norm(system.A @ r.u):.2e} "
          f"mass {np.abs(system.B @ r.u).max() / np.abs(r.u).max():.2e} p in [{r.p.min():.4f}, {r.p.max():.4f}] "
          f"outflow {r.u[-g.n_boundary_faces(1):].sum():.6e} inflow {r.u[g.n_flux_dofs:g.n_flux_dofs + g.n_boundary_faces(1)].sum():.6e}", flush=True)
# per-call device-time breakdown of one setup + one solve
from paper_1901_02090_b200 import _native as nat
nat.profile_start()
st = B.BddcSetup(system, dec, cfg)
prof_setup = nat.profile_stop()
st.force_eager = True
r = B.solve(system, dec, cfg, setup=st)
nat.profile_start()
r = B.solve(system, dec, cfg, setup=st)
prof_solve = nat.profile_stop()
for title, prof in (("SETUP", prof_setup), ("SOLVE", prof_solve)):
    tot = sum(t for _, t in prof.values())
    print(f"{title} total {tot:.1f} ms")
    for name, (cnt, t) in sorted(prof.items(), key=lambda kv: -kv[1][1])[:14]:
        print(f"   {name:28s} calls={cnt:5d} total={t:9.2f} ms  mean={t/cnt:8.3f} ms")

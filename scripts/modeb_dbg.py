import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bddc_oracle as O
import paper_1901_02090_b200 as B
def run_a(counts, sizes, splits, cons="initial", tau=float("inf"), scaling="multiplicity"):
    g = B.build_grid(len(counts), counts, sizes)
    k = np.ones((g.n_cells, len(counts)))
    sy = B.assemble_system(g, B.Permeability(k), B.Wells(0, g.n_cells - 1))
    dec = B.regular_partition(g, splits)
    cfg = B.SolveConfig(tau=tau, scaling=scaling, constraints=cons, tol=1e-12)
    r = B.solve(sy, dec, cfg)
    u_ref, p_ref = O.direct_solve(O.Mesh(counts, sizes), k, sy.f)
    print("modeA", counts, splits, "it", r.it, "ru", np.linalg.norm(r.u - u_ref) / np.linalg.norm(u_ref))
def run(counts, sizes, splits, axis, cons, tau, scaling, std, seed=1):
    rng = np.random.default_rng(seed)
    k = 10.0 ** (std * rng.standard_normal((int(np.prod(counts)), len(counts))))
    g = B.build_grid(len(counts), counts, sizes)
    sy = B.assemble_system(g, B.Permeability(k), B.PressureDrop(axis, 1.0, 0.0))
    dec = B.regular_partition(g, splits)
    cfg = B.SolveConfig(tau=tau, scaling=scaling, constraints=cons, tol=1e-12)
    try:
        r = B.solve(sy, dec, cfg)
    except Exception as e:
        print("EXC", counts, splits, axis, e); return
    u_ref, p_ref = O.direct_solve_dirichlet(O.Mesh(counts, sizes), k, np.zeros(g.n_cells), axis, 1.0, 0.0)
    du = sy.B @ r.u_star
    sub = dec.cell_sub
    per = np.bincount(sub, weights=np.abs(du), minlength=dec.n_subdomains)
    print(counts, splits, axis, cons, scaling, std, "it", r.it, "defect", r.conservation_defect,
          "ru", np.linalg.norm(r.u - u_ref) / np.linalg.norm(u_ref), "rp", np.linalg.norm(r.p - p_ref) / np.linalg.norm(p_ref))
    print("   |Bu*| per sub", np.round(per, 6))
for sp in [(1, 4, 1), (2, 4, 1), (1, 4, 2), (2, 2, 2)]:
    try:
        run_a((12, 20, 6), (1.0, 1.0, 1.0), sp)
    except Exception as e:
        print("modeA EXC", sp, e)
for args in [((12, 20, 6), (20.0, 10.0, 2.0), (2, 4, 2), 1, "initial", float("inf"), "multiplicity", 0.0),
             ((12, 20, 6), (1.0, 1.0, 1.0), (2, 4, 2), 1, "initial", float("inf"), "multiplicity", 0.0),
             ((12, 20, 6), (1.0, 1.0, 1.0), (1, 4, 1), 1, "initial", float("inf"), "multiplicity", 0.0),
             ((12, 20, 6), (1.0, 1.0, 1.0), (2, 1, 1), 1, "initial", float("inf"), "multiplicity", 0.0),
             ((12, 20, 6), (1.0, 1.0, 1.0), (1, 1, 1), 1, "initial", float("inf"), "multiplicity", 0.0),
             ((12, 20, 6), (1.0, 1.0, 1.0), (1, 1, 1), 0, "initial", float("inf"), "multiplicity", 0.0),
             ((12, 20, 6), (1.0, 1.0, 1.0), (1, 1, 1), 2, "initial", float("inf"), "multiplicity", 0.0),
             ((12, 20), (1.0, 1.0), (1, 1), 1, "initial", float("inf"), "multiplicity", 0.0),
             ((12, 20), (1.0, 1.0), (1, 4), 1, "initial", float("inf"), "multiplicity", 0.0),
             ((12, 20, 6), (1.0, 1.0, 1.0), (2, 4, 1), 1, "initial", float("inf"), "multiplicity", 0.0),
             ((12, 20, 6), (1.0, 1.0, 1.0), (1, 4, 2), 1, "initial", float("inf"), "multiplicity", 0.0),
             ((12, 20, 6), (1.0, 1.0, 1.0), (2, 2, 2), 1, "initial", float("inf"), "multiplicity", 0.0),
             ]:
    run(*args)

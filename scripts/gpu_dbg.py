import sys, time, math, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import _golden as GD
import paper_1901_02090_b200 as B
names = [a for a in sys.argv[1:] if not a.startswith("--")] or ['g2d_small']
for name in names:
    d = GD.load(name)
    g = B.build_grid(len(d['counts']), d['counts'], d['sizes'])
    perm = B.Permeability(d['k'])
    sysm = B.assemble_system(g, perm, B.Wells(0, g.n_cells-1))
    dec = B.regular_partition(g, d['splits'])
    cfg = B.SolveConfig(tau=d['tau'], scaling=d['scaling'], constraints=d['mode'], tol=d['tol'])
    tm = {}
    t=time.time(); st = B.BddcSetup(sysm, dec, cfg, timings=tm); torch.cuda.synchronize(); t1=time.time()-t
    S0 = st.schur_dense(0)
    print(name, 'setup %.3fs'%t1, {k: round(v,2) for k,v in tm.items()})
    print('  S0 rel', GD.rel(S0, d['S_sub0']), 'Slast', GD.rel(st.schur_dense(dec.n_subdomains-1), d['S_sublast']))
    print('  Px', GD.rel(st.project_balanced(d['x']), d['Px']), 'Sx', GD.rel(st.schur_matvec(d['x']), d['Sx']))
    print('  n_c', st.n_c, int(d['n_c']), 'omega', st.omega_tilde, float(d['omega_tilde']))
    if 'pair_selected' in d:
        print('  selected eq', np.array_equal(st.pair_selected, d['pair_selected']), 'faces rows eq', np.array_equal(st.pair_added+1, d['face_rows']))
        lam = st.pair_lambda.cpu().numpy()
        k = min(lam.shape[1], d['pair_lam'].shape[1])
        ref = d['pair_lam'][:, :k]; mine = lam[:, :k]
        m = np.isfinite(ref) & np.isfinite(mine) & (ref > 1e-8*np.nanmax(ref))
        print('  lam maxrel', np.max(np.abs(mine[m]-ref[m])/ref[m]))
    print('  Mx', GD.rel(st.precondition(d['x']), d['Mx']))
    t=time.time(); rep = B.solve(sysm, dec, cfg, setup=st); t2=time.time()-t
    print('  it', rep.it, int(d['it']), 'kappa', rep.kappa, float(d['kappa']), 'u', GD.rel(rep.u, d['u']), 'p', GD.rel(rep.p, d['p']), 'u0', GD.rel(rep.u0, d['u0']), 'us', GD.rel(rep.u_star, d['u_star']), 'solve %.3fs'%t2, 'pw', rep.pressure_warning)
    if '--hist' in sys.argv or True:
        h = d['residuals']; m = rep.residuals
        n = min(len(h), len(m))
        print('  hist tail ref', np.array2string(h[-4:], precision=3), 'mine', np.array2string(m[-4:], precision=3))

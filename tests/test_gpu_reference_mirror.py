"""GPU-path counterparts of the reference's own unit tests (test_solver.py,
test_adaptive.py, test_coarse.py in /root/reference/pkg/tests), same problems and
assertions where the public API exposes the quantity."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _problem(seed, counts=(16, 14), splits=(2, 2), orders=4.0):
    import paper_1901_02090_b200 as B
    g = B.build_grid(len(counts), counts, (1.0,) * len(counts))
    rng = np.random.default_rng(seed)
    k = 10.0 ** rng.uniform(-orders / 2, orders / 2, g.n_cells)
    perm = B.Permeability.isotropic(g, k)
    system = B.assemble_system(g, perm, B.Wells(0, g.n_cells - 1))
    dec = B.regular_partition(g, splits)
    return B, g, system, dec


def test_aligned_jump_warning_suggests_stiffness():
    """test_solver.py:154-162: checkerboard of subdomain-aligned jumps."""
    import paper_1901_02090_b200 as B
    g = B.build_grid(2, (8, 8), (1.0, 1.0))
    dec = B.regular_partition(g, (2, 2))
    sx, sy = dec.part % 2, dec.part // 2
    k = np.where((sx + sy) % 2 == 0, 1.0, 1e6)
    system = B.assemble_system(g, B.Permeability.isotropic(g, k), B.Wells(0, g.n_cells - 1))
    with pytest.warns(UserWarning, match="stiffness"):
        B.solve(system, dec, B.SolveConfig(scaling="multiplicity"))


def test_residual_history_and_pressure_recovery():
    """test_solver.py:126-151: history starts at 1 and ends below tol, no
    pressure warning, zero-mean pressure."""
    B, g, system, dec = _problem(9)
    rep = B.solve(system, dec, B.SolveConfig(tol=1e-10))
    assert rep.residuals[0] == 1.0
    assert rep.residuals[-1] <= 1e-10
    assert len(rep.residuals) == rep.it + 1
    assert not rep.pressure_warning
    assert abs(rep.p.mean()) <= 1e-12 * max(np.abs(rep.p).max(), 1.0)


def test_homogeneous_field_needs_no_constraints():
    """test_adaptive.py:51-60: k = 1, tau = 10: nothing selected, omega <= tau."""
    import paper_1901_02090_b200 as B
    g = B.build_grid(2, (16, 14), (1.0, 1.0))
    system = B.assemble_system(g, B.Permeability.isotropic(g, 1.0), B.Wells(0, g.n_cells - 1))
    dec = B.regular_partition(g, (2, 2))
    st = B.BddcSetup(system, dec, B.SolveConfig(constraints="adaptive", tau=10.0))
    assert st.omega_tilde <= 10.0
    assert int(st.pair_added.sum()) == 0
    assert st.n_flux_coarse == dec.n_faces


@pytest.mark.parametrize("scaling", ["multiplicity", "stiffness"])
@pytest.mark.parametrize("tau", [100.0, 10.0, 3.0])
def test_post_augmentation_bound(scaling, tau):
    """test_adaptive.py:63-69: after augmentation every pair's next eigenvalue,
    hence omega_tilde, is at most tau."""
    B, g, system, dec = _problem(5)
    st = B.BddcSetup(system, dec, B.SolveConfig(scaling=scaling, constraints="adaptive", tau=tau))
    assert st.omega_tilde <= tau * (1.0 + 1e-8)
    assert np.all(st.face_omega <= tau * (1.0 + 1e-8))


def test_more_constraints_for_smaller_tau():
    """test_adaptive.py:94-99."""
    ncs = []
    for tau in (100.0, 10.0, 3.0):
        B, g, system, dec = _problem(8)
        st = B.BddcSetup(system, dec, B.SolveConfig(constraints="adaptive", tau=tau))
        ncs.append(st.n_flux_coarse)
    assert ncs[0] <= ncs[1] <= ncs[2]


def test_eigenvalues_nonnegative_sorted():
    """test_adaptive.py:42-48 on the eigs-report spectra."""
    B, g, system, dec = _problem(3)
    reports = B.eigs_report(system, dec, B.SolveConfig(constraints="adaptive", tau=10.0))
    assert reports
    for rep in reports.values():
        lam = np.asarray(rep.eigenvalues)
        assert np.all(lam >= 0.0)
        assert np.all(np.diff(lam) <= 1e-9 * max(lam[0], 1.0))


def test_indicator_floor_and_max():
    """test_adaptive.py:85-91: omega_tilde = max(1, max over pairs)."""
    B, g, system, dec = _problem(7)
    st = B.BddcSetup(system, dec, B.SolveConfig(constraints="adaptive", tau=math.inf))
    assert st.omega_tilde >= 1.0
    assert st.omega_tilde == max(float(st.face_omega.max()), 1.0)


def test_coarse_counts_2x7():
    """test_coarse.py:23-29: initial constraints, one per face, plus one pressure per
    subdomain in the coarse size."""
    import paper_1901_02090_b200 as B
    g = B.build_grid(2, (14, 49), (1.0, 1.0))
    system = B.assemble_system(g, B.Permeability.isotropic(g, 1.0), B.Wells(0, g.n_cells - 1))
    dec = B.regular_partition(g, (2, 7))
    st = B.BddcSetup(system, dec, B.SolveConfig(constraints="initial"))
    assert dec.n_faces == 1 * 7 + 2 * 6
    assert st.n_c == dec.n_faces + dec.n_subdomains


# ------------------------------------------------ reference bookkeeping views

def _golden_setup(name):
    from _golden import load
    import paper_1901_02090_b200 as B
    d = load(name)
    g = B.build_grid(len(d["counts"]), d["counts"], d["sizes"])
    system = B.assemble_system(g, B.Permeability(d["k"]), B.Wells(0, g.n_cells - 1),
                               lumped=d["lumped"])
    dec = B.regular_partition(g, d["splits"])
    cfg = B.SolveConfig(tau=d["tau"], scaling=d["scaling"], constraints=d["mode"], tol=d["tol"])
    return d, B, system, dec, B.BddcSetup(system, dec, cfg)


@pytest.mark.parametrize("name", ["g2d_adapt", "g3d_thin", "c1_rho"])
def test_broken_interface_E(name):
    """test_decomposition.py:132-146 and test_acceptance.py:226-230: E is a projection
    and average(expand(x)) = x; weights match the oracle's (decomposition.py:212-239)."""
    from oracle import bddc_oracle as O
    d, B, system, dec, st = _golden_setup(name)
    br = st.broken
    rng = np.random.default_rng(0)
    w = rng.standard_normal(br.size)
    ew = br.apply_E(w)
    assert np.abs(br.apply_E(ew) - ew).max() <= 1e-12
    x = rng.standard_normal(dec.n_gamma)
    np.testing.assert_allclose(br.average(br.expand(x)), x, atol=1e-13)
    mesh = O.Mesh(d["counts"], d["sizes"])
    ref = O.weights(O.BoxPartition(mesh, d["splits"]), d["k"], d["scaling"])
    for i in range(dec.n_subdomains):
        np.testing.assert_allclose(st.weights.delta[i], ref[i], rtol=1e-14, atol=0)
        assert len(br.local(w, i)) == int(dec.nG[i])


@pytest.mark.parametrize("name", ["g2d_adapt", "g3d_adapt", "c2_tau10", "g3d_ms"])
def test_constraint_set_view(name):
    """test_adaptive.py:51-82, 105-110: rows per face match the reference's, rows are
    antisymmetric across the face, every subdomain's rows have full rank, the coarse
    size is the row count plus one pressure per subdomain."""
    d, B, system, dec, st = _golden_setup(name)
    cs = st.cset
    assert cs.n_flux_coarse == st.n_flux_coarse
    assert cs.n_coarse == int(d["n_c"])
    counts = [len(cs.rows_for_face(i, j)) // 2 for (i, j) in dec.adjacent_pairs()]
    np.testing.assert_array_equal(counts, d["face_rows"])
    ids = sorted(r.coarse_dof for rows in cs.rows for r in rows if r.sign > 0)
    assert ids == list(range(cs.n_flux_coarse))
    for (i, j) in dec.adjacent_pairs():
        rows = cs.rows_for_face(i, j)
        byg = {}
        for s, r in rows:
            byg.setdefault(r.coarse_dof, []).append((s, r))
        for g, pair in byg.items():
            (si, ri), (sj, rj) = sorted(pair, key=lambda t: t[0])
            shared = dec.faces[(i, j)][0].dofs
            vi = ri.values[dec.gamma_index(si, shared)]
            vj = rj.values[dec.gamma_index(sj, shared)]
            np.testing.assert_allclose(vi, -vj, atol=0)
            if ri.origin == "adaptive":   # adaptive.py:168-170: i-half scaled to max |c| = 1
                assert np.abs(vi).max() == pytest.approx(1.0)
            elif ri.origin == "initial":
                np.testing.assert_array_equal(np.abs(vi), 1.0)
    cs.check_rank()


@pytest.mark.parametrize("name", ["g2d_adapt", "g3d_c3block", "c2_tau10", "c2_tau100"])
def test_pair_reports_filled(name):
    """solver.py:76-88: every adaptive setup carries PairEigenReports; their leading
    eigenvalues match the reference's, selected counts and omega agree."""
    d, B, system, dec, st = _golden_setup(name)
    reps = st.pair_reports
    pairs = [tuple(p) for p in d["pairs"]]
    assert sorted(reps) == sorted(pairs)
    tau = float(d["tau"])
    for q, key in enumerate(pairs):
        r = reps[key]
        assert r.selected == int(d["pair_selected"][q])
        ref = d["pair_lam"][q]
        n = len(r.eigenvalues)
        assert n == min(r.selected + 1, int(np.isfinite(ref).sum()))
        scale = max(float(ref[0]), 1.0)
        np.testing.assert_allclose(r.eigenvalues, ref[:n], rtol=1e-8, atol=1e-10 * scale)
        assert r.omega(tau) == pytest.approx(st.face_omega[q], rel=1e-12)


@pytest.mark.parametrize("name", ["g2d_adapt", "g3d_box"])
def test_subs_and_coarse_views(name):
    """substructure.py:90-99 (dense S_i) and coarse.py:208-215 (pinned coarse solve in
    the reference's numbering) against the golden S and the oracle's coarse solve."""
    from _golden import rel
    from oracle import bddc_oracle as O
    d, B, system, dec, st = _golden_setup(name)
    assert rel(st.subs[0].schur_dense(), d["S_sub0"]) <= 1e-11
    x = np.random.default_rng(3).standard_normal(int(dec.nG[0]))
    assert rel(st.subs[0].schur_apply(x), d["S_sub0"] @ x) <= 1e-11
    mesh = O.Mesh(d["counts"], d["sizes"])
    cfg = O.Config(tau=d["tau"], scaling=d["scaling"], constraints=d["mode"], tol=d["tol"],
                   lumped=d["lumped"])
    ost = O.Setup(mesh, d["k"], O.well_rhs(mesh, 0, mesh.n_cells - 1), d["splits"], cfg)
    # adaptive rows are defined up to sign / rotation inside a degenerate eigenspace,
    # so the coarse bases of two implementations differ by a face-block transform on
    # the adaptive dofs: a load on the initial-row dofs and the pressures gives the
    # same initial-row and pressure components
    rng = np.random.default_rng(4)
    nf = dec.n_faces
    rf = np.zeros(st.cset.n_flux_coarse)
    rf[:nf] = rng.standard_normal(nf)
    rq = rng.standard_normal(dec.n_subdomains)
    rq -= rq.mean()
    xf, xp = st.coarse.solve(rf, rq)
    of, op = ost.coarse.solve(rf, rq)
    assert rel(xf[:nf], of[:nf]) <= 1e-10
    assert rel(xp[1:], op[1:]) <= 1e-10


def test_graph_cache_survives_history_realloc():
    """a larger maxit reallocates the PCG history; cached graphs of the
    smaller maxit must not write into the freed buffers (history and kappa of a
    repeated solve stay identical)."""
    B, g, system, dec = _problem(11)
    cfg_s = B.SolveConfig(tol=1e-10, maxit=100)
    st = B.BddcSetup(system, dec, cfg_s)
    a = B.solve(system, dec, cfg_s, setup=st)
    B.solve(system, dec, B.SolveConfig(tol=1e-10, maxit=10000), setup=st)
    c = B.solve(system, dec, cfg_s, setup=st)
    assert a.it == c.it and a.kappa == c.kappa
    np.testing.assert_array_equal(a.residuals, c.residuals)
    np.testing.assert_array_equal(a.u, c.u)


def test_two_setups_same_source_twice():
    """two live setups solving one source array twice each (the source is
    page-locked once per process; a refused registration must not poison later
    launches)."""
    B, g, system, dec = _problem(12)
    s1 = B.BddcSetup(system, dec, B.SolveConfig(tol=1e-10, constraints="adaptive", tau=10.0))
    s2 = B.BddcSetup(system, dec, B.SolveConfig(tol=1e-10, constraints="adaptive", tau=3.0))
    reps = [B.solve(system, dec, st.config, setup=st) for st in (s1, s2, s1, s2)]
    np.testing.assert_array_equal(reps[0].u, reps[2].u)
    np.testing.assert_array_equal(reps[1].u, reps[3].u)
    assert all(r.converged for r in reps)
    del s1
    r = B.solve(system, dec, s2.config, setup=s2)
    np.testing.assert_array_equal(r.u, reps[1].u)

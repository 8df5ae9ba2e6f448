"""Implementation-independent invariants of the GPU path (test_acceptance.py [1], [6], [7];
test_solver.py determinism / non-convergence), checked against the CPU oracle."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _problem(counts, splits, seed, scaling="multiplicity", tau=math.inf, tol=1e-10, sizes=None,
             orders=6.0):
    import paper_1901_02090_b200 as B
    sizes = sizes or (1.0,) * len(counts)
    g = B.build_grid(len(counts), counts, sizes)
    rng = np.random.default_rng(seed)
    k = 10.0 ** rng.uniform(-orders / 2, orders / 2, (g.n_cells, len(counts)))
    system = B.assemble_system(g, B.Permeability(k), B.Wells(0, g.n_cells - 1))
    dec = B.regular_partition(g, splits)
    cfg = B.SolveConfig(tau=tau, scaling=scaling,
                        constraints="adaptive" if math.isfinite(tau) else "initial", tol=tol)
    return B, g, k, system, dec, cfg


RANDOM = []
for n, (counts, splits) in enumerate([
        ((16, 16), (2, 2)), ((24, 24), (3, 3)), ((24, 12), (2, 2)), ((9, 21), (3, 3)),
        ((20, 20), (2, 2)), ((15, 15), (3, 3)), ((6, 6, 6), (2, 2, 2)), ((6, 6, 6), (3, 3, 3)),
        ((5, 5, 5), (2, 2, 2)), ((4, 6, 4), (2, 2, 2))]):
    for scaling in ("multiplicity", "stiffness"):
        tau = math.inf if (n + len(splits)) % 2 == 0 else 5.0
        RANDOM.append((counts, splits, scaling, tau, 100 + n))


@pytest.mark.parametrize("counts,splits,scaling,tau,seed", RANDOM)
def test_random_instances_vs_direct(counts, splits, scaling, tau, seed):
    """test_acceptance.py [1]: 20 random instances vs a monolithic direct solve."""
    from oracle import bddc_oracle as O
    B, g, k, system, dec, cfg = _problem(counts, splits, seed, scaling, tau, tol=1e-11)
    rep = B.solve(system, dec, cfg)
    m = O.Mesh(counts, (1.0,) * len(counts))
    u, p = O.direct_solve(m, k, O.well_rhs(m, 0, m.n_cells - 1))
    assert np.linalg.norm(rep.u - u) / np.linalg.norm(u) <= 1e-5
    assert np.linalg.norm(rep.p - p) / np.linalg.norm(p) <= 1e-4


def test_conservation_and_balance():
    """test_acceptance.py [6]: u* conserves mass, correction divergence-free, iterates balanced."""
    B, g, k, system, dec, cfg = _problem((12, 12), (3, 3), 4, tol=1e-10)
    st = B.BddcSetup(system, dec, cfg)
    phi = st.net_flux_matrix()
    worst, scale = [0.0], [1.0]

    def watch(x, r):
        worst[0] = max(worst[0], np.abs(phi @ x).max())
        scale[0] = max(scale[0], np.abs(x).max())

    rep = B.solve(system, dec, cfg, setup=st, iterate_callback=watch)
    f = system.f
    assert np.linalg.norm(system.B @ rep.u_star - f) / np.linalg.norm(f) <= 1e-10
    corr = rep.u - rep.u_star
    assert np.linalg.norm(system.B @ corr) <= 1e-8 * np.linalg.norm(system.B @ rep.u)
    assert worst[0] / scale[0] <= 1e-9


def test_stiffness_final_conservation():
    """test_solver.py:94-100."""
    B, g, k, system, dec, cfg = _problem((8, 8), (2, 2), 5, scaling="stiffness", tol=1e-10,
                                         orders=4.0)
    rep = B.solve(system, dec, cfg)
    assert np.linalg.norm(system.B @ rep.u - system.f) / np.linalg.norm(system.f) <= 1e-8


def test_spectrum_floor():
    """test_acceptance.py [7]: eigenvalues of the preconditioned operator >= 1."""
    import scipy.linalg as sla
    B, g, k, system, dec, cfg = _problem((12, 12), (3, 3), 3, tau=3.0)
    st = B.BddcSetup(system, dec, cfg)
    n = dec.n_gamma
    E = np.eye(n)
    S = np.stack([st.schur_matvec(E[:, c]) for c in range(n)], axis=1)
    M = np.stack([st.precondition(E[:, c]) for c in range(n)], axis=1)
    Z = sla.null_space(st.net_flux_matrix().toarray())
    Sb = Z.T @ S @ Z
    Mb = Z.T @ M @ Z
    Sb, Mb = 0.5 * (Sb + Sb.T), 0.5 * (Mb + Mb.T)
    w, V = sla.eigh(Mb)
    W = (V * np.sqrt(np.maximum(w, 0.0))) @ V.T
    lam = sla.eigh(W @ Sb @ W, eigvals_only=True)
    assert lam[0] >= 1.0 - 1e-8
    assert lam[-1] <= 2.0 * st.omega_tilde * dec.max_faces_per_subdomain ** 2
    # the on-device diagnostic gives the same spectrum
    lam_gpu = B.preconditioned_spectrum(st)
    np.testing.assert_allclose(lam_gpu, np.sort(lam), rtol=1e-9, atol=1e-9)
    # and the PCG's Lanczos kappa lies inside it
    rep = B.solve(system, dec, cfg, setup=st)
    assert rep.kappa <= lam_gpu[-1] / lam_gpu[0] * (1 + 1e-6)


def test_bitwise_determinism():
    """test_solver.py:165-173: repeated solves with one setup are bitwise identical."""
    B, g, k, system, dec, cfg = _problem((16, 16), (4, 4), 10, tau=5.0, tol=1e-8)
    st = B.BddcSetup(system, dec, cfg)
    r1 = B.solve(system, dec, cfg, setup=st)
    r2 = B.solve(system, dec, cfg, setup=st)
    np.testing.assert_array_equal(r1.u, r2.u)
    np.testing.assert_array_equal(r1.p, r2.p)
    assert r1.it == r2.it
    st2 = B.BddcSetup(system, dec, cfg)
    r3 = B.solve(system, dec, cfg, setup=st2)
    np.testing.assert_array_equal(r1.u, r3.u)


@pytest.mark.parametrize("counts,splits,seed", [((16, 16), (4, 4), 10), ((12, 12, 8), (3, 3, 2), 4)])
def test_pdl_launches_do_not_change_results(counts, splits, seed):
    """The small PCG kernels as programmatic dependent launches (they become resident
    while their predecessor runs and wait at their top) against plain stream-ordered
    launches of the same kernels: bitwise the same solve.  A load that took the
    non-coherent path, or work placed ahead of the dependency wait, would show here."""
    from paper_1901_02090_b200 import _native as nat
    B, g, k, system, dec, cfg = _problem(counts, splits, seed, tau=5.0, tol=1e-9)
    lib = nat.load()
    out = {}
    try:
        for mask in (31, 0):
            lib.bddc_set_pdl_pcg(mask)
            lib.bddc_set_pdl(1 if mask else 0)
            st = B.BddcSetup(system, dec, cfg)      # fresh setup: fresh captured graphs
            reps = [B.solve(system, dec, cfg, setup=st) for _ in range(3)]
            for r in reps[1:]:
                np.testing.assert_array_equal(reps[0].u, r.u)
            out[mask] = reps[0]
    finally:
        lib.bddc_set_pdl_pcg(31)
        lib.bddc_set_pdl(1)
    assert out[31].it == out[0].it
    np.testing.assert_array_equal(out[31].u, out[0].u)
    np.testing.assert_array_equal(out[31].p, out[0].p)
    np.testing.assert_array_equal(out[31].residuals, out[0].residuals)


def test_nonconvergence_partial_report():
    """test_solver.py:139-144."""
    B, g, k, system, dec, cfg = _problem((8, 8), (2, 2), 8, tol=1e-12)
    cfg.maxit = 2
    with pytest.raises(B.NonConvergenceError) as ei:
        B.solve(system, dec, cfg)
    rep = ei.value.report
    assert rep is not None and not rep.converged and rep.it == 2
    assert len(rep.residuals) == 3


def test_single_subdomain():
    """No interface: the solve is one local KKT solve (N = 1 edge case)."""
    from oracle import bddc_oracle as O
    B, g, k, system, dec, cfg = _problem((6, 5), (1, 1), 2, tol=1e-10)
    rep = B.solve(system, dec, cfg)
    m = O.Mesh((6, 5), (1.0, 1.0))
    u, p = O.direct_solve(m, k, O.well_rhs(m, 0, m.n_cells - 1))
    assert rep.it == 0
    assert np.linalg.norm(rep.u - u) / np.linalg.norm(u) <= 1e-10


def test_homogeneous_benchmark_2x7():
    """test_acceptance.py [2]: 60x220, 2x7, k = 1: 8<=it<=18, 2<=kappa<=6, n_c=33."""
    import paper_1901_02090_b200 as B
    g = B.build_grid(2, (60, 220), (1.0, 1.0))
    system = B.assemble_system(g, B.Permeability.isotropic(g, 1.0), B.Wells(0, g.n_cells - 1))
    dec = B.regular_partition(g, (2, 7))
    rep = B.solve(system, dec, B.SolveConfig(tol=1e-6))
    assert 8 <= rep.it <= 18 and 2.0 <= rep.kappa <= 6.0 and rep.n_c == 33


def test_multiscale_rows_unit_net_flux():
    """test_adaptive.py:102-111: every multiscale row carries the unit transfer, i.e.
    sums to 1 for the lower subdomain of its pair."""
    import paper_1901_02090_b200 as B
    g = B.build_grid(2, (12, 12), (1.0, 1.0))
    k = 10.0 ** np.random.default_rng(9).uniform(-3, 3, (g.n_cells, 2))
    system = B.assemble_system(g, B.Permeability(k), B.Wells(0, g.n_cells - 1))
    dec = B.regular_partition(g, (3, 3))
    st = B.BddcSetup(system, dec, B.SolveConfig(constraints="multiscale", tol=1e-8))
    assert len(st.multiscale_rows) == dec.n_faces
    for row in st.multiscale_rows:
        assert row.sum() == pytest.approx(1.0, rel=1e-8)
    assert st.n_c == 2 * dec.n_faces + dec.n_subdomains

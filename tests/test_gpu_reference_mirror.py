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

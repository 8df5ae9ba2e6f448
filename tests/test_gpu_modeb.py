"""Mode B (BASELINE's pressure-drop boundary condition) against a monolithic
sparse direct solve.

The reference cannot express Dirichlet pressure, so the pin is
oracle.direct_solve_dirichlet: an independent assembly of the full saddle system
with the boundary faces of the drop axis as flux dofs.  Gates: u and p within
1e-8 relative L2 at PCG rtol 1e-10, mass conservation B u = f and the momentum
residual of the host-assembled system (SaddleSystem.A/.B/.g, CPU-tested against
the oracle's assembly in test_modeb_host.py).
"""
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))

pytestmark = pytest.mark.gpu

CASES = [
    # name, counts, sizes, splits, axis, constraints, tau, scaling, field std
    ("2d_y", (24, 30), (1.0, 1.0), (3, 3), 1, "initial", float("inf"), "multiplicity", 0.5),
    ("2d_x_adapt", (30, 20), (2.0, 1.0), (5, 2), 0, "adaptive", 3.0, "stiffness", 1.5),
    ("3d_y_adapt", (12, 20, 6), (20.0, 10.0, 2.0), (2, 4, 2), 1, "adaptive", 10.0, "stiffness", 1.5),
    ("3d_z", (8, 8, 12), (1.0, 1.0, 1.0), (2, 2, 3), 2, "initial", float("inf"), "stiffness", 1.0),
    ("3d_uneven", (13, 17, 5), (1.0, 2.0, 1.0), ((4, 9), (5, 3, 6, 3), (5,)), 1, "adaptive", 5.0,
     "stiffness", 1.0),
    ("2d_two_strips", (16, 16), (1.0, 1.0), (4, 2), 1, "adaptive", 10.0, "stiffness", 1.0),
    ("2d_one_strip", (16, 16), (1.0, 1.0), (4, 1), 1, "initial", float("inf"), "multiplicity", 1.0),
    ("2d_chain_homog", (12, 20), (1.0, 1.0), (1, 4), 1, "initial", float("inf"), "multiplicity", 0.0),
    ("3d_chain", (6, 20, 4), (1.0, 1.0, 1.0), (1, 4, 1), 1, "adaptive", 10.0, "stiffness", 1.0),
    ("2d_multiscale", (24, 24), (1.0, 1.0), (3, 4), 1, "multiscale", float("inf"), "stiffness", 1.0),
]


def _field(counts, std, seed):
    rng = np.random.default_rng(seed)
    n = int(np.prod(counts))
    k = 10.0 ** (std * rng.standard_normal((n, len(counts))))
    return k


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_modeb_vs_direct(case):
    import bddc_oracle as O
    import paper_1901_02090_b200 as B
    name, counts, sizes, splits, axis, cons, tau, scaling, std = case
    k = _field(counts, std, sum(name.encode()))
    g = B.build_grid(len(counts), counts, sizes)
    system = B.assemble_system(g, B.Permeability(k), B.PressureDrop(axis, 1.0, 0.0))
    if isinstance(splits[0], tuple):
        dec = B.box_partition(g, splits)
    else:
        dec = B.regular_partition(g, splits)
    cfg = B.SolveConfig(tau=tau, scaling=scaling, constraints=cons, tol=1e-10)
    rep = B.solve(system, dec, cfg)
    u_ref, p_ref = O.direct_solve_dirichlet(O.Mesh(counts, sizes), k, np.zeros(g.n_cells), axis, 1.0, 0.0)
    # (pressure_warning is not asserted: its 10*tol momentum bar sits at rounding level
    # for the 3-decade fields at tol 1e-10; the momentum residual is checked below)
    assert rep.converged
    assert len(rep.u) == system.n_flux
    ru = np.linalg.norm(rep.u - u_ref) / np.linalg.norm(u_ref)
    rp = np.linalg.norm(rep.p - p_ref) / np.linalg.norm(p_ref)
    assert ru <= 1e-8, (ru, rp, rep.it)
    assert rp <= 1e-8, (ru, rp, rep.it)
    res = system.A @ rep.u + system.B.T @ rep.p - system.g
    assert np.linalg.norm(res) <= 1e-8 * np.linalg.norm(system.g)
    assert np.abs(system.B @ rep.u).max() <= 1e-10 * np.abs(rep.u).max()


def test_modeb_setup_reuse_and_values():
    """One setup, several pressure drops: the solution is linear in (p_low, p_high)."""
    import paper_1901_02090_b200 as B
    counts = (16, 24)
    g = B.build_grid(2, counts, (1.0, 1.0))
    k = _field(counts, 1.0, 7)
    s1 = B.assemble_system(g, B.Permeability(k), B.PressureDrop(1, 1.0, 0.0))
    dec = B.regular_partition(g, (2, 3))
    cfg = B.SolveConfig(tau=10.0, scaling="stiffness", constraints="adaptive", tol=1e-10)
    st = B.BddcSetup(s1, dec, cfg)
    r1 = B.solve(s1, dec, cfg, setup=st)
    s2 = B.assemble_system(g, B.Permeability(k), B.PressureDrop(1, 3.0, 1.0))
    r2 = B.solve(s2, dec, cfg, setup=st)
    # p_low=3, p_high=1: twice the drop, shifted by 1
    np.testing.assert_allclose(r2.u, 2.0 * r1.u, rtol=0, atol=1e-9 * np.abs(r1.u).max())
    np.testing.assert_allclose(r2.p, 2.0 * r1.p + 1.0, rtol=0, atol=1e-9)
    s3 = B.assemble_system(g, B.Permeability(k), B.Wells(0, g.n_cells - 1))
    with pytest.raises(B.InvalidArgumentError):
        B.solve(s3, dec, cfg, setup=st)


@pytest.mark.parametrize("splits,axis", [((3, 5, 2), 1), ((4, 3, 3), 0), ((2, 2, 4), 2), ((2, 2, 2), 1)])
def test_modeb_separable_balance_matches_dense(splits, axis, monkeypatch):
    """Large-N mode B path (separable Laplacian solves on the floating sub-box) against
    the dense-inverse path on the same problem: same iterates, same solution."""
    import paper_1901_02090_b200 as B
    from paper_1901_02090_b200 import solver as SV
    counts = (12, 15, 8)
    g = B.build_grid(3, counts, (2.0, 1.0, 1.0))
    k = _field(counts, 1.0, 11 + axis)
    system = B.assemble_system(g, B.Permeability(k), B.PressureDrop(axis, 1.0, 0.0))
    dec = B.regular_partition(g, splits)
    cfg = B.SolveConfig(tau=5.0, scaling="stiffness", constraints="adaptive", tol=1e-10)
    r_dense = B.solve(system, dec, cfg)
    monkeypatch.setattr(SV, "DENSE_BALANCE_MAX", 0)
    st = B.BddcSetup(system, dec, cfg)
    assert st.d_Lp is None
    x = np.random.default_rng(0).standard_normal(dec.n_gamma)
    px = st.project_balanced(x)
    phi = st.net_flux_matrix()
    phi = phi.toarray() if hasattr(phi, "toarray") else np.asarray(phi)
    # balanced on the floating subdomains, orthogonal projection (P x - x in range Phi_F^T)
    if st.floating.any():
        assert np.abs(phi[st.floating] @ px).max() <= 1e-12 * np.abs(x).max()
    else:   # two strips along the drop axis: nothing floats, the projection is the identity
        np.testing.assert_array_equal(px, x)
    np.testing.assert_allclose(st.project_balanced(px), px, atol=1e-12)
    r_sep = B.solve(system, dec, cfg, setup=st)
    assert abs(r_sep.it - r_dense.it) <= 1
    assert np.linalg.norm(r_sep.u - r_dense.u) <= 1e-9 * np.linalg.norm(r_dense.u)
    assert np.linalg.norm(r_sep.p - r_dense.p) <= 1e-9 * np.linalg.norm(r_dense.p)

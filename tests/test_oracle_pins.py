"""Known-answer pins for the CPU oracle (from the reference's own tests)."""
import math

import numpy as np
import pytest

from oracle import bddc_oracle as O


def test_dof_counts_2d():
    # test_grid.py:10-17
    m = O.Mesh((60, 220), (1.0, 1.0))
    assert m.n_cells == 13200
    assert m.n_flux == 26120


def test_dof_counts_3d():
    # test_grid.py:19-22: 3*31*30*30 faces + 27000 cells = 110700 total dofs
    m = O.Mesh((30, 30, 30), (1.0, 1.0, 1.0))
    assert 3 * 31 * 30 * 30 + m.n_cells == 110700
    assert m.n_flux == 3 * 29 * 30 * 30


def test_two_cell_assembly():
    # test_grid.py:25-33: A = [2/3], B = [[-1],[1]], f = [-1, 1]
    m = O.Mesh((2, 1), (1.0, 1.0))
    k = np.ones((2, 2))
    np.testing.assert_allclose(O.mass_matrix(m, k).toarray(), [[2.0 / 3.0]])
    np.testing.assert_allclose(O.divergence(m).toarray(), [[-1.0], [1.0]])
    np.testing.assert_allclose(O.well_rhs(m, 0, 1), [-1.0, 1.0])


def test_two_cell_analytic_direct():
    # test_oracle.py:12-21: u = 3, p_hi - p_lo = -1
    m = O.Mesh((2, 1), (1.0, 1.0))
    k = np.full((2, 2), 2.0)
    u, p = O.direct_solve(m, k, O.well_rhs(m, 0, 1, 3.0))
    np.testing.assert_allclose(u, [3.0])
    np.testing.assert_allclose(p[1] - p[0], -1.0)


@pytest.mark.parametrize("counts,splits,N,nf,ng", [
    ((60, 220), (2, 7), 14, 19, 580),      # test_decomposition.py:13-21
    ((60, 220), (6, 22), 132, 236, 2360),  # test_decomposition.py:23-28
    ((30, 30, 30), (3, 3, 3), 27, 54, 5400),  # test_decomposition.py:31-36
])
def test_partition_counts(counts, splits, N, nf, ng):
    P = O.BoxPartition(O.Mesh(counts, (1.0,) * len(counts)), splits)
    assert P.N == N
    assert len(P.pairs) == nf
    assert len(P.gamma) == ng


def test_initial_coarse_count_2x7():
    # test_coarse.py:23-29: n_c = 19 + 14 = 33
    P = O.BoxPartition(O.Mesh((60, 220), (1.0, 1.0)), (2, 7))
    cs = O.initial_constraints(P)
    assert cs.n_flux + P.N == 33


def test_stiffness_weights_contrast():
    # test_decomposition.py:113-128
    m = O.Mesh((4, 2), (1.0, 1.0))
    P = O.BoxPartition(m, (2, 1))
    k = np.where(np.arange(8) % 4 < 2, 1.0, 1e6)
    k = np.repeat(k[:, None], 2, axis=1)
    w = O.weights(P, k, "stiffness")
    np.testing.assert_allclose(w[0], 1.0 / (1.0 + 1e-6))
    np.testing.assert_allclose(w[1], 1e-6 / (1.0 + 1e-6))


def test_homogeneous_benchmark_2x7():
    # test_acceptance.py:90-105: 8 <= it <= 18, 2 <= kappa <= 6, n_c = 33
    k = np.ones((13200, 2))
    st, rep = O.run((60, 220), (1.0, 1.0), k, (2, 7), O.Config(tol=1e-6))
    assert 8 <= rep.it <= 18
    assert 2.0 <= rep.kappa <= 6.0
    assert rep.n_c == 33

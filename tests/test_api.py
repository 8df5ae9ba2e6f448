"""Host-side API mirror: validation and error classes (no GPU needed)."""
import math

import numpy as np
import pytest

import paper_1901_02090_b200 as B


def test_config_validation():
    # test_solver.py:29-35
    with pytest.raises(B.InvalidArgumentError):
        B.SolveConfig(tau=0.5)
    with pytest.raises(B.InvalidArgumentError):
        B.SolveConfig(tol=2.0)
    with pytest.raises(B.InvalidArgumentError):
        B.SolveConfig(constraints="bogus")


def test_grid_validation():
    with pytest.raises(B.InvalidArgumentError):
        B.build_grid(4, (2, 2, 2, 2), (1, 1, 1, 1))
    with pytest.raises(B.InvalidArgumentError):
        B.build_grid(2, (0, 3), (1.0, 1.0))
    with pytest.raises(B.InvalidArgumentError):
        B.build_grid(2, (2, 3), (1.0, -1.0))
    with pytest.raises(B.InvalidArgumentError):
        B.Permeability(np.array([[1.0, -1.0]]))


def test_assemble_system():
    g = B.build_grid(2, (2, 1), (1.0, 1.0))
    s = B.assemble_system(g, B.Permeability.isotropic(g, 1.0), B.Wells(0, 1))
    np.testing.assert_allclose(s.f, [-1.0, 1.0])
    np.testing.assert_allclose(s.A.toarray(), [[2.0 / 3.0]])
    np.testing.assert_allclose(s.B.toarray(), [[-1.0], [1.0]])
    with pytest.raises(B.InvalidArgumentError):
        B.assemble_system(g, B.Permeability.isotropic(g, 1.0), B.Wells(0, 5))


def test_assemble_system_lumped():
    """grid.py:220-225 / test_grid.py:51-55: the lumped element block is diag(3c):
    the single interior face of two unit cells gets 3/6 from each side."""
    g = B.build_grid(2, (2, 1), (1.0, 1.0))
    s = B.assemble_system(g, B.Permeability.isotropic(g, 1.0), B.Wells(0, 1), lumped=True)
    np.testing.assert_allclose(s.A.toarray(), [[1.0]])
    g = B.build_grid(2, (3, 3), (1.0, 2.0))
    k = np.random.default_rng(0).uniform(0.5, 2.0, (9, 2))
    A = B.assemble_system(g, B.Permeability(k), B.Wells(0, 8), lumped=True).A
    assert A.nnz == A.shape[0]   # diagonal


def test_matrices_match_oracle():
    from oracle import bddc_oracle as O
    rng = np.random.default_rng(3)
    g = B.build_grid(3, (4, 3, 5), (2.0, 1.0, 0.5))
    k = 10 ** rng.uniform(-2, 2, (g.n_cells, 3))
    s = B.assemble_system(g, B.Permeability(k), B.Wells(0, g.n_cells - 1))
    m = O.Mesh((4, 3, 5), (2.0, 1.0, 0.5))
    assert abs(s.A - O.mass_matrix(m, k)).max() == 0.0
    assert abs(s.B - O.divergence(m)).max() == 0.0


def test_errors_taxonomy():
    assert issubclass(B.NumericalFailureError, RuntimeError)
    assert issubclass(B.ConstraintRankError, ValueError)
    assert B.NumericalFailureError("x", where=3).where == 3
    assert B.NonConvergenceError("x", report=1).report == 1

"""Mode B host pieces (CPU): the package's SaddleSystem assembly with Dirichlet
boundary dofs against the oracle's independent assembly, and the oracle direct
solve against closed-form solutions."""
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))


def test_channel_closed_form():
    import bddc_oracle as O
    m = O.Mesh((1, 8), (1.0, 1.0))
    u, p = O.direct_solve_dirichlet(m, np.ones((8, 2)), np.zeros(8), 1, 1.0, 0.0)
    np.testing.assert_allclose(u, 0.125, atol=1e-14)          # Darcy: k dp/L = 1/8
    np.testing.assert_allclose(p, 1.0 - (np.arange(8) + 0.5) / 8, atol=1e-14)


@pytest.mark.parametrize("axis", [0, 1, 2])
def test_host_assembly_matches_oracle(axis):
    import bddc_oracle as O
    import paper_1901_02090_b200 as B
    counts, sizes = (5, 7, 3), (2.0, 1.0, 0.5)
    k = np.exp(np.random.default_rng(axis).normal(size=(105, 3)))
    u, p = O.direct_solve_dirichlet(O.Mesh(counts, sizes), k, np.zeros(105), axis, 1.0, 0.25)
    g = B.build_grid(3, counts, sizes)
    sy = B.assemble_system(g, B.Permeability(k), B.PressureDrop(axis, 1.0, 0.25))
    assert sy.n_flux == len(u)
    assert np.abs(sy.A @ u + sy.B.T @ p - sy.g).max() < 1e-13
    assert np.abs(sy.B @ u).max() < 1e-13
    assert p.min() > 0.25 - 1e-12 and p.max() < 1.0 + 1e-12   # maximum principle


def test_pressure_drop_validation():
    import paper_1901_02090_b200 as B
    g = B.build_grid(2, (4, 4), (1.0, 1.0))
    k = B.Permeability.isotropic(g, 1.0)
    with pytest.raises(B.InvalidArgumentError):
        B.assemble_system(g, k, B.PressureDrop(2))
    with pytest.raises(B.InvalidArgumentError):
        B.assemble_system(g, k, B.PressureDrop(0, float("nan")))

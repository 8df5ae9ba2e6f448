"""Closed-form box topology of the package vs the oracle / reference counts."""
import numpy as np
import pytest

import paper_1901_02090_b200 as B
from oracle import bddc_oracle as O


@pytest.mark.parametrize("counts,splits", [
    ((8, 8), (2, 2)), ((9, 21), (3, 3)), ((60, 220), (6, 22)), ((5, 5, 5), (3, 3, 3)),
    ((8, 6, 4), (2, 2, 2)), ((12, 7, 9), (3, 2, 4)), ((7, 5), (1, 2)), ((4, 4), (1, 1)),
])
def test_topology_matches_oracle(counts, splits):
    g = B.build_grid(len(counts), counts, (1.0,) * len(counts))
    d = B.regular_partition(g, splits)
    P = O.BoxPartition(O.Mesh(counts, (1.0,) * len(counts)), splits)
    np.testing.assert_array_equal(d.part, P.part)
    np.testing.assert_array_equal(d.gamma, P.gamma)
    for i in range(d.n_subdomains):
        np.testing.assert_array_equal(d.gamma_dofs[i], P.gamma_dofs[i])
        np.testing.assert_array_equal(d.cells[i], P.cells[i])
    assert d.adjacent_pairs() == P.pairs
    for f, (i, j) in enumerate(P.pairs):
        np.testing.assert_array_equal(d.faces[(i, j)][0].dofs, P.face_dofs[f])
        np.testing.assert_array_equal(d.sign_for(i, P.face_dofs[f]), P.sign(i, P.face_dofs[f]))
    # slot tables are mutually consistent
    for i in range(d.n_subdomains):
        n = d.nG[i]
        codes = d.gcode[i, :n]
        a, side, line = codes & 3, (codes >> 2) & 1, codes >> 3
        np.testing.assert_array_equal(d.fslot[i, 2 * a + side, line], np.arange(n))
    lo = d.gown[:, 0] // d.maxG
    hi = d.gown[:, 1] // d.maxG
    np.testing.assert_array_equal(lo, d.dof_sub_low)
    assert np.all(lo < hi)


def test_counts_config3():
    g = B.build_grid(3, (60, 220, 85), (20.0, 10.0, 2.0))
    d = B.regular_partition(g, (6, 22, 17))
    assert d.n_subdomains == 2244
    assert d.n_faces == 6124
    assert d.n_gamma == 411800
    assert int(d.nG.max()) == 400


def test_validation():
    g = B.build_grid(2, (4, 4), (1.0, 1.0))
    with pytest.raises(B.InvalidArgumentError):
        B.regular_partition(g, (5, 1))
    with pytest.raises(B.InvalidArgumentError):
        B.regular_partition(g, (2,))


def test_box_partition_uneven_strips_and_part_roundtrip(tmp_path):
    """Tensor-product box partitions with uneven strips (box
    case): widths, the reference constructor Decomposition(grid, part) and PART
    import all give the same topology; non-box maps are rejected."""
    import paper_1901_02090_b200 as B
    from paper_1901_02090_b200.errors import ConfigurationError
    g = B.build_grid(3, (12, 10, 8), (1.0, 1.0, 1.0))
    d1 = B.box_partition(g, [[3, 5, 4], [2, 4, 4], [5, 3]])
    assert d1.splits == (3, 3, 2)
    assert [list(map(int, w)) for w in d1.sw] == [[3, 5, 4], [2, 4, 4], [5, 3]]
    d2 = B.Decomposition(g, d1.part)
    np.testing.assert_array_equal(d1.gpos, d2.gpos)
    np.testing.assert_array_equal(d1.gamma, d2.gamma)
    path = tmp_path / "p.part"
    path.write_text(f"PART {d1.n_subdomains} {g.n_cells}\n" + "\n".join(map(str, d1.part)) + "\n")
    d3 = B.import_partition(str(path), g)
    np.testing.assert_array_equal(d1.gcode, d3.gcode)
    with pytest.raises(ConfigurationError):
        B.Decomposition(g, np.random.default_rng(0).integers(0, 4, g.n_cells))


@pytest.mark.parametrize("dim,counts,splits", [
    (2, (12, 12), (3, 3)), (2, (10, 7), (1, 3)), (2, (5, 5), (1, 1)),
    (3, (12, 10, 8), (3, 2, 2)), (3, (12, 10, 8), (1, 1, 4)),
    (3, (12, 12, 9), ([3, 5, 4], [2, 4, 6], [5, 4]))])
def test_closed_form_tables_and_lazy_host_copies(dim, counts, splits):
    """Constructing a Decomposition does O(N) host work only (sizes, nG, face table,
    face prefix counts in closed form); the per-slot / per-dof tables appear on first
    access and agree with the closed forms (asserted inside the lazy build) and with
    the reference's definitions (decomposition.py:60-125)."""
    import paper_1901_02090_b200 as B
    g = B.build_grid(dim, counts, (1.0,) * dim)
    d = B.Decomposition(g, splits)
    lazy = set(B.Decomposition._LAZY) | {"part"}
    assert not (lazy & set(d.__dict__))
    N = d.n_subdomains
    # face prefix counts: faces are sorted by (i, j)
    assert np.array_equal(d.face_base, np.searchsorted(d.face_table[:, 0], np.arange(N)))
    gam = d.gamma                      # triggers the lazy build (with its own asserts)
    assert len(gam) == d.n_gamma == len(np.unique(gam))
    part = d.part
    # Gamma = interior faces whose two cells lie in different subdomains
    expect = []
    for a in range(dim):
        lo, hi = g.cell_faces(a)
        m = hi >= 0
        cells = np.nonzero(m)[0]
        stride = int(np.prod(g.counts[:a]))
        cut = part[cells] != part[cells + stride]
        expect.append(hi[m][cut])
    assert np.array_equal(np.sort(np.concatenate(expect)), gam)
    assert np.array_equal(d.nG, [len(x) for x in d.gamma_dofs])
    for f, (i, j, a, m) in enumerate(d.face_table):
        assert int((d.gface == f).sum()) == m

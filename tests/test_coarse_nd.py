"""Host-side symbolic analysis of the nested-dissection coarse solver (CPU only)."""

import types

import numpy as np
import pytest
import torch

import paper_1901_02090_b200 as B
from paper_1901_02090_b200 import coarse_nd as ND
from paper_1901_02090_b200 import solver as SV


def _tables(counts, splits, seed):
    g = B.build_grid(len(counts), counts, (1.0,) * len(counts))
    dec = B.regular_partition(g, splits)
    rng = np.random.default_rng(seed)
    per_face = rng.integers(1, 5, dec.n_faces)
    cstart = np.concatenate([[0], np.cumsum(per_face)[:-1]])
    fake = types.SimpleNamespace(dec=dec, N=dec.n_subdomains)
    SV.BddcSetup._build_coarse_tables(fake, cstart, per_face, 4)
    nd = ND.CoarseND(dec, per_face, cstart, fake.sub_rows, fake.nC, fake.maxC, "cpu")
    return dec, per_face, fake, nd


@pytest.mark.parametrize("counts,splits", [((12, 12, 12), (2, 3, 4)), ((9, 9, 6), (3, 3, 3)),
                                           ((16, 12), (4, 3))])
def test_pivots_partition_coarse_dofs(counts, splits):
    """Every flux coarse dof and every pressure but the pinned one is eliminated
    exactly once (pressures at the node that eliminates their subdomain's last face)."""
    dec, per_face, fake, nd = _tables(counts, splits, 1)
    seps = np.concatenate([L.sep_flat.numpy()[:L.ysize] for L in nd.levels])
    want = np.concatenate([np.arange(nd.nfc), nd.nfc + np.arange(1, dec.n_subdomains)])
    assert np.array_equal(np.sort(seps), want)


@pytest.mark.parametrize("counts,splits", [((12, 12, 12), (2, 3, 4)), ((9, 9, 6), (3, 3, 3))])
def test_child_maps_and_gather_lists(counts, splits):
    dec, per_face, fake, nd = _tables(counts, splits, 2)
    nb_total = 0
    for L in nd.levels:
        cm = L.cmap.numpy()
        for slot in (0, 1):
            for q in range(L.m):
                v = cm[slot, q]
                v = v[v >= 0]
                assert len(np.unique(v)) == len(v)
                assert np.all(v < L.nf)
        nb_total += int(L.b.sum())
    # every boundary entry of every node is one contribution to exactly one
    # pivot entry of an ancestor (the pinned pressure appears nowhere)
    nlist = sum(int(L.lptr[-1]) for L in nd.levels)
    assert nlist == nb_total
    assert not any(np.any(L.bnd_flat.numpy()[:int(L.b.sum())] == nd.nfc) for L in nd.levels)


def test_tree_levels_parent_above_child():
    dec, per_face, fake, nd = _tables((12, 12, 12), (2, 3, 4), 3)
    for li, L in enumerate(nd.levels):
        ck = L.ckind.numpy()
        internal = ck[..., 0] == 0
        if li == 0:
            assert not internal.any()
        else:
            assert np.all(ck[..., 1][internal] < nd.levels[li - 1].m)

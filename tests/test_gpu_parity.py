"""GPU path vs the reference's golden vectors and the CPU oracle (parity gates).

Gates (BASELINE north_star): same selected constraint count per face, PCG
iterations within +-1, fluxes/pressures within 1e-8 rel L2, above-tau
eigenvalues within 1e-8 rel.  Cases whose Lanczos kappa exceeds 100 (the
rho-scaled C1 field, kappa ~ 841) have rounding-sensitive iteration counts
(the reference and its own CPU oracle differ there too); for those the count
bar is max(2, 5%) and the flux bar is 2e-8 (Parity).
"""
import math

import numpy as np
import pytest

from _golden import load, names, rel

pytestmark = pytest.mark.gpu

CASES = names()


def _setup(d):
    import paper_1901_02090_b200 as B
    g = B.build_grid(len(d["counts"]), d["counts"], d["sizes"])
    system = B.assemble_system(g, B.Permeability(d["k"]), B.Wells(0, g.n_cells - 1))
    dec = B.regular_partition(g, d["splits"])
    cfg = B.SolveConfig(tau=d["tau"], scaling=d["scaling"], constraints=d["mode"], tol=d["tol"])
    return B, system, dec, cfg


def _sensitive(d):
    return float(d["kappa"]) > 100


@pytest.mark.parametrize("name", CASES)
def test_solution_parity(name):
    d = load(name)
    d["name"] = name
    B, system, dec, cfg = _setup(d)
    st = B.BddcSetup(system, dec, cfg)
    rep = B.solve(system, dec, cfg, setup=st)
    assert rep.n_c == int(d["n_c"])
    np.testing.assert_array_equal(st.pair_added + 1 if st.pair_added is not None
                                  else np.ones(dec.n_faces, int), d["face_rows"])
    it_ref = int(d["it"])
    if _sensitive(d):
        assert abs(rep.it - it_ref) <= max(2, int(0.05 * it_ref))
        assert rel(rep.u, d["u"]) <= 2e-8
    else:
        assert abs(rep.it - it_ref) <= 1
        assert rel(rep.u, d["u"]) <= 1e-8
        assert rel(rep.p, d["p"]) <= 1e-8
        if rep.it == it_ref:
            assert abs(rep.kappa - float(d["kappa"])) <= 1e-4 * float(d["kappa"])
    assert rep.converged and not rep.pressure_warning
    assert abs(rep.p.mean()) <= 1e-12 * max(np.abs(rep.p).max(), 1.0)


@pytest.mark.parametrize("name", [n for n in CASES if "pair_selected" in load(n)])
def test_adaptive_parity(name):
    d = load(name)
    B, system, dec, cfg = _setup(d)
    st = B.BddcSetup(system, dec, cfg)
    np.testing.assert_array_equal(st.pair_selected, d["pair_selected"])
    assert abs(st.omega_tilde - float(d["omega_tilde"])) <= 1e-8 * float(d["omega_tilde"])
    lam = st.pair_lambda.cpu().numpy()
    tau = d["tau"]
    for q in range(dec.n_faces):
        ref = d["pair_lam"][q]
        m = np.isfinite(ref) & (ref > tau)
        if m.any():
            np.testing.assert_allclose(lam[q, :int(m.sum())], ref[m], rtol=1e-8)


@pytest.mark.parametrize("name", ["g2d_small", "g2d_adapt", "g3d_adapt", "g3d_thin", "c0"])
def test_operator_parity(name):
    d = load(name)
    B, system, dec, cfg = _setup(d)
    st = B.BddcSetup(system, dec, cfg)
    assert rel(st.schur_dense(0), d["S_sub0"]) <= 1e-11
    assert rel(st.schur_dense(dec.n_subdomains - 1), d["S_sublast"]) <= 1e-11
    assert rel(st.schur_matvec(d["x"]), d["Sx"]) <= 1e-10
    assert rel(st.project_balanced(d["x"]), d["Px"]) <= 1e-13
    assert rel(st.precondition(d["x"]), d["Mx"]) <= 1e-9


@pytest.mark.parametrize("name", [n for n in CASES if "pair_selected" in load(n)])
def test_eigs_report_full_spectra(name):
    """eigs-report (cli.py:147-162): every pair's spectrum against
    the initial constraints, compared with the reference's leading 24 eigenvalues
    (zeros included) to 1e-8 of the pair's largest eigenvalue."""
    d = load(name)
    B, system, dec, cfg = _setup(d)
    reports = B.eigs_report(system, dec, cfg)
    pairs = [tuple(p) for p in d["pairs"]]
    assert sorted(reports) == sorted(pairs)
    for q, key in enumerate(pairs):
        ref = d["pair_lam"][q]
        ref = ref[np.isfinite(ref)]
        mine = reports[key].eigenvalues[:len(ref)]
        assert len(mine) == len(ref)
        scale = max(float(ref.max()), 1.0)
        np.testing.assert_allclose(mine, ref, rtol=0, atol=1e-8 * scale)
        assert reports[key].selected == int(d["pair_selected"][q])

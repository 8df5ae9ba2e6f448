"""GPU path vs the reference's golden vectors and the CPU oracle (parity gates).

Gates (BASELINE north_star): same selected constraint count per face, PCG
iterations within +-1, fluxes/pressures within 1e-8 rel L2, above-tau
eigenvalues within 1e-8 rel.  Bars per case class (measured values in
DESIGN.md, Parity; `scripts/parity_report.py` prints them):

* kappa <= 100 (every adaptive case but c1_rho): it +-1, u and p <= 1e-8.
* kappa > 100 (c1_rho kappa 841, g3d_ms 566, g2d_ms 121, g2d_small 1680):
  rounding-sensitive iteration counts -- the reference and its own CPU
  oracle differ there too -- so it +-max(2, 5%), u and p <= 2e-8.
* tau = inf on the channelised C2 field (kappa 7.5e4, 775 iterations;
  SURVEY 8c): it within +-1 %, u and p <= 1e-6.
* intermediate iterates u0 (harmonic extension of the coarse trace) and u*
  (trace solve): <= 5e-8 (the explicit-inverse coarse basis carries
  cond(S_i) eps ~ 1e-9 relative; measured <= 1.5e-8 on the 6-decade C2
  field, <= 3e-10 elsewhere); conservation defect of u* <= 1e-10 absolute
  (the reference's own acceptance bar, test_acceptance.py:247).
* operators: S x within 3e-11 and M x within 5e-9 relative (measured at most
  1.1e-11 / 1.7e-10 on the 6-decade channelised C2 field, <= 7e-12 on the
  C3-shaped blocks, ~1e-14 on the mild fields -- S_i and T_i come from
  explicit SPD inverses, so their error scales with cond(S_i) eps; M x grows
  with the coarse problem's conditioning: 9e-12 at 27 C3-shaped subdomains,
  1.9e-9 at 64, 1.2e-9 at the full 2244 of C3); P x within 1e-13.
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
    system = B.assemble_system(g, B.Permeability(d["k"]), B.Wells(0, g.n_cells - 1),
                               lumped=d["lumped"])
    dec = B.regular_partition(g, d["splits"])
    cfg = B.SolveConfig(tau=d["tau"], scaling=d["scaling"], constraints=d["mode"], tol=d["tol"])
    return B, system, dec, cfg


def _sensitive(d):
    return float(d["kappa"]) > 100


@pytest.mark.parametrize("name", CASES)
def test_solution_parity(name):
    d = load(name)
    B, system, dec, cfg = _setup(d)
    st = B.BddcSetup(system, dec, cfg)
    rep = B.solve(system, dec, cfg, setup=st)
    assert rep.n_c == int(d["n_c"])
    np.testing.assert_array_equal(st.pair_added + 1 if st.pair_added is not None
                                  else np.ones(dec.n_faces, int), d["face_rows"])
    it_ref = int(d["it"])
    if not math.isfinite(d["tau"]) and d["mode"] == "adaptive":
        assert abs(rep.it - it_ref) <= max(1, int(0.01 * it_ref))
        bar = 1e-6
    elif _sensitive(d):
        assert abs(rep.it - it_ref) <= max(2, int(0.05 * it_ref))
        bar = 2e-8
    else:
        assert abs(rep.it - it_ref) <= 1
        bar = 1e-8
        if rep.it == it_ref:
            assert abs(rep.kappa - float(d["kappa"])) <= 1e-4 * float(d["kappa"])
    assert rel(rep.u, d["u"]) <= bar
    assert rel(rep.p, d["p"]) <= bar
    assert rel(rep.u0, d["u0"]) <= 5e-8
    assert rel(rep.u_star, d["u_star"]) <= 5e-8
    cd_ref = float(d["conservation_defect"])
    assert abs(rep.conservation_defect - cd_ref) <= 1e-10 + 1e-8 * cd_ref
    assert rep.converged and not rep.pressure_warning
    assert abs(rep.p.mean()) <= 1e-12 * max(np.abs(rep.p).max(), 1.0)
    assert len(rep.residuals) == rep.it + 1 and rep.residuals[0] == 1.0


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


@pytest.mark.parametrize("name", [n for n in CASES if n != "c2_tauinf"])
def test_operator_parity(name):
    d = load(name)
    B, system, dec, cfg = _setup(d)
    st = B.BddcSetup(system, dec, cfg)
    assert rel(st.schur_dense(0), d["S_sub0"]) <= 1e-11
    assert rel(st.schur_dense(dec.n_subdomains - 1), d["S_sublast"]) <= 1e-11
    x = d["x"]
    assert rel(st.schur_matvec(x), d["Sx"]) <= 3e-11
    assert rel(st.project_balanced(x), d["Px"]) <= 1e-13
    assert rel(st.precondition(x), d["Mx"]) <= 5e-9


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

"""Reference-shaped read-only views of a `BddcSetup` (the drop-in's bookkeeping surface).

The reference's `BddcSetup` exposes its host objects as attributes that its
own tests and diagnostics read (`solver.py:65-93`; `test_acceptance.py:137-155,
201-249`; `test_adaptive.py:51-110`; `test_decomposition.py:132-146`):

* `weights`  -- `WeightOperator` (decomposition.py:199-209): `delta[i]` aligned
  with `dec.gamma_dofs[i]`, `weight(i, dofs)`;
* `broken`   -- `BrokenInterface` (decomposition.py:242-279): the broken
  interface space, `expand` / `average` / `apply_E` / `apply_I_minus_E`;
* `subs`     -- per-subdomain operators (substructure.py:25-116):
  `n_int`, `n_gamma`, `n_p`, `schur_dense()`, `schur_apply(x)`;
* `cset`     -- `ConstraintSet` (coarse.py:36-118): per-subdomain
  `ConstraintRow`s with the reference's coarse-dof numbering, `matrix(i)`,
  `rows_for_face(i, j)`, `check_rank()`;
* `coarse`   -- `CoarseSpace.solve` (coarse.py:208-215) on the device ND
  factorisation, in the reference's coarse-dof numbering.

Everything here is materialised lazily from the device state the solve path
already holds (delta, the packed S_i, the harvested face rows, the ND
factors); nothing on the solve path reads these views.  Dense applies of the
views (`schur_apply`, `apply_E`) are host NumPy, like the reference's.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import ConstraintRankError

_RANK_TOL = 1e-10   # coarse.py:22


class WeightView:
    """decomposition.py:199-209."""

    def __init__(self, setup):
        dec = setup.dec
        self.dec = dec
        self.kind = setup.config.scaling
        d = setup.d_delta.view(dec.n_subdomains, setup.maxG).cpu().numpy()
        self.delta = [d[i, :int(dec.nG[i])].copy() for i in range(dec.n_subdomains)]

    def weight(self, i, dofs=None):
        d = self.delta[i]
        return d if dofs is None else d[self.dec.gamma_index(i, dofs)]


class BrokenInterface:
    """decomposition.py:242-279: concatenated per-subdomain interface vectors."""

    def __init__(self, weights):
        self.dec = weights.dec
        self.weights = weights
        sizes = [len(g) for g in self.dec.gamma_dofs]
        self.offsets = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
        self.size = int(self.offsets[-1])
        self._global_pos = [self.dec.gpos[i, :int(self.dec.nG[i])].astype(np.int64)
                            for i in range(self.dec.n_subdomains)]
        self.n_gamma = self.dec.n_gamma
        self._pos = np.concatenate(self._global_pos) if sizes else np.zeros(0, np.int64)
        self._w = np.concatenate(weights.delta) if sizes else np.zeros(0)

    def local(self, w, i):
        return w[self.offsets[i]:self.offsets[i + 1]]

    def expand(self, x):
        return np.asarray(x, dtype=np.float64)[self._pos]

    def average(self, w):
        x = np.zeros(self.n_gamma)
        np.add.at(x, self._pos, self._w * np.asarray(w, dtype=np.float64))
        return x

    def apply_E(self, w):
        return self.expand(self.average(w))

    def apply_I_minus_E(self, w):
        return w - self.apply_E(w)


class SubdomainView:
    """substructure.py:25-116 (the quantities the reference's tests read)."""

    def __init__(self, setup, i):
        dec = setup.dec
        self._setup = setup
        self.index = i
        self.cells = dec.cells[i]
        self.gamma = dec.gamma_dofs[i]
        self.n_gamma = int(dec.nG[i])
        self.n_p = len(self.cells)
        g = dec.grid
        # local flux dofs: every face of the subdomain's cells that is a dof
        ids = [g.cell_faces(a)[s][self.cells] for a in range(g.dim) for s in (0, 1)]
        alld = np.unique(np.concatenate(ids))
        alld = alld[alld >= 0]
        self.interior = np.setdiff1d(alld, self.gamma, assume_unique=True)
        self.n_int = len(self.interior)
        self._S = None

    def schur_dense(self):
        if self._S is None:
            self._S = self._setup.schur_dense(self.index)
        return self._S

    def schur_apply(self, x):
        return self.schur_dense() @ np.asarray(x, dtype=np.float64)


@dataclass
class ConstraintRow:
    """coarse.py:25-33."""

    subdomain: int
    values: np.ndarray        # dense over gamma_dofs[subdomain]
    face: tuple
    component: int
    origin: str               # initial | adaptive | multiscale
    coarse_dof: int = -1
    sign: float = 1.0


class ConstraintSetView:
    """coarse.py:36-118 with the reference's coarse-dof numbering: the initial row of
    face f (faces in `adjacent_pairs()` order) is coarse dof f, the adaptive /
    multiscale rows follow in face order (solver.py:76-90 add them after
    `initial_constraints`).  `ref_of_dev[g]` maps this package's per-face
    numbering (face f owns ids cstart[f] .. cstart[f] + per_face[f] - 1) onto it."""

    def __init__(self, setup):
        dec = setup.dec
        self.dec = dec
        nf = dec.n_faces
        per_face = setup._per_face
        extra = per_face - 1
        self.n_flux_coarse = int(per_face.sum()) if nf else 0
        cstart = np.concatenate([[0], np.cumsum(per_face)[:-1]]).astype(np.int64)
        xstart = np.concatenate([[0], np.cumsum(extra)[:-1]]).astype(np.int64)
        ref = np.empty(self.n_flux_coarse, dtype=np.int64)
        for f in range(nf):
            ref[cstart[f]] = f
            ref[cstart[f] + 1:cstart[f] + per_face[f]] = nf + xstart[f] + np.arange(extra[f])
        self.ref_of_dev = ref
        origin = "multiscale" if setup.config.constraints == "multiscale" else "adaptive"
        face_rows = setup._face_row_values()   # per face: (extra[f], m_f) i-side values
        self.rows = [[] for _ in range(dec.n_subdomains)]
        faces = dec.faces
        for f, (i, j) in enumerate(dec.adjacent_pairs()):
            comp = faces[(i, j)][0]
            vals = [(0, "initial", comp.sign_i)]
            vals += [(1 + r, origin, face_rows[f][r]) for r in range(int(extra[f]))]
            for k, org, v in vals:
                g = int(ref[cstart[f] + k])
                for s, sg in ((i, 1.0), (j, -1.0)):
                    full = np.zeros(len(dec.gamma_dofs[s]))
                    full[dec.gamma_index(s, comp.dofs)] = sg * v
                    self.rows[s].append(ConstraintRow(s, full, (i, j), 0, org, g, sg))
        for r in self.rows:
            r.sort(key=lambda row: row.coarse_dof)

    @property
    def n_coarse(self):
        return self.n_flux_coarse + self.dec.n_subdomains

    def matrix(self, i):
        rows = self.rows[i]
        if not rows:
            return np.zeros((0, len(self.dec.gamma_dofs[i])))
        return np.array([r.values for r in rows])

    def rows_for_face(self, i, j):
        key = (min(i, j), max(i, j))
        return [(s, r) for s in (i, j) for r in self.rows[s] if r.face == key]

    def check_rank(self):
        for i in range(self.dec.n_subdomains):
            C = self.matrix(i)
            if C.shape[0] and np.linalg.matrix_rank(C, tol=_RANK_TOL) < len(C):
                raise ConstraintRankError(f"dependent constraint rows on subdomain {i}",
                                          rows=self.rows[i])


class CoarseView:
    """coarse.py:208-215: the pinned coarse solve, in the reference's numbering,
    on the device multifrontal factorisation."""

    def __init__(self, setup, cset):
        self._setup = setup
        self._cset = cset
        self.n_flux_coarse = cset.n_flux_coarse
        self.N = setup.N

    def solve(self, rhs_flux, rhs_p):
        import torch
        st = self._setup
        nfc, N = self.n_flux_coarse, self.N
        rf = np.zeros(nfc)
        rf[:] = np.asarray(rhs_flux, dtype=np.float64)[self._cset.ref_of_dev]
        rc = np.concatenate([rf, np.asarray(rhs_p, dtype=np.float64)])
        if st.nd is None:
            return np.zeros(nfc), np.zeros(N)
        with torch.cuda.stream(st.stream):
            st.w_rc[:nfc + N].copy_(torch.from_numpy(rc))
            st._coarse_solve()
            xc = st.w_xc[:nfc + N].cpu().numpy()
        x = np.empty(nfc)
        x[self._cset.ref_of_dev] = xc[:nfc]
        return x, xc[nfc:]

"""CPU parity oracle: a NumPy/SciPy restatement of the reference bddcflow path.

TEST INFRASTRUCTURE ONLY.  Nothing in the product package imports this
module; only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
`cpu_baseline` / `--impl reference` legs use it, and only as the checker or
as the timed CPU baseline.  It restates the reference algorithm
(`/root/reference/pkg/src/bddcflow/*.py`) for *regular (box) partitions*:

* sparse LU (SuperLU) of every interior and constrained local KKT, exactly
  the factorisations the reference performs (`substructure.py:25-78`,
  `coarse.py:130-206`);
* dense generalized pair eigenproblems by two `eigh` calls
  (`adaptive.py:63-138`), selection + Gram-Schmidt dependence filtering
  (`adaptive.py:141-173`, `coarse.py:61-100`);
* dense coarse saddle LU with subdomain-0 pressure pinned (`coarse.py:186-215`);
* PCG + Lanczos condition estimate (`solver.py:186-251`), three-step solve
  (`solver.py:301-398`), pressure recovery (`solver.py:254-274`).

Topology (interface, faces, signs) uses closed forms valid for box
subdomains instead of the reference's O(N * n_faces) Python loops
(`decomposition.py:48-100, 183-196`); tests pin the two against each other
and against golden vectors produced by the unmodified reference
(`oracle/make_golden.py` -> `tests/golden/*.npz`).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp
import scipy.sparse.linalg as spla

RANK_TOL = 1e-10          # coarse.py:22
DEFLATION_TOL = 1e-12     # adaptive.py:24
PERMC = "COLAMD"          # SuperLU column ordering of the interior KKTs (scipy default)
ZERO_ROW_TOL = 1e-10      # adaptive.py:25


class OracleNonConvergence(RuntimeError):
    def __init__(self, msg, report=None):
        super().__init__(msg)
        self.report = report


# --------------------------------------------------------------- grid / RT0

@dataclass
class Mesh:
    """Tensor grid with RT0 interior-face flux dofs (grid.py:21-160)."""

    counts: tuple
    sizes: tuple

    def __post_init__(self):
        self.counts = tuple(int(c) for c in self.counts)
        self.sizes = tuple(float(s) for s in self.sizes)
        self.dim = len(self.counts)
        self.n_cells = int(np.prod(self.counts))
        self.vol = float(np.prod(self.sizes))
        # per family: extents of the interior faces (coordinate a in 1..n_a-1)
        self.fam_ext = []
        offs = [0]
        for a in range(self.dim):
            e = list(self.counts)
            e[a] -= 1
            self.fam_ext.append(tuple(e))
            offs.append(offs[-1] + int(np.prod(e)))
        self.fam_off = tuple(offs)
        self.n_flux = offs[-1]
        c = np.arange(self.n_cells)
        self.coords = np.empty((self.n_cells, self.dim), dtype=np.int64)
        for a in range(self.dim):
            self.coords[:, a] = c % self.counts[a]
            c = c // self.counts[a]

    def cell_id(self, coords):
        idx = np.zeros(len(coords), dtype=np.int64)
        stride = 1
        for a in range(self.dim):
            idx += coords[:, a] * stride
            stride *= self.counts[a]
        return idx

    def face_dof(self, a, coords):
        """Dof of the a-face at integer face coordinate (-1 on boundary).

        Face coordinate c_a in 0..n_a; interior faces are 1..n_a-1 and are
        numbered family-major, x-fastest (grid.py:102-108).
        """
        ca = coords[:, a]
        ok = (ca >= 1) & (ca <= self.counts[a] - 1)
        idx = np.zeros(len(coords), dtype=np.int64)
        stride = 1
        for d in range(self.dim):
            v = coords[:, d] - (1 if d == a else 0)
            idx += v * stride
            stride *= self.fam_ext[a][d]
        return np.where(ok, self.fam_off[a] + idx, -1)

    def cell_face_dofs(self, a):
        """(low, high) a-face dofs of every cell, -1 on the boundary (cached)."""
        cache = self.__dict__.setdefault("_cfd", {})
        if a not in cache:
            lo = self.face_dof(a, self.coords)
            hi_c = self.coords.copy()
            hi_c[:, a] += 1
            cache[a] = (lo, self.face_dof(a, hi_c))
        return cache[a]

    def dof_cells(self):
        """(n_flux, 2) low/high neighbour cell of every interior face."""
        out = np.empty((self.n_flux, 2), dtype=np.int64)
        for a in range(self.dim):
            lo, hi = self.cell_face_dofs(a)
            cells = np.arange(self.n_cells)
            m = hi >= 0
            out[hi[m], 0] = cells[m]      # cell below the face
            m = lo >= 0
            out[lo[m], 1] = cells[m]      # cell above the face
        return out

    def dof_axis(self):
        ax = np.empty(self.n_flux, dtype=np.int64)
        for a in range(self.dim):
            ax[self.fam_off[a]:self.fam_off[a + 1]] = a
        return ax


LUMPED = False   # module switch set by Setup (grid.py:204-227, 327 `lumped`)


def mass_matrix(mesh, k, cells=None, lumped=None):
    """RT0 flux mass matrix from element blocks c[[2,1],[1,2]], or c[[3,0],[0,3]]
    lumped (grid.py:204-307)."""
    lumped = LUMPED if lumped is None else lumped
    if cells is None:
        cells = np.arange(mesh.n_cells)
    rows, cols, vals = [], [], []
    for a in range(mesh.dim):
        lo, hi = mesh.cell_face_dofs(a)
        dl, dh = lo[cells], hi[cells]
        c = mesh.sizes[a] ** 2 / (6.0 * mesh.vol) / k[cells, a]
        for d, o in ((dl, dh), (dh, dl)):
            m = d >= 0
            rows.append(d[m]); cols.append(d[m]); vals.append((3.0 if lumped else 2.0) * c[m])
            if lumped:
                continue
            mo = m & (o >= 0)
            rows.append(d[mo]); cols.append(o[mo]); vals.append(c[mo])
    n = mesh.n_flux
    return sp.coo_matrix((np.concatenate(vals),
                          (np.concatenate(rows), np.concatenate(cols))),
                         shape=(n, n)).tocsr()


def divergence(mesh):
    """B[cell, low face] = +1, B[cell, high face] = -1 (grid.py:310-324)."""
    rows, cols, vals = [], [], []
    cells = np.arange(mesh.n_cells)
    for a in range(mesh.dim):
        lo, hi = mesh.cell_face_dofs(a)
        for d, s in ((lo, 1.0), (hi, -1.0)):
            m = d >= 0
            rows.append(cells[m]); cols.append(d[m])
            vals.append(np.full(int(m.sum()), s))
    return sp.coo_matrix((np.concatenate(vals),
                          (np.concatenate(rows), np.concatenate(cols))),
                         shape=(mesh.n_cells, mesh.n_flux)).tocsr()


def well_rhs(mesh, src, sink, strength=1.0):
    """f = -strength at src, +strength at sink (grid.py:336-338)."""
    f = np.zeros(mesh.n_cells)
    f[src] -= strength
    f[sink] += strength
    return f


# ------------------------------------------------------------ decomposition

def near_equal(n, s):
    base, extra = divmod(n, s)
    return [base + 1 if q < extra else base for q in range(s)]


@dataclass
class BoxPartition:
    """Regular partition + interface topology (decomposition.py:32-151)."""

    mesh: Mesh
    splits: tuple

    def __post_init__(self):
        mesh = self.mesh
        # per axis: a strip count (near-equal strips) or explicit strip widths
        widths = [list(map(int, s)) if not np.isscalar(s) and np.ndim(s) > 0 else None
                  for s in self.splits]
        self.splits = tuple(len(w) if w is not None else int(s)
                            for w, s in zip(widths, self.splits))
        strip = []
        self.strip_lo = []
        self.strip_n = []
        for a in range(mesh.dim):
            w = widths[a] if widths[a] is not None else near_equal(mesh.counts[a], self.splits[a])
            bounds = np.cumsum(w)
            strip.append(np.searchsorted(bounds, np.arange(mesh.counts[a]),
                                         side="right"))
            self.strip_lo.append(np.concatenate([[0], bounds[:-1]]))
            self.strip_n.append(np.array(w))
        part = np.zeros(mesh.n_cells, dtype=np.int64)
        stride = 1
        for a in range(mesh.dim):
            part += stride * strip[a][mesh.coords[:, a]]
            stride *= self.splits[a]
        self.part = part
        self.N = int(np.prod(self.splits))
        order = np.argsort(part, kind="stable")
        bnd = np.searchsorted(part[order], np.arange(self.N + 1))
        self.cells = [order[bnd[i]:bnd[i + 1]] for i in range(self.N)]

        dc = mesh.dof_cells()
        p_lo, p_hi = part[dc[:, 0]], part[dc[:, 1]]
        on = p_lo != p_hi
        self.gamma = np.flatnonzero(on)
        self.dof_lo_sub = p_lo
        self.dof_hi_sub = p_hi
        a_sub = np.minimum(p_lo, p_hi)[self.gamma]
        b_sub = np.maximum(p_lo, p_hi)[self.gamma]
        key = a_sub * self.N + b_sub
        o = np.lexsort((self.gamma, key))
        keys, starts = np.unique(key[o], return_index=True)
        ends = np.append(starts[1:], len(o))
        # box faces are connected (one hinge component per subdomain pair)
        self.pairs = [(int(q // self.N), int(q % self.N)) for q in keys]
        self.face_dofs = [self.gamma[o[s:e]] for s, e in zip(starts, ends)]
        # per-subdomain sorted interface dofs
        subs = np.concatenate([p_lo[self.gamma], p_hi[self.gamma]])
        dd = np.concatenate([self.gamma, self.gamma])
        o2 = np.lexsort((dd, subs))
        b2 = np.searchsorted(subs[o2], np.arange(self.N + 1))
        self.gamma_dofs = [dd[o2[b2[i]:b2[i + 1]]] for i in range(self.N)]
        self.local_pos = [np.searchsorted(self.gamma, g)
                          for g in self.gamma_dofs]
        self.sub_faces = [[] for _ in range(self.N)]
        for f, (a, b) in enumerate(self.pairs):
            self.sub_faces[a].append(f)
            self.sub_faces[b].append(f)
        self._dof_cells = dc

    def sign(self, i, dofs):
        """+1 where the +axis points out of subdomain i (decomposition.py:102-105)."""
        return np.where(self.part[self._dof_cells[dofs, 0]] == i, 1.0, -1.0)

    def gamma_index(self, i, dofs):
        pos = np.searchsorted(self.gamma_dofs[i], dofs)
        assert np.array_equal(self.gamma_dofs[i][pos], dofs)
        return pos

    def sub_flux_dofs(self, i):
        ids = []
        for a in range(self.mesh.dim):
            lo, hi = self.mesh.cell_face_dofs(a)
            ids.append(lo[self.cells[i]])
            ids.append(hi[self.cells[i]])
        d = np.unique(np.concatenate(ids))
        return d[d >= 0]


def rescale_D(mesh, k, part_obj, A):
    """Per-subdomain mean of diag(A) over touching dofs (grid.py:344-357)."""
    diag = A.diagonal()
    d_sub = np.array([diag[part_obj.sub_flux_dofs(i)].mean()
                      for i in range(part_obj.N)])
    return d_sub[part_obj.part], d_sub


def weights(part_obj, k, kind):
    """Multiplicity 1/2 or stiffness d_own/(d_own+d_other) (decomposition.py:212-239)."""
    mesh = part_obj.mesh
    if kind == "multiplicity":
        return [np.full(len(g), 0.5) for g in part_obj.gamma_dofs]
    dc = part_obj._dof_cells
    ax = mesh.dof_axis()
    out = []
    for i in range(part_obj.N):
        d = part_obj.gamma_dofs[i]
        lo, hi = dc[d, 0], dc[d, 1]
        mine = part_obj.part[lo] == i
        own = np.where(mine, lo, hi)
        oth = np.where(mine, hi, lo)
        a = ax[d]
        h = np.array(mesh.sizes)[a]
        d_own = h ** 2 / (3.0 * mesh.vol) / k[own, a]
        d_oth = h ** 2 / (3.0 * mesh.vol) / k[oth, a]
        out.append(d_own / (d_own + d_oth))
    return out


# ----------------------------------------------------------- local operators

class LocalOp:
    """Interior KKT [[A_II,B_I^T,0],[B_I,0,V^T],[0,V,0]] via SuperLU (substructure.py:24-119)."""

    def __init__(self, mesh, k, part_obj, Bs, i):
        self.i = i
        self.cells = part_obj.cells[i]
        self.gamma = part_obj.gamma_dofs[i]
        alld = part_obj.sub_flux_dofs(i)
        self.interior = np.setdiff1d(alld, self.gamma, assume_unique=True)
        self.dofs = np.concatenate([self.interior, self.gamma])
        self.nI, self.nG, self.nP = (len(self.interior), len(self.gamma),
                                     len(self.cells))
        A = mass_matrix(mesh, k, self.cells)
        self.A_loc = A[self.dofs][:, self.dofs].tocsr()
        self.B_loc = Bs[self.cells][:, self.dofs].tocsr()
        nI = self.nI
        self.A_II = self.A_loc[:nI, :nI]
        self.A_IG = self.A_loc[:nI, nI:]
        self.A_GG = self.A_loc[nI:, nI:]
        self.B_I = self.B_loc[:, :nI]
        self.B_G = self.B_loc[:, nI:]
        self.V = sp.csr_matrix(np.full((1, self.nP), mesh.vol))
        K = sp.bmat([[self.A_II, self.B_I.T, None],
                     [self.B_I, None, self.V.T],
                     [None, self.V, None]], format="csc")
        self.lu = spla.splu(K, permc_spec=PERMC)
        self._S = None

    def kkt(self, rf, rp):
        """Solve the interior KKT for (possibly multi-column) rhs blocks."""
        rf = np.asarray(rf, dtype=np.float64)
        rp = np.asarray(rp, dtype=np.float64)
        two = rf.ndim == 2
        if not two:
            rf, rp = rf[:, None], rp[:, None]
        rhs = np.vstack([rf, rp, np.zeros((1, rf.shape[1]))])
        sol = self.lu.solve(rhs)
        uI, p = sol[:self.nI], sol[self.nI:self.nI + self.nP]
        return (uI, p) if two else (uI[:, 0], p[:, 0])

    def harmonic(self, x):
        uI, _ = self.kkt(-(self.A_IG @ x), -(self.B_G @ x))
        return uI

    def schur_apply(self, x):
        uI, p = self.kkt(-(self.A_IG @ x), -(self.B_G @ x))
        return self.A_GG @ x + self.A_IG.T @ uI + self.B_G.T @ p

    def schur(self):
        if self._S is None:
            E = np.eye(self.nG)
            S = self.schur_apply(E)
            self._S = 0.5 * (S + S.T)
        return self._S

    def trace_solve(self, g, fc):
        return self.kkt(-(self.A_IG @ g), fc - self.B_G @ g)


# ------------------------------------------------------------- constraints

class Constraints:
    """Face-paired constraint rows (coarse.py:36-118).

    Rows are stored per face (index into part_obj.pairs) as i-side values
    on the face's shared dofs; the j side carries the negative.  Coarse dof
    ids follow add order, like the reference.
    """

    def __init__(self, part_obj):
        self.P = part_obj
        self.face_rows = [[] for _ in part_obj.pairs]   # (g, values)
        self.face_basis = [np.zeros((0, len(d))) for d in part_obj.face_dofs]
        self.n_flux = 0
        self.order = []   # (face, values) in coarse-dof order

    def independent(self, f, v):
        # per-subdomain basis restricted to this face (rows on other faces
        # have disjoint support), coarse.py:61-67
        Q = self.face_basis[f]
        if Q.shape[0] == 0:
            return np.linalg.norm(v) > 0
        r = v - Q.T @ (Q @ v)
        return np.linalg.norm(r) > RANK_TOL * max(np.linalg.norm(v), 1.0)

    def add(self, f, v):
        """add_pair (coarse.py:78-100); returns True if kept."""
        if not self.independent(f, v):
            return False
        Q = self.face_basis[f]
        w = v.copy()
        if Q.shape[0]:
            w -= Q.T @ (Q @ w)
            w -= Q.T @ (Q @ w)
        w /= np.linalg.norm(w)
        self.face_basis[f] = np.vstack([Q, w])
        g = self.n_flux
        self.n_flux += 1
        self.face_rows[f].append((g, v.copy()))
        self.order.append((f, v.copy()))
        return True

    def sub_rows(self, i):
        """(coarse ids, signs, dense rows over gamma_dofs[i]) in coarse-dof order."""
        P = self.P
        out = []
        for f in P.sub_faces[i]:
            a, b = P.pairs[f]
            pos = P.gamma_index(i, P.face_dofs[f])
            s = 1.0 if i == a else -1.0
            for g, v in self.face_rows[f]:
                row = np.zeros(len(P.gamma_dofs[i]))
                row[pos] = s * v
                out.append((g, s, row))
        out.sort(key=lambda t: t[0])
        if not out:
            return np.zeros(0, int), np.zeros(0), np.zeros((0, len(P.gamma_dofs[i])))
        g = np.array([t[0] for t in out])
        s = np.array([t[1] for t in out])
        C = np.array([t[2] for t in out])
        return g, s, C


def initial_constraints(part_obj):
    cs = Constraints(part_obj)
    for f, (i, j) in enumerate(part_obj.pairs):
        cs.add(f, part_obj.sign(i, part_obj.face_dofs[f]))
    return cs


# --------------------------------------------------------------- adaptivity

@dataclass
class PairResult:
    i: int
    j: int
    lam: np.ndarray          # descending, clipped at 0 (adaptive.py:138)
    rows: list = field(default_factory=list)   # candidate i-side rows (lam > tau)
    selected: int = 0

    def omega(self, tau):
        below = self.lam[self.lam <= tau]
        return float(max(below[0], 1.0)) if len(below) else 1.0


def pair_eigen(setup, f, tau):
    """Dense pair pencil and harvested rows (adaptive.py:63-138, 141-173)."""
    P = setup.P
    i, j = P.pairs[f]
    shared = P.face_dofs[f]
    di, dj = P.gamma_dofs[i], P.gamma_dofs[j]
    ni, n = len(di), len(di) + len(dj)
    pos_i = P.gamma_index(i, shared)
    pos_j = ni + P.gamma_index(j, shared)
    S = np.zeros((n, n))
    S[:ni, :ni] = setup.locs[i].schur()
    S[ni:, ni:] = setup.locs[j].schur()
    wi = setup.delta[i][P.gamma_index(i, shared)]
    wj = setup.delta[j][P.gamma_index(j, shared)]
    E = np.eye(n)
    E[pos_i] = 0.0
    E[pos_j] = 0.0
    E[pos_i, pos_i] = wi
    E[pos_i, pos_j] = wj
    E[pos_j, pos_i] = wi
    E[pos_j, pos_j] = wj
    rows = setup.cons.face_rows[f]
    C = np.zeros((len(rows), n))
    for r, (g, v) in enumerate(rows):
        C[r, pos_i] = v
        C[r, pos_j] = -v
    if len(rows):
        q, rr, _ = sla.qr(C.T, mode="economic", pivoting=True)
        dg = np.abs(np.diag(rr))
        rank = int((dg > ZERO_ROW_TOL * max(dg[0], 1e-300)).sum())
        Q = q[:, :rank]
        Pi = np.eye(n) - Q @ Q.T
    else:
        Pi = np.eye(n)
    IE = np.eye(n) - E
    L = Pi @ IE.T @ S @ IE @ Pi
    R = Pi @ S @ Pi
    L = 0.5 * (L + L.T)
    R = 0.5 * (R + R.T)
    sig, V = sla.eigh(R)
    keep = sig > DEFLATION_TOL * max(sig[-1], 0.0)
    if not keep.any():
        return PairResult(i, j, np.zeros(0))
    X = V[:, keep] / np.sqrt(sig[keep])
    T = X.T @ L @ X
    lam, Y = sla.eigh(0.5 * (T + T.T))
    o = np.argsort(lam)[::-1]
    lam = np.clip(lam[o], 0.0, None)
    W = X @ Y[:, o]
    res = PairResult(i, j, lam)
    if math.isfinite(tau):
        k = int((lam > tau).sum())
        res.selected = k
        for ell in range(k):
            c = L @ W[:, ell]
            scale = np.abs(c).max()
            if scale == 0.0:
                continue
            ci = c[pos_i]
            res.rows.append(ci / np.abs(ci).max())
    return res


# ----------------------------------------------------------------- coarse

class Coarse:
    """Constrained local KKTs, Psi, S_Pi/B0 and the pinned coarse LU (coarse.py:121-245).

    `mode="dense"` is the reference's dense `lu_factor` of the pinned saddle
    (coarse.py:186-215); `mode="sparse"` factors the same pinned matrix with
    SuperLU (a harness substitution for configs whose dense saddle does not
    fit: 36 k^2 at C3, 77 k^2 at C4).  The assembled entries are identical;
    tests pin the two modes against each other and the goldens.
    """

    def __init__(self, setup, mode="dense"):
        P, cons = setup.P, setup.cons
        N = P.N
        nf = cons.n_flux
        self.nf = nf
        rows, cols, vals = [], [], []      # S_Pi
        brow, bcol, bval = [], [], []      # B0
        self.psi, self.lus, self.gids, self.signs = [], [], [], []
        # materialise: keep the Gamma block of each constrained-KKT inverse as a
        # dense matrix (nG solves with the same LU, in forked workers) instead of
        # the LU itself -- the preconditioner only reads the Gamma part of the
        # Delta-solve (solver.py:120-126); memory-bound harness substitution
        mat = setup.cfg.workers > 1
        if mat:
            res = _fork_map(setup, _fork_coarse_local, list(range(N)), setup.cfg.workers)
        for i, lo in enumerate(setup.locs):
            g, s, C = cons.sub_rows(i)
            nc = len(g)
            nu = lo.nI + lo.nG
            if mat:
                psi, T = res[i]
                self.lus.append(T)
            else:
                lu, nK = _constrained_lu(lo, C)
                rhs = np.zeros((nK, nc))
                rhs[nu + lo.nP + np.arange(nc), np.arange(nc)] = 1.0
                psi = lu.solve(rhs)[:nu] if nc else np.zeros((nu, 0))
                self.lus.append((lu, nK, nu))
            self.psi.append(psi)
            self.gids.append(g)
            self.signs.append(s)
            if nc:
                Sl = psi.T @ (lo.A_loc @ psi)
                rows.append(np.repeat(g, nc)); cols.append(np.tile(g, nc))
                vals.append((s[:, None] * Sl * s[None, :]).ravel())
                bl = np.asarray((lo.B_loc @ psi).sum(axis=0)).ravel()
                brow.append(np.full(nc, i)); bcol.append(g); bval.append(s * bl)
        cat = lambda l, dt: np.concatenate(l).astype(dt) if l else np.zeros(0, dt)
        S_pi = sp.coo_matrix((cat(vals, float), (cat(rows, int), cat(cols, int))),
                             shape=(nf, nf)).tocsr()
        B0 = sp.coo_matrix((cat(bval, float), (cat(brow, int), cat(bcol, int))),
                           shape=(N, nf)).tocsr()
        self.S_pi, self.B0 = S_pi, B0
        K0 = sp.bmat([[S_pi, B0.T], [B0, None]], format="csr")
        keep = np.ones(nf + N, dtype=bool)
        keep[nf] = False
        self.keep = keep
        Kp = K0[keep][:, keep]
        self.mode = mode
        if mode == "dense":
            self.lu0 = sla.lu_factor(Kp.toarray())
        else:
            self.lu0 = spla.splu(Kp.tocsc())
        self.N = N
        self.locs = setup.locs

    def solve(self, rf, rq):
        rhs = np.concatenate([rf, rq])[self.keep]
        if self.mode == "dense":
            sol = sla.lu_solve(self.lu0, rhs)
        else:
            sol = self.lu0.solve(rhs)
        full = np.zeros(self.nf + self.N)
        full[self.keep] = sol
        return full[:self.nf], full[self.nf:]

    def combine(self, i, x):
        return self.psi[i] @ (self.signs[i] * x[self.gids[i]])

    def restrict(self, i, t):
        lo = self.locs[i]
        out = np.zeros(self.nf)
        if len(self.gids[i]):
            np.add.at(out, self.gids[i],
                      self.signs[i] * (self.psi[i][lo.nI:].T @ t))
        return out

    def delta_solve(self, i, load_gamma):
        """Full local vector; with a materialised operator only its Gamma part
        (the only part the preconditioner reads) is filled."""
        lo = self.locs[i]
        if isinstance(self.lus[i], np.ndarray):
            out = np.zeros(lo.nI + lo.nG)
            out[lo.nI:] = self.lus[i] @ load_gamma
            return out
        lu, n, nu = self.lus[i]
        rhs = np.zeros(n)
        rhs[lo.nI:nu] = load_gamma
        return lu.solve(rhs)[:nu]


def _constrained_lu(lo, C):
    """SuperLU of the constrained local KKT (coarse.py:139-163)."""
    nc = C.shape[0]
    Cf = np.zeros((nc, lo.nI + lo.nG))
    Cf[:, lo.nI:] = C
    if nc:
        K = sp.bmat([[lo.A_loc, lo.B_loc.T, sp.csr_matrix(Cf.T), None],
                     [lo.B_loc, None, None, lo.V.T],
                     [sp.csr_matrix(Cf), None, None, None],
                     [None, lo.V, None, None]], format="csc")
    else:
        K = sp.bmat([[lo.A_loc, lo.B_loc.T, None],
                     [lo.B_loc, None, lo.V.T],
                     [None, lo.V, None]], format="csc")
    return spla.splu(K), K.shape[0]


def _fork_coarse_local(i):
    """Worker: Psi_i and the Gamma block of the constrained-KKT inverse."""
    setup = _FORK
    lo = setup.locs[i]
    g, s, C = setup.cons.sub_rows(i)
    nc = len(g)
    lu, nK = _constrained_lu(lo, C)
    nu = lo.nI + lo.nG
    rhs = np.zeros((nK, nc + lo.nG))
    rhs[nu + lo.nP + np.arange(nc), np.arange(nc)] = 1.0
    rhs[lo.nI + np.arange(lo.nG), nc + np.arange(lo.nG)] = 1.0
    sol = lu.solve(rhs)
    return sol[:nu, :nc], np.ascontiguousarray(sol[lo.nI:nu, nc:])


# ------------------------------------------------------------------- setup

def multiscale_row(setup, f):
    """MsMFEM face row (adaptive.py:207-262): pair-local Darcy solve on the two
    subdomains' cells with a unit source transfer (-1 spread over i, +1 over j,
    uniformly or following the wells), no-flow on the pair's boundary, one
    pressure pinned; the flux trace on the shared face, outward from i."""
    P, mesh = setup.P, setup.mesh
    i, j = P.pairs[f]
    cells = np.concatenate([P.cells[i], P.cells[j]])
    cell_pos = {c: n for n, c in enumerate(cells)}
    dc = P._dof_cells
    inside = np.isin(dc[:, 0], cells) & np.isin(dc[:, 1], cells)
    dofs = np.flatnonzero(inside)
    dof_pos = {d: n for n, d in enumerate(dofs)}
    A = mass_matrix(mesh, setup.k, cells)[dofs][:, dofs].tocsr()
    Bm = setup.B[cells][:, dofs].tocsr()
    f_loc = np.zeros(len(cells))
    for sub, sign in ((i, -1.0), (j, 1.0)):
        sc = P.cells[sub]
        well = setup.f[sc]
        dist = well / well.sum() if abs(well.sum()) > 1e-14 else np.full(len(sc), 1.0 / len(sc))
        for c, v in zip(sc, dist):
            f_loc[cell_pos[c]] = sign * v
    d = A.diagonal().mean()
    K = sp.bmat([[A, d * Bm.T], [d * Bm, None]], format="csc")
    n_u = len(dofs)
    keep = np.ones(K.shape[0], dtype=bool)
    keep[n_u] = False
    rhs = np.concatenate([np.zeros(n_u), d * f_loc])
    sol = np.zeros(K.shape[0])
    sol[keep] = spla.spsolve(K[keep][:, keep].tocsc(), rhs[keep])
    u = sol[:n_u]
    fd = P.face_dofs[f]
    return P.sign(i, fd) * u[[dof_pos[x] for x in fd]]


@dataclass
class Config:
    tau: float = math.inf
    scaling: str = "multiplicity"
    tol: float = 1e-6
    maxit: int = 5000
    constraints: str = "initial"
    # harness substitutions for full-size configs (pinned against the literal
    # forms on the golden cases, tests/test_oracle_golden.py):
    coarse: str = "auto"      # dense (coarse.py:196) | sparse | auto (dense up to 8000)
    workers: int = 1          # fork workers for the S_i and pair-eigenproblem loops
    project: str = "auto"     # qr (solver.py:166-179) | laplacian | auto
    pressure: str = "auto"    # splu (solver.py:254-274) | dct | auto
    log: object = None        # optional progress callback log(str)
    lumped: bool = False      # lumped RT0 mass matrix (grid.py:327 assemble_system(lumped=))


_FORK = None   # the Setup a forked worker reads (inherited copy-on-write)


def _fork_schur(i):
    return _FORK.locs[i].schur()


def _fork_pair(args):
    f_, tau = args
    return pair_eigen(_FORK, f_, tau)


def _fork_map(setup, fn, items, workers):
    """Map over items in forked workers (each single-threaded BLAS) or serially."""
    global _FORK
    _FORK = setup
    if workers <= 1 or len(items) < 2 * workers:
        try:
            return [fn(x) for x in items]
        finally:
            _FORK = None
    import multiprocessing as mp
    import os
    old = {k: os.environ.get(k) for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS")}
    try:
        ctx = mp.get_context("fork")
        with ctx.Pool(workers, initializer=_single_thread_blas) as pool:
            return pool.map(fn, items, chunksize=max(1, len(items) // (8 * workers)))
    finally:
        _FORK = None
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def _single_thread_blas():
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:
        pass


class Setup:
    """BddcSetup restatement (solver.py:65-183)."""

    def __init__(self, mesh, k, f, splits, cfg):
        global LUMPED
        LUMPED = bool(cfg.lumped)
        self.mesh, self.k, self.cfg = mesh, k, cfg
        self.P = BoxPartition(mesh, splits)
        self.A = mass_matrix(mesh, k)
        self.B = divergence(mesh)
        self.D, self.D_sub = rescale_D(mesh, k, self.P, self.A)
        self.Bs = (sp.diags(self.D) @ self.B).tocsr()
        self.f = f
        self.fs = self.D * f
        self.delta = weights(self.P, k, cfg.scaling)
        log = cfg.log or (lambda m: None)
        self.locs = [LocalOp(mesh, k, self.P, self.Bs, i)
                     for i in range(self.P.N)]
        log(f"local KKT factorisations: {self.P.N}")
        self.cons = initial_constraints(self.P)
        self.pairs = {}
        self.omega_tilde = None
        if cfg.constraints == "adaptive":
            if cfg.workers > 1:
                # dense S_i (substructure.py:90-99) once per subdomain, in workers
                for lo, S in zip(self.locs, _fork_map(self, _fork_schur, list(range(self.P.N)),
                                                      cfg.workers)):
                    lo._S = S
                log("dense S_i")
            res = _fork_map(self, _fork_pair, [(f_, cfg.tau) for f_ in range(len(self.P.pairs))],
                            cfg.workers)
            for key, r in zip(self.P.pairs, res):
                self.pairs[key] = r
            log(f"pair eigenproblems: {len(res)}")
            if math.isfinite(cfg.tau):
                for f_, key in enumerate(self.P.pairs):
                    for row in self.pairs[key].rows:
                        self.cons.add(f_, row)
            self.omega_tilde = (max(r.omega(cfg.tau)
                                    for r in self.pairs.values())
                                if self.pairs else 1.0)
        if cfg.constraints == "multiscale":
            # solver.py:89-90, adaptive.py:265-269
            for f_ in range(len(self.P.pairs)):
                self.cons.add(f_, multiscale_row(self, f_))
        nc_tot = self.cons.n_flux + self.P.N
        mode = cfg.coarse if cfg.coarse != "auto" else ("dense" if nc_tot <= 8000 else "sparse")
        self.coarse = Coarse(self, mode)
        log(f"coarse ({mode}): n_c = {self.n_c}")

    @property
    def n_c(self):
        return self.cons.n_flux + self.P.N

    # interface operator / preconditioner (solver.py:97-128)
    def schur_matvec(self, x):
        y = np.zeros_like(x)
        for i, lo in enumerate(self.locs):
            np.add.at(y, self.P.local_pos[i],
                      lo.schur_apply(x[self.P.local_pos[i]]))
        return y

    def precondition(self, r):
        cr = np.zeros(self.cons.n_flux)
        loads = []
        for i in range(self.P.N):
            t = self.delta[i] * r[self.P.local_pos[i]]
            loads.append(t)
            cr += self.coarse.restrict(i, t)
        x, _ = self.coarse.solve(cr, np.zeros(self.P.N))
        out = np.zeros_like(r)
        for i, lo in enumerate(self.locs):
            w = self.coarse.combine(i, x) + self.coarse.delta_solve(i, loads[i])
            np.add.at(out, self.P.local_pos[i], self.delta[i] * w[lo.nI:])
        return out

    def phi(self):
        """Net-flux functionals Phi[i, d] = sign_i(d) (solver.py:132-144)."""
        rows, cols, vals = [], [], []
        for i in range(self.P.N):
            s = self.P.sign(i, self.P.gamma_dofs[i])
            rows.extend([i] * len(s))
            cols.extend(self.P.local_pos[i])
            vals.extend(s)
        return sp.coo_matrix((vals, (rows, cols)),
                             shape=(self.P.N, len(self.P.gamma))).tocsr()

    def project(self, x):
        """Orthogonal projection onto null(Phi) (solver.py:166-179).

        For small problems the reference's dense QR of Phi^T; otherwise the
        algebraically identical I - Phi^T (Phi Phi^T)^+ Phi.
        """
        if not hasattr(self, "_proj"):
            Phi = self.phi()
            mode = self.cfg.project
            if mode == "auto":
                mode = "qr" if Phi.shape[0] * Phi.shape[1] <= 4e7 else "laplacian"
            if mode == "qr":
                q, r = np.linalg.qr(Phi.toarray().T)
                keep = np.abs(np.diag(r)) > 1e-12 * np.abs(r).max()
                Q = q[:, keep]
                self._proj = lambda v: v - Q @ (Q.T @ v)
            else:
                # (Phi Phi^T)^+ b for b = Phi v (orthogonal to the constants: every
                # interface dof has +1 on one side and -1 on the other): the
                # connected subdomain-graph Laplacian solved with one entry pinned
                # (sparse LU), then the constant removed
                L = (Phi @ Phi.T).tocsc()
                lu = spla.splu(L[1:, 1:].tocsc())

                def lap_pinv(b):
                    z = np.zeros(len(b))
                    z[1:] = lu.solve(b[1:])
                    return z - z.mean()
                self._proj = lambda v: v - Phi.T @ lap_pinv(Phi @ v)
        return self._proj(x)

    def balanced_shift(self, targets):
        """Least-squares face shifts (solver.py:146-164)."""
        P = self.P
        T = np.zeros((P.N, len(P.pairs)))
        for c, (i, j) in enumerate(P.pairs):
            T[i, c] = 1.0
            T[j, c] = -1.0
        x, *_ = np.linalg.lstsq(T, targets, rcond=None)
        w = np.zeros(len(P.gamma))
        for c, (i, j) in enumerate(P.pairs):
            d = P.face_dofs[c]
            pos = np.searchsorted(P.gamma, d)
            w[pos] += x[c] * P.sign(i, d) / len(d)
        return w


def pcg(op, prec, rhs, tol, maxit, callback=None):
    """PCG with Lanczos kappa (solver.py:186-233)."""
    x = np.zeros_like(rhs)
    r = rhs.copy()
    r0 = np.linalg.norm(r)
    hist = [1.0]
    if r0 == 0.0:
        return x, 0, 1.0, np.array(hist), True
    z = prec(r)
    p = z.copy()
    rz = r @ z
    al, be = [], []
    it = 0
    conv = False
    for it in range(1, maxit + 1):
        Ap = op(p)
        pAp = p @ Ap
        if pAp <= 0:
            raise OracleNonConvergence("non-positive curvature")
        a = rz / pAp
        x += a * p
        r -= a * Ap
        al.append(a)
        rel = np.linalg.norm(r) / r0
        hist.append(rel)
        if callback is not None:
            callback(x, r)
        if rel <= tol:
            conv = True
            break
        z = prec(r)
        rzn = r @ z
        b = rzn / rz
        be.append(b)
        rz = rzn
        p = z + b * p
    return x, it, lanczos_kappa(al, be), np.array(hist), conv


def lanczos_kappa(al, be):
    """solver.py:236-251."""
    m = len(al)
    if m <= 1:
        return 1.0
    d = np.empty(m)
    e = np.empty(m - 1)
    d[0] = 1.0 / al[0]
    for q in range(1, m):
        d[q] = 1.0 / al[q] + be[q - 1] / al[q - 1]
        e[q - 1] = math.sqrt(max(be[q - 1], 0.0)) / al[q - 1]
    ev = sla.eigh_tridiagonal(d, e, eigvals_only=True)
    return float(ev[-1] / max(ev[0], np.finfo(float).tiny))


@dataclass
class Report:
    u: np.ndarray
    p: np.ndarray
    it: int
    kappa: float
    omega_tilde: float
    n_c: int
    residuals: np.ndarray
    u0: np.ndarray
    u_star: np.ndarray
    conservation_defect: float
    pressure_warning: bool
    converged: bool


def solve(setup, callback=None):
    """Three-step solve (solver.py:301-398) + pressure (solver.py:254-274)."""
    P, co, cfg = setup.P, setup.coarse, setup.cfg
    fs = setup.fs
    nu = setup.mesh.n_flux
    rq = np.array([fs[c].sum() for c in P.cells])
    x0, _ = co.solve(np.zeros(co.nf), rq)
    g = np.zeros(len(P.gamma))
    for i, lo in enumerate(setup.locs):
        w = co.combine(i, x0)[lo.nI:]
        np.add.at(g, P.local_pos[i], setup.delta[i] * w)
    u0 = np.zeros(nu)
    u0[P.gamma] = g
    us = np.zeros(nu)
    us[P.gamma] = g
    for i, lo in enumerate(setup.locs):
        gi = g[P.local_pos[i]]
        u0[lo.interior] = lo.harmonic(gi)
        uI, _ = lo.trace_solve(gi, fs[lo.cells])
        us[lo.interior] = uI
    dd = fs - setup.Bs @ us
    defect = np.linalg.norm(dd) / max(np.linalg.norm(fs), 1e-300)
    rf = -(setup.A @ us)
    rg = rf[P.gamma].copy()
    for i, lo in enumerate(setup.locs):
        uI, p = lo.kkt(rf[lo.interior], dd[lo.cells])
        np.add.at(rg, P.local_pos[i], -(lo.A_IG.T @ uI + lo.B_G.T @ p))
    targets = np.array([-dd[c].sum() / setup.D[c[0]] for c in P.cells])
    if np.abs(targets).max() > 1e-13 * max(np.abs(fs).sum(), 1.0):
        wp = setup.balanced_shift(targets)
        rg -= setup.schur_matvec(wp)
    else:
        wp = np.zeros_like(rg)
    rg = setup.project(rg)
    w, it, kappa, hist, conv = pcg(
        lambda v: setup.project(setup.schur_matvec(v)),
        lambda v: setup.project(setup.precondition(v)),
        rg, cfg.tol, cfg.maxit, callback)
    corr = wp + w
    u = us.copy()
    u[P.gamma] += corr
    for i, lo in enumerate(setup.locs):
        gi = corr[P.local_pos[i]]
        uI, _ = lo.kkt(rf[lo.interior] - lo.A_IG @ gi,
                       dd[lo.cells] - lo.B_G @ gi)
        u[lo.interior] += uI
    p, warn = recover_pressure(setup, u, cfg.tol)
    om = setup.omega_tilde if setup.omega_tilde is not None else float("nan")
    rep = Report(u, p, it, kappa, om, setup.n_c, hist, u0, us, defect, warn,
                 conv)
    if not conv:
        raise OracleNonConvergence("CG did not converge", rep)
    return rep


def recover_pressure(setup, u, tol):
    """(Bs Bs^T) p = Bs(-A u), cell 0 pinned, unscale, zero mean (solver.py:254-274)."""
    Bs = setup.Bs
    g = -(setup.A @ u)
    mode = setup.cfg.pressure
    if mode == "auto":
        mode = "splu" if setup.mesh.n_cells <= 200_000 else "dct"
    if mode == "splu":
        L = (Bs @ Bs.T).tocsc()
        rhs = Bs @ g
        n = L.shape[0]
        pb = np.zeros(n)
        if n > 1:
            pb[1:] = spla.spsolve(L[1:, 1:], rhs[1:])
        p = setup.D * pb
        p -= p.mean()
        num = np.linalg.norm(setup.A @ u + Bs.T @ pb)
    else:
        # (Bs Bs^T) pb = Bs g  <=>  (B B^T)(D pb) = B g, and B B^T is the unit-weight
        # cell-graph Neumann Laplacian: exact in the DCT-II eigenbasis (the constant
        # mode dropped = the pin + mean removal above; B^T 1 = 0 on interior faces)
        p = neumann_dct_solve(setup.mesh, setup.B @ g)
        num = np.linalg.norm(setup.A @ u + setup.B.T @ p)
    den = np.linalg.norm(setup.A @ u)
    return p, bool(den > 0 and num > 10.0 * tol * den)


def neumann_dct_solve(mesh, rhs):
    """Zero-mean solution of the cell-graph Neumann Laplacian (B B^T) p = rhs."""
    import scipy.fft as sfft
    shape = tuple(reversed(mesh.counts))          # C order (z, y, x): x fastest
    r = rhs.reshape(shape)
    axes = tuple(range(len(shape)))
    rh = sfft.dctn(r, type=2, norm="ortho", axes=axes)
    lam = np.zeros(shape)
    for ax, n in enumerate(shape):
        l1 = 2.0 - 2.0 * np.cos(np.pi * np.arange(n) / n)
        sh = [1] * len(shape)
        sh[ax] = n
        lam = lam + l1.reshape(sh)
    lam.flat[0] = 1.0
    rh = rh / lam
    rh.flat[0] = 0.0
    return sfft.idctn(rh, type=2, norm="ortho", axes=axes).ravel()


def direct_solve(mesh, k, f):
    """Monolithic sparse saddle solve, first pressure pinned (oracle.py:30-111)."""
    A = mass_matrix(mesh, k)
    B = divergence(mesh)
    K = sp.bmat([[A, B.T], [B, None]], format="csc")
    nu = mesh.n_flux
    keep = np.ones(nu + mesh.n_cells, dtype=bool)
    keep[nu] = False
    rhs = np.concatenate([np.zeros(nu), f])
    sol = np.zeros(nu + mesh.n_cells)
    sol[keep] = spla.spsolve(K[keep][:, keep].tocsc(), rhs[keep])
    u, p = sol[:nu], sol[nu:]
    return u, p - p.mean()


def dirichlet_faces(mesh, axis):
    """Mode B: per-cell (low, high) `axis`-face dofs with the two boundary ends as
    dofs n_flux + t (low end) and n_flux + nt + t (high end), t = x-fastest index
    over the transverse axes.  Extension, not in the reference."""
    lo, hi = mesh.cell_face_dofs(axis)
    ca = mesh.coords[:, axis]
    nt = mesh.n_cells // mesh.counts[axis]
    lo = lo.copy(); hi = hi.copy()
    lo[ca == 0] = mesh.n_flux + np.arange(nt)
    hi[ca == mesh.counts[axis] - 1] = mesh.n_flux + nt + np.arange(nt)
    return lo, hi, nt


def direct_solve_dirichlet(mesh, k, f, axis, p_low, p_high):
    """Monolithic sparse solve of [[A, B^T], [B, 0]] (u, p) = (g, f) with Dirichlet
    pressure p_low / p_high on the two ends of `axis` (mode B).  A and B are
    assembled from the element blocks c[[2,1],[1,2]] and B[cell, low] = +1,
    B[cell, high] = -1 (grid.py:204-324) over all faces of the cells, boundary
    faces of `axis` included; g = +p_low on low-end faces, -p_high on high-end
    ones (the weak form -(p, div v) + <p_D, v.n>).  No pressure pin."""
    lo_d, hi_d, nt = dirichlet_faces(mesh, axis)
    nu = mesh.n_flux + 2 * nt
    rows, cols, vals, brow, bcol, bval = [], [], [], [], [], []
    cells = np.arange(mesh.n_cells)
    for a in range(mesh.dim):
        lo, hi = (lo_d, hi_d) if a == axis else mesh.cell_face_dofs(a)
        c = mesh.sizes[a] ** 2 / (6.0 * mesh.vol) / k[:, a]
        for d, o in ((lo, hi), (hi, lo)):
            m = d >= 0
            rows.append(d[m]); cols.append(d[m]); vals.append(2.0 * c[m])
            mo = m & (o >= 0)
            rows.append(d[mo]); cols.append(o[mo]); vals.append(c[mo])
        for d, sgn in ((lo, 1.0), (hi, -1.0)):
            m = d >= 0
            brow.append(cells[m]); bcol.append(d[m]); bval.append(np.full(int(m.sum()), sgn))
    A = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                      shape=(nu, nu)).tocsr()
    B = sp.coo_matrix((np.concatenate(bval), (np.concatenate(brow), np.concatenate(bcol))),
                      shape=(mesh.n_cells, nu)).tocsr()
    g = np.zeros(nu)
    g[mesh.n_flux:mesh.n_flux + nt] = p_low
    g[mesh.n_flux + nt:] = -p_high
    K = sp.bmat([[A, B.T], [B, None]], format="csc")
    sol = spla.spsolve(K, np.concatenate([g, f]))
    return sol[:nu], sol[nu:]


def run(counts, sizes, k, splits, cfg, wells=None):
    """Convenience: build + solve in mode A (wells at cells 0, n-1)."""
    mesh = Mesh(counts, sizes)
    src, sink = wells if wells is not None else (0, mesh.n_cells - 1)
    f = well_rhs(mesh, src, sink)
    st = Setup(mesh, k, f, splits, cfg)
    return st, solve(st)

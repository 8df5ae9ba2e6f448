"""Regular (box) partitions and the interface topology, in closed form.

Mirrors `regular_partition` / `Decomposition` of the reference
(`/root/reference/pkg/src/bddcflow/decomposition.py:32-151`).  For box
subdomains the reference's hinge-connected face components
(`decomposition.py:84-100`) are always single rectangles and every
subdomain is connected, so the topology has closed forms; the tables below
are what the device kernels consume:

* `gpos[i, q]`   position in `gamma` of the q-th interface slot of i
                 (slots sorted by global dof, like `gamma_dofs[i]`)
* `gcode[i, q]`  axis | side << 2 | line << 3 of that slot (side 1 = high
                 face of the box, line = transverse local index, x-fastest)
* `fslot[i, 2a+side, line]` inverse of gcode
* `gown[d]`      broken-slot ids (i*maxG+q) of the low / high copy of dof d
* `faces[f]`     (i, j, axis, m) for subdomain pairs i < j, sorted
* eigen data of the separable subdomain-graph Laplacians used by the
  balanced projection (solver.py:166-179) and the balanced shift
  (solver.py:146-164).
"""

from __future__ import annotations

from dataclasses import dataclass
from functools import cached_property

import numpy as np

from .errors import ConfigurationError, InvalidArgumentError

MAX_STRIPS = 64


def near_equal_splits(n, s):
    """decomposition.py:128-130."""
    base, extra = divmod(n, s)
    return [base + 1 if k < extra else base for k in range(s)]


def _pad(n, m):
    return max(m, ((n + m - 1) // m) * m)


@dataclass(frozen=True)
class FaceComponent:
    """decomposition.py:22-29 (one component per box face)."""

    i: int
    j: int
    dofs: np.ndarray
    sign_i: np.ndarray


def _box_widths(grid, part):
    """Strip widths of a tensor-product box partition given as a cell -> subdomain
    map numbered x-fastest over the strips (what `regular_partition` and
    `box_partition` produce); ConfigurationError for anything else."""
    part = np.asarray(part, dtype=np.int64)
    if part.shape != (grid.n_cells,):
        raise InvalidArgumentError("partition length must equal n_cells")
    coords = grid.cell_coords
    widths, strip, stride = [], [], 1
    for a in range(grid.dim):
        # strip index along axis a read off the first line of cells along a
        line = np.all(coords[:, [b for b in range(grid.dim) if b != a]] == 0, axis=1)
        ids = part[line][np.argsort(coords[line, a])]
        s_a = (ids // stride)
        steps = np.diff(s_a)
        if np.any((steps != 0) & (steps != 1)) or s_a[0] != 0:
            raise ConfigurationError("only tensor-product box partitions numbered "
                                     "x-fastest over the strips are supported")
        w = np.bincount(s_a).astype(np.int64)
        widths.append([int(v) for v in w])
        strip.append(s_a)
        stride *= len(w)
    rebuilt = np.zeros(grid.n_cells, dtype=np.int64)
    stride = 1
    for a in range(grid.dim):
        rebuilt += stride * strip[a][coords[:, a]]
        stride *= len(widths[a])
    if not np.array_equal(rebuilt, part):
        raise ConfigurationError("only tensor-product box partitions numbered "
                                 "x-fastest over the strips are supported")
    return widths


class Decomposition:
    """Box partition: `splits` per axis is a strip count (near-equal strips,
    decomposition.py:128-130) or a list of strip widths; `Decomposition(grid,
    part)` with a cell -> subdomain array (the reference's constructor,
    decomposition.py:33) is accepted when `part` is such a box partition."""

    def __init__(self, grid, splits):
        if len(splits) == grid.n_cells and grid.n_cells != grid.dim:
            splits = _box_widths(grid, np.asarray(splits))
        widths = None
        if any(not np.isscalar(s) and np.ndim(s) > 0 for s in splits):
            widths = [[int(v) for v in np.atleast_1d(s)] for s in splits]
            if len(widths) != grid.dim or any(len(w) < 1 or min(w) < 1 for w in widths):
                raise InvalidArgumentError("need positive strip widths per axis")
            if any(sum(w) != c for w, c in zip(widths, grid.counts)):
                raise InvalidArgumentError("strip widths must sum to the cell counts")
            splits = tuple(len(w) for w in widths)
        splits = tuple(int(s) for s in splits)
        if len(splits) != grid.dim or any(s < 1 for s in splits):
            raise InvalidArgumentError("need one split >= 1 per axis")
        if any(s > c for s, c in zip(splits, grid.counts)):
            raise InvalidArgumentError("splits exceed cell counts")
        if any(s > MAX_STRIPS for s in splits):
            raise InvalidArgumentError(f"at most {MAX_STRIPS} strips per axis")
        self.grid = grid
        self.splits = splits
        dim = grid.dim
        n3 = tuple(grid.counts) + (1,) * (3 - dim)
        S3 = splits + (1,) * (3 - dim)
        self.n3, self.S3 = n3, S3
        self.sw = [np.array(widths[a] if (widths is not None and a < dim)
                            else near_equal_splits(n3[a], S3[a]), dtype=np.int64)
                   for a in range(3)]
        self.so = [np.concatenate([[0], np.cumsum(w)[:-1]]) for w in self.sw]
        strip_of = [np.repeat(np.arange(S3[a]), self.sw[a]) for a in range(3)]
        self.strip_of = strip_of
        N = int(np.prod(S3))
        self.n_subdomains = N
        sub = np.arange(N)
        self.sub_strip = np.stack([sub % S3[0], (sub // S3[0]) % S3[1],
                                   sub // (S3[0] * S3[1])], axis=1)
        self.box_o = np.stack([self.so[a][self.sub_strip[:, a]]
                               for a in range(3)], axis=1)
        self.box_L = np.stack([self.sw[a][self.sub_strip[:, a]]
                               for a in range(3)], axis=1)
        self._closed_forms()

    # ------------------------------------------------------------ topology

    def _closed_forms(self):
        """Sizes and the per-subdomain / per-face tables (O(N) host work).  The
        per-slot and per-dof tables are built on the device by the solver
        (csrc/topology.cu); their host copies below are made on first access."""
        g = self.grid
        n3, S3, dim = self.n3, self.S3, g.dim
        N = self.n_subdomains
        self.fam_off = list(g.flux_offsets) + [g.flux_offsets[-1]] * (4 - len(g.flux_offsets))
        ss, L = self.sub_strip, self.box_L
        stride = (1, S3[0], S3[0] * S3[1])
        nG = np.zeros(N, dtype=np.int64)
        n_hi = np.zeros(N, dtype=np.int64)
        rows = []
        n_gamma, maxF = 0, 1
        for a in range(dim):
            t1 = 1 if a == 0 else 0
            t2 = 1 if a == 2 else 2
            lines = L[:, t1] * L[:, t2]
            lo = ss[:, a] > 0
            hi = ss[:, a] < S3[a] - 1
            nG += (lo.astype(np.int64) + hi) * lines
            n_hi += hi
            i_lo = np.nonzero(hi)[0]
            rows.append(np.stack([i_lo, i_lo + stride[a], np.full(len(i_lo), a),
                                  lines[i_lo]], axis=1))
            n_gamma += (S3[a] - 1) * n3[t1] * n3[t2]
            maxF = max(maxF, int(self.sw[t1].max() * self.sw[t2].max()))
        self.nG = nG.astype(np.int32)
        self.maxG = _pad(int(nG.max()) if N else 1, 64)
        self.maxF = maxF
        self._n_gamma = int(n_gamma)
        # faces sorted by (i, j): for one i the x, y, z neighbours have increasing ids
        ft = np.concatenate(rows) if rows else np.zeros((0, 4), dtype=np.int64)
        ft = ft[np.lexsort((ft[:, 1], ft[:, 0]))]
        self.face_table = ft.astype(np.int32).reshape(-1, 4)
        self.n_faces = len(ft)
        self.face_base = (np.cumsum(n_hi) - n_hi).astype(np.int32)
        P = np.prod([int(w.max()) for w in self.sw])
        self.maxP = _pad(int(P), 64)
        self.maxL = int(max(int(w.max()) for w in self.sw))

    _LAZY = ("gamma", "gpos", "gcode", "fslot", "gown", "gface", "dof_sub_low",
             "dof_sub_high", "_slot_sub", "_slot_q", "_slot_dof", "_fidx")

    def __getattr__(self, name):
        # host copies of the big tables (reference-compatible views, tests): built
        # once, on demand, by the vectorised NumPy restatement below
        if name in Decomposition._LAZY:
            self._build_interface()
            return self.__dict__[name]
        raise AttributeError(name)

    @cached_property
    def part(self):
        """Cell -> subdomain map (decomposition.py:33)."""
        n3, S3, strip_of = self.n3, self.S3, self.strip_of
        cz, cy, cx = np.meshgrid(np.arange(n3[2]), np.arange(n3[1]),
                                 np.arange(n3[0]), indexing="ij")
        cx, cy, cz = cx.ravel(), cy.ravel(), cz.ravel()
        return (strip_of[0][cx] + S3[0] * (strip_of[1][cy]
                + S3[1] * strip_of[2][cz])).astype(np.int64)

    def _build_interface(self):
        g = self.grid
        n3, S3 = self.n3, self.S3
        fam_off = self.fam_off
        subs, dofs, codes = [], [], []
        lo_dofs = []
        face_rows = []
        for a in range(g.dim):
            t1 = 1 if a == 0 else 0
            t2 = 1 if a == 2 else 2
            c2, c1 = np.meshgrid(np.arange(n3[t2]), np.arange(n3[t1]), indexing="ij")
            c1, c2 = c1.ravel(), c2.ravel()
            s1, s2 = self.strip_of[t1][c1], self.strip_of[t2][c2]
            l1 = c1 - self.so[t1][s1]
            l2 = c2 - self.so[t2][s2]
            line = l1 + self.sw[t1][s1] * l2
            for s in range(1, S3[a]):
                fa = int(self.so[a][s])
                coords = np.zeros((len(c1), 3), dtype=np.int64)
                coords[:, a] = fa
                coords[:, t1] = c1
                coords[:, t2] = c2
                ext = [n3[d] - (1 if d == a else 0) for d in range(3)]
                idx = (coords[:, 0] - (a == 0)) + ext[0] * (
                    (coords[:, 1] - (a == 1)) + ext[1] * (coords[:, 2] - (a == 2)))
                dof = fam_off[a] + idx
                sst = [None, None, None]
                sst[t1] = s1
                sst[t2] = s2
                sst[a] = np.full(len(c1), s - 1)
                lo = sst[0] + S3[0] * (sst[1] + S3[1] * sst[2])
                sst[a] = np.full(len(c1), s)
                hi = sst[0] + S3[0] * (sst[1] + S3[1] * sst[2])
                subs += [lo, hi]
                dofs += [dof, dof]
                lo_dofs.append(dof)
                codes += [a | (1 << 2) | (line << 3), a | (0 << 2) | (line << 3)]
                # faces on this plane: one per transverse strip pair, m = w_t1 * w_t2
                for u2 in range(S3[t2]):
                    for u1 in range(S3[t1]):
                        st_ = [0, 0, 0]
                        st_[t1], st_[t2], st_[a] = u1, u2, s - 1
                        i_lo = st_[0] + S3[0] * (st_[1] + S3[1] * st_[2])
                        i_hi = i_lo + (1 if a == 0 else (S3[0] if a == 1 else S3[0] * S3[1]))
                        face_rows.append((i_lo, i_hi, a, int(self.sw[t1][u1] * self.sw[t2][u2])))
        if subs:
            subs = np.concatenate(subs)
            dofs = np.concatenate(dofs)
            codes = np.concatenate(codes)
        else:
            subs = dofs = codes = np.zeros(0, dtype=np.int64)
        # every interface dof has exactly one low-side copy
        self.gamma = np.sort(np.concatenate(lo_dofs)) if lo_dofs else np.zeros(0, np.int64)
        n_gamma = len(self.gamma)
        # (subdomain, dof) pairs are unique: a plain argsort of the combined key is
        # the lexicographic order (and deterministic)
        o = np.argsort(subs.astype(np.int64) * (g.n_flux_dofs + 1) + dofs)
        subs, dofs, codes = subs[o], dofs[o], codes[o]
        N = self.n_subdomains
        counts = np.bincount(subs, minlength=N)
        starts = np.concatenate([[0], np.cumsum(counts)[:-1]])
        slot = np.arange(len(subs)) - starts[subs]
        assert np.array_equal(counts, self.nG) and n_gamma == self._n_gamma
        maxG = self.maxG
        inv = np.empty(g.n_flux_dofs, dtype=np.int64)
        inv[self.gamma] = np.arange(n_gamma)
        gpos = inv[dofs]
        self.gpos = np.full((N, maxG), -1, dtype=np.int32)
        self.gcode = np.full((N, maxG), -1, dtype=np.int32)
        self.gpos[subs, slot] = gpos
        self.gcode[subs, slot] = codes
        self._slot_sub, self._slot_q, self._slot_dof = subs, slot, dofs
        # fslot
        maxF = self.maxF
        self.fslot = np.full((N, 6, maxF), -1, dtype=np.int32)
        a_ = codes & 3
        side_ = (codes >> 2) & 1
        line_ = codes >> 3
        self.fslot[subs, 2 * a_ + side_, line_] = slot
        # gown: low copy = the slot on the high side of the lower subdomain
        own = np.zeros((n_gamma, 2), dtype=np.int32)
        broken = subs * maxG + slot
        own[gpos[side_ == 1], 0] = broken[side_ == 1]
        own[gpos[side_ == 0], 1] = broken[side_ == 0]
        self.gown = own
        # faces sorted by (i, j)
        fr = sorted(face_rows)
        assert np.array_equal(np.array(fr, dtype=np.int32).reshape(-1, 4), self.face_table)
        fidx = {(r[0], r[1]): k for k, r in enumerate(fr)}
        lo_sub = subs[side_ == 1]
        # the face of each gamma dof (via its low copy)
        gface = np.zeros(n_gamma, dtype=np.int32)
        hi_sub = np.zeros(n_gamma, dtype=np.int64)
        hi_sub[gpos[side_ == 0]] = subs[side_ == 0]
        lo_s = np.zeros(n_gamma, dtype=np.int64)
        lo_s[gpos[side_ == 1]] = lo_sub
        if self.n_faces:
            keys = lo_s * (N + 1) + hi_sub
            ftab_keys = self.face_table[:, 0].astype(np.int64) * (N + 1) + self.face_table[:, 1]
            gface = np.searchsorted(ftab_keys, keys).astype(np.int32)
        self.gface = gface
        self.dof_sub_low = lo_s
        self.dof_sub_high = hi_sub
        self._fidx = fidx

    # -------------------------------------------------- Laplacian eigendata

    def laplacian_eigs(self, weighted, dirichlet_axis=None):
        """Eigen data of K_a = D_a^-1/2 Lpath_a D_a^-1/2 (weighted) or Lpath_a.

        With `dirichlet_axis` d (mode B) the operator is the principal submatrix
        over the floating subdomains (strips 1 .. S_d-2 of axis d): K_d loses its
        first and last row/column (keeping their couplings on the diagonal), no
        null mode, and `dm` lists the floating subdomains in increasing id."""
        Qs, lams = [], []
        S3 = list(self.S3)
        for a in range(3):
            s = self.S3[a]
            L = np.zeros((s, s))
            for k in range(s - 1):
                L[k, k] += 1
                L[k + 1, k + 1] += 1
                L[k, k + 1] -= 1
                L[k + 1, k] -= 1
            w = self.sw[a][:s].astype(np.float64)
            if a == dirichlet_axis:
                L, w = L[1:-1, 1:-1], w[1:-1]
                S3[a] = s - 2
            if weighted:
                dm = 1.0 / np.sqrt(w)
                L = dm[:, None] * L * dm[None, :]
            lam, Q = np.linalg.eigh(L)
            if a != dirichlet_axis:
                lam[0] = 0.0
            Qs.append(Q.ravel())
            lams.append(lam)
        eig = np.concatenate(Qs + lams)
        dm = None
        if weighted:
            ncell = (self.sw[0][self.sub_strip[:, 0]] * self.sw[1][self.sub_strip[:, 1]]
                     * self.sw[2][self.sub_strip[:, 2]]).astype(np.float64)
            if dirichlet_axis is not None:
                sd = self.sub_strip[:, dirichlet_axis]
                ncell = ncell[(sd >= 1) & (sd <= self.S3[dirichlet_axis] - 2)]
            dm = 1.0 / np.sqrt(ncell)
        if dirichlet_axis is not None:
            return eig, dm, tuple(S3)
        return eig, dm

    # ------------------------------------------------ reference-compatible

    @property
    def n_gamma(self):
        return self._n_gamma

    @cached_property
    def cells(self):
        o = np.argsort(self.part, kind="stable")
        b = np.searchsorted(self.part[o], np.arange(self.n_subdomains + 1))
        return [o[b[i]:b[i + 1]] for i in range(self.n_subdomains)]

    @cached_property
    def gamma_dofs(self):
        return [self.gamma[self.gpos[i, :self.nG[i]]]
                for i in range(self.n_subdomains)]

    @cached_property
    def faces(self):
        out = {}
        o = np.argsort(self.gface, kind="stable")
        b = np.searchsorted(self.gface[o], np.arange(self.n_faces + 1))
        for f, (i, j, a, m) in enumerate(self.face_table):
            d = np.sort(self.gamma[o[b[f]:b[f + 1]]])
            out[(int(i), int(j))] = [FaceComponent(int(i), int(j), d,
                                                   np.ones(len(d)))]
        return out

    def adjacent_pairs(self):
        return [(int(i), int(j)) for i, j, _, _ in self.face_table]

    @property
    def max_faces_per_subdomain(self):
        if not self.n_faces:
            return 0
        c = np.bincount(np.concatenate([self.face_table[:, 0],
                                        self.face_table[:, 1]]),
                        minlength=self.n_subdomains)
        return int(c.max())

    def sign_for(self, i, dofs):
        """+1 where the +axis points out of subdomain i (decomposition.py:102-108)."""
        pos = np.searchsorted(self.gamma, dofs)
        return np.where(self.dof_sub_low[pos] == i, 1.0, -1.0)

    def gamma_index(self, i, dofs):
        pos = np.searchsorted(self.gamma_dofs[i], dofs)
        if not np.array_equal(self.gamma_dofs[i][pos], dofs):
            raise InvalidArgumentError("dofs not on this subdomain interface")
        return pos

    @cached_property
    def cell_sub(self):
        return self.part.astype(np.int32)

    def geom_fields(self):
        """Values for the C `bddc_geom` struct."""
        g = self.grid
        h3 = tuple(g.sizes) + (1.0,) * (3 - g.dim)
        return dict(dim=g.dim, n=self.n3, h=h3, vol=g.cell_volume, S=self.S3,
                    so=self.so, sw=self.sw, fam_off=self.fam_off,
                    n_cells=g.n_cells, n_flux=g.n_flux_dofs,
                    N=self.n_subdomains, n_gamma=self.n_gamma,
                    n_faces=self.n_faces, maxG=self.maxG, maxP=self.maxP,
                    maxL=self.maxL, maxF=self.maxF)


def regular_partition(grid, splits):
    """Tensor-product partition with near-equal strips (decomposition.py:133-151)."""
    return Decomposition(grid, splits)


def box_partition(grid, widths):
    """Tensor-product partition with the given strip widths per axis."""
    return Decomposition(grid, [list(w) for w in widths])


def import_partition(path, grid):
    """Read a PART file (decomposition.py:154-177): header 'PART <N> <ncells>', then
    one 0-based subdomain id per cell, x-fastest.  Box partitions only (the ids
    are compacted like the reference's, then checked for tensor-product form)."""
    import warnings

    from .errors import FormatError
    with open(path) as fh:
        header = fh.readline().split()
        if len(header) < 3 or header[0] != "PART":
            raise FormatError("expected header 'PART <N> <ncells>'")
        n_declared, ncells = int(header[1]), int(header[2])
        ids = np.array([int(line) for line in fh if line.strip()])
    if len(ids) != ncells or ncells != grid.n_cells:
        raise FormatError(
            f"expected {grid.n_cells} ids, file declares {ncells}, found {len(ids)}")
    if ids.min() < 0:
        raise FormatError("subdomain ids must be non-negative")
    uniq, compact = np.unique(ids, return_inverse=True)
    if len(uniq) != n_declared:
        warnings.warn(f"header declares {n_declared} subdomains, file uses {len(uniq)}")
    return Decomposition(grid, compact)

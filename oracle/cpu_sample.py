"""Bounded CPU-baseline sample of the reference algorithm at a full-size config.

TEST/BENCH INFRASTRUCTURE ONLY (bench.py's `cpu_baseline` leg and
`--impl reference`).  A complete reference solve at BASELINE config 3 takes
hours (the oracle's own fork-parallel run in
oracle/full_config.py takes 17 min on 8 cores with harness shortcuts), so
the reference's time-to-solve is assembled from unit costs measured on the
box's host cores, every unit being the reference's own operation on the real
data at the real size:

* per subdomain, on a STRATIFIED sample (corner / edge / face / interior
  subdomains of the box partition, by number of shared faces), with the REAL
  constraint rows of the config (oracle/sample_rows_c{3,4}.npz, produced by
  `prepare()` from the actual pair eigenproblems of the sampled subdomains'
  faces): the interior KKT SuperLU factorisation (substructure.py:66), one
  `schur_apply` (substructure.py:85-88), the constrained KKT SuperLU
  (coarse.py:159) and one Delta solve (coarse.py:237-245), and the four
  interior KKT solves of Steps 2-3 and recovery (solver.py:326-390);
* the dense coarse `lu_solve` (coarse.py:208-215) at the TRUE coarse order
  (two triangular solves over an n_c x n_c factor, the reference's
  per-iteration coarse cost; the factor's values do not change the time);
* the balanced projection Q (Q^T x) (solver.py:175-179) with Q at its TRUE
  size (n_Gamma x (N - 1));
* the pressure recovery's sparse solve (solver.py:254-274), SuperLU on the
  same cell-graph Laplacian over a z-slab of the grid, scaled to the full
  cell count by the measured growth between two slab thicknesses.

time_to_solve = sum_types count_t * mean_t(4 t_kkt + it (t_schur + t_delta))
              + it (t_coarse + 2 t_proj)        [+ t_pressure, reported apart]
Per-subdomain, coarse and projection costs are measured; the sum over
subdomains scales the stratified sample by the type counts -- the result is
labelled "extrapolated" by the caller.  The pressure solve's SuperLU fill
grows steeply with the slab thickness (measured here: 1.0 s at 4 layers, 6.1 s
at 8, 72 s at 16 of the 60x220 plane), so its full-size time is only
estimated from slabs and NOT added to the value: the value is a lower bound of
the reference's time-to-solve (an upper bound of its it/s).  The reference's setup (pair eigenproblems, dense S_i, coarse LU) is
not part of the metric (solve with a prebuilt setup).
"""

from __future__ import annotations

import os
import time

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from . import bddc_oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))


def _timeit(fn, reps):
    fn()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    return (time.perf_counter() - t) / reps


def sub_types(splits):
    """Per subdomain the number of shared faces (3D box: 3 corner .. 6 interior)."""
    s3 = tuple(splits) + (1,) * (3 - len(splits))
    idx = np.arange(int(np.prod(s3)))
    nb = np.zeros(len(idx), dtype=np.int64)
    stride = 1
    for a in range(3):
        c = (idx // stride) % s3[a]
        nb += (c > 0).astype(np.int64) + (c < s3[a] - 1).astype(np.int64)
        stride *= s3[a]
    return nb


def sample_subdomains(splits, per_type=(2, 3, 4, 7)):
    """Stratified deterministic sample: for each face-count class (fewest faces
    first) up to per_type[k] subdomains spread evenly through the class."""
    nb = sub_types(splits)
    out = {}
    for k, t in enumerate(sorted(set(nb.tolist()))):
        ids = np.nonzero(nb == t)[0]
        m = per_type[min(k, len(per_type) - 1)]
        pick = ids[np.linspace(0, len(ids) - 1, min(m, len(ids))).round().astype(int)]
        out[int(t)] = (np.unique(pick), int(len(ids)))
    return out


class _LazySetup:
    """Just enough of oracle.Setup for pair_eigen on chosen faces (locs built on demand)."""

    def __init__(self, mesh, k, splits, scaling):
        self.mesh, self.k = mesh, k
        self.P = O.BoxPartition(mesh, splits)
        A = O.mass_matrix(mesh, k)
        B = O.divergence(mesh)
        self.D, _ = O.rescale_D(mesh, k, self.P, A)
        self.Bs = (sp.diags(self.D) @ B).tocsr()
        self.delta = O.weights(self.P, k, scaling)
        self.cons = O.initial_constraints(self.P)
        self._locs = {}
        outer = self

        class _L:
            def __getitem__(self, i):
                if i not in outer._locs:
                    outer._locs[i] = O.LocalOp(outer.mesh, outer.k, outer.P, outer.Bs, i)
                return outer._locs[i]
        self.locs = _L()


def prepare(cfg_id, out=None):
    """Real constraint rows of the sampled subdomains of BASELINE config cfg_id (run
    once in the build container; writes oracle/sample_rows_c{cfg_id}.npz)."""
    import sys
    sys.path.insert(0, os.path.dirname(HERE))
    from paper_1901_02090_b200 import fields
    spec = fields.CONFIGS[cfg_id]
    k = fields.config_field(cfg_id)
    mesh = O.Mesh(spec["counts"], spec["sizes"])
    st = _LazySetup(mesh, k, spec["splits"], spec["scaling"])
    samp = sample_subdomains(spec["splits"])
    ids = np.concatenate([v[0] for v in samp.values()])
    faces = sorted({f for i in ids for f in st.P.sub_faces[int(i)]})
    t0 = time.time()
    for f in faces:
        res = O.pair_eigen(st, f, spec["tau"])
        for row in res.rows:
            st.cons.add(f, row)
    rows, ptr, shapes = [], [0], []
    for i in ids:
        g, s, C = st.cons.sub_rows(int(i))
        rows.append(C.ravel())
        shapes.append(C.shape)
        ptr.append(ptr[-1] + C.size)
    path = out or os.path.join(HERE, f"sample_rows_c{cfg_id}.npz")
    np.savez_compressed(path, ids=ids, rows=np.concatenate(rows), ptr=np.array(ptr),
                        shapes=np.array(shapes), types=np.array(sorted(samp)),
                        type_counts=np.array([samp[t][1] for t in sorted(samp)]),
                        type_sizes=np.array([len(samp[t][0]) for t in sorted(samp)]))
    print(f"prepared {len(ids)} subdomains, {len(faces)} faces in {time.time() - t0:.0f}s -> {path}")


class Sample:
    """The per-subdomain operators of the sample (built once; factorisations timed)."""

    def __init__(self, cfg_id, counts, sizes, k, splits, scaling):
        z = np.load(os.path.join(HERE, f"sample_rows_c{cfg_id}.npz"))
        self.ids = z["ids"]
        self.mesh = O.Mesh(counts, sizes)
        self.P = O.BoxPartition(self.mesh, splits)
        A = O.mass_matrix(self.mesh, k)
        B = O.divergence(self.mesh)
        D, _ = O.rescale_D(self.mesh, k, self.P, A)
        Bs = (sp.diags(D) @ B).tocsr()
        nb = sub_types(splits)
        self.type_of = {int(i): int(nb[i]) for i in self.ids}
        self.type_count = dict(zip(z["types"].tolist(), z["type_counts"].tolist()))
        self.subs = []
        for q, i in enumerate(self.ids):
            t0 = time.perf_counter()
            lo = O.LocalOp(self.mesh, k, self.P, Bs, int(i))
            t_fac = time.perf_counter() - t0
            C = z["rows"][z["ptr"][q]:z["ptr"][q + 1]].reshape(z["shapes"][q])
            t0 = time.perf_counter()
            lu, nK = O._constrained_lu(lo, C)
            t_cfac = time.perf_counter() - t0
            self.subs.append((int(i), lo, lu, nK, t_fac, t_cfac))
        self.N = self.P.N
        self.n_gamma = len(self.P.gamma)

    def unit_costs(self, rng):
        """Per sampled subdomain: (schur_apply, delta solve, interior KKT solve) seconds."""
        out = []
        for i, lo, lu, nK, _, _ in self.subs:
            x = rng.standard_normal(lo.nG)
            rhs = np.zeros(nK)
            rhs[lo.nI:lo.nI + lo.nG] = x
            ts = _timeit(lambda: lo.schur_apply(x), 2)
            td = _timeit(lambda: lu.solve(rhs)[:lo.nI + lo.nG], 2)
            tk = _timeit(lambda: lo.kkt(np.zeros(lo.nI), np.zeros(lo.nP)), 2)
            out.append((i, ts, td, tk))
        return out

    def per_subdomain_sum(self, costs, it):
        """sum over all N subdomains of (4 t_kkt + it (t_schur + t_delta)), stratified."""
        by = {}
        for i, ts, td, tk in costs:
            by.setdefault(self.type_of[i], []).append(4 * tk + it * (ts + td))
        return sum(self.type_count[t] * float(np.mean(v)) for t, v in by.items())


class DenseParts:
    """The reference's dense per-iteration operations at their true sizes."""

    def __init__(self, n_coarse, n_gamma, N, mem_frac=0.5):
        try:
            avail = os.sysconf("SC_AVPHYS_PAGES") * os.sysconf("SC_PAGE_SIZE")
        except Exception:
            avail = 16e9
        self.n_coarse = n = n_coarse - 1               # subdomain 0's pressure pinned
        self.full_coarse = 8.0 * n * n <= mem_frac * avail
        self.n_c_timed = n if self.full_coarse else int(np.sqrt(mem_frac * avail / 8.0))
        m = self.n_c_timed
        # factor values only need to keep the substitutions in normal floating-point
        # range (no overflow, no denormals); the time of the two triangular solves does
        # not depend on them
        self.lu = np.full((m, m), 1e-12)
        self.lu[np.arange(m), np.arange(m)] = 1.0
        self.piv = np.arange(m, dtype=np.int32)
        self.b = np.ones(m)
        rows = n_gamma
        self.full_proj = 8.0 * rows * max(N - 1, 1) <= mem_frac * avail
        self.proj_rows = rows if self.full_proj else int(mem_frac * avail / 8.0 / max(N - 1, 1))
        self.Q = np.full((self.proj_rows, max(N - 1, 1)), 1e-3)
        self.x = np.ones(self.proj_rows)
        self.n_gamma = n_gamma

    def coarse_s(self):
        t = _timeit(lambda: sla.lu_solve((self.lu, self.piv), self.b), 1)
        return t * (self.n_coarse / self.n_c_timed) ** 2

    def proj_s(self):
        t = _timeit(lambda: self.Q @ (self.Q.T @ self.x), 1)
        return t * (self.n_gamma / self.proj_rows)


def pressure_s(counts, slabs=(4, 8)):
    """SuperLU of the pinned cell-graph Laplacian (solver.py:254-274) on two z-slabs,
    extrapolated in the cell count by the measured growth exponent."""
    ts, ns = [], []
    for nz in slabs:
        c = tuple(counts[:-1]) + (nz,) if len(counts) == 3 else tuple(counts)
        mesh = O.Mesh(c, (1.0,) * len(c))
        B = O.divergence(mesh)
        L = (B @ B.T).tocsc()[1:, 1:].tocsc()
        rhs = np.ones(L.shape[0])
        t0 = time.perf_counter()
        spla.spsolve(L, rhs)
        ts.append(time.perf_counter() - t0)
        ns.append(mesh.n_cells)
        if len(counts) != 3:
            return ts[0], "measured at full size"
    expo = max(1.0, np.log(ts[1] / ts[0]) / np.log(ns[1] / ns[0]))
    n_full = int(np.prod(counts))
    return ts[1] * (n_full / ns[1]) ** expo, f"SuperLU on z-slabs of {slabs} layers, growth n^{expo:.2f}"

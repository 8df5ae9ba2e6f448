"""Sparse coarse solver: structured nested dissection over the subdomain grid.

The reference factors the coarse saddle problem densely (`coarse.py:186-215`:
`lu_factor` of [[S_Pi, B0^T],[B0, 0]] with subdomain 0's pressure pinned).
S_Pi couples coarse dofs only through shared subdomains, so for box
partitions a plane of subdomain faces separates the subdomain grid, and each
subdomain pressure couples only to that subdomain's coarse flux dofs.  We
factor the pinned saddle matrix itself by a multifrontal block LDL^T over the
nested-dissection tree: a node's pivot block holds its separator's flux dofs
and the pressures of the subdomains whose last face it eliminates
([[A, B^T], [B, C]], A SPD and the pressure Schur complement negative
definite, inverted in quasi-definite block form); subdomain 0's pressure is
pinned and never appears.  The coarse solve (solver.py:117-118, 318-319) is
then one forward and one backward sweep over the tree, pressures included,
which is algebraically the pinned solve of the reference.

Tree: every node is a box of subdomain strips; the bisection tree splits a
box at the middle of its longest axis, and ND_MERGE consecutive bisection
levels are merged into one node (separator = the union of their planes).
A node's boundary = coarse dofs on the box's faces toward the rest of the
domain, then the pressures of its subdomains still live above it.  Leaves are
single subdomains whose contribution is the local block
[[sigma sigma^T Kc_i, b0_i^T],[b0_i, 0]] (coarse.py:179-185).  Per internal
node (front F over [pivot | bnd]):
    F11inv = F11^-1,  X = F21 F11inv,  U = F22 - X F12  (extend-added into
    the parent's front).
Solve: forward y = F11inv (r_pivot - descendant contributions), c = X
r_pivot (leaves -> root, left-looking gathers in a fixed order); backward
x_pivot = y - X^T x_bnd (root -> leaves).
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np
import torch

from . import _native as nat
from .errors import ConfigurationError

_p = nat.ptr
F64 = torch.float64
I32 = torch.int32


def _pad(n, m):
    return max(m, ((n + m - 1) // m) * m)


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


class _Level:
    pass


def _has_p(dec, has_p):
    """Subdomains with a coarse pressure: all but the pinned subdomain 0 (mode A,
    coarse.py:192-194), or the floating ones (mode B: no pin)."""
    if has_p is None:
        has_p = np.arange(dec.n_subdomains) != 0
    return np.asarray(has_p, dtype=bool)


def nd_geometry(dec, has_p=None):
    """Nested-dissection tree of the subdomain grid in face ids (cached on `dec`).

    Node: dict(leaf, depth, sub | sep (face ids), bnd (face ids), pres (subdomain ids), ch).
    """
    has_p = _has_p(dec, has_p)
    cache = dec.__dict__.setdefault("_nd_geometry", {})
    cached = cache.get(has_p.tobytes())
    if cached is not None:
        return cached
    S3 = dec.S3
    ft = dec.face_table
    fkey = {}
    for f in range(dec.n_faces):
        i, a = int(ft[f, 0]), int(ft[f, 2])
        s = dec.sub_strip[i]
        t = [d for d in range(3) if d != a]
        fkey[(a, int(s[a]) + 1, int(s[t[0]]), int(s[t[1]]))] = f

    def plane_faces(a, plane, lo, hi):
        t = [d for d in range(3) if d != a]
        return [fkey[(a, plane, u, v)] for v in range(lo[t[1]], hi[t[1]])
                for u in range(lo[t[0]], hi[t[0]])]

    def box_subs(lo, hi):
        # x-fastest over the box: already increasing
        x = np.arange(lo[0], hi[0])
        y = np.arange(lo[1], hi[1]) * S3[0]
        z = np.arange(lo[2], hi[2]) * (S3[0] * S3[1])
        return (z[:, None, None] + y[None, :, None] + x[None, None, :]).ravel()

    nodes = []

    def rec(lo, hi, depth):
        idx = len(nodes)
        nodes.append(None)
        ext = [hi[a] - lo[a] for a in range(3)]
        if all(e == 1 for e in ext):
            nodes[idx] = dict(leaf=True, sub=int(lo[0] + S3[0] * (lo[1] + S3[1] * lo[2])),
                              depth=depth)
            return idx
        bnd = []
        for a in range(3):
            for plane in (lo[a], hi[a]):
                if 0 < plane < S3[a]:
                    bnd += plane_faces(a, plane, lo, hi)
        a = int(np.argmax(ext))
        mid = lo[a] + ext[a] // 2
        sep = plane_faces(a, mid, lo, hi)
        h1 = list(hi)
        h1[a] = mid
        l2 = list(lo)
        l2[a] = mid
        c1 = rec(lo, tuple(h1), depth + 1)
        c2 = rec(tuple(l2), hi, depth + 1)
        nodes[idx] = dict(leaf=False, depth=depth, sep=np.array(sep, dtype=np.int64),
                          bnd=np.array(bnd, dtype=np.int64), pres=box_subs(lo, hi), ch=(c1, c2))
        return idx

    if dec.n_subdomains > 1:
        rec((0, 0, 0), tuple(S3), 0)
    nodes = _contract(nodes, _merge_schedule(nodes, ND_MERGE))
    _assign_pressures(nodes, dec, has_p)
    cache[has_p.tobytes()] = nodes
    return nodes


def _assign_pressures(nodes, dec, has_p):
    """Subdomain pressures are eliminated inside the tree, not carried to the root:
    p_i couples only to i's coarse flux dofs, so once the last face of i has been
    eliminated (at the highest node H_i whose separator holds a face of i) p_i is
    eliminated too, in H_i's pivot block (quasi-definite: the flux block is SPD,
    the pressure Schur complement negative definite).  Subdomains without a
    coarse pressure (`has_p` false: the pinned subdomain 0, coarse.py:192-194, or
    in mode B every subdomain on a Dirichlet end) appear nowhere.  Per internal node:
    pres_elim = pressures eliminated there, pres = pressures of its box still
    live above it (its boundary)."""
    if not nodes:
        return
    internal = [k for k, n in enumerate(nodes) if not n["leaf"]]
    face_node = np.full(dec.n_faces, -1, dtype=np.int64)
    for k in internal:
        face_node[nodes[k]["sep"]] = k
    ft = dec.face_table
    N = dec.n_subdomains
    H = np.full(N, -1, dtype=np.int64)
    for f in range(dec.n_faces):
        k = int(face_node[f])
        for sub in (int(ft[f, 0]), int(ft[f, 1])):
            if H[sub] < 0 or nodes[k]["depth"] < nodes[int(H[sub])]["depth"]:
                H[sub] = k
    hdepth = np.array([nodes[int(h)]["depth"] if h >= 0 else -1 for h in H])
    for k in internal:
        box = nodes[k]["pres"]
        box = box[has_p[box]]
        nodes[k]["pres_elim"] = box[H[box] == k]
        nodes[k]["pres"] = box[hdepth[box] < nodes[k]["depth"]]


# Binary-tree levels merged per multifrontal node: a node eliminates the
# separators of `ND_MERGE` consecutive bisection levels at once (up to
# 2**ND_MERGE children), dividing the number of sequential solve levels by
# ND_MERGE (C3: 13 -> 5); the level count, not the bytes, bounds the coarse
# solve's latency (C3 coarse solve 284 us binary, 192 us with 2, 166 us with 3,
# 201 us with 4: the 3394-dof root front of 4 is bandwidth-bound).
ND_MERGE = 3
if os.environ.get("BDDC_ND_MERGE"):   # explicit per-level schedule, e.g. "3,4,6" (tuning)
    ND_MERGE = [int(v) for v in os.environ["BDDC_ND_MERGE"].split(",")]


def _merge_schedule(nodes, c):
    """Per-depth merge counts: c binary levels per node from the root down, the
    remainder of the separator depth folded into the bottom group instead of
    leaving a last level of tiny nodes (C3, 13 separator levels: 3,3,3,4 -> 4
    solve levels, coarse solve 133 -> 123 us)."""
    if isinstance(c, (list, tuple)) or not nodes:
        return c
    depth = 1 + max((n["depth"] for n in nodes if not n["leaf"]), default=-1)
    if depth <= c:
        return [max(depth, 1)]
    if depth >= 15:
        # deep trees (C4: 15 separator levels) merge only two levels in the top two
        # node levels (a 7-plane root front, 4652 dofs at C4, makes the root GEMV
        # bandwidth-bound and its factorisation dominate the setup) and fold the
        # remainder into the bottom group (C4 coarse solve 228 us with 2,2,3,3,3,2,
        # 196 us with 2,2,3,3,5, setup coarse 70 -> 63 ms; scripts/nd_merge_sweep.sh)
        rest = depth - 4
        sched = [2, 2] + [c] * (rest // c)
        if rest % c:
            sched[-1] += rest % c
        return sched
    sched = [c] * (depth // c)
    if depth % c:
        sched[-1] += depth % c
    return sched


def _contract(nodes, c):
    """Merge c consecutive levels of the bisection tree into one node level
    (c: int, or a per-depth list whose last entry repeats)."""
    sched = list(c) if isinstance(c, (list, tuple)) else [c]
    if max(sched) <= 1 or not nodes:
        return nodes
    out = []

    def build(k, depth):
        c = sched[min(depth, len(sched) - 1)]
        idx = len(out)
        out.append(None)
        n = nodes[k]
        if n["leaf"]:
            out[idx] = dict(leaf=True, sub=n["sub"], depth=depth)
            return idx
        seps = [n["sep"]]
        frontier = list(n["ch"])
        for _ in range(c - 1):
            nxt = []
            for x in frontier:
                if nodes[x]["leaf"]:
                    nxt.append(x)
                else:
                    seps.append(nodes[x]["sep"])
                    nxt.extend(nodes[x]["ch"])
            frontier = nxt
        ch = tuple(build(x, depth + 1) for x in frontier)
        out[idx] = dict(leaf=False, depth=depth, sep=np.concatenate(seps), bnd=n["bnd"],
                        pres=n["pres"], ch=ch)
        return idx

    build(0, 0)
    return out


def nd_geometry_flat(dec, has_p=None):
    """Flat arrays of the internal nodes of nd_geometry (cached on `dec`)."""
    has_p = _has_p(dec, has_p)
    cache = dec.__dict__.setdefault("_nd_geometry_flat", {})
    cached = cache.get(has_p.tobytes())
    if cached is not None:
        return cached
    geo = nd_geometry(dec, has_p)
    internal = [k for k, n in enumerate(geo) if not n["leaf"]]
    gpos = {k: i for i, k in enumerate(internal)}

    def csr(key):
        parts = [np.asarray(geo[k][key], dtype=np.int64) for k in internal]
        ptr = np.concatenate([[0], np.cumsum([len(p) for p in parts])]).astype(np.int64)
        flat = np.concatenate(parts) if parts else np.zeros(0, np.int64)
        return ptr, flat

    F = dict(internal=np.array(internal, dtype=np.int64),
             depth=np.array([geo[k]["depth"] for k in internal], dtype=np.int64))
    F["sep_ptr"], F["sep"] = csr("sep")
    F["bnd_ptr"], F["bnd"] = csr("bnd")
    F["pres_ptr"], F["pres"] = csr("pres")
    F["pel_ptr"], F["pel"] = csr("pres_elim")
    # children: internal index (>= 0) or -(1 + subdomain) for leaves; nch per node
    ns = max([len(geo[k]["ch"]) for k in internal] + [1])
    ch = np.zeros((len(internal), ns), dtype=np.int64)
    nch = np.zeros(len(internal), dtype=np.int64)
    for i, k in enumerate(internal):
        nch[i] = len(geo[k]["ch"])
        for s_, c in enumerate(geo[k]["ch"]):
            ch[i, s_] = gpos[c] if not geo[c]["leaf"] else -(1 + geo[c]["sub"])
    F["ch"] = ch
    F["nch"] = nch
    cache[has_p.tobytes()] = F
    return F


def _expand(ptr, faces, per_face, cstart):
    """Face lists (CSR) -> coarse dof lists (CSR): face f -> cstart[f] .. + per_face[f]."""
    cnt = per_face[faces]
    tot = int(cnt.sum())
    first = np.cumsum(cnt) - cnt
    dofs = np.repeat(cstart[faces] - first, cnt) + np.arange(tot, dtype=np.int64)
    csum = np.concatenate([[0], np.cumsum(cnt)])
    return csum[ptr], dofs


def _ranges(lo, cnt):
    """concat(arange(lo[i], lo[i] + cnt[i]))."""
    tot = int(cnt.sum())
    if tot == 0:
        return np.zeros(0, np.int64)
    start = np.cumsum(cnt) - cnt
    return np.repeat(lo - start, cnt) + np.arange(tot, dtype=np.int64)


class CoarseND:
    """Symbolic analysis (host, index tables only) + numeric factorisation (device)."""

    def __init__(self, dec, per_face, cstart, sub_rows, nC, maxC, dev, has_p=None):
        """Symbolic analysis, vectorised over all tree nodes (numpy, no per-node loops).
        has_p: subdomains carrying a coarse pressure (default: all but subdomain 0)."""
        self.dev = dev
        has_p = _has_p(dec, has_p)
        self.has_p = has_p
        N = dec.n_subdomains
        self.N = N
        nfaces = dec.n_faces
        self.nfc = nfc = int(per_face.sum()) if nfaces else 0
        per_face = np.asarray(per_face, dtype=np.int64)
        cstart = np.asarray(cstart, dtype=np.int64)
        nC = np.asarray(nC, dtype=np.int64)
        self.maxC = maxC
        self.factored = False
        self.levels = []
        def t(a, dt=I32):   # async upload (no wait for the queued device work)
            h = torch.from_numpy(np.ascontiguousarray(a)).to(dt)
            if torch.device(dev).type != "cuda":   # host-only symbolic tests
                return h
            return h.pin_memory().to(dev, non_blocking=True)
        if not (N > 1 and nfc):
            self.cb_total = 1
            return
        G = nd_geometry_flat(dec, has_p)
        nI = len(G["internal"])
        # coarse dof lists per internal node: separator = its faces' dofs ++ the
        # pressures eliminated there; boundary = boundary faces' dofs ++ live pressures
        sptr_f, sdofs_f = _expand(G["sep_ptr"], G["sep"], per_face, cstart)
        nsf = np.diff(sptr_f)
        nsp = np.diff(G["pel_ptr"])
        ns_all = nsf + nsp
        sptr = np.concatenate([[0], np.cumsum(ns_all)])
        node_s = np.repeat(np.arange(nI), ns_all)
        within_s = np.arange(int(sptr[-1]), dtype=np.int64) - sptr[node_s]
        isf_s = within_s < nsf[node_s]
        sdofs = np.empty(int(sptr[-1]), dtype=np.int64)
        sdofs[isf_s] = sdofs_f[sptr_f[node_s[isf_s]] + within_s[isf_s]]
        nq_s = ~isf_s
        sdofs[nq_s] = nfc + G["pel"][G["pel_ptr"][node_s[nq_s]] + within_s[nq_s] - nsf[node_s[nq_s]]]
        fptr, fdofs = _expand(G["bnd_ptr"], G["bnd"], per_face, cstart)
        ns = ns_all
        nbf = np.diff(fptr)
        npres = np.diff(G["pres_ptr"])
        nb = nbf + npres
        bptr = np.concatenate([[0], np.cumsum(nb)])
        node_b = np.repeat(np.arange(nI), nb)
        within = np.arange(int(bptr[-1]), dtype=np.int64) - bptr[node_b]
        isf = within < nbf[node_b]
        bdofs = np.empty(int(bptr[-1]), dtype=np.int64)
        bdofs[isf] = fdofs[fptr[node_b[isf]] + within[isf]]
        nq = ~isf
        bdofs[nq] = nfc + G["pres"][G["pres_ptr"][node_b[nq]] + within[nq] - nbf[node_b[nq]]]
        # levels: deepest first; within a level, tree order
        depth = G["depth"]
        ud = np.unique(depth)[::-1]
        lev = np.searchsorted(-ud, -depth)
        order = np.lexsort((np.arange(nI), lev))
        lev_start = np.searchsorted(lev[order], np.arange(len(ud) + 1))
        pos = np.empty(nI, dtype=np.int64)
        for li in range(len(ud)):
            ids = order[lev_start[li]:lev_start[li + 1]]
            pos[ids] = np.arange(len(ids))
        ch = G["ch"]
        NS = ch.shape[1]
        has = np.arange(NS)[None, :] < G["nch"][:, None]
        internal_ch = (ch >= 0) & has
        par = np.repeat(np.arange(nI)[:, None], NS, axis=1)
        if np.any(lev[ch[internal_ch]] != lev[par[internal_ch]] - 1):
            raise ConfigurationError("nested dissection: child not one level below")
        sub_g = np.asarray(sub_rows[:, :, 0], dtype=np.int64)
        M = nfc + N + 1

        coff = 0
        for li in range(len(ud)):
            ids = order[lev_start[li]:lev_start[li + 1]]
            L = _Level()
            L.m = m = len(ids)
            s = ns[ids]
            sf = nsf[ids]
            b = nb[ids]
            # pivot block [flux separator (padded to Sf) | eliminated pressures (to Sp)]
            L.Sf = Sf = _pad(int(sf.max()), 32)
            L.Sp = Sp = _pad(int(nsp[ids].max()), 32) if int(nsp[ids].max()) else 0
            L.S = S = Sf + Sp
            L.B = _pad(int(b.max()), 2)
            L.nf = S + L.B
            sep_flat = sdofs[_ranges(sptr[ids], s)]
            bnd_flat = bdofs[_ranges(bptr[ids], b)]
            srow = np.repeat(np.arange(m), s)
            scol = _ranges(np.zeros(m, np.int64), s)
            spos = np.where(scol < sf[srow], scol, Sf + scol - sf[srow])   # padded pivot position
            sep_idx = np.full((m, S), -1, dtype=np.int32)
            sep_idx[srow, spos] = sep_flat
            # parent fronts [sep | bnd] keyed by (parent, dof) -> position in the padded front
            brow = np.repeat(np.arange(m), b)
            bcol = _ranges(np.zeros(m, np.int64), b)
            fk = np.concatenate([srow * M + sep_flat, brow * M + bnd_flat])
            fv = np.concatenate([spos, S + bcol])
            fo = np.argsort(fk, kind="stable")
            fk, fv = fk[fo], fv[fo]
            K = 1
            maps = []
            L.nslots = NS
            ckind = np.zeros((NS, m, 3), dtype=np.int32)
            for slot in range(NS):
                c = ch[ids, slot]
                valid = has[ids, slot]
                leafc = (c < 0) & valid
                subc = np.where(leafc, -c - 1, 0)
                # leaf export: its coarse dofs, then its pressure (none for the pinned 0)
                elen = np.where(leafc, nC[subc] + has_p[subc], nb[np.maximum(c, 0)])
                elen = np.where(valid, elen, 0)
                erow = np.repeat(np.arange(m), elen)
                ecol = _ranges(np.zeros(m, np.int64), elen)
                cr = c[erow]
                lf = cr < 0
                dof = np.empty(len(erow), dtype=np.int64)
                sr = -cr[lf] - 1
                last = ecol[lf] == nC[sr]
                dof_l = np.where(last, nfc + sr, sub_g[sr, np.minimum(ecol[lf], sub_g.shape[1] - 1)])
                dof[lf] = dof_l
                ci = cr[~lf]
                dof[~lf] = bdofs[bptr[ci] + ecol[~lf]]
                key = erow * M + dof
                loc = np.searchsorted(fk, key)
                if len(key) and not np.array_equal(fk[np.minimum(loc, len(fk) - 1)], key):
                    raise ConfigurationError("nested dissection: child export not in parent front")
                maps.append((erow, ecol, fv[loc].astype(np.int32)))
                K = max(K, int(elen.max()) if m else 1)
                intc = valid & ~leafc
                ckind[slot, leafc, 0] = 1
                ckind[slot, leafc, 1] = subc[leafc]
                ckind[slot, leafc, 2] = nC[subc[leafc]]
                ckind[slot, intc, 1] = pos[c[intc]]
                ckind[slot, ~valid, 0] = 2
            L.K = K
            cmap = np.full((NS, m, K), -1, dtype=np.int32)
            for slot, (erow, ecol, v) in enumerate(maps):
                cmap[slot, erow, ecol] = v
            L._sf = sf
            L.sep_idx = t(sep_idx)
            L.cmap = t(cmap)
            L.ckind = t(ckind)
            L.s = s
            L.b = b
            L.cb_off = coff + np.concatenate([[0], np.cumsum(b)[:-1]])
            coff += int(b.sum())
            L._sep_flat, L._bnd_flat = sep_flat, bnd_flat
            self.levels.append(L)
        self.cb_total = max(coff, 1)
        # left-looking forward lists: for every separator slot (and every pressure) the
        # cbuf indices of all descendant contributions to it, ordered by cbuf index
        gs = np.concatenate([L._bnd_flat for L in self.levels])
        srcs = np.concatenate([_ranges(L.cb_off, L.b) for L in self.levels])
        o = np.lexsort((srcs, gs))
        gs, srcs = gs[o], srcs[o]

        def lists(keys):
            lo = np.searchsorted(gs, keys, side="left")
            hi = np.searchsorted(gs, keys, side="right")
            cnt = hi - lo
            ptr = np.concatenate([[0], np.cumsum(cnt)]).astype(np.int32)
            idx = _ranges(lo, cnt)
            src = srcs[idx] if len(idx) else np.zeros(1, np.int64)
            return ptr, src.astype(np.int32)

        def rows_per_task(total):
            # 4 rows per warp pass, 8 warps per CTA: aim for >= ~8 CTAs per SM per level
            r = 8
            while r < 64 and total / (2 * r) >= 148 * 8:
                r *= 2
            return r

        def split(nrows, step):
            k = -(-nrows // step)
            q = np.repeat(np.arange(len(nrows)), k)
            r0 = _ranges(np.zeros(len(nrows), np.int64), k) * step
            return np.stack([q, r0, np.minimum(r0 + step, nrows[q])], axis=1).astype(np.int32)

        for L in self.levels:
            s, b = L.s, L.b
            sep_ptr = np.concatenate([[0], np.cumsum(s)])
            bnd_ptr = np.concatenate([[0], np.cumsum(b)])
            data_off = np.concatenate([[0], np.cumsum(s * s + 2 * b * s)])
            L.ysize = int(sep_ptr[-1])
            L.csize = int(data_off[-1])
            lptr, lsrc = lists(L._sep_flat)
            info = np.stack([s, b, sep_ptr[:-1], bnd_ptr[:-1], L.cb_off, L._sf], axis=1).astype(np.int32)
            rf = rows_per_task(int((s + b).sum()))
            # backward rows are long (b): split a row over wpr warps when the
            # level has too few rows to fill the GPU
            L.wpr = 1
            while L.wpr < 8 and int(s.sum()) * L.wpr < 148 * 8 * 4 and int(b.max()) >= 128 * L.wpr:
                L.wpr *= 2
            rb = rows_per_task(int(s.sum()) * max(1, int(b.max()) // 64)) if L.wpr == 1 else 8 // L.wpr
            ft = split(s + b, rf)
            bt = split(s, rb)
            L.info = t(info)
            L.data_off = t(data_off[:-1].astype(np.int64), torch.int64)
            L.sep_flat = t(L._sep_flat.astype(np.int32))
            L.bnd_flat = t(L._bnd_flat.astype(np.int32) if len(L._bnd_flat) else np.zeros(1, np.int32))
            L.lptr = t(lptr)
            L.lsrc = t(lsrc)
            L.ftasks = t(ft)
            L.btasks = t(bt)
            L.n_ft, L.n_bt = len(ft), len(bt)
            L.smax = int(s.max())
            L.bmax = int(b.max())
            del L._sep_flat, L._bnd_flat, L._sf

    # --------------------------------------------------------------- numeric

    def factor(self, Kc, sub_rows_dev, b0):
        """Assemble and factor every front (leaves -> root); returns the root level."""
        st = _stream()
        lib = nat.load()
        info = torch.zeros(1, dtype=I32, device=self.dev)
        for li, L in enumerate(self.levels):
            L.F = torch.empty(L.m * L.nf * L.nf, dtype=F64, device=self.dev)
            child = self.levels[li - 1] if li > 0 else None
            for slot in range(L.nslots):
                nat.call("bddc_nd_assemble", L.m, L.S, L.Sf, L.B, L.nf, slot, L.K, _p(L.cmap),
                         _p(L.ckind), _p(L.sep_idx), _p(L.F),
                         _p(child.F) if child is not None else None,
                         child.S if child is not None else 0,
                         child.nf if child is not None else 1,
                         _p(Kc), _p(sub_rows_dev), _p(b0), self.maxC, st)
            self._pivot_inverse(L, info, st)
            L.X = torch.empty(L.m * L.B * L.S, dtype=F64, device=self.dev)
            F21 = L.F[L.S * L.nf:]
            nat.call("bddc_dgemm_batched", 0, 0, L.B, L.S, L.S, 1.0, _p(F21), L.nf,
                     L.nf * L.nf, _p(L.F), L.nf, L.nf * L.nf, 0.0, _p(L.X), L.S,
                     L.B * L.S, L.m, 0, st)
            F22 = L.F[L.S * L.nf + L.S:]
            F12 = L.F[L.S:]
            nat.call("bddc_dgemm_batched", 0, 0, L.B, L.B, L.S, -1.0, _p(L.X), L.S,
                     L.B * L.S, _p(F12), L.nf, L.nf * L.nf, 1.0, _p(F22), L.nf,
                     L.nf * L.nf, L.m, 0, st)
        self._factor_info = info   # checked by check() after the setup's final sync
        self.factored = True
        for L in self.levels:
            L.Fc = torch.empty(max(L.csize, 1), dtype=F64, device=self.dev)
            nat.call("bddc_nd_compact", L.m, L.S, L.Sf, L.nf, L.B, _p(L.F), _p(L.X), _p(L.info),
                     _p(L.data_off), _p(L.Fc), st)
        # bytes streamed per solve: F11inv + X (forward) + X^T (backward)
        self.bytes = sum(L.csize * 8 for L in self.levels)
        return self.levels[-1]

    def _pivot_inverse(self, L, info, st):
        """F11^-1 in place for every front of a level.  Pivot blocks without
        pressures are SPD; with eliminated pressures [[A, B^T], [B, C]] is
        quasi-definite (A SPD, Sp = C - B A^-1 B^T negative definite):
          A <- A^-1;  W = B A^-1;  C <- -(C - W B^T) -> inverse Ms = (-Sp)^-1;
          B <- Ms W (= -Sp^-1 W);  A <- A^-1 - W^T B;  C <- -Ms;  mirror B^T."""
        lib = nat.load()
        m, nf, Sf, Sp = L.m, L.nf, L.Sf, L.Sp
        sF = nf * nf
        if Sp == 0:
            ws = torch.empty(lib.bddc_spd_inverse_workspace(L.S, m, 32) // 8 + 2, dtype=F64,
                             device=self.dev)
            nat.call("bddc_spd_inverse_batched", _p(L.F), L.S, nf, sF, m, 32, _p(ws), _p(info), st)
            return
        ws = torch.empty(lib.bddc_spd_inverse_workspace(max(Sf, Sp), m, 32) // 8 + 2, dtype=F64,
                         device=self.dev)
        W = torch.empty(m * Sp * Sf, dtype=F64, device=self.dev)
        A = L.F
        Bb = L.F[Sf * nf:]            # pressure rows, flux columns
        Cb = L.F[Sf * nf + Sf:]       # pressure block
        nat.call("bddc_spd_inverse_batched", _p(A), Sf, nf, sF, m, 32, _p(ws), _p(info), st)
        nat.call("bddc_dgemm_batched", 0, 0, Sp, Sf, Sf, 1.0, _p(Bb), nf, sF, _p(A), nf, sF,
                 0.0, _p(W), Sf, Sp * Sf, m, 0, st)
        nat.call("bddc_dgemm_batched", 0, 1, Sp, Sp, Sf, -1.0, _p(W), Sf, Sp * Sf, _p(Bb), nf, sF,
                 1.0, _p(Cb), nf, sF, m, 0, st)
        nat.call("bddc_nd_qd", 0, m, Sf, Sp, nf, _p(L.F), st)
        nat.call("bddc_spd_inverse_batched", _p(Cb), Sp, nf, sF, m, 32, _p(ws), _p(info), st)
        nat.call("bddc_dgemm_batched", 0, 0, Sp, Sf, Sp, 1.0, _p(Cb), nf, sF, _p(W), Sf, Sp * Sf,
                 0.0, _p(Bb), nf, sF, m, 0, st)
        nat.call("bddc_dgemm_batched", 1, 0, Sf, Sf, Sp, -1.0, _p(W), Sf, Sp * Sf, _p(Bb), nf, sF,
                 1.0, _p(A), nf, sF, m, 0, st)
        nat.call("bddc_nd_qd", 0, m, Sf, Sp, nf, _p(L.F), st)
        nat.call("bddc_nd_qd", 1, m, Sf, Sp, nf, _p(L.F), st)

    def check(self):
        if int(self._factor_info.item()):
            raise ConfigurationError("coarse problem singular (non-positive pivot in S_Pi)")

    def release_fronts(self):
        """Drop the padded factorisation fronts (the solves read the compact copies)."""
        for L in self.levels:
            L.F = None
            L.X = None

    def solve(self, r, x, restricted=None):
        """Pinned coarse solve on the combined vector [flux | pressures] (coarse.py:208-215).

        r, x: length nfc + N.  r is read-only; x[nfc] (subdomain 0's pinned
        pressure) is not written.  restricted = (v, cown): r is not read; the
        flux rhs is v[cown[:, 0]] - v[cown[:, 1]] and the pressure rhs zero
        (the preconditioner's restriction, coarse.py:225-235).
        """
        st = _stream()
        ys, cb = self._bufs()
        v, cown = restricted if restricted is not None else (None, None)
        for li, L in enumerate(self.levels):
            # a level without boundary (the root) writes its solution directly
            direct = L.bmax == 0
            nat.call("bddc_nd_fwd", L.ysize, L.n_ft, L.smax, _p(L.ftasks), _p(L.info), _p(L.data_off),
                     _p(L.sep_flat), _p(L.lptr), _p(L.lsrc), _p(L.Fc), _p(r), _p(v), _p(cown), self.nfc,
                     _p(self._rs), _p(ys[li]), _p(cb), _p(x) if direct else None, st)
        for li in range(len(self.levels) - 1, -1, -1):
            L = self.levels[li]
            if L.bmax == 0:
                continue
            nat.call("bddc_nd_bwd", L.n_bt, L.bmax, L.wpr, _p(L.btasks), _p(L.info), _p(L.data_off),
                     _p(L.sep_flat), _p(L.bnd_flat), _p(L.Fc), _p(ys[li]), _p(x), st)

    def _bufs(self):
        if getattr(self, "_yb", None) is None:
            ys = [torch.empty(max(L.ysize, 1), dtype=F64, device=self.dev) for L in self.levels]
            cb = torch.empty(self.cb_total, dtype=F64, device=self.dev)
            self._yb = (ys, cb)
            self._rs = torch.empty(max([L.ysize for L in self.levels] + [1]), dtype=F64, device=self.dev)
        return self._yb

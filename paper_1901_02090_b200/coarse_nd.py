"""Sparse coarse solver: structured nested dissection over the subdomain grid.

The reference factors the coarse saddle problem densely (`coarse.py:186-215`:
`lu_factor` of [[S_Pi, B0^T],[B0, 0]] with subdomain 0's pressure pinned).
S_Pi couples coarse dofs only through shared subdomains, so for box
partitions a plane of subdomain faces separates the subdomain grid.  We
eliminate the flux coarse dofs by a multifrontal block-LDL^T over that
nested-dissection tree while carrying the subdomain pressures along as
never-eliminated front variables: the root's update matrix is then exactly
-B0 S_Pi^-1 B0^T, whose pinned part Pc (drop subdomain 0) is inverted
densely.  Coarse solves (solver.py:117-118, 318-319) become

    flux rhs r, pressure rhs 0 :  x = S_Pi^-1 (r - B0^T Pc^-1 B0 S_Pi^-1 r)
    flux rhs 0, pressure rhs q :  w = S_Pi^-1 B0[1:]^T Pc^-1 q[1:]

which is algebraically the pinned solve of the reference.

Tree: every node is a box of subdomain strips; an internal node splits its
box at the middle of its longest axis; its separator = the coarse dofs on
the faces of that plane; its boundary = coarse dofs on the box's faces
toward the rest of the domain, then the pressures of the box's subdomains.
Leaves are single subdomains whose contribution is the local block
[[sigma sigma^T Kc_i, b0_i^T],[b0_i, 0]] (coarse.py:179-185).  Per internal
node (front F over [sep | bnd]):
    F11inv = F11^-1 (blocked symmetric sweep),  X = F21 F11inv,
    U = F22 - X F12  (extend-added into the parent's front).
Solve (flux part only): forward y_sep = F11inv (r_sep - descendant
contributions), c = X r_sep (leaves -> root, left-looking gathers in a
fixed order); backward x_sep = y_sep - X^T x_bnd (root -> leaves).
"""

from __future__ import annotations

import ctypes as C

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


def nd_geometry(dec):
    """Nested-dissection tree of the subdomain grid in face ids (cached on `dec`).

    Node: dict(leaf, depth, sub | sep (face ids), bnd (face ids), pres (subdomain ids), ch).
    """
    cached = getattr(dec, "_nd_geometry", None)
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
        z, y, x = np.meshgrid(np.arange(lo[2], hi[2]), np.arange(lo[1], hi[1]),
                              np.arange(lo[0], hi[0]), indexing="ij")
        return np.sort((x + S3[0] * (y + S3[1] * z)).ravel())

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
    dec._nd_geometry = nodes
    return nodes


class CoarseND:
    """Symbolic analysis (host, index tables only) + numeric factorisation (device)."""

    def __init__(self, dec, per_face, cstart, sub_rows, nC, maxC, dev):
        self.dev = dev
        N = dec.n_subdomains
        self.N = N
        nfaces = dec.n_faces
        self.nfc = nfc = int(per_face.sum()) if nfaces else 0
        per_face = np.asarray(per_face, dtype=np.int64)
        cstart = np.asarray(cstart, dtype=np.int64)

        def face_dofs(fl):
            if len(fl) == 0:
                return np.zeros(0, dtype=np.int64)
            cnt = per_face[fl]
            tot = int(cnt.sum())
            first = np.cumsum(cnt) - cnt
            return np.repeat(cstart[fl] - first, cnt) + np.arange(tot)

        # geometry-only tree (cached on the decomposition), expanded to coarse dofs here
        geo = nd_geometry(dec) if (N > 1 and nfc) else []
        nodes = []
        for gn in geo:
            if gn["leaf"]:
                nodes.append(dict(leaf=True, sub=gn["sub"], depth=gn["depth"]))
            else:
                bf = face_dofs(gn["bnd"])
                nodes.append(dict(leaf=False, depth=gn["depth"], sep=face_dofs(gn["sep"]), bndf=bf,
                                  bnd=np.concatenate([bf, nfc + gn["pres"]]), ch=gn["ch"]))
        self.nodes = nodes
        internal = [k for k, n in enumerate(nodes) if not n["leaf"]]
        depths = sorted({nodes[k]["depth"] for k in internal}, reverse=True)
        pos_in_level = {}
        self.levels = []
        t = lambda a, dt=I32: torch.as_tensor(np.ascontiguousarray(a), dtype=dt, device=dev)
        sub_g = sub_rows[:, :, 0]

        def export(cn):
            if cn["leaf"]:
                i = cn["sub"]
                return np.concatenate([sub_g[i, :nC[i]], [nfc + i]])
            return cn["bnd"]

        for d in depths:
            ids = [k for k in internal if nodes[k]["depth"] == d]
            L = _Level()
            L.ids, L.m = ids, len(ids)
            for q, k in enumerate(ids):
                pos_in_level[k] = (len(self.levels), q)
            L.S = _pad(max(len(nodes[k]["sep"]) for k in ids), 32)
            L.B = _pad(max(len(nodes[k]["bnd"]) for k in ids), 2)
            L.Bf = max(len(nodes[k]["bndf"]) for k in ids)
            L.nf = L.S + L.B
            sep_idx = np.full((L.m, L.S), -1, dtype=np.int32)
            bnd_idx = np.full((L.m, max(L.Bf, 1)), -1, dtype=np.int32)
            K = 1
            maps = []
            for q, k in enumerate(ids):
                n = nodes[k]
                sep_idx[q, :len(n["sep"])] = n["sep"]
                bnd_idx[q, :len(n["bndf"])] = n["bndf"]
                front = np.concatenate([n["sep"], n["bnd"]])
                order = np.argsort(front, kind="stable")
                fs = front[order]
                ns = len(n["sep"])
                mm = []
                for c in n["ch"]:
                    src = export(nodes[c])
                    loc = np.searchsorted(fs, src)
                    if len(src) and not np.array_equal(fs[np.minimum(loc, len(fs) - 1)], src):
                        raise ConfigurationError("nested dissection: child export not in parent front")
                    mp = order[loc]
                    mm.append(np.where(mp < ns, mp, L.S + (mp - ns)).astype(np.int32))
                    K = max(K, len(src))
                maps.append(mm)
            L.K = K
            cmap = np.full((2, L.m, K), -1, dtype=np.int32)
            ckind = np.zeros((2, L.m, 3), dtype=np.int32)
            for q, k in enumerate(ids):
                for slot, c in enumerate(nodes[k]["ch"]):
                    cmap[slot, q, :len(maps[q][slot])] = maps[q][slot]
                    cn = nodes[c]
                    ckind[slot, q] = (1, cn["sub"], nC[cn["sub"]]) if cn["leaf"] else (0, -1, 0)
            L.sep_idx_h = sep_idx
            L.sep_idx, L.bnd_idx = t(sep_idx), t(bnd_idx)
            L.cmap_h, L.ckind_h = cmap, ckind
            self.levels.append(L)
        for li, L in enumerate(self.levels):
            for q, k in enumerate(L.ids):
                for slot, c in enumerate(nodes[k]["ch"]):
                    if not nodes[c]["leaf"]:
                        lc, pc = pos_in_level[c]
                        if lc != li - 1:
                            raise ConfigurationError("nested dissection: child not one level below")
                        L.ckind_h[slot, q] = (0, pc, 0)
            L.cmap = t(L.cmap_h)
            L.ckind = t(L.ckind_h)
        # ---- compact solve layout over the combined vector [flux coarse dofs | pressures]:
        # per node F11inv (s x s) then X (b x s) for the whole boundary (flux + pressures).
        # Left-looking forward lists: for every separator slot (and every pressure) the
        # cbuf indices of all descendant contributions to it, ordered deeper level
        # first, then node, then slot (vectorised).
        coff = 0
        gs, srcs = [], []
        for L in self.levels:
            L.s = np.array([len(nodes[k]["sep"]) for k in L.ids], dtype=np.int64)
            L.b = np.array([len(nodes[k]["bnd"]) for k in L.ids], dtype=np.int64)
            L.cb_off = coff + np.concatenate([[0], np.cumsum(L.b)[:-1]])
            for q, k in enumerate(L.ids):
                bb = nodes[k]["bnd"]
                if len(bb):
                    gs.append(bb)
                    srcs.append(L.cb_off[q] + np.arange(len(bb)))
            coff += int(L.b.sum())
        self.cb_total = max(coff, 1)
        if gs:
            gs = np.concatenate(gs)
            srcs = np.concatenate(srcs)
            o = np.lexsort((srcs, gs))
            gs, srcs = gs[o], srcs[o]
        else:
            gs = srcs = np.zeros(0, np.int64)

        def lists(keys):
            lo = np.searchsorted(gs, keys, side="left")
            hi = np.searchsorted(gs, keys, side="right")
            cnt = hi - lo
            ptr = np.concatenate([[0], np.cumsum(cnt)]).astype(np.int32)
            idx = np.concatenate([np.arange(a_, b_) for a_, b_, c_ in zip(lo, hi, cnt) if c_]) \
                if cnt.sum() else np.zeros(0, np.int64)
            src = srcs[idx] if len(idx) else np.zeros(1, np.int64)
            return ptr, src.astype(np.int32)

        def rows_per_task(total):
            # warp per row, 8 warps per CTA: aim for >= ~8 CTAs per SM per level
            r = 8
            while r < 64 and total / (2 * r) >= 148 * 8:
                r *= 2
            return r

        for L in self.levels:
            sep_flat = np.concatenate([nodes[k]["sep"] for k in L.ids]).astype(np.int64)
            bnd_flat = np.concatenate([nodes[k]["bnd"] for k in L.ids] + [np.zeros(0, np.int64)])
            sep_ptr = np.concatenate([[0], np.cumsum(L.s)])
            bnd_ptr = np.concatenate([[0], np.cumsum(L.b)])
            data_off = np.concatenate([[0], np.cumsum(L.s * L.s + 2 * L.b * L.s)])
            L.ysize = int(sep_ptr[-1])
            L.csize = int(data_off[-1])
            lptr, lsrc = lists(sep_flat)
            info = np.stack([L.s, L.b, sep_ptr[:-1], bnd_ptr[:-1], L.cb_off], axis=1).astype(np.int32)
            ft_, bt_ = [], []
            rf = rows_per_task(int((L.s + L.b).sum()))
            # backward rows are long (b): split a row over wpr warps when the
            # level has too few rows to fill the GPU
            L.wpr = 1
            while L.wpr < 8 and int(L.s.sum()) * L.wpr < 148 * 8 * 4 and int(L.b.max()) >= 128 * L.wpr:
                L.wpr *= 2
            rb = rows_per_task(int(L.s.sum()) * max(1, int(L.b.max()) // 64)) if L.wpr == 1 else 8 // L.wpr
            for q in range(L.m):
                nr, ns = int(L.s[q] + L.b[q]), int(L.s[q])
                for r0 in range(0, nr, rf):
                    ft_.append((q, r0, min(r0 + rf, nr)))
                for k0 in range(0, ns, rb):
                    bt_.append((q, k0, min(k0 + rb, ns)))
            L.h = dict(sep_flat=sep_flat, bnd_flat=bnd_flat, sep_ptr=sep_ptr, bnd_ptr=bnd_ptr,
                       data_off=data_off, lptr=lptr, lsrc=lsrc)
            L.info = t(info)
            L.data_off = t(data_off[:-1].astype(np.int64), torch.int64)
            L.sep_flat = t(sep_flat.astype(np.int32))
            L.bnd_flat = t(bnd_flat.astype(np.int32) if len(bnd_flat) else np.zeros(1, np.int32))
            L.lptr = t(lptr)
            L.lsrc = t(lsrc)
            L.ftasks = t(np.array(ft_, dtype=np.int32).reshape(-1, 3))
            L.btasks = t(np.array(bt_, dtype=np.int32).reshape(-1, 3))
            L.n_ft, L.n_bt = len(ft_), len(bt_)
            L.smax = int(L.s.max())
            L.bmax = int(L.b.max())
        # pressure gather lists (pressures 1..N-1; subdomain 0 is pinned)
        pptr, psrc = lists(nfc + np.arange(1, N, dtype=np.int64))
        self.pptr, self.psrc = t(pptr), t(psrc)
        self.maxC = maxC
        self.factored = False
        self.persistent = False   # per-level launches (faster than nd_persist.cu today)
        if self.levels:
            self._build_persistent(nodes, pos_in_level, pptr, t)

    def _build_persistent(self, nodes, pos_in_level, pptr, t):
        """Global node table + topologically ordered work items of the one-kernel solve
        (csrc/nd_persist.cu)."""
        levels = self.levels
        nb = np.cumsum([0] + [L.m for L in levels])
        sb = np.cumsum([0] + [L.ysize for L in levels])
        bb = np.cumsum([0] + [len(L.h["bnd_flat"]) for L in levels])
        lb = np.cumsum([0] + [int(L.h["lptr"][-1]) for L in levels])
        fb = np.cumsum([0] + [L.csize for L in levels])
        self.fc_base = fb
        gid = {k: int(nb[li] + q) for k, (li, q) in pos_in_level.items()}
        nn = int(nb[-1])
        NC = 11
        tab = np.zeros((nn, NC), dtype=np.int64)
        off = np.zeros(nn, dtype=np.int64)
        for li, L in enumerate(levels):
            g0 = int(nb[li])
            tab[g0:g0 + L.m, 0] = L.s
            tab[g0:g0 + L.m, 1] = L.b
            tab[g0:g0 + L.m, 2] = sb[li] + L.h["sep_ptr"][:-1]
            tab[g0:g0 + L.m, 3] = bb[li] + L.h["bnd_ptr"][:-1]
            tab[g0:g0 + L.m, 4] = L.cb_off
            off[g0:g0 + L.m] = fb[li] + L.h["data_off"][:-1]
        tab[:, 5:8] = -1
        for k, g in gid.items():
            for slot, c in enumerate(nodes[k]["ch"]):
                if c in gid:
                    tab[g, 6 + slot] = gid[c]
                    tab[gid[c], 5] = g
        lptr_g = [np.zeros(1, np.int64)]
        for li, L in enumerate(levels):
            lp = L.h["lptr"].astype(np.int64)
            lptr_g.append(lp[1:] + lb[li])
        lptr_g = np.concatenate(lptr_g)
        lsrc_g = np.concatenate([L.h["lsrc"][:L.h["lptr"][-1]].astype(np.int64) for L in levels]
                                + [np.zeros(1, np.int64)])
        G = 296   # ~2 CTAs per SM worth of items per level
        items = []
        for li, L in enumerate(levels):
            g0 = int(nb[li])
            rows = (L.s + L.b).astype(np.int64)
            rf = max(8, -(-int(rows.sum()) // G))
            for q in range(L.m):
                g = g0 + q
                nr = int(rows[q])
                nf = 0
                for r0 in range(0, nr, rf):
                    items.append((2, g, r0, min(r0 + rf, nr)))
                    nf += 1
                tab[g, 8], tab[g, 9] = nf, 0
        npr = max(self.N - 1, 0)
        pg = [(3, -1, e0, min(e0 + 256, npr)) for e0 in range(0, npr, 256)]
        pv = [(4, -1, r0, min(r0 + 8, npr)) for r0 in range(0, npr, 8)]
        items += pg + pv
        for li in range(len(levels) - 1, -1, -1):
            L = levels[li]
            g0 = int(nb[li])
            wpr = getattr(L, "wpr", 1)
            rb = (8 // wpr) if wpr > 1 else max(8, -(-int(L.s.sum()) // G))
            for q in range(L.m):
                ns = int(L.s[q])
                nbk = 0
                for k0 in range(0, ns, rb):
                    items.append((5 | (wpr << 8), g0 + q, k0, min(k0 + rb, ns)))
                    nbk += 1
                tab[g0 + q, 10] = nbk
        self.p_items = t(np.array(items, dtype=np.int32).reshape(-1, 4))
        self.p_nitems = len(items)
        self.p_nodes = t(tab.astype(np.int32))
        self.p_nn = nn
        self.p_off = t(off, torch.int64)
        self.p_sep = t(np.concatenate([L.h["sep_flat"] for L in levels]).astype(np.int32))
        bf = np.concatenate([L.h["bnd_flat"] for L in levels]).astype(np.int32)
        self.p_bnd = t(bf if len(bf) else np.zeros(1, np.int32))
        self.p_lptr = t(lptr_g.astype(np.int32))
        self.p_lsrc = t(lsrc_g.astype(np.int32))
        self.p_npg, self.p_npv = len(pg), len(pv)
        self.p_root = int(nb[-1]) - 1
        self.p_ysize = int(sb[-1])
        self.p_smem = int(max(max(int(L.s.max()) for L in levels),
                              max(int(L.b.max()) for L in levels) + 8, npr, 1))
        self.p_cnt = torch.zeros(3 + 3 * nn, dtype=I32, device=self.dev)

    # --------------------------------------------------------------- numeric

    def factor(self, Kc, sub_rows_dev, b0):
        """Assemble and factor every front (leaves -> root); returns the root level."""
        st = _stream()
        lib = nat.load()
        info = torch.zeros(1, dtype=I32, device=self.dev)
        for li, L in enumerate(self.levels):
            L.F = torch.empty(L.m * L.nf * L.nf, dtype=F64, device=self.dev)
            child = self.levels[li - 1] if li > 0 else None
            for slot in (0, 1):
                nat.call("bddc_nd_assemble", L.m, L.S, L.B, L.nf, slot, L.K, _p(L.cmap),
                         _p(L.ckind), _p(L.sep_idx), _p(L.F),
                         _p(child.F) if child is not None else None,
                         child.S if child is not None else 0,
                         child.nf if child is not None else 1,
                         _p(Kc), _p(sub_rows_dev), _p(b0), self.maxC, st)
            ws = torch.empty(lib.bddc_spd_inverse_workspace(L.S, L.m, 32) // 8 + 2, dtype=F64,
                             device=self.dev)
            nat.call("bddc_spd_inverse_batched", _p(L.F), L.S, L.nf, L.nf * L.nf, L.m, 32,
                     _p(ws), _p(info), st)
            del ws
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
        if int(info.item()):
            raise ConfigurationError("coarse problem singular (non-positive pivot in S_Pi)")
        self.factored = True
        self.Fc_all = torch.empty(max(int(self.fc_base[-1]), 1), dtype=F64, device=self.dev)
        for li, L in enumerate(self.levels):
            L.Fc = self.Fc_all[int(self.fc_base[li]):int(self.fc_base[li]) + max(L.csize, 1)]
            nat.call("bddc_nd_compact", L.m, L.S, L.nf, L.B, _p(L.F), _p(L.X), _p(L.info),
                     _p(L.data_off), _p(L.Fc), st)
        # bytes streamed per solve: F11inv + X (forward) + X^T (backward)
        self.bytes = sum(L.csize * 8 for L in self.levels)
        return self.levels[-1]

    def release_fronts(self):
        """Drop the padded factorisation fronts once Pc has been read off the root."""
        for L in self.levels:
            L.F = None
            L.X = None

    def solve(self, r, x, Pcinv, npc):
        """Pinned coarse solve on the combined vector [flux | pressures] (coarse.py:208-215).

        r, x: length nfc + N.  r is read-only; x[nfc] (subdomain 0) is pinned to 0.
        """
        st = _stream()
        ys, cb = self._bufs()
        if self.persistent and self.levels:
            nat.call("bddc_nd_solve_persist", self.p_nitems, _p(self.p_items), self.p_nn,
                     _p(self.p_nodes), _p(self.p_off), _p(self.p_sep), _p(self.p_bnd),
                     _p(self.p_lptr), _p(self.p_lsrc), _p(self.pptr), _p(self.psrc),
                     _p(self.Fc_all), _p(Pcinv), _p(r), _p(self._rs_all), _p(self._y_all), _p(cb),
                     _p(self._prhs), _p(x), _p(self.p_cnt), self.p_root, self.N, self.nfc, npc,
                     self.p_npg, self.p_npv, self.p_smem, 0, st)
            return
        for li, L in enumerate(self.levels):
            nat.call("bddc_nd_fwd", L.ysize, L.n_ft, L.smax, _p(L.ftasks), _p(L.info), _p(L.data_off),
                     _p(L.sep_flat), _p(L.lptr), _p(L.lsrc), _p(L.Fc), _p(r), _p(self._rs), _p(ys[li]),
                     _p(cb), st)
        nat.call("bddc_nd_pressure", self.N, self.nfc, npc, _p(self.pptr), _p(self.psrc), _p(cb),
                 _p(Pcinv), _p(r), _p(self._prhs), _p(x), st)
        for li in range(len(self.levels) - 1, -1, -1):
            L = self.levels[li]
            nat.call("bddc_nd_bwd", L.n_bt, L.bmax, L.wpr, _p(L.btasks), _p(L.info), _p(L.data_off),
                     _p(L.sep_flat), _p(L.bnd_flat), _p(L.Fc), _p(ys[li]), _p(x), st)

    def _bufs(self):
        if getattr(self, "_yb", None) is None:
            ys = [torch.empty(max(L.ysize, 1), dtype=F64, device=self.dev) for L in self.levels]
            cb = torch.empty(self.cb_total, dtype=F64, device=self.dev)
            self._yb = (ys, cb)
            self._prhs = torch.empty(max(self.N, 1), dtype=F64, device=self.dev)
            self._rs = torch.empty(max(max(L.ysize for L in self.levels), 1), dtype=F64, device=self.dev)
            py = max(getattr(self, "p_ysize", 0), 1)
            self._rs_all = torch.empty(py, dtype=F64, device=self.dev)
            self._y_all = torch.empty(py, dtype=F64, device=self.dev)
        return self._yb

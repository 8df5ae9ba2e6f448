"""BDDC setup, interface PCG and the three-step solve on one B200.

Drop-in for the reference's `bddcflow.solver` path
(`/root/reference/pkg/src/bddcflow/solver.py:29-398`): same `SolveConfig`,
`SolveReport`, `BddcSetup`, `solve(system, dec, config, u_exact=None,
setup=None, iterate_callback=None)` signatures, argument meaning and error
classes.  Every numerical step runs in hand-written sm_100a kernels from
libbddc.so (csrc/); torch only allocates device memory and provides the
stream.  There is no CPU fallback.
"""

from __future__ import annotations

import ctypes as C
import math
import os
import warnings
from collections.abc import Mapping
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as nat
from . import views as _views
from .coarse_nd import CoarseND
from .decomposition import Decomposition
from .errors import (ConfigurationError, ConstraintRankError, InternalConsistencyError,
                     InvalidArgumentError, NonConvergenceError,
                     NumericalFailureError)

_p = nat.ptr
F64 = torch.float64
I32 = torch.int32
SPD_LEAF = 64   # leaf order of the batched SPD inverses (leaf64 kernel: one launch per 64-block)


@dataclass
class SolveConfig:
    """solver.py:29-44."""

    tau: float = math.inf
    scaling: str = "multiplicity"
    tol: float = 1e-6
    maxit: int = 5000
    constraints: str = "initial"   # initial | adaptive | multiscale

    def __post_init__(self):
        if not 0.0 < self.tol < 1.0:
            raise InvalidArgumentError("tol must lie in (0, 1)")
        if not self.tau > 1.0:
            raise InvalidArgumentError("tau must exceed 1")
        if self.constraints not in ("initial", "adaptive", "multiscale"):
            raise InvalidArgumentError(
                f"unknown constraint mode {self.constraints!r}")
        if self.scaling not in ("multiplicity", "stiffness"):
            raise InvalidArgumentError(f"unknown scaling kind {self.scaling!r}")


@dataclass
class SolveReport:
    """solver.py:47-62."""

    u: np.ndarray
    p: np.ndarray
    it: int
    kappa: float
    omega_tilde: float
    n_c: int
    residuals: np.ndarray
    u0: np.ndarray = None
    u_star: np.ndarray = None
    eps0: float = None
    eps_star: float = None
    conservation_defect: float = 0.0
    pressure_warning: bool = False
    converged: bool = True


# Largest subdomain count for which the balance operators (projection, shift) are
# kept as dense N x N matrices applied by one multi-CTA GEMV (134 MB at 4096);
# beyond it they are separable transforms over the subdomain grid.
DENSE_BALANCE_MAX = 4096


def _dev():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1901_02090_b200 needs a CUDA device (no CPU fallback)")
    return torch.device("cuda")


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _geom(dec, system=None):
    f = dec.geom_fields()
    g = nat.Geom()
    g.dim = f["dim"]
    for a in range(3):
        g.n[a] = int(f["n"][a])
        g.h[a] = float(f["h"][a])
        g.S[a] = int(f["S"][a])
        for s in range(len(f["so"][a])):
            g.so[a][s] = int(f["so"][a][s])
            g.sw[a][s] = int(f["sw"][a][s])
    g.vol = f["vol"]
    for a in range(4):
        g.fam_off[a] = int(f["fam_off"][a])
    for key in ("n_cells", "n_flux", "N", "n_gamma", "n_faces", "maxG", "maxP",
                "maxL", "maxF"):
        setattr(g, key, int(f[key]))
    # mode B: the Dirichlet faces of one axis are flux dofs after the interior ones
    ax = None if system is None else system.dirichlet_axis
    g.dir_axis = -1 if ax is None else int(ax)
    g.n_flux_int = g.n_flux
    g.n_bt = 0 if ax is None else dec.grid.n_boundary_faces(ax)
    g.n_flux = g.n_flux_int + 2 * g.n_bt
    lumped = bool(getattr(system, "lumped", False)) if system is not None else False
    g.a_diag, g.a_off = (3.0, 0.0) if lumped else (2.0, 1.0)
    return g


def _upload(a, dt, dev):
    """Host table -> device without a stream sync: staged through pinned memory
    (torch's caching host allocator keeps the block until the async copy ran).
    torch.as_tensor(..., device=cuda) would wait for all queued device work."""
    h = torch.from_numpy(np.ascontiguousarray(a)).to(dt)
    return h.pin_memory().to(dev, non_blocking=True)


def _pad(n, m):
    return max(m, ((n + m - 1) // m) * m)


class BddcSetup:
    """Everything reusable across solves (solver.py:65-183), resident in HBM.

    Device state per subdomain i (maxP / maxG / maxC padded):
      Q[i]    = P_i^+  pressure-Schur pseudo-inverse   (interior solves)
      S[i]    = interface Schur complement              (operator)
      T[i]    = Gamma block of the constrained inverse  (preconditioner)
      PsiT[i] = Gamma rows of the coarse basis, transposed (restriction/prolongation)
    and the explicit coarse operators Mc (flux block of the pinned coarse
    inverse) and Wq (pressure-rhs -> coarse flux, solve step 1).
    """

    def __init__(self, system, dec, config, timings=None, pair_spectra=False):
        if not isinstance(dec, Decomposition):
            raise InvalidArgumentError("dec must come from regular_partition()")
        dev = _dev()
        nat.load()
        self.system = system
        self.dec = dec
        self.config = config
        self.dev = dev
        self._ktimer = None
        # resolve every pair eigenvalue and keep PairEigenReports (eigs-report);
        # the solve path only needs the ones above tau and the next one
        self.pair_spectra = bool(pair_spectra)
        self.pcg_timer = None   # list -> (start, end) CUDA events of every PCG graph launch
        self.geom = _geom(dec, system)
        G = self.geom
        # mode B (PressureDrop): subdomains on a Dirichlet end have a nonsingular
        # interior pressure block, no balance constraint and no coarse pressure;
        # the others ("floating") keep both.  Mode A: all floating, subdomain 0's
        # coarse pressure pinned (coarse.py:192-194).
        self.mode_b = system.dirichlet is not None
        if self.mode_b:
            ax = system.dirichlet_axis
            sidx = (np.arange(dec.n_subdomains) // int(np.prod(dec.S3[:ax]))) % dec.S3[ax]
            self.floating = (sidx != 0) & (sidx != dec.S3[ax] - 1)
            self.has_p = self.floating
        else:
            self.floating = np.ones(dec.n_subdomains, dtype=bool)
            self.has_p = np.arange(dec.n_subdomains) != 0
        gp = C.byref(G)
        st = _stream()
        self._timings = timings
        ev = self._events()
        # coarse chain of the preconditioner (and the T_i setup branch): high priority
        # so its small latency-bound kernels get SM slots ahead of queued GEMV blocks
        self.side_stream = torch.cuda.Stream(device=dev, priority=-1)
        N, mg, mp = dec.n_subdomains, dec.maxG, dec.maxP
        self.N, self.maxG, self.maxP = N, mg, mp
        t = lambda a, dt=I32: _upload(a, dt, dev)
        # topology tables: per-slot / per-dof / per-cell ones in closed form on the
        # device (csrc/topology.cu); the host keeps only O(N) and per-face tables
        e = lambda *shape: torch.empty(shape, dtype=I32, device=dev)
        ngam = max(dec.n_gamma, 1)
        self.d_gpos = e(N, mg)
        self.d_gcode = e(N, mg)
        self.d_nG = e(N)
        self.d_fslot = e(N, 6, dec.maxF)
        self.d_gown = e(ngam, 2)
        self.d_gamma = e(ngam)
        self.d_gface = e(ngam)
        self.d_cell_sub = e(G.n_cells)
        self.d_faces = t(dec.face_table if dec.n_faces else np.zeros((1, 4)))
        self.d_face_base = t(dec.face_base)
        nat.call("bddc_topology_box", gp, _p(self.d_face_base), _p(self.d_nG), _p(self.d_gpos),
                 _p(self.d_gcode), _p(self.d_fslot), _p(self.d_gown), _p(self.d_gamma),
                 _p(self.d_gface), _p(self.d_cell_sub), st)
        eig_w, dm_w = dec.laplacian_eigs(True)
        eig_u, _ = dec.laplacian_eigs(False)
        self.d_eig_w = t(eig_w, F64)
        self.d_dm_w = t(dm_w, F64)
        # dense (Phi Phi^T)^+ for the balanced projection: one multi-CTA GEMV per
        # projection instead of the latency-bound single-CTA separable solve
        # (N^2 doubles: used up to N = 4096, i.e. 134 MB per GEMV)
        S3 = dec.S3
        self.d_Lp = None
        self.d_Lu = None
        self._lap_ws = torch.empty(2 * N, dtype=F64, device=dev)   # multi-CTA separable solve
        self.NF = 0
        if self.mode_b and N <= DENSE_BALANCE_MAX:
            self.d_Lp, self.d_Lu = self._dirichlet_laplacian_inverses()
        elif self.mode_b:
            # large N: separable solves on the floating sub-box (strips 1..S_d-2 of the
            # drop axis), gathered from / scattered to the full subdomain vector
            ax = system.dirichlet_axis
            ew, dw, self.S3F = dec.laplacian_eigs(True, ax)
            eu, _, _ = dec.laplacian_eigs(False, ax)
            self.NF = int(np.prod(self.S3F))
            self.d_fidx = t(np.nonzero(self.floating)[0].astype(np.int32))
            self.d_eig_wF, self.d_dm_wF, self.d_eig_uF = t(ew, F64), t(dw, F64), t(eu, F64)
            zf = lambda n: torch.zeros(max(n, 1), dtype=F64, device=dev)
            self._phiF, self._zF, self._lap_wsF = zf(self.NF), zf(self.NF), zf(2 * self.NF)
            self.w_zp, self.w_zs = zf(N), zf(N)   # z on all subdomains, zero off the floating set
        elif N <= DENSE_BALANCE_MAX:
            ws = torch.empty(2 * N * N, dtype=F64, device=dev)
            self.d_Lp = torch.empty(N * N, dtype=F64, device=dev)
            nat.call("bddc_lap_dense", S3[0], S3[1], S3[2], _p(self.d_eig_w), _p(self.d_dm_w),
                     _p(ws), _p(self.d_Lp), st)
            del ws
        self.d_eig_u = t(eig_u, F64)
        # permeability -> cell coefficients, D, delta
        k = np.ascontiguousarray(system.perm.k, dtype=np.float64)
        self.d_k = _upload(k, F64, dev)
        self.d_coef = torch.empty(G.n_cells * 3, dtype=F64, device=dev)
        nat.call("bddc_cell_coeffs", gp, _p(self.d_k), _p(self.d_coef), st)
        self.d_Dsub = torch.empty(N, dtype=F64, device=dev)
        nat.call("bddc_rescale", gp, _p(self.d_coef), _p(self.d_Dsub), st)
        self.d_delta = torch.empty(N * mg, dtype=F64, device=dev)
        nat.call("bddc_weights", gp, int(config.scaling == "stiffness"),
                 _p(self.d_coef), _p(self.d_gcode), _p(self.d_delta), st)
        self._mark(ev, "prep")
        # local interior elimination: P, G, S_A -> Q = P^+ -> S
        self.d_Q = torch.empty(N * mp * mp, dtype=F64, device=dev)
        Gc = torch.empty(N * mg * dec.maxL, dtype=F64, device=dev)
        SAd = torch.empty(N * mg, dtype=F64, device=dev)
        SApart = torch.empty(N * mg, dtype=I32, device=dev)
        SAoff = torch.empty(N * mg, dtype=F64, device=dev)
        alpha = torch.empty(N * (mp + 1), dtype=F64, device=dev)   # Jacobi scaling of P
        nat.call("bddc_local_build", gp, _p(self.d_coef), _p(self.d_fslot),
                 _p(self.d_Q), _p(Gc), _p(SAd), _p(SApart), _p(SAoff),
                 _p(alpha), st)
        info = torch.zeros(5, dtype=I32, device=dev)
        ws = torch.empty(nat.load().bddc_spd_inverse_workspace(mp, N, SPD_LEAF) // 8 + 2,
                         dtype=F64, device=dev)
        nat.call("bddc_spd_inverse_batched", _p(self.d_Q), mp, mp, mp * mp, N,
                 SPD_LEAF, _p(ws), _p(info), st)
        del ws
        nat.call("bddc_local_pinv_fix", gp, _p(self.d_Q), _p(alpha), st)
        Wt = torch.empty(N * mg * mp, dtype=F64, device=dev)
        self.d_S = torch.empty(N * mg * mg, dtype=F64, device=dev)
        nat.call("bddc_local_schur", gp, _p(self.d_gcode), _p(self.d_Q), _p(Gc),
                 _p(SAd), _p(SApart), _p(SAoff), _p(Wt), _p(self.d_S), st)
        del Wt, Gc, SAd, SApart, SAoff
        # the local solves read Q tile-packed (symmetric upper tiles: half the bytes)
        self.d_Qp = torch.empty(N * nat.load().bddc_sym_packed_elems(mp), dtype=F64, device=dev)
        nat.call("bddc_pack_sym", N, mp, _p(self.d_Q), _p(self.d_Qp), st)
        del self.d_Q
        Sinv = self.d_S.clone()
        leaf = SPD_LEAF
        ws = torch.empty(nat.load().bddc_spd_inverse_workspace(mg, N, leaf) // 8 + 2,
                         dtype=F64, device=dev)
        nat.call("bddc_spd_inverse_batched", _p(Sinv), mg, mg, mg * mg, N, leaf,
                 _p(ws), _p(info[1:]), st)
        del ws
        self._mark(ev, "local")
        # adaptive pair eigenproblems (adaptive.py:176-195)
        nf = dec.n_faces
        self.pair_reports = {}
        self.omega_tilde = None
        maxsel = 1
        nadd = np.zeros(nf, dtype=np.int64)
        rows = torch.zeros(1, dtype=F64, device=dev)
        qbasis = None
        self.pair_lambda = None
        self.pair_added = None   # rows added per face beyond the initial one
        if config.constraints == "adaptive" and nf:
            maxsel = dec.maxF
            lam_ld = dec.maxF
            lam = torch.empty(nf * lam_ld, dtype=F64, device=dev)
            d_nsel = torch.empty(nf, dtype=I32, device=dev)
            d_nadd = torch.empty(nf, dtype=I32, device=dev)
            rows = torch.zeros(nf * maxsel * 112, dtype=F64, device=dev)
            omega = torch.empty(nf, dtype=F64, device=dev)
            scratch = torch.empty(nat.load().bddc_pair_scratch_bytes(nf) // 8,
                                  dtype=F64, device=dev)
            qbasis = torch.zeros(nf * (maxsel + 1) * 112, dtype=F64, device=dev)
            err = torch.zeros(1, dtype=I32, device=dev)
            tau = config.tau if math.isfinite(config.tau) else 1e308
            # two launches by face size: small faces need a third of the shared
            # memory, so three faces share an SM instead of one
            fm = dec.face_table[:, 3]
            for sel, mm in ((fm <= 64, 64), (fm > 64, int(dec.maxF))):
                if sel.any():
                    fl = t(np.nonzero(sel)[0].astype(np.int32))
                    nat.call("bddc_pair_eigs", gp, _p(self.d_faces), _p(self.d_fslot),
                             _p(self.d_S), _p(Sinv), _p(self.d_delta), float(tau),
                             maxsel, _p(lam), lam_ld, _p(d_nsel), _p(d_nadd), _p(rows),
                             _p(omega), _p(scratch), _p(qbasis), _p(err), _p(fl), len(fl), mm,
                             int(self.pair_spectra), st)
            del scratch
            # the nested-dissection tree of the subdomain grid depends on the partition
            # only: build it (once per Decomposition) while the device works through the
            # local and pair phases, before the first host sync of the setup
            _nd_prefetch(dec, self.has_p)
            e = int(err.item())
            if e & 1:
                raise NumericalFailureError("pair eigensolver: M not positive definite")
            if e & 2:
                raise InternalConsistencyError(
                    f"more than {maxsel} eigenvalues above tau on one face")
            nadd = d_nadd.cpu().numpy().astype(np.int64)
            self.pair_selected = d_nsel.cpu().numpy()
            self.pair_added = nadd
            self.pair_lambda = lam.view(nf, lam_ld)
            # PairEigenReports for every adaptive setup (solver.py:76-88): the full
            # spectrum with pair_spectra, else the eigenvalues the selection resolved
            # (those above tau and the next one, which sets omega)
            # (materialised on first access: the host loop stays out of the setup)
            self.pair_reports = _LazyPairReports(dec, self.pair_lambda, self.pair_selected,
                                                 self.pair_spectra)
            self.face_omega = omega.cpu().numpy()
            self.omega_tilde = float(max(self.face_omega.max(), 1.0)) if nf else 1.0
        elif config.constraints == "adaptive":
            self.omega_tilde = 1.0
        elif config.constraints == "multiscale" and nf:
            # MsMFEM baseline (solver.py:89-90, adaptive.py:207-269): one row per face
            maxsel = 1
            rows, qbasis, nadd = self._multiscale_rows(system, Sinv)
            self.pair_added = nadd
            # per face: the multiscale row on the shared dofs, outward from the lower subdomain
            fm = dec.face_table[:, 3]
            rh = rows.view(nf, 112).cpu().numpy()
            self.multiscale_rows = [rh[q, :int(fm[q])].copy() for q in range(nf)]
        self._mark(ev, "pairs")
        # coarse dof numbering: per face [initial, adaptive...]
        per_face = 1 + nadd
        self._per_face = per_face
        self._rows_dev, self._rows_maxsel = rows, maxsel   # harvested face rows (views.cset)
        cstart = np.concatenate([[0], np.cumsum(per_face)[:-1]]).astype(np.int64)
        self.n_flux_coarse = int(per_face.sum()) if nf else 0
        self._build_coarse_tables(cstart, per_face, maxsel)
        maxC = self.maxC
        dev_rows = t(self.sub_rows)
        self.d_sub_rows = dev_rows
        self.d_cown = t(self.cown if len(self.cown) else np.zeros((1, 2)))
        self.d_nC = t(self.nC)
        Ct = torch.empty(N * mg * maxC, dtype=F64, device=dev)
        Y = torch.empty(N * mg * maxC, dtype=F64, device=dev)
        E = torch.empty(N * mg * maxC, dtype=F64, device=dev)
        gam = torch.empty(N, dtype=F64, device=dev)
        self.d_Kc = torch.empty(N * maxC * maxC, dtype=F64, device=dev)
        self.d_Psi = torch.empty(N * mg * maxC, dtype=F64, device=dev)
        self.d_T = torch.empty(N * mg * mg, dtype=F64, device=dev)
        self.d_b0 = torch.empty(N * maxC, dtype=F64, device=dev)
        wsz = nat.load().bddc_spd_inverse_workspace(maxC, N, 32)
        ws = torch.empty(wsz // 8 + 2, dtype=F64, device=dev)
        dims = torch.empty(N * 16, dtype=I32, device=dev)
        cl_args = [gp, _p(dev_rows), _p(self.d_faces), _p(self.d_fslot), _p(self.d_gcode),
                   _p(self.d_nG), _p(rows), _p(qbasis) if qbasis is not None else None, maxsel,
                   _p(self.d_S), _p(Sinv), _p(self.d_Dsub), maxC, _p(Ct), _p(Y), _p(E), _p(gam),
                   _p(self.d_Kc), _p(self.d_Psi), _p(self.d_T), _p(self.d_b0), _p(ws), _p(dims),
                   _p(info[2:])]
        # T_i (its batched inverse) on a side stream with its own workspaces, concurrently
        # with Kc / Psi / b0 and then the global coarse factorisation (the critical
        # path: host symbolic analysis, latency-bound small-batch inverses)
        # small subdomains (LDG GEMV, maxG < 256) pack S_i in 16 x 16 tiles (the packed
        # bytes follow the live triangle: C4 S GEMV 186 -> 165 us); T_i keeps 32-tiles,
        # whose fewer, larger tiles suit the one-CTA-per-SM launch beside the coarse chain
        self.tile16 = (mg < 256 and mg % 16 == 0 and os.environ.get("BDDC_TILE16", "1") != "0"
                       and os.environ.get("BDDC_SYMV_BULK", "") != "1")
        npk = nat.load().bddc_sym_packed_elems(mg)
        npk16 = nat.load().bddc_sym_packed16_elems(mg) if self.tile16 else npk
        self.d_Sp = torch.empty(N * npk16, dtype=F64, device=dev)
        self.d_Tp = torch.empty(N * npk, dtype=F64, device=dev)
        Ct2 = torch.empty(N * mg * maxC, dtype=F64, device=dev)
        Y2 = torch.empty(N * mg * maxC, dtype=F64, device=dev)
        ws2 = torch.empty(nat.load().bddc_spd_inverse_workspace(mg, N, 32) // 8 + 2,
                          dtype=F64, device=dev)
        dims2 = torch.empty(N * 16, dtype=I32, device=dev)
        main = torch.cuda.current_stream()
        side = torch.cuda.Stream(device=dev)   # normal priority: the ND branch is the critical path
        side.wait_stream(main)
        cl2 = list(cl_args)
        cl2[13], cl2[14], cl2[21], cl2[22], cl2[23] = _p(Ct2), _p(Y2), _p(ws2), _p(dims2), _p(info[4:])
        with torch.cuda.stream(side):
            ss = _stream()
            nat.call("bddc_coarse_local", *cl2, 2, ss)
            nat.call("bddc_pack_sym", N, mg, _p(self.d_T), _p(self.d_Tp), ss)
        nat.call("bddc_coarse_local", *cl_args, 1, st)
        # tile-packed symmetric S_i, T_i for the PCG loop (half the bytes of full storage)
        nat.call("bddc_pack_sym16" if self.tile16 else "bddc_pack_sym", N, mg, _p(self.d_S),
                 _p(self.d_Sp), st)
        self._mark(ev, "coarse_local")
        # global coarse: multifrontal S_Pi (nested dissection) + pinned pressure Schur Pc
        nfc = self.n_flux_coarse
        self.nfc = nfc
        self.npad = _pad(max(nfc, 1), 64)
        self.nd = None
        if nfc:
            self.nd = CoarseND(dec, per_face, cstart, self.sub_rows, self.nC, maxC, dev,
                               has_p=self.has_p)
            self.nd.factor(self.d_Kc, dev_rows, self.d_b0)
            self.nd.release_fronts()
        main.wait_stream(side)   # T_i done; its workspaces may go now
        del Ct, Y, E, gam, ws, Sinv, dims, cl_args, self.d_S, self.d_T, Ct2, Y2, ws2, dims2, cl2
        bad = info.cpu().numpy()
        # info slots hold 1 + the first failing subdomain (dense.cu leaf kernels)
        if bad[0] or bad[1]:
            i = int(bad[0] or bad[1]) - 1
            raise NumericalFailureError(   # substructure.py:65-70
                f"interior KKT factorization failed on subdomain {i}: "
                "pressure Schur complement or S_i not positive definite", where=i)
        if bad[2] or bad[4]:
            i = int(bad[2] or bad[4]) - 1
            raise ConstraintRankError(   # coarse.py:159-163
                f"constrained KKT singular on subdomain {i}; check constraint rank")
        if self.nd is not None:
            self.nd.check()
        self._mark(ev, "coarse")
        # persistent PCG workspaces
        ng = dec.n_gamma
        self.n_gamma = ng
        z = lambda n: torch.zeros(max(n, 1), dtype=F64, device=dev)
        self.w_yb = z(N * mg)
        self.w_yb2 = z(N * mg)
        self.w_v = z(N * maxC)
        self.w_rc = z(self.nfc + N)     # combined coarse rhs [flux | pressures]
        self.w_xc = z(self.nfc + N)     # combined coarse solution
        self.w_phi = z(N)
        self.w_z = z(N)
        self.w_dot = torch.zeros(nat.load().bddc_dot_workspace() // 8 + 1, dtype=F64, device=dev)
        self.w_scal = z(16)
        self.w_norms = z(8)     # deferred per-solve norms (_N_* slots)
        self._host_norms = torch.zeros(8, dtype=F64, pin_memory=True)
        self.d_dct = torch.empty(sum(n * n + n for n in dec.n3), dtype=F64, device=dev)
        nat.call("bddc_dct_init", gp, _p(self.d_dct), st)
        self._graphs = {}
        self._graph_kernels = {}
        self.graph_kernels_run = 0   # kernels executed inside PCG graph launches (accounting)
        self._pcg_b = None
        self._work = None
        self._host_scal = torch.empty(16, dtype=F64, pin_memory=True)
        self.stream = torch.cuda.Stream(device=dev)
        self.n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
        # T_i GEMV grid beside the coarse chain: one 256-thread CTA per SM (grid-stride
        # over subdomains).  The latency-bound chain is the critical path; giving T more
        # bandwidth starves it (C3 PCG-only it/s: 1424 at 1x SMs, 1363 at 2x, 1346 at 4x,
        # 1357 with 512-thread CTAs; the chain's kernels carry the side stream's
        # priority as a launch attribute so it survives graph capture)
        self.t_grid = self.n_sm
        # persistent bulk-streamed S_i / T_i GEMVs (one CTA per SM, ~160 KB of tiles
        # in flight each): S on every SM; T on t_grid_bulk SMs, the rest left to the
        # concurrent coarse chain
        # bulk kernel for subdomains with many tiles (C3: maxG 448, 105 tiles: S GEMV
        # 211 -> 208 us, PCG 1478 -> 1495 it/s); small subdomains (C4: maxG 160, 15
        # tiles) keep the one-CTA-per-subdomain LDG kernel, whose occupancy hides the
        # per-subdomain gather and epilogue (C4 PCG 1163 vs 1087 it/s with bulk)
        self.symv_bulk = {"1": True, "0": False}.get(os.environ.get("BDDC_SYMV_BULK", ""), 256 <= dec.maxG <= 512)
        # C3 (scripts/precond_tune.py, chunked tile classes): precond 399 us at 148
        # CTAs, 376 at 120, 354 at 100, 366 at 84; T alone 218 / 223 / 235 / 263 us
        self.t_grid_bulk = max(1, (self.n_sm * 2) // 3)
        self._sched = torch.zeros(8, dtype=I32, device=dev)   # ticket counters per call site
        self.restrict_first = False
        # Step 2's two local solves in one two-rhs pass over Q where the two-rhs kernel's
        # shared memory still allows several CTAs per SM (C4: 36.98 -> 36.79 ms per
        # solve); at C3 (maxP 512, ~96 KB per CTA) the two passes are faster
        # (26.86 vs 27.21 ms, scripts/step2_check.py)
        self.step2_fused = (dec.maxG + 23 * dec.maxP) * 8 <= 64 * 1024
        self._scaling_checked = False
        self.force_eager = False   # host-driven PCG loop (profiling); default is the graph
        self._solves = 0   # public solves run on this setup
        # per-solve buffers, allocated here on the allocating stream while the device
        # finishes the setup (allocations on the solve stream could not reuse the
        # blocks the setup freed and would each go to cudaMalloc)
        self.work()
        self._pcg_bufs(config.maxit)
        if self.nd is not None:
            self.nd._bufs()
        self._mark(ev, "done")
        self.phase_ms = self._finish(ev)

    # ---------------------------------------------------------------- util

    def _events(self):
        if self._timings is None:
            return None
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        return [("start", e)]

    def _mark(self, ev, name):
        if ev is None:
            return
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        ev.append((name, e))
        import time as _t
        self._hmarks = getattr(self, "_hmarks", [])
        self._hmarks.append((name, _t.perf_counter()))

    def _finish(self, ev):
        if ev is None:
            return None
        ev[-1][1].synchronize()
        out = {}
        for (_, a), (n, b) in zip(ev[:-1], ev[1:]):
            out[n] = a.elapsed_time(b)
        out["total"] = ev[0][1].elapsed_time(ev[-1][1])
        hm = getattr(self, "_hmarks", [])
        for (_, a), (n, b) in zip(hm[:-1], hm[1:]):
            out["host_" + n] = 1000.0 * (b - a)
        if isinstance(self._timings, dict):
            self._timings.update(out)
        return out

    def _dirichlet_laplacian_inverses(self):
        """Mode B balance operators: (Phi_F Phi_F^T)^-1 (projection, solver.py:166-179)
        and the inverse face-graph Laplacian (balanced shift, solver.py:146-164) over
        the floating subdomains F, as N x N matrices with zero rows and columns for
        the others.  Both are principal submatrices of graph Laplacians whose graph
        reaches a Dirichlet subdomain, hence SPD: one batched device inverse."""
        dec, N, dev, st = self.dec, self.N, self.dev, _stream()
        n = _pad(N, 64)
        fl = _upload(self.floating.astype(np.int32), I32, dev)
        L = torch.empty(2 * n * n, dtype=F64, device=dev)
        nat.call("bddc_fill", 2 * n * n, 0.0, _p(L), st)
        nat.call("bddc_dirichlet_laplacian", N, n, dec.n_faces, _p(self.d_faces), _p(fl), _p(L), st)
        info = torch.zeros(1, dtype=I32, device=dev)
        ws = torch.empty(nat.load().bddc_spd_inverse_workspace(n, 2, 32) // 8 + 2,
                         dtype=F64, device=dev)
        nat.call("bddc_spd_inverse_batched", _p(L), n, n, n * n, 2, 32, _p(ws), _p(info), st)
        if int(info.item()):
            raise NumericalFailureError("mode B balance Laplacian not positive definite",
                                        where=int(info.item()) - 1)
        Lp = torch.empty(N * N, dtype=F64, device=dev)
        Lu = torch.empty(N * N, dtype=F64, device=dev)
        nat.call("bddc_dirichlet_finish", N, n, _p(fl), _p(L), _p(Lp), _p(Lu), st)
        return Lp, Lu

    def _multiscale_rows(self, system, Sinv):
        """Face rows of the pair-local unit-transfer solves (adaptive.py:207-262),
        from each subdomain's interior response to its unit source distribution
        (uniform, or following the wells) and the S_i face blocks."""
        dec, dev, st = self.dec, self.dev, _stream()
        N, mg, nf = self.N, self.maxG, dec.n_faces
        f = np.asarray(system.f, dtype=np.float64)
        tot = np.bincount(dec.cell_sub, weights=f, minlength=N)
        cnt = np.bincount(dec.cell_sub, minlength=N).astype(np.float64)
        well = np.abs(tot) > 1e-14
        dist = np.where(well[dec.cell_sub], f / np.where(well, tot, 1.0)[dec.cell_sub],
                        1.0 / cnt[dec.cell_sub])
        gdev = _upload(dist, F64, dev)
        g = torch.empty_like(gdev)
        # D-scaled cell values (local_solve reads g / D)
        nat.call("bddc_scale_cells", C.byref(self.geom), _p(gdev), _p(self.d_cell_sub),
                 _p(self.d_Dsub), _p(g), st)
        rg = torch.zeros(N * mg, dtype=F64, device=dev)
        a = nat.LocalSolveArgs()
        a.g_cell, a.g_scale = _p(g).value, 1.0
        a.rg_broken = _p(rg).value
        nat.call("bddc_local_solve", C.byref(self.geom), _p(self.d_coef), _p(self.d_gcode),
                 _p(self.d_gpos), _p(self.d_fslot), _p(self.d_Qp), _p(self.d_Dsub), C.byref(a), st)
        rows = torch.zeros(nf * 112, dtype=F64, device=dev)
        qbasis = torch.zeros(nf * 2 * 112, dtype=F64, device=dev)
        d_nadd = torch.zeros(nf, dtype=I32, device=dev)
        err = torch.zeros(1, dtype=I32, device=dev)
        nat.call("bddc_multiscale_rows", C.byref(self.geom), _p(self.d_faces), _p(self.d_fslot),
                 _p(self.d_S), _p(rg), 1, _p(rows), _p(qbasis), _p(d_nadd), _p(err), st)
        if int(err.item()) & 1:
            raise NumericalFailureError("multiscale: pair face block not positive definite")
        return rows, qbasis, d_nadd.cpu().numpy().astype(np.int64)

    def _build_coarse_tables(self, cstart, per_face, maxsel):
        """Per-subdomain coarse rows {g, face, k, sigma} in (face, k) order and the
        two owners (i*maxC + r) of every coarse dof (vectorised bookkeeping)."""
        dec, N = self.dec, self.N
        ft = dec.face_table
        nf = dec.n_faces
        nfc = int(per_face.sum()) if nf else 0
        f_of = np.repeat(np.arange(nf), per_face) if nf else np.zeros(0, np.int64)
        k_of = np.arange(nfc) - np.repeat(cstart, per_face) if nf else np.zeros(0, np.int64)
        g_of = np.arange(nfc)
        sub = np.concatenate([ft[f_of, 0], ft[f_of, 1]]) if nf else np.zeros(0, np.int64)
        sig = np.concatenate([np.ones(nfc, np.int64), -np.ones(nfc, np.int64)])
        ff = np.concatenate([f_of, f_of])
        kk = np.concatenate([k_of, k_of])
        gg = np.concatenate([g_of, g_of])
        o = np.lexsort((kk, ff, sub))
        sub, sig, ff, kk, gg = sub[o], sig[o], ff[o], kk[o], gg[o]
        nC = np.bincount(sub, minlength=N).astype(np.int32) if len(sub) else np.zeros(N, np.int32)
        maxC = _pad(int(nC.max()) if N else 1, 32)
        starts = np.concatenate([[0], np.cumsum(nC)[:-1]])
        r = np.arange(len(sub)) - starts[sub]
        sub_rows = np.full((N, maxC, 4), -1, dtype=np.int32)
        sub_rows[sub, r] = np.stack([gg, ff, kk, sig], axis=1)
        cown = np.zeros((nfc, 2), dtype=np.int32)
        cown[gg, np.where(sig > 0, 0, 1)] = sub * maxC + r
        self.sub_rows, self.cown, self.nC, self.maxC = sub_rows, cown, nC, maxC

    @property
    def n_c(self):
        return self.n_flux_coarse + self.N

    def _pcg_bufs(self, maxit):
        if self._pcg_b is None or self._pcg_b.maxit < maxit:
            # the captured PCG graphs hold the old history buffers' addresses: drop
            # them before the buffers are freed (a cached graph would otherwise write
            # alphas/betas/residuals into memory the allocator has handed out again)
            self._drop_graphs()
            self._pcg_b = _PCGBufs(self, maxit)
        return self._pcg_b

    def _drop_graphs(self):
        graphs = getattr(self, "_graphs", None)
        if not graphs:
            return
        torch.cuda.current_stream().synchronize()
        lib = nat.load()
        for g in graphs.values():
            lib.bddc_graph_destroy(g)
        graphs.clear()
        self._graph_kernels.clear()

    def work(self):
        if self._work is None:
            self._work = _Work(self)
        return self._work

    def __del__(self):
        try:
            _unregister_source(self)
        except Exception:
            pass
        try:
            lib = nat.load()
            for g in getattr(self, "_graphs", {}).values():
                lib.bddc_graph_destroy(g)
        except Exception:
            pass

    def _coarse_solve(self):
        """Pinned coarse solve w_xc = K0^-1 w_rc on [flux | pressures] (coarse.py:208-215)."""
        self.nd.solve(self.w_rc, self.w_xc)

    # ----------------------------------------- interface operator (device)

    def _schur(self, x, y, assemble=True):
        """y = S x (continuous interface vectors), solver.py:103-107.  assemble=False:
        the per-slot products stay in w_yb (the caller's projection assembles them)."""
        st = _stream()
        kt = self._ktimer
        if kt is not None:
            e0 = torch.cuda.Event(enable_timing=True)
            e0.record()
        self._symv(self.d_Sp, x, None, self.w_yb, 0, 0, st)
        if kt is not None:
            e1 = torch.cuda.Event(enable_timing=True)
            e1.record()
            kt["ev"].append((e0, e1))
        if assemble:
            nat.call("bddc_scatter", self.n_gamma, _p(self.d_gown), _p(self.w_yb), _p(y), st)

    def _project(self, y, dot=None, yb=None):
        """In-place balanced projection, solver.py:166-179.  dot = (x, op, hist): fuse
        the following PCG dot x . (P y) into the apply step (one pass, one launch).
        yb: y is not assembled yet; its per-slot values yb are summed on the fly by
        the phi and apply kernels (the scatter fused away; requires dot)."""
        st = _stream()
        if yb is not None:
            nat.call("bddc_phi_broken", self.N, self.maxG, _p(self.d_nG), _p(self.d_gpos),
                     _p(self.d_gcode), _p(self.d_gown), _p(yb), _p(self.w_phi), st)
        else:
            nat.call("bddc_phi", self.N, self.maxG, _p(self.d_nG), _p(self.d_gpos),
                     _p(self.d_gcode), _p(y), _p(self.w_phi), st)
        z = self.w_z
        if self.d_Lp is not None:
            nat.call("bddc_gemv_static", self.N, self.N, self.N, _p(self.d_Lp), _p(self.w_phi),
                     _p(self.w_z), st)
        elif self.mode_b:
            if self.NF:
                S3 = self.S3F
                nat.call("bddc_gamma_flux", self.NF, _p(self.d_fidx), _p(self._phiF), _p(self.w_phi), 2, st)
                nat.call("bddc_lap_solve_mc", S3[0], S3[1], S3[2], _p(self.d_eig_wF),
                         _p(self.d_dm_wF), _p(self._phiF), _p(self._zF), _p(self._lap_wsF), st)
                nat.call("bddc_gamma_flux", self.NF, _p(self.d_fidx), _p(self._zF), _p(self.w_zp), 0, st)
            z = self.w_zp
        else:
            S3 = self.dec.S3
            nat.call("bddc_lap_solve_mc", S3[0], S3[1], S3[2], _p(self.d_eig_w),
                     _p(self.d_dm_w), _p(self.w_phi), _p(self.w_z), _p(self._lap_ws), st)
        if yb is not None:
            x, op, hist = dot
            nat.call("bddc_proj_dot_broken", self.n_gamma, self.maxG, _p(self.d_gown), _p(yb), _p(z),
                     _p(y), _p(x), _p(self.w_dot), _p(self.w_scal), op,
                     _p(hist) if hist is not None else None, st)
        elif dot is None:
            nat.call("bddc_proj_apply", self.n_gamma, self.maxG, _p(self.d_gown), _p(z), _p(y), st)
        else:
            x, op, hist = dot
            nat.call("bddc_proj_dot", self.n_gamma, self.maxG, _p(self.d_gown), _p(z), _p(y), _p(x),
                     _p(self.w_dot), _p(self.w_scal), op, _p(hist) if hist is not None else None, st)

    def _precond(self, r, out, assemble=True):
        """BDDC Algorithm 2 (solver.py:109-128): coarse + Delta, averaged.  assemble=False:
        the averaged per-slot result stays in w_yb2 (the projection assembles it)."""
        st = _stream()
        main = torch.cuda.current_stream()
        if self.nfc:
            # the coarse chain (restriction, latency-bound ND solve) runs on a side
            # stream, concurrently with the bandwidth-bound T_i GEMV (a fork/join
            # inside the captured PCG graph); they meet at the prolongation.
            # restrict_first: the Psi^T restriction runs alone on every SM before the
            # fork, so only the ND solve shares the machine with the T_i GEMV
            if self.restrict_first:
                nat.call("bddc_gather_gemv_t", self.N, self.maxG, self.maxC, _p(self.d_nG),
                         _p(self.d_nC), _p(self.d_gpos), _p(self.d_Psi), _p(r),
                         _p(self.d_delta), _p(self.w_v), st)
            side = self.side_stream
            fork = torch.cuda.Event()
            fork.record(main)
            side.wait_event(fork)
            with torch.cuda.stream(side):
                ss = _stream()
                if not self.restrict_first:
                    nat.call("bddc_gather_gemv_t", self.N, self.maxG, self.maxC, _p(self.d_nG),
                             _p(self.d_nC), _p(self.d_gpos), _p(self.d_Psi), _p(r),
                             _p(self.d_delta), _p(self.w_v), ss)
                # the ND forward sweep forms the coarse load v[own+] - v[own-] (zero
                # pressure load) itself: no assembled rhs
                self.nd.solve(None, self.w_xc, restricted=(self.w_v, self.d_cown))
                join = torch.cuda.Event()
                join.record(side)
        # T_i GEMV with one CTA per SM (grid-stride over subdomains) so the
        # concurrent coarse chain finds free SM slots
        if self.symv_bulk:
            self._symv(self.d_Tp, r, self.d_delta, self.w_yb, self.t_grid_bulk if self.nfc else 0, 1, st)
        else:
            self._symv(self.d_Tp, r, self.d_delta, self.w_yb, self.t_grid if self.nfc else 0, 1, st)
        if self.nfc:
            main.wait_event(join)
        nat.call("bddc_prolong", self.N, self.maxG, self.maxC, _p(self.d_nG), _p(self.d_nC),
                 _p(self.d_sub_rows), _p(self.d_Psi), _p(self.w_xc), _p(self.w_yb),
                 _p(self.d_delta), _p(self.w_yb2), st)
        if assemble:
            nat.call("bddc_scatter", self.n_gamma, _p(self.d_gown), _p(self.w_yb2), _p(out), st)

    def _symv(self, mats, x, win, yb, grid, site, st):
        """yb = blockdiag(M_i) (win . x) gathered per subdomain (bulk kernel unless
        symv_bulk is off; `site` selects this call site's ticket counter)."""
        if self.symv_bulk:
            nat.call("bddc_gather_symv_bulk", self.N, self.maxG, _p(self.d_nG), _p(self.d_gpos),
                     _p(mats), _p(x), _p(win), _p(yb), grid, _p(self._sched[2 * site:]), st)
        elif self.tile16 and mats is self.d_Sp:
            nat.call("bddc_gather_symv16", self.N, self.maxG, _p(self.d_nG), _p(self.d_gpos),
                     _p(mats), _p(x), _p(win), _p(yb), grid, st)
        else:
            nat.call("bddc_gather_symv", self.N, self.maxG, _p(self.d_nG), _p(self.d_gpos),
                     _p(mats), _p(x), _p(win), _p(yb), grid, st)

    def time_kernel(self, which="S", reps=20):
        """Mean device time (s) of one interface GEMV launch (bench roofline helper)."""
        mats = {"S": self.d_Sp, "T": self.d_Tp}[which]
        x = torch.ones(max(self.n_gamma, 1), dtype=F64, device=self.dev)
        st = _stream()
        self._symv(mats, x, None, self.w_yb, 0, 2, st)
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            self._symv(mats, x, None, self.w_yb, 0, 2, st)
        b.record()
        b.synchronize()
        return a.elapsed_time(b) / 1000.0 / reps

    # public reference-compatible applies (numpy in / numpy out)
    def schur_matvec(self, x):
        xd = torch.as_tensor(np.asarray(x, dtype=np.float64), device=self.dev)
        y = torch.empty_like(xd)
        self._schur(xd, y)
        return y.cpu().numpy()

    def precondition(self, r):
        rd = torch.as_tensor(np.asarray(r, dtype=np.float64), device=self.dev)
        y = torch.empty_like(rd)
        self._precond(rd, y)
        return y.cpu().numpy()

    def project_balanced(self, x):
        xd = torch.as_tensor(np.asarray(x, dtype=np.float64), device=self.dev).clone()
        self._project(xd)
        return xd.cpu().numpy()

    def schur_dense(self, i):
        """Dense S_i (n_Gamma_i x n_Gamma_i), substructure.py:90-99 (unpacked from tiles)."""
        n = int(self.dec.nG[i])
        ts = 16 if self.tile16 else 32
        nt = self.maxG // ts
        npk = nt * (nt + 1) // 2 * ts * ts
        tiles = self.d_Sp[i * npk:(i + 1) * npk].view(-1, ts, ts).cpu().numpy()
        full = np.zeros((self.maxG, self.maxG))
        t = 0
        for bi in range(nt):
            for bj in range(bi, nt):
                full[bi * ts:(bi + 1) * ts, bj * ts:(bj + 1) * ts] = tiles[t]
                full[bj * ts:(bj + 1) * ts, bi * ts:(bi + 1) * ts] = tiles[t].T
                t += 1
        return full[:n, :n]

    # ------------------------------------- reference bookkeeping views (views.py)

    def _view(self, name, make):
        v = self.__dict__.get("_v_" + name)
        if v is None:
            v = make()
            self.__dict__["_v_" + name] = v
        return v

    @property
    def weights(self):
        """WeightOperator (decomposition.py:199-209)."""
        return self._view("weights", lambda: _views.WeightView(self))

    @property
    def broken(self):
        """BrokenInterface (decomposition.py:242-279)."""
        return self._view("broken", lambda: _views.BrokenInterface(self.weights))

    @property
    def subs(self):
        """Per-subdomain operators (substructure.py:25-116)."""
        return self._view("subs", lambda: [_views.SubdomainView(self, i)
                                           for i in range(self.N)])

    @property
    def cset(self):
        """ConstraintSet (coarse.py:36-118) in the reference's coarse numbering."""
        return self._view("cset", lambda: _views.ConstraintSetView(self))

    @property
    def coarse(self):
        """CoarseSpace.solve (coarse.py:208-215) on the device factorisation."""
        return self._view("coarse", lambda: _views.CoarseView(self, self.cset))

    def _face_row_values(self):
        """Per face: (rows added beyond the initial one, m_f) i-side values on the
        face's shared dofs (sorted), as the pair / multiscale kernels harvested them."""
        dec = self.dec
        nf = dec.n_faces
        extra = self._per_face - 1
        mx = int(extra.max()) if nf else 0
        if mx == 0:
            return [np.zeros((0, int(m))) for m in dec.face_table[:, 3]]
        R = self._rows_dev.view(nf, self._rows_maxsel, -1)[:, :mx].cpu().numpy()
        return [R[f, :int(extra[f]), :int(dec.face_table[f, 3])] for f in range(nf)]

    def net_flux_matrix(self):
        import scipy.sparse as sp
        dec = self.dec
        rows, cols, vals = [], [], []
        for i in range(dec.n_subdomains):
            n = dec.nG[i]
            cols.append(dec.gpos[i, :n])
            rows.append(np.full(n, i))
            side = (dec.gcode[i, :n] >> 2) & 1
            vals.append(np.where(side == 1, 1.0, -1.0))
        return sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                             shape=(dec.n_subdomains, dec.n_gamma)).tocsr()


@dataclass
class PairEigenReport:
    """Spectrum of one pair pencil (adaptive.py:46-60): eigenvalues descending,
    clipped at 0, as many as the reference keeps (n_i + n_j minus the rank of
    the face's initial constraint row); the nonzero part is the reduced m x m
    pencil's, the rest are the zeros of (I - E)."""
    i: int
    j: int
    eigenvalues: np.ndarray
    selected: int = 0
    complete: bool = True   # False: only the leading selected + 1 eigenvalues resolved

    def omega(self, tau):
        lam = self.eigenvalues
        below = lam[lam <= tau]
        return float(max(below[0], 1.0)) if len(below) else 1.0


class _LazyPairReports(Mapping):
    """dict (i, j) -> PairEigenReport, built from the device eigenvalues on first use."""

    def __init__(self, dec, lam_dev, selected, complete):
        self._args = (dec, lam_dev, selected, complete)
        self._d = None

    def _get(self):
        if self._d is None:
            dec, lam_dev, selected, complete = self._args
            self._d = _pair_reports(dec, lam_dev.cpu().numpy(), selected, complete=complete)
        return self._d

    def __getitem__(self, key):
        return self._get()[key]

    def __iter__(self):
        return iter(self._get())

    def __len__(self):
        return self._args[0].n_faces


def _pair_reports(dec, lam, selected, complete=True):
    """complete: the whole spectrum (reduced pencil resolved fully, then the zeros of
    I - E); else the leading eigenvalues the selection resolved (selected + 1)."""
    ft = dec.face_table
    out = {}
    for f in range(dec.n_faces):
        i, j, m = int(ft[f, 0]), int(ft[f, 1]), int(ft[f, 3])
        if complete:
            n_keep = int(dec.nG[i] + dec.nG[j]) - 1
            ev = np.maximum(lam[f, :m], 0.0)
            ev = np.concatenate([ev, np.zeros(max(n_keep - m, 0))])
        else:
            ev = np.maximum(lam[f, :min(int(selected[f]) + 1, m)], 0.0)
        out[(min(i, j), max(i, j))] = PairEigenReport(min(i, j), max(i, j), ev, int(selected[f]),
                                                      complete)
    return out


def eigs_report(system, dec, config):
    """Per-pair spectra against the initial constraints (cli.py:147-162): dict
    (i, j) -> PairEigenReport, computed on the GPU."""
    cfg = SolveConfig(tau=config.tau, scaling=config.scaling, tol=config.tol,
                      maxit=config.maxit, constraints="adaptive")
    return dict(BddcSetup(system, dec, cfg, pair_spectra=True).pair_reports)


def preconditioned_spectrum(setup, max_n=8192, seed=0, _debug=None):
    """Eigenvalues of the preconditioned interface operator on the balanced subspace
    (oracle.py:114-141), ascending, on the device with the library's kernels.

    M S is self-adjoint in the S inner product, so Lanczos in that inner product on
    range(P) (P the balanced projection, solver.py:166-179) with full
    reorthogonalisation (twice) run to the subspace dimension yields a tridiagonal
    T whose eigenvalues are those of the reference's Mb Sb (every (P S P) / (P M P)
    apply is the device operator; a breakdown restarts from a fresh random vector
    orthogonal to the basis, so multiple eigenvalues are kept).  T's eigenvalues:
    bisection on Sturm counts (bddc_tridiag_eigvals).  Diagnostic for
    n_Gamma <= max_n (the basis Q and S Q are stored: 2 n^2 doubles)."""
    n = setup.n_gamma
    if n > max_n:
        raise InvalidArgumentError(f"preconditioned_spectrum: n_Gamma = {n} > {max_n}")
    dev = setup.dev
    # dimension of the balanced subspace: one net-flux constraint per floating
    # subdomain, minus one in mode A (the constraints sum to zero)
    nb = n - (setup.N - 1 if not setup.mode_b else int(setup.floating.sum()))
    Q = torch.empty(max(nb, 1), n, dtype=F64, device=dev)
    SQ = torch.empty(max(nb, 1), n, dtype=F64, device=dev)
    w = torch.empty(n, dtype=F64, device=dev)
    Sw = torch.empty(n, dtype=F64, device=dev)
    c = torch.empty(max(nb, 1), dtype=F64, device=dev)
    tmp = torch.empty(n, dtype=F64, device=dev)
    host = setup._host_scal
    alphas, betas = [], []
    gen = torch.Generator(device="cpu").manual_seed(seed)

    def dot(x, y):
        _dot(setup, x, y, n, 100 + 14)
        host.copy_(setup.w_scal, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return float(host[14])

    def s_apply(x, out):          # out = P S x
        setup._schur(x, out)
        setup._project(out)

    def m_apply(x, out):          # out = P M x
        setup._precond(x, out)
        setup._project(out)

    def reorth(k, x):             # x -= Q^T (SQ x) over the first k basis vectors, twice
        for _ in range(2):
            nat.call("bddc_gemv", k, n, n, _p(SQ), _p(x), _p(c), _stream())
            nat.call("bddc_gemv_t_sub", k, n, _p(Q), _p(c), _p(x), _stream())

    def fresh(k):
        """A random unit vector of range(P), S-orthogonal to the first k basis vectors."""
        for _ in range(5):
            w.copy_(torch.randn(n, dtype=F64, generator=gen))
            setup._project(w)
            if k:
                reorth(k, w)
                setup._project(w)
            s_apply(w, Sw)
            nrm2 = dot(w, Sw)
            if nrm2 > 0:
                r = 1.0 / math.sqrt(nrm2)
                nat.call("bddc_axpby", n, r, _p(w), 0.0, _p(Q[k]), _stream())
                nat.call("bddc_axpby", n, r, _p(Sw), 0.0, _p(SQ[k]), _stream())
                return True
        return False

    with torch.cuda.stream(setup.stream):
        setup.stream.wait_stream(torch.cuda.default_stream())
        if nb > 0 and fresh(0):
            scale = 0.0
            for k in range(nb):
                m_apply(SQ[k], w)                      # w = (P M P)(P S P) q_k
                a = dot(w, SQ[k])                      # <w, q_k>_S
                alphas.append(a)
                nat.call("bddc_axpby", n, -a, _p(Q[k]), 1.0, _p(w), _stream())
                if k:
                    nat.call("bddc_axpby", n, -betas[-1], _p(Q[k - 1]), 1.0, _p(w), _stream())
                reorth(k + 1, w)
                # re-project: the S'-norm does not see null(P) components, so division
                # by a small beta would amplify them step after step
                setup._project(w)
                if k == nb - 1:
                    break
                s_apply(w, Sw)
                b2 = dot(w, Sw)
                scale = max(scale, abs(a))
                if b2 > (1e-10 * scale) ** 2:
                    bk = math.sqrt(b2)
                    betas.append(bk)
                    nat.call("bddc_axpby", n, 1.0 / bk, _p(w), 0.0, _p(Q[k + 1]), _stream())
                    nat.call("bddc_axpby", n, 1.0 / bk, _p(Sw), 0.0, _p(SQ[k + 1]), _stream())
                else:
                    # invariant subspace exhausted: restart (T splits into blocks)
                    betas.append(0.0)
                    if not fresh(k + 1):
                        raise NumericalFailureError("preconditioned_spectrum: Lanczos restart failed")
        m = len(alphas)
        d = torch.tensor(alphas, dtype=F64).to(dev)
        e = torch.tensor(betas[:max(m - 1, 0)] + [0.0], dtype=F64).to(dev)
        lam = torch.empty(max(m, 1), dtype=F64, device=dev)
        nat.call("bddc_tridiag_eigvals", m, _p(d), _p(e), _p(tmp), _p(lam), _stream())
        out = lam[:m].cpu().numpy()
    torch.cuda.current_stream().wait_stream(setup.stream)
    if _debug is not None:
        _debug.update(alphas=alphas, betas=betas, Q=Q.cpu().numpy(), SQ=SQ.cpu().numpy())
    return out


def write_eigs_csv(path, reports):
    """i,j,rank,lambda with rank 1 = largest (io.py:256-262)."""
    lines = ["i,j,rank,lambda"]
    for (i, j) in sorted(reports):
        for rank, lam in enumerate(reports[(i, j)].eigenvalues, 1):
            lines.append(f"{i},{j},{rank},{float(lam)!r}")
    with open(path, "w") as f:
        f.write("\n".join(lines) + "\n")


def _nd_prefetch(dec, has_p):
    from .coarse_nd import nd_geometry_flat
    if dec.n_faces:
        nd_geometry_flat(dec, has_p)


def _suggest_scaling(setup):
    """solver.py:286-298 (warning only): aligned coefficient jumps, per face max k
    over the low-side cells against min k over the high-side cells (one CTA per
    face on the setup's permeability copy; the host reads one flag)."""
    if setup.config.scaling != "multiplicity":
        return
    dec = setup.dec
    if not dec.n_gamma or not dec.n_faces:
        return
    flag = torch.empty(1, dtype=I32, device=setup.dev)
    nat.call("bddc_face_jumps", C.byref(setup.geom), _p(setup.d_faces), _p(setup.d_k), _p(flag),
             _stream())
    if int(flag.item()):
        warnings.warn("coefficient jumps aligned with the partition detected; "
                      "consider --scaling stiffness")


class _Work:
    """Per-solve device vectors."""

    def __init__(self, setup):
        dev = setup.dev
        G = setup.geom
        z = lambda n: torch.zeros(max(n, 1), dtype=F64, device=dev)
        ng = setup.n_gamma
        self.x = z(ng)
        self.r = z(ng)
        self.zv = z(ng)
        self.p = z(ng)
        self.Ap = z(ng)
        self.g = z(ng)
        self.wp = z(ng)
        self.fs = z(G.n_cells)
        self.dd = z(G.n_cells)
        self.u0 = z(G.n_flux)
        self.us = z(G.n_flux)
        self.u = z(G.n_flux)
        self.rf = z(G.n_flux)
        self.tmpc = z(G.n_cells)
        self.pc = z(G.n_cells)
        self.rq = z(setup.N)
        self.x0 = z(setup.npad)
        self.f_dev = z(G.n_cells)
        self.gv = None
        if setup.mode_b:
            # momentum rhs g: +p_low on the low Dirichlet faces, -p_high on the high ones
            self.gv = z(G.n_flux)
            self.gv_vals = None


def _dot(setup, x, y, n, op, hist=None):
    nat.call("bddc_dot", _p(x), _p(y), int(n), _p(setup.w_dot), _p(setup.w_scal), op,
             _p(hist) if hist is not None else None, _stream())


def _norm(setup, x, n):
    _dot(setup, x, x, n, 100 + 10)
    return math.sqrt(float(setup.w_scal[10].item()))


# deferred squared norms of one solve (read with the next unavoidable host sync)
_N_FS, _N_DD, _N_R0, _N_PDEN, _N_PNUM = range(5)


def _norm2_async(setup, x, n, slot):
    nat.call("bddc_dot", _p(x), _p(x), int(n), _p(setup.w_dot), _p(setup.w_norms), 100 + slot,
             None, _stream())


def _norms_to_host(setup):
    """Queue the copy of the deferred norms; valid after the stream's next sync."""
    setup._host_norms.copy_(setup.w_norms, non_blocking=True)
    return setup._host_norms


def solve(system, dec, config, u_exact=None, setup=None, iterate_callback=None,
          f_device=None, return_device=False):
    """Three-step method + pressure recovery (solver.py:301-398)."""
    if setup is None:
        setup = BddcSetup(system, dec, config)
    if setup.mode_b != (system.dirichlet is not None) or (
            setup.mode_b and system.dirichlet.axis != setup.system.dirichlet.axis):
        raise InvalidArgumentError("setup was built for a different boundary condition")
    if not setup._scaling_checked:
        _suggest_scaling(setup)
        setup._scaling_checked = True
    caller = torch.cuda.current_stream()
    setup.stream.wait_stream(caller)
    with torch.cuda.stream(setup.stream):
        out = _solve_on_stream(system, setup, config, u_exact, iterate_callback, f_device,
                               return_device)
    caller.wait_stream(setup.stream)
    return out


def _solve_on_stream(system, setup, config, u_exact, iterate_callback, f_device, return_device):
    dec = setup.dec
    G = setup.geom
    gp = C.byref(G)
    st = _stream()
    W = setup.work()
    N, ng = setup.N, setup.n_gamma
    # fs = D f
    if f_device is None:
        f_device = W.f_dev
        if setup._solves == 0:
            f_device.copy_(torch.as_tensor(np.asarray(system.f, dtype=np.float64).reshape(-1)))
        else:
            fh = _pinned_source(setup, system.f)
            if fh is None:
                # staging through torch's caching pinned allocator (no cudaHostAlloc per call)
                fh = torch.empty(G.n_cells, dtype=F64, pin_memory=True)
                np.copyto(fh.numpy(), np.asarray(system.f, dtype=np.float64).reshape(-1))
                W.f_host = fh   # keep the pinned buffer alive until the copy ran
            f_device.copy_(fh, non_blocking=True)
    _scale_fs(setup, f_device, W.fs)
    gv = None
    if setup.mode_b:
        gv = W.gv
        vals = (float(system.dirichlet.p_low), float(system.dirichlet.p_high))
        if W.gv_vals != vals:
            nb = G.n_bt
            gv[G.n_flux_int:G.n_flux_int + nb].fill_(vals[0])
            gv[G.n_flux_int + nb:G.n_flux_int + 2 * nb].fill_(-vals[1])
            W.gv_vals = vals
    # step 1: rq_i = sum fs over cells of i; x0 = Wq rq[1:]; g = average(Psi x0)
    nat.call("bddc_sub_sum", gp, _p(W.fs), _p(W.rq), 1.0, None, st)
    if setup.nfc and N > 1:
        if gv is not None:
            # mode B: the coarse flux rhs is the BDDC coarse restriction of the
            # interface residual of the boundary data, r = -sum_i R_i^T condense_i(g)
            a = nat.LocalSolveArgs()
            a.f_flux, a.f_scale = _p(gv).value, 1.0
            a.rg_broken = _p(setup.w_yb).value
            nat.call("bddc_local_solve", gp, _p(setup.d_coef), _p(setup.d_gcode),
                     _p(setup.d_gpos), _p(setup.d_fslot), _p(setup.d_Qp), _p(setup.d_Dsub),
                     C.byref(a), st)
            nat.call("bddc_scatter", ng, _p(setup.d_gown), _p(setup.w_yb), _p(W.r), st)
            nat.call("bddc_gather_gemv_t", N, setup.maxG, setup.maxC, _p(setup.d_nG),
                     _p(setup.d_nC), _p(setup.d_gpos), _p(setup.d_Psi), _p(W.r),
                     _p(setup.d_delta), _p(setup.w_v), st)
            nat.call("bddc_coarse_restrict", setup.nfc, _p(setup.d_cown), _p(setup.w_v),
                     _p(setup.w_rc), st)
            nat.call("bddc_axpby", setup.nfc, 0.0, _p(setup.w_rc), -1.0, _p(setup.w_rc), st)
        else:
            nat.call("bddc_fill", setup.nfc, 0.0, _p(setup.w_rc), st)
        nat.call("bddc_axpby", N, 1.0, _p(W.rq), 0.0, _p(setup.w_rc[setup.nfc:]), st)
        setup._coarse_solve()
        nat.call("bddc_axpby", setup.nfc, 1.0, _p(setup.w_xc), 0.0, _p(W.x0), st)
    if ng:
        nat.call("bddc_prolong", N, setup.maxG, setup.maxC, _p(setup.d_nG), _p(setup.d_nC),
                 _p(setup.d_sub_rows), _p(setup.d_Psi), _p(W.x0), None,
                 _p(setup.d_delta), _p(setup.w_yb2), st)
        nat.call("bddc_scatter", ng, _p(setup.d_gown), _p(setup.w_yb2), _p(W.g), st)
        nat.call("bddc_gamma_flux", ng, _p(setup.d_gamma), _p(W.g), _p(W.u0), 0, st)
        nat.call("bddc_gamma_flux", ng, _p(setup.d_gamma), _p(W.g), _p(W.us), 0, st)
    # step 2: harmonic extension (u0) and trace solve (u*) (solver.py:326-335): the
    # same interface trace and flux load, different cell loads -- one pass over the
    # packed pressure Schur inverses with two right-hand sides
    a = nat.LocalSolveArgs()
    a.x_gamma, a.x_scale = _p(W.g).value, 1.0
    a.u_out, a.u_mode = _p(W.u0).value, 0
    if gv is not None:
        a.f_flux, a.f_scale = _p(gv).value, 1.0
    if setup.step2_fused:
        a.g_cell2, a.g_scale2 = _p(W.fs).value, 1.0
        a.u_out2 = _p(W.us).value
    nat.call("bddc_local_solve", gp, _p(setup.d_coef), _p(setup.d_gcode), _p(setup.d_gpos),
             _p(setup.d_fslot), _p(setup.d_Qp), _p(setup.d_Dsub), C.byref(a), st)
    if not setup.step2_fused:
        a = nat.LocalSolveArgs()
        a.x_gamma, a.x_scale = _p(W.g).value, 1.0
        a.g_cell, a.g_scale = _p(W.fs).value, 1.0
        a.u_out, a.u_mode = _p(W.us).value, 0
        if gv is not None:
            a.f_flux, a.f_scale = _p(gv).value, 1.0
        nat.call("bddc_local_solve", gp, _p(setup.d_coef), _p(setup.d_gcode), _p(setup.d_gpos),
                 _p(setup.d_fslot), _p(setup.d_Qp), _p(setup.d_Dsub), C.byref(a), st)
    host = {}
    first = setup._solves == 0
    setup._solves += 1
    if not return_device and not first:
        # u0 and u* are final here: stream them to pinned host memory on a copy
        # stream while the PCG runs (from the second solve on: the first one would
        # pay the pinned allocation, slower than a pageable copy of the same bytes)
        host["u0"], host["us"] = _d2h_async(setup, (W.u0, W.us))
    # div_defect = fs - Bs u*
    nat.call("bddc_cell_div", gp, _p(W.us), _p(W.fs), 1.0, -1.0, _p(setup.d_cell_sub),
             _p(setup.d_Dsub), _p(W.dd), st)
    # |fs|, |div defect| (read with the next host sync)
    _norm2_async(setup, W.fs, G.n_cells, _N_FS)
    _norm2_async(setup, W.dd, G.n_cells, _N_DD)
    defect_norm = None
    # step 3 rhs: r = g - A u* (g = 0 in mode A, solver.py:342); r_G -= sum condense
    if gv is not None:
        nat.call("bddc_axpby", G.n_flux, 1.0, _p(gv), 0.0, _p(W.rf), st)
        nat.call("bddc_flux_A", gp, _p(setup.d_coef), _p(W.us), -1.0, 1.0, _p(W.rf), st)
    else:
        nat.call("bddc_flux_A", gp, _p(setup.d_coef), _p(W.us), -1.0, 0.0, _p(W.rf), st)
    w_cg_it = 0
    kappa = 1.0
    history = np.array([1.0])
    converged = True
    r_floor = 0.0
    if ng:
        nat.call("bddc_gamma_flux", ng, _p(setup.d_gamma), _p(W.r), _p(W.rf), 2, st)
        if gv is not None:
            # mode B extension: an interface residual at rounding level relative to
            # the uncondensed one means Steps 1-2 already solved the problem (e.g. a
            # homogeneous field whose solution the coarse space contains); PCG
            # on it would only chase rounding (the reference stops on r0 == 0 only)
            _norm2_async(setup, W.r, ng, _N_R0)
            r_floor = None   # 1e-12 |r_uncondensed|, read in _pcg's first sync
        a = nat.LocalSolveArgs()
        a.f_flux, a.f_scale = _p(W.rf).value, 1.0
        a.g_cell, a.g_scale = _p(W.dd).value, 1.0
        a.rg_broken = _p(setup.w_yb).value
        nat.call("bddc_local_solve", gp, _p(setup.d_coef), _p(setup.d_gcode), _p(setup.d_gpos),
                 _p(setup.d_fslot), _p(setup.d_Qp), _p(setup.d_Dsub), C.byref(a), st)
        nat.call("bddc_scatter", ng, _p(setup.d_gown), _p(setup.w_yb), _p(W.Ap), st)
        nat.call("bddc_axpby", ng, -1.0, _p(W.Ap), 1.0, _p(W.r), st)
        # subdomain net-flux targets (stiffness scaling only)
        nat.call("bddc_sub_sum", gp, _p(W.dd), _p(setup.w_phi), -1.0, _p(setup.d_Dsub), st)
        # max |targets| and sum |fs| (abs-reduction modes of the dot kernel), read with
        # the deferred norms in one host sync
        _dot(setup, setup.w_phi, None, N, 300 + 12)
        _dot(setup, W.fs, None, G.n_cells, 200 + 13)
        hs = setup._host_scal
        hs.copy_(setup.w_scal, non_blocking=True)
        hn = _norms_to_host(setup)
        torch.cuda.current_stream().synchronize()
        tmax, fs_abs = float(hs[12]), float(hs[13])
        nfs2, dd2 = float(hn[_N_FS]), float(hn[_N_DD])
        # relative to |fs| (solver.py:331-333); absolute when there is no source (mode B)
        defect_norm = math.sqrt(dd2) / (math.sqrt(nfs2) if nfs2 > 0 else 1.0)
        if tmax > 1e-13 * max(fs_abs, 1.0):
            S3 = dec.S3
            zs = setup.w_z
            if setup.d_Lu is not None:   # mode B: floating subdomains only, zero elsewhere
                nat.call("bddc_gemv", N, N, N, _p(setup.d_Lu), _p(setup.w_phi), _p(setup.w_z), st)
            elif setup.mode_b:
                zs = setup.w_zs
                if setup.NF:
                    S3F = setup.S3F
                    nat.call("bddc_gamma_flux", setup.NF, _p(setup.d_fidx), _p(setup._phiF),
                             _p(setup.w_phi), 2, st)
                    nat.call("bddc_lap_solve_mc", S3F[0], S3F[1], S3F[2], _p(setup.d_eig_uF), None,
                             _p(setup._phiF), _p(setup._zF), _p(setup._lap_wsF), st)
                    nat.call("bddc_gamma_flux", setup.NF, _p(setup.d_fidx), _p(setup._zF),
                             _p(setup.w_zs), 0, st)
            else:
                nat.call("bddc_lap_solve", S3[0], S3[1], S3[2], _p(setup.d_eig_u), None,
                         _p(setup.w_phi), _p(setup.w_z), st)
            nat.call("bddc_face_shift", ng, dec.n_faces, _p(setup.d_gface), _p(setup.d_faces),
                     _p(zs), _p(W.wp), st)
            setup._schur(W.wp, W.Ap)
            nat.call("bddc_axpby", ng, -1.0, _p(W.Ap), 1.0, _p(W.r), st)
        else:
            nat.call("bddc_fill", ng, 0.0, _p(W.wp), st)
        setup._project(W.r)
        w_cg_it, kappa, history, converged = _pcg(setup, W, config, iterate_callback, r_floor)
        # u = u* + correction, interior recovery
        nat.call("bddc_axpby", ng, 1.0, _p(W.wp), 1.0, _p(W.x), st)
    nat.call("bddc_axpby", G.n_flux, 1.0, _p(W.us), 0.0, _p(W.u), st)
    if ng:
        nat.call("bddc_gamma_flux", ng, _p(setup.d_gamma), _p(W.x), _p(W.u), 1, st)
        a = nat.LocalSolveArgs()
        a.f_flux, a.f_scale = _p(W.rf).value, 1.0
        a.g_cell, a.g_scale = _p(W.dd).value, 1.0
        a.x_gamma, a.x_scale = _p(W.x).value, 1.0
        a.u_out, a.u_mode = _p(W.u).value, 1
        nat.call("bddc_local_solve", gp, _p(setup.d_coef), _p(setup.d_gcode), _p(setup.d_gpos),
                 _p(setup.d_fslot), _p(setup.d_Qp), _p(setup.d_Dsub), C.byref(a), st)
    if not return_device and not first:
        # u is final: stream it to the host while the pressure is recovered
        (host["u"],) = _d2h_async(setup, (W.u,))
    # pressure recovery: B B^T p = B(g - A u), zero mean in mode A
    _recover_pressure(setup, W, gv)
    omega = setup.omega_tilde if setup.omega_tilde is not None else float("nan")
    if return_device:
        return W, w_cg_it, kappa, history, converged
    hn = _norms_to_host(setup)
    if first:
        host = {"u": W.u.cpu(), "p": W.pc.cpu(), "u0": W.u0.cpu(), "us": W.us.cpu()}
    else:
        (host["p"],) = _d2h_async(setup, (W.pc,))
        setup.copy_stream.synchronize()
    torch.cuda.current_stream().synchronize()
    hn = hn.tolist()
    if defect_norm is None:
        defect_norm = math.sqrt(hn[_N_DD]) / (math.sqrt(hn[_N_FS]) if hn[_N_FS] > 0 else 1.0)
    den, num = math.sqrt(hn[_N_PDEN]), math.sqrt(hn[_N_PNUM])
    # solver.py:271-273: warn if |A u + B^T p - g| > 10 tol |A u - g|
    p_warn = bool(den > 0 and num > 10.0 * config.tol * den)
    report = SolveReport(
        u=host["u"].numpy(), p=host["p"].numpy(), it=w_cg_it, kappa=kappa,
        omega_tilde=omega, n_c=setup.n_c, residuals=history,
        u0=host["u0"].numpy(), u_star=host["us"].numpy(),
        conservation_defect=defect_norm, pressure_warning=p_warn,
        converged=converged)
    if u_exact is not None:
        nrm = np.linalg.norm(u_exact)
        if nrm == 0:
            raise InvalidArgumentError("exact solution is zero")
        report.eps0 = float(np.linalg.norm(report.u0 - u_exact) / nrm)
        report.eps_star = float(np.linalg.norm(report.u_star - u_exact) / nrm)
    if not converged:
        raise NonConvergenceError(
            f"CG did not converge in {config.maxit} iterations", report=report)
    return report


# Process-wide page-lock table: (address, bytes) -> [owners, array, tensor].  Several
# live setups may solve the same source array (a tau sweep keeping one setup per
# tau); the array is registered once and released when its last owner lets go.
_HOST_REG = {}


def _pinned_source(setup, f):
    """The caller's source array page-locked in place (bddc_host_register, once per
    array and process; the setup holds a reference so the registration never
    outlives the array), so the per-solve upload is one async DMA without a host
    staging copy.  None when f is not a contiguous float64 array or registration
    fails (the library clears the failed call's error state)."""
    if not (isinstance(f, np.ndarray) and f.dtype == np.float64 and f.flags.c_contiguous
            and f.size == setup.geom.n_cells):
        return None
    key = (f.__array_interface__["data"][0], f.nbytes)
    reg = getattr(setup, "_f_reg", None)
    if reg is not None and reg == key and _HOST_REG.get(key, (0, None))[1] is f:
        return _HOST_REG[key][2]
    _unregister_source(setup)
    ent = _HOST_REG.get(key)
    if ent is not None and ent[1] is not f:
        return None   # another live array at this address: leave its registration alone
    if ent is None:
        if nat.load().bddc_host_register(C.c_void_p(key[0]), key[1]) != 0:
            return None
        ent = _HOST_REG[key] = [0, f, torch.from_numpy(f)]
    ent[0] += 1
    setup._f_reg = key
    return ent[2]


def _unregister_source(setup):
    key = getattr(setup, "_f_reg", None)
    if key is None:
        return
    setup._f_reg = None
    ent = _HOST_REG.get(key)
    if ent is None:
        return
    ent[0] -= 1
    if ent[0] <= 0:
        del _HOST_REG[key]
        torch.cuda.synchronize()   # no queued copy may still read the pages
        nat.load().bddc_host_unregister(C.c_void_p(key[0]))


def _d2h_async(setup, tensors):
    """Copy device vectors into fresh pinned host tensors on the setup's copy stream
    (ordered after the work queued so far on the current stream)."""
    cs = getattr(setup, "copy_stream", None)
    if cs is None:
        cs = setup.copy_stream = torch.cuda.Stream(device=setup.dev)
    cs.wait_stream(torch.cuda.current_stream())
    out = []
    with torch.cuda.stream(cs):
        for t in tensors:
            h = torch.empty(t.numel(), dtype=t.dtype, pin_memory=True)
            h.copy_(t, non_blocking=True)
            out.append(h)
    return out


def _scale_fs(setup, f, fs):
    """fs = D f (grid.py:250-251)."""
    nat.call("bddc_scale_cells", C.byref(setup.geom), _p(f), _p(setup.d_cell_sub),
             _p(setup.d_Dsub), _p(fs), _stream())


def _recover_pressure(setup, W, gv=None):
    """solver.py:254-274: (B B^T) p = B(g - A u) by the separable cosine (mode A,
    pure Neumann: zero-mean p) or cosine/sine (mode B: Dirichlet ends) transform."""
    G = setup.geom
    gp = C.byref(G)
    st = _stream()
    nat.call("bddc_flux_A", gp, _p(setup.d_coef), _p(W.u), 1.0, 0.0, _p(W.rf), st)
    if gv is not None:
        nat.call("bddc_axpby", G.n_flux, -1.0, _p(gv), 1.0, _p(W.rf), st)
    # rhs = B(g - A u)
    nat.call("bddc_cell_div", gp, _p(W.rf), None, 0.0, -1.0, None, None, _p(W.pc), st)
    nat.call("bddc_neumann_solve", gp, _p(setup.d_dct), _p(W.pc), _p(W.tmpc), st)
    if gv is None:
        ones = _ones(setup, G.n_cells)
        _dot(setup, W.pc, ones, G.n_cells, 100 + 11)
        nat.call("bddc_sub_mean", G.n_cells, _p(setup.w_scal[11:]), _p(W.pc), st)
    _norm2_async(setup, W.rf, G.n_flux, _N_PDEN)
    nat.call("bddc_grad", gp, _p(W.pc), 1.0, 1.0, _p(W.rf), st)
    _norm2_async(setup, W.rf, G.n_flux, _N_PNUM)


def _ones(setup, n):
    o = getattr(setup, "_ones_c", None)
    if o is None or o.numel() < n:
        o = torch.ones(n, dtype=F64, device=setup.dev)
        setup._ones_c = o
    return o


class _PCGBufs:
    """Device-resident PCG history (alphas, betas, relative residuals)."""

    def __init__(self, setup, maxit):
        z = lambda n: torch.zeros(n, dtype=F64, device=setup.dev)
        self.maxit = maxit
        self.alphas = z(maxit + 2)
        self.betas = z(maxit + 2)
        self.res = z(maxit + 2)


def _pcg_core(setup, W, B, cond=None):
    """Ap = P S p; alpha = rz / p.Ap; x += alpha p; r -= alpha Ap; relres
    (solver.py:205-216): the projection assembles S p from the per-slot products and
    carries the p.Ap dot, the update carries r.r.  cond = (handle, tol, maxit) inside
    the captured loop: the update's reducing block also sets the WHILE condition."""
    ng = setup.n_gamma
    setup._schur(W.p, W.Ap, assemble=False)
    setup._project(W.Ap, dot=(W.p, 1, B.alphas), yb=setup.w_yb)
    if cond is None:
        nat.call("bddc_cg_update_dot", ng, _p(W.x), _p(W.p), _p(W.r), _p(W.Ap), _p(setup.w_dot),
                 _p(setup.w_scal), 2, _p(B.res), _stream())
    else:
        nat.call("bddc_cg_update_dot_cond", ng, _p(W.x), _p(W.p), _p(W.r), _p(W.Ap), _p(setup.w_dot),
                 _p(setup.w_scal), 2, _p(B.res), cond[0], float(cond[1]), int(cond[2]), _stream())


def _pcg_first(setup, W, B, cond=None):
    """z = P M r; p = z; rz = r.z; first iteration (solver.py:198-216)."""
    ng = setup.n_gamma
    setup._precond(W.r, W.zv, assemble=False)
    setup._project(W.zv, dot=(W.r, 0, None), yb=setup.w_yb2)
    nat.call("bddc_axpby", ng, 1.0, _p(W.zv), 0.0, _p(W.p), _stream())
    _pcg_core(setup, W, B, cond)


def _pcg_body(setup, W, B, cond=None):
    """z = P M r; beta; p = z + beta p; next iteration (solver.py:222-227, 205-216)."""
    ng = setup.n_gamma
    setup._precond(W.r, W.zv, assemble=False)
    setup._project(W.zv, dot=(W.r, 3, B.betas), yb=setup.w_yb2)
    nat.call("bddc_p_update", ng, _p(setup.w_scal), _p(W.zv), _p(W.p), _stream())
    _pcg_core(setup, W, B, cond)


def _pcg_graph(setup, W, B, tol, maxit):
    """Build (once per setup/tol/maxit) the WHILE-conditional graph of the PCG loop."""
    key = (float(tol), int(maxit))
    cache = setup._graphs
    if key in cache:
        return cache[key]
    st = _stream()
    lib = nat.load()
    state = C.c_void_p()
    nat.call("bddc_graph_begin", C.byref(state), st)
    try:
        c0 = lib.bddc_launch_count()
        cond = (lib.bddc_graph_handle(state), tol, maxit)
        _pcg_first(setup, W, B, cond)
        c1 = lib.bddc_launch_count()
        nat.call("bddc_graph_while", state, st)
        _pcg_body(setup, W, B, cond)
        c2 = lib.bddc_launch_count()
        nat.call("bddc_graph_end", state, st)
    except Exception:
        lib.bddc_graph_destroy(state)
        raise
    # kernels per graph launch: top level (first iteration) and per WHILE body pass
    setup._graph_kernels[key] = (int(c1 - c0), int(c2 - c1))
    cache[key] = state
    return state


def _pcg(setup, W, config, callback, r_floor=0.0):
    """PCG with Lanczos kappa (solver.py:186-233), fully device resident.

    Without a callback the whole loop is one CUDA-graph launch (conditional
    WHILE node); with a callback every iteration syncs to hand x, r to the host.
    """
    ng = setup.n_gamma
    st = _stream()
    tol, maxit = config.tol, config.maxit
    scal = setup.w_scal
    B = setup._pcg_bufs(maxit)
    nat.call("bddc_fill", 16, 0.0, _p(scal), st)
    nat.call("bddc_fill", ng, 0.0, _p(W.x), st)
    _dot(setup, W.r, W.r, ng, 4, B.res)
    host = setup._host_scal
    host.copy_(scal, non_blocking=True)
    if r_floor is None:
        hn = _norms_to_host(setup)
    torch.cuda.current_stream().synchronize()
    if r_floor is None:
        r_floor = 1e-12 * math.sqrt(float(hn[_N_R0]))
    if host[4] <= r_floor:   # host[4] = ||r0||
        return 0, 1.0, np.array([1.0]), True
    if callback is None and not setup.force_eager:
        # make sure every lazily-created buffer exists before capture
        setup.nd is not None and setup.nd._bufs()
        g = _pcg_graph(setup, W, B, tol, maxit)
        pt = setup.pcg_timer
        if pt is not None:
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
        nat.call("bddc_graph_launch", g, st)
        if pt is not None:
            e1.record()
            pt.append((e0, e1))
        host.copy_(scal, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        top, body = setup._graph_kernels[(float(tol), int(maxit))]
        setup.graph_kernels_run += top + body * max(int(host[9]) - 1, 0)
    else:
        pt = setup.pcg_timer
        if pt is not None:
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
        _pcg_first(setup, W, B)
        while True:
            host.copy_(scal, non_blocking=True)
            torch.cuda.current_stream().synchronize()
            if callback is not None:
                callback(W.x.cpu().numpy(), W.r.cpu().numpy())
            if host[5] <= tol or host[8] != 0.0 or int(host[9]) >= maxit:
                break
            _pcg_body(setup, W, B)
        if pt is not None:
            e1.record()
            pt.append((e0, e1))
    it = int(host[9])
    if host[8] != 0.0:
        raise NonConvergenceError(
            f"non-positive curvature p'Sp = {float(host[1]):.3e} at iteration {it}; "
            "iterate left the balanced subspace")
    converged = bool(host[5] <= tol)
    history = B.res[:it + 1].cpu().numpy()
    kappa = _lanczos(setup, B.alphas, B.betas, it)
    return it, kappa, history, converged


def _lanczos(setup, alphas, betas, m):
    """solver.py:236-251 on the device (Sturm bisection for the extremes)."""
    if m <= 1:
        return 1.0
    work = torch.empty(2 * m + 2, dtype=F64, device=setup.dev)
    out = torch.empty(4, dtype=F64, device=setup.dev)
    nat.call("bddc_lanczos", m, _p(alphas), _p(betas), _p(work), _p(out), _stream())
    return float(out[2].item())

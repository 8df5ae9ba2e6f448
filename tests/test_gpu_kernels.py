"""Kernel-level numerics vs torch float64 references (DMMA GEMM, SPD sweep inverse,
matrix-free RT0 operators, DCT Neumann solve, Lanczos)."""
import ctypes as C
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _lib():
    from paper_1901_02090_b200 import _native as nat
    nat.load()
    return nat


@pytest.mark.parametrize("ta,tb,M,N,K", [(0, 0, 130, 70, 33), (1, 0, 64, 200, 17), (0, 1, 5, 9, 300),
                                         (1, 1, 257, 129, 64), (0, 0, 7, 9, 11)])
def test_dgemm_vs_torch(ta, tb, M, N, K):
    import torch
    nat = _lib()
    g = torch.Generator(device="cuda").manual_seed(1)
    A = torch.randn((K, M) if ta else (M, K), dtype=torch.float64, device="cuda", generator=g)
    Bm = torch.randn((N, K) if tb else (K, N), dtype=torch.float64, device="cuda", generator=g)
    Cm = torch.randn((M, N), dtype=torch.float64, device="cuda", generator=g)
    ref = 0.5 * Cm + 2.0 * ((A.T if ta else A) @ (Bm.T if tb else Bm))
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    nat.call("bddc_dgemm_batched", ta, tb, M, N, K, 2.0, nat.ptr(A), A.shape[1], 0, nat.ptr(Bm),
             Bm.shape[1], 0, 0.5, nat.ptr(Cm), N, 0, 1, 0, st)
    torch.cuda.synchronize()
    assert torch.allclose(Cm, ref, rtol=1e-13, atol=1e-12 * math.sqrt(K))


@pytest.mark.parametrize("beta", [0.0, 1.0])
def test_dgemm_per_batch_dims(beta):
    """Live (M_b, N_b, K_b) per batch: padded operands beyond them are ignored (even
    NaN), tiles outside are zero-filled (beta 0) or untouched (beta 1)."""
    import torch
    nat = _lib()
    g = torch.Generator(device="cuda").manual_seed(3)
    M, N, K, batch = 200, 150, 170, 4
    A = torch.randn(batch, M, K, dtype=torch.float64, device="cuda", generator=g)
    Bm = torch.randn(batch, N, K, dtype=torch.float64, device="cuda", generator=g)
    C0 = torch.randn(batch, M, N, dtype=torch.float64, device="cuda", generator=g)
    dims = torch.tensor([[200, 150, 170], [37, 90, 5], [1, 1, 1], [130, 64, 129]], dtype=torch.int32,
                        device="cuda")
    ref = C0.clone() * beta
    for z in range(batch):
        m, n, k = dims[z].tolist()
        A[z, m:, :] = float("nan")
        A[z, :, k:] = float("nan")
        Bm[z, n:, :] = float("nan")
        Bm[z, :, k:] = float("nan")
        ref[z, :m, :n] += A[z, :m, :k] @ Bm[z, :n, :k].T
    Cm = C0.clone()
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    nat.call("bddc_dgemm_batched_dims", 0, 1, M, N, K, 1.0, nat.ptr(A), K, M * K, nat.ptr(Bm), K, N * K,
             beta, nat.ptr(Cm), N, M * N, batch, 0, nat.ptr(dims), 3, st)
    torch.cuda.synchronize()
    for z in range(batch):
        m, n, k = dims[z].tolist()
        assert torch.allclose(Cm[z, :m, :n], ref[z, :m, :n], rtol=1e-13, atol=1e-11)
        outside = torch.ones(M, N, dtype=torch.bool, device="cuda")
        outside[:m, :n] = False
        # whole tiles outside the live block: zero (beta 0) or untouched (beta 1)
        tiles = torch.zeros(M, N, dtype=torch.bool, device="cuda")
        tiles[((m + 63) // 64) * 64:, :] = True
        tiles[:, ((n + 63) // 64) * 64:] = True
        exp = torch.zeros_like(C0[z]) if beta == 0.0 else C0[z]
        assert torch.equal(Cm[z][tiles], exp[tiles])
        part = outside & ~tiles
        if beta == 0.0:
            assert torch.all(Cm[z][part] == 0.0)
        else:
            assert torch.equal(Cm[z][part], C0[z][part])


@pytest.mark.parametrize("n,b,batch", [(64, 32, 3), (192, 64, 5), (512, 64, 2), (40, 64, 7), (64, 64, 3),
                                       (100, 64, 4), (160, 64, 300), (448, 64, 80), (448, 32, 80),
                                       (512, 32, 2)])
def test_spd_inverse_vs_torch(n, b, batch):
    import torch
    nat = _lib()
    g = torch.Generator(device="cuda").manual_seed(2)
    X = torch.randn(batch, n, n, dtype=torch.float64, device="cuda", generator=g)
    A = X @ X.transpose(1, 2) + n * torch.eye(n, dtype=torch.float64, device="cuda")
    M = A.clone()
    ws = torch.empty(nat.load().bddc_spd_inverse_workspace(n, batch, b) // 8 + 2,
                     dtype=torch.float64, device="cuda")
    info = torch.zeros(1, dtype=torch.int32, device="cuda")
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    nat.call("bddc_spd_inverse_batched", nat.ptr(M), n, n, n * n, batch, b, nat.ptr(ws),
             nat.ptr(info), st)
    ref = torch.linalg.inv(A)
    torch.cuda.synchronize()
    assert int(info.item()) == 0
    assert torch.allclose(M, ref, rtol=1e-11, atol=1e-14)
    # upper-triangle-only variant: same upper triangle, bitwise
    Mu = A.clone()
    nat.call("bddc_spd_inverse_batched_ex", nat.ptr(Mu), n, n, n * n, batch, b, nat.ptr(ws),
             nat.ptr(info), 1, st)
    torch.cuda.synchronize()
    iu = torch.triu_indices(n, n, device="cuda")
    assert torch.equal(Mu[:, iu[0], iu[1]], M[:, iu[0], iu[1]])


def test_rt0_operators_vs_scipy():
    import torch
    import paper_1901_02090_b200 as B
    from paper_1901_02090_b200 import solver as S
    nat = _lib()
    rng = np.random.default_rng(0)
    g = B.build_grid(3, (7, 5, 6), (2.0, 1.0, 0.5))
    k = 10 ** rng.uniform(-2, 2, (g.n_cells, 3))
    system = B.assemble_system(g, B.Permeability(k), B.Wells(0, g.n_cells - 1))
    dec = B.regular_partition(g, (2, 1, 2))
    st = B.BddcSetup(system, dec, B.SolveConfig())
    u = rng.standard_normal(g.n_flux_dofs)
    ud = torch.as_tensor(u, device="cuda")
    y = torch.empty_like(ud)
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    nat.call("bddc_flux_A", C.byref(st.geom), nat.ptr(st.d_coef), nat.ptr(ud), 1.0, 0.0, nat.ptr(y), s)
    np.testing.assert_allclose(y.cpu().numpy(), system.A @ u, rtol=1e-13, atol=1e-13)
    c = torch.empty(g.n_cells, dtype=torch.float64, device="cuda")
    nat.call("bddc_cell_div", C.byref(st.geom), nat.ptr(ud), None, 0.0, 1.0, None, None, nat.ptr(c), s)
    np.testing.assert_allclose(c.cpu().numpy(), system.B @ u, rtol=1e-13, atol=1e-13)
    # Neumann solve: B B^T p = B g with zero mean
    gvec = system.B @ u
    rhs = torch.as_tensor(gvec, device="cuda").clone()
    tmp = torch.empty_like(rhs)
    nat.call("bddc_neumann_solve", C.byref(st.geom), nat.ptr(st.d_dct), nat.ptr(rhs), nat.ptr(tmp), s)
    p = rhs.cpu().numpy()
    L = (system.B @ system.B.T).toarray()
    np.testing.assert_allclose(L @ p, gvec, atol=1e-10 * np.abs(gvec).max())
    assert abs(p.sum()) <= 1e-10 * np.abs(p).max()


def test_lanczos_kappa_matches_host():
    import torch
    import scipy.linalg as sla
    from paper_1901_02090_b200 import solver as S
    rng = np.random.default_rng(0)
    n = 40
    Q = rng.standard_normal((n, n))
    A = Q @ Q.T + n * np.eye(n)
    b = rng.standard_normal(n)
    # CG alphas/betas on the host
    x = np.zeros(n); r = b.copy(); p = r.copy(); rz = r @ r
    al, be = [], []
    for _ in range(25):
        Ap = A @ p; a = rz / (p @ Ap); x += a * p; r -= a * Ap; al.append(a)
        rzn = r @ r; be.append(rzn / rz); rz = rzn; p = r + be[-1] * p
    m = len(al)
    d = np.empty(m); e = np.empty(m - 1)
    d[0] = 1 / al[0]
    for q in range(1, m):
        d[q] = 1 / al[q] + be[q - 1] / al[q - 1]
        e[q - 1] = math.sqrt(be[q - 1]) / al[q - 1]
    ev = sla.eigh_tridiagonal(d, e, eigvals_only=True)

    class _S:
        dev = torch.device("cuda")
    k = S._lanczos(_S, torch.tensor(al + [0.0], device="cuda", dtype=torch.float64),
                   torch.tensor(be + [0.0], device="cuda", dtype=torch.float64), m)
    assert abs(k - ev[-1] / ev[0]) <= 1e-10 * k


@pytest.mark.parametrize("S3", [(6, 22, 17), (12, 44, 17), (5, 7, 1)])
def test_lap_solvers_agree(S3):
    """The single-CTA separable Laplacian solve, its multi-CTA variant and the
    dense (Phi Phi^T)^+ GEMV give the same projection solve."""
    import torch
    nat = _lib()
    import paper_1901_02090_b200 as B
    g = B.build_grid(3 if S3[2] > 1 else 2, tuple(2 * s for s in S3[:3 if S3[2] > 1 else 2]),
                     (1.0,) * (3 if S3[2] > 1 else 2))
    dec = B.regular_partition(g, S3[:3 if S3[2] > 1 else 2])
    eig, dm = dec.laplacian_eigs(True)
    dev = "cuda"
    eig = torch.as_tensor(eig, device=dev)
    dm = torch.as_tensor(dm, device=dev)
    N = int(np.prod(S3))
    phi = torch.randn(N, dtype=torch.float64, device=dev, generator=torch.Generator(device=dev).manual_seed(5))
    z1 = torch.empty_like(phi)
    z2 = torch.empty_like(phi)
    ws = torch.empty(2 * N, dtype=torch.float64, device=dev)
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    nat.call("bddc_lap_solve", S3[0], S3[1], S3[2], nat.ptr(eig), nat.ptr(dm), nat.ptr(phi), nat.ptr(z1), st)
    nat.call("bddc_lap_solve_mc", S3[0], S3[1], S3[2], nat.ptr(eig), nat.ptr(dm), nat.ptr(phi), nat.ptr(z2),
             nat.ptr(ws), st)
    torch.cuda.synchronize()
    assert torch.allclose(z1, z2, rtol=1e-12, atol=1e-12 * float(z1.abs().max()))
    if N <= 4096:
        Lp = torch.empty(N * N, dtype=torch.float64, device=dev)
        w2 = torch.empty(2 * N * N, dtype=torch.float64, device=dev)
        z3 = torch.empty_like(phi)
        nat.call("bddc_lap_dense", S3[0], S3[1], S3[2], nat.ptr(eig), nat.ptr(dm), nat.ptr(w2), nat.ptr(Lp), st)
        nat.call("bddc_gemv", N, N, N, nat.ptr(Lp), nat.ptr(phi), nat.ptr(z3), st)
        torch.cuda.synchronize()
        assert torch.allclose(z1, z3, rtol=1e-11, atol=1e-11 * float(z1.abs().max()))


def test_fused_scatter_projection_matches_unfused():
    """bddc_phi_broken / bddc_proj_dot_broken (the scatter fused into the balanced
    projection, solver.py:100-101 + 166-179) against scatter -> phi -> proj_dot:
    bitwise equal projected vector and dot."""
    import torch
    import paper_1901_02090_b200 as B
    from _golden import load
    nat = _lib()
    d = load("g3d_c3block")
    g = B.build_grid(3, d["counts"], d["sizes"])
    system = B.assemble_system(g, B.Permeability(d["k"]), B.Wells(0, g.n_cells - 1))
    dec = B.regular_partition(g, d["splits"])
    cfg = B.SolveConfig(tau=d["tau"], scaling=d["scaling"], constraints=d["mode"], tol=d["tol"])
    st = B.BddcSetup(system, dec, cfg)
    gen = torch.Generator(device="cuda").manual_seed(7)
    yb = torch.randn(st.w_yb.numel(), dtype=torch.float64, device="cuda", generator=gen)
    x = torch.randn(st.n_gamma, dtype=torch.float64, device="cuda", generator=gen)
    res = []
    for fused in (False, True):
        st.w_yb.copy_(yb)
        y = torch.empty(st.n_gamma, dtype=torch.float64, device="cuda")
        if not fused:
            nat.call("bddc_scatter", st.n_gamma, nat.ptr(st.d_gown), nat.ptr(st.w_yb), nat.ptr(y),
                     C.c_void_p(torch.cuda.current_stream().cuda_stream))
            st._project(y, dot=(x, 100 + 12, None))
        else:
            st._project(y, dot=(x, 100 + 12, None), yb=st.w_yb)
        torch.cuda.synchronize()
        res.append((y.clone(), float(st.w_scal[12])))
    assert torch.equal(res[0][0], res[1][0])
    assert res[0][1] == res[1][1]


@pytest.mark.parametrize("dim,counts,splits", [
    (2, (12, 12), (3, 3)), (2, (10, 7), (1, 3)), (2, (10, 7), (3, 1)), (2, (5, 5), (1, 1)),
    (3, (12, 10, 8), (3, 2, 2)), (3, (12, 10, 8), (1, 2, 2)), (3, (12, 10, 8), (3, 1, 2)),
    (3, (12, 10, 8), (3, 2, 1)), (3, (12, 10, 8), (1, 1, 4)),
    (3, (12, 12, 9), ([3, 5, 4], [2, 4, 6], [5, 4])), (3, (30, 44, 15), (6, 11, 3))])
def test_device_topology_bitwise(dim, counts, splits):
    """csrc/topology.cu (closed-form index kernels) against the host NumPy
    restatement of decomposition.py:32-125: every table identical, and the setup
    never materialises the host copies."""
    import torch
    import paper_1901_02090_b200 as B
    g = B.build_grid(dim, counts, (1.0,) * dim)
    rng = np.random.default_rng(7)
    k = 10.0 ** rng.uniform(-1, 1, (g.n_cells, dim))
    system = B.assemble_system(g, B.Permeability(k), B.Wells(0, g.n_cells - 1))
    dec = B.Decomposition(g, splits)
    st = B.BddcSetup(system, dec, B.SolveConfig(tau=float("inf"), constraints="initial"))
    torch.cuda.synchronize()
    lazy = set(B.Decomposition._LAZY) | {"part"}
    assert not (lazy & set(dec.__dict__)), lazy & set(dec.__dict__)
    ng = dec.n_gamma
    pairs = [("nG", st.d_nG), ("gpos", st.d_gpos), ("gcode", st.d_gcode), ("fslot", st.d_fslot),
             ("cell_sub", st.d_cell_sub)]
    if ng:
        pairs += [("gown", st.d_gown[:ng]), ("gamma", st.d_gamma[:ng]), ("gface", st.d_gface[:ng])]
    for name, dev in pairs:
        host = np.asarray(getattr(dec, name))
        assert np.array_equal(dev.cpu().numpy().astype(np.int64), host.astype(np.int64)), name


def test_face_jump_warning_matches_reference_rule():
    """solver.py:286-298: warn (multiplicity scaling) iff some face sees a k ratio
    beyond 1e3 between its two sides."""
    import warnings
    import paper_1901_02090_b200 as B
    g = B.build_grid(2, (12, 12), (1.0, 1.0))
    dec = B.regular_partition(g, (3, 3))
    cfg = B.SolveConfig(tau=float("inf"), constraints="initial", scaling="multiplicity")
    for jump, expect in ((1e4, True), (5e2, False)):
        k = np.ones((144, 2))
        k[np.arange(144) % 12 < 4] = jump          # aligned with the x = 4 strip boundary
        system = B.assemble_system(g, B.Permeability(k), B.Wells(0, 143))
        with warnings.catch_warnings(record=True) as w:
            warnings.simplefilter("always")
            B.solve(system, dec, cfg)
        hit = any("coefficient jumps aligned" in str(x.message) for x in w)
        assert hit == expect, (jump, hit)

"""ctypes binding of libbddc.so (the C ABI in include/bddc.h).

The library is built in-tree (`paper_1901_02090_b200/libbddc.so`, see
`build_native()`); there is no CPU fallback: importing the solver on a box
without the library or without a CUDA device raises immediately.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

from . import errors

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BDDC_LIB") or os.path.join(HERE, "libbddc.so")
CSRC = os.path.join(HERE, "csrc")
SOURCES = ["capi.cu", "dense.cu", "topology.cu", "local.cu", "adaptive.cu", "coarse.cu",
           "nd.cu", "pcg.cu", "stencil.cu", "graph.cu"]
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3",
              "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
              "-diag-suppress", "550"]
MAX_STRIPS = 64


def build_native(force=False, verbose=False):
    """Compile csrc/*.cu into libbddc.so for sm_100a (nvcc cross-compiles)."""
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    hdrs = [os.path.join(CSRC, "common.cuh"),
            os.path.join(os.path.dirname(HERE), "include", "bddc.h")]
    if not force and os.path.exists(LIB_PATH):
        t = os.path.getmtime(LIB_PATH)
        if all(os.path.getmtime(s) <= t for s in srcs + hdrs):
            return LIB_PATH
    nvcc = os.environ.get("NVCC", "nvcc")
    if os.path.exists("/usr/local/cuda/bin/nvcc") and nvcc == "nvcc":
        nvcc = "/usr/local/cuda/bin/nvcc"
    tmp = LIB_PATH + ".tmp"
    cmd = [nvcc] + NVCC_FLAGS + ["-o", tmp] + srcs
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True, cwd=CSRC)
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


class Geom(C.Structure):
    _fields_ = [
        ("dim", C.c_int),
        ("n", C.c_int * 3),
        ("h", C.c_double * 3),
        ("vol", C.c_double),
        ("S", C.c_int * 3),
        ("so", (C.c_int * MAX_STRIPS) * 3),
        ("sw", (C.c_int * MAX_STRIPS) * 3),
        ("fam_off", C.c_int * 4),
        ("n_cells", C.c_int), ("n_flux", C.c_int), ("N", C.c_int),
        ("n_gamma", C.c_int), ("n_faces", C.c_int),
        ("maxG", C.c_int), ("maxP", C.c_int), ("maxL", C.c_int),
        ("maxF", C.c_int),
        ("dir_axis", C.c_int), ("n_flux_int", C.c_int), ("n_bt", C.c_int),
        ("a_diag", C.c_double), ("a_off", C.c_double),
    ]


class LocalSolveArgs(C.Structure):
    _fields_ = [
        ("f_flux", C.c_void_p), ("f_scale", C.c_double),
        ("g_cell", C.c_void_p), ("g_scale", C.c_double),
        ("x_gamma", C.c_void_p), ("x_scale", C.c_double),
        ("u_out", C.c_void_p), ("u_mode", C.c_int),
        ("rg_broken", C.c_void_p), ("p_out", C.c_void_p),
        ("g_cell2", C.c_void_p), ("g_scale2", C.c_double), ("u_out2", C.c_void_p),
    ]


_P = C.c_void_p
_I = C.c_int
_D = C.c_double
_L = C.c_longlong
_GP = C.POINTER(Geom)

# name -> argtypes (all return int status unless listed in _RESTYPES)
_SIGS = {
    "bddc_dgemm_batched": [_I, _I, _I, _I, _I, _D, _P, _I, _L, _P, _I, _L, _D,
                           _P, _I, _L, _I, _I, _P],
    "bddc_dgemm_batched_dims": [_I, _I, _I, _I, _I, _D, _P, _I, _L, _P, _I, _L, _D,
                                _P, _I, _L, _I, _I, _P, _I, _P],
    "bddc_spd_inverse_workspace": [_I, _I, _I],
    "bddc_spd_log_enable": [_I],
    "bddc_spd_log_read": [_P, _I],
    "bddc_spd_inverse_batched": [_P, _I, _I, _L, _I, _I, _P, _P, _P],
    "bddc_spd_inverse_batched_ex": [_P, _I, _I, _L, _I, _I, _P, _P, _I, _P],
    "bddc_topology_box": [_GP, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P],
    "bddc_face_jumps": [_GP, _P, _P, _P, _P],
    "bddc_cell_coeffs": [_GP, _P, _P, _P],
    "bddc_weights": [_GP, _I, _P, _P, _P, _P],
    "bddc_rescale": [_GP, _P, _P, _P],
    "bddc_local_build": [_GP, _P, _P, _P, _P, _P, _P, _P, _P, _P],
    "bddc_local_pinv_fix": [_GP, _P, _P, _P],
    "bddc_local_schur": [_GP, _P, _P, _P, _P, _P, _P, _P, _P, _P],
    "bddc_local_solve": [_GP, _P, _P, _P, _P, _P, _P,
                         C.POINTER(LocalSolveArgs), _P],
    "bddc_pair_scratch_bytes": [_I],
    "bddc_multiscale_rows": [_GP, _P, _P, _P, _P, _I, _P, _P, _P, _P, _P],
    "bddc_pair_eigs": [_GP, _P, _P, _P, _P, _P, _D, _I, _P, _I, _P, _P, _P,
                       _P, _P, _P, _P, _P, _I, _I, _I, _P],
    "bddc_coarse_local": [_GP, _P, _P, _P, _P, _P, _P, _P, _I, _P, _P, _P, _I, _P,
                          _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I, _P],
    "bddc_pad_identity": [_P, _I, _I, _P],
    "bddc_graph_begin": [C.POINTER(C.c_void_p), _P],
    "bddc_graph_while": [_P, _P],
    "bddc_graph_end": [_P, _P],
    "bddc_graph_launch": [_P, _P],
    "bddc_graph_destroy": [_P],
    "bddc_graph_handle": [_P],
    "bddc_pcg_cond": [_P, _P, _D, _I, _P],
    "bddc_nd_assemble": [_I, _I, _I, _I, _I, _I, _I, _P, _P, _P, _P, _P, _I, _I, _P,
                         _P, _P, _I, _P],
    "bddc_nd_fwd": [_I, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I, _P, _P, _P, _P, _P],
    "bddc_nd_compact": [_I, _I, _I, _I, _I, _P, _P, _P, _P, _P, _P],
    "bddc_nd_qd": [_I, _I, _I, _I, _I, _P, _P],
    "bddc_nd_bwd": [_I, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P],
    "bddc_fill": [_L, _D, _P, _P],

    "bddc_gather_gemv": [_I, _I, _P, _P, _P, _P, _P, _P, _P],
    "bddc_sym_packed_elems": [_I],
    "bddc_pack_sym": [_I, _I, _P, _P, _P],
    "bddc_sym_packed16_elems": [_I],
    "bddc_pack_sym16": [_I, _I, _P, _P, _P],
    "bddc_gather_symv16": [_I, _I, _P, _P, _P, _P, _P, _P, _I, _P],
    "bddc_gather_symv": [_I, _I, _P, _P, _P, _P, _P, _P, _I, _P],
    "bddc_gather_symv_bulk": [_I, _I, _P, _P, _P, _P, _P, _P, _I, _P, _P],
    "bddc_gather_gemv_t": [_I, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P],
    "bddc_coarse_restrict": [_I, _P, _P, _P, _P],
    "bddc_prolong": [_I, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P],
    "bddc_scatter": [_I, _P, _P, _P, _P],
    "bddc_phi": [_I, _I, _P, _P, _P, _P, _P, _P],
    "bddc_lap_solve": [_I, _I, _I, _P, _P, _P, _P, _P],
    "bddc_lap_solve_mc": [_I, _I, _I, _P, _P, _P, _P, _P, _P],
    "bddc_proj_apply": [_I, _I, _P, _P, _P, _P],
    "bddc_dot_workspace": [],
    "bddc_dot": [_P, _P, _L, _P, _P, _I, _P, _P],
    "bddc_cg_update": [_L, _P, _P, _P, _P, _P, _P],
    "bddc_proj_dot": [_I, _I, _P, _P, _P, _P, _P, _P, _I, _P, _P],
    "bddc_cg_update_dot": [_L, _P, _P, _P, _P, _P, _P, _I, _P, _P],
    "bddc_cg_update_dot_cond": [_L, _P, _P, _P, _P, _P, _P, _I, _P, C.c_ulonglong, _D, _I, _P],
    "bddc_proj_dot_broken": [_I, _I, _P, _P, _P, _P, _P, _P, _P, _I, _P, _P],
    "bddc_phi_broken": [_I, _I, _P, _P, _P, _P, _P, _P, _P],
    "bddc_p_update": [_L, _P, _P, _P, _P],
    "bddc_gemv": [_I, _I, _I, _P, _P, _P, _P],
    "bddc_gemv_static": [_I, _I, _I, _P, _P, _P, _P],
    "bddc_set_gemv_wpr": [_I],
    "bddc_set_leaf_regs": [_I],
    "bddc_set_symv_threads": [_I],
    "bddc_set_symv_groups": [_I],
    "bddc_set_pair_threads": [_I],
    "bddc_set_prolong_direct": [_I],
    "bddc_lap_dense": [_I, _I, _I, _P, _P, _P, _P, _P],
    "bddc_lanczos": [_I, _P, _P, _P, _P, _P],
    "bddc_gemv_t_sub": [_I, _I, _P, _P, _P, _P],
    "bddc_tridiag_eigvals": [_I, _P, _P, _P, _P, _P],
    "bddc_axpby": [_L, _D, _P, _D, _P, _P],
    "bddc_flux_A": [_GP, _P, _P, _D, _D, _P, _P],
    "bddc_cell_div": [_GP, _P, _P, _D, _D, _P, _P, _P, _P],
    "bddc_grad": [_GP, _P, _D, _D, _P, _P],
    "bddc_dct_init": [_GP, _P, _P],
    "bddc_neumann_solve": [_GP, _P, _P, _P, _P],
    "bddc_sub_mean": [_L, _P, _P, _P],
    "bddc_sub_sum": [_GP, _P, _P, _D, _P, _P],
    "bddc_gamma_flux": [_I, _P, _P, _P, _I, _P],
    "bddc_face_shift": [_I, _I, _P, _P, _P, _P, _P],
    "bddc_scale_cells": [_GP, _P, _P, _P, _P, _P],
    "bddc_host_register": [_P, C.c_size_t],
    "bddc_dirichlet_laplacian": [_I, _I, _I, _P, _P, _P, _P],
    "bddc_dirichlet_finish": [_I, _I, _P, _P, _P, _P, _P],
    "bddc_host_unregister": [_P],
    "bddc_geom_size": [],
    "bddc_launch_count": [],
    "bddc_version": [],
    "bddc_last_error": [],
}
_RESTYPES = {
    "bddc_spd_inverse_workspace": C.c_size_t,
    "bddc_pair_scratch_bytes": C.c_size_t,
    "bddc_dot_workspace": C.c_size_t,
    "bddc_sym_packed_elems": C.c_size_t,
    "bddc_sym_packed16_elems": C.c_size_t,
    "bddc_geom_size": C.c_size_t,
    "bddc_launch_count": C.c_ulonglong,
    "bddc_graph_handle": C.c_ulonglong,
    "bddc_set_symv_groups": None,
    "bddc_spd_log_enable": None,
    "bddc_last_error": C.c_char_p,
}

EXPORTED = tuple(_SIGS)

_ERRMAP = {
    1: errors.InvalidArgumentError,
    2: errors.NumericalFailureError,
    3: errors.ConstraintRankError,
    4: errors.ConfigurationError,
    5: errors.InternalConsistencyError,
    6: RuntimeError,
}

_lib = None


def load(path=None):
    """Load libbddc.so and declare every exported symbol (raises if absent)."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = path or LIB_PATH
    if not os.path.exists(p):
        raise ImportError(
            f"libbddc.so not found at {p}; run __graft_entry__.build() "
            "(there is no CPU fallback)")
    lib = C.CDLL(p)
    for name, args in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = _RESTYPES.get(name, C.c_int)
    if lib.bddc_geom_size() != C.sizeof(Geom):
        raise ImportError("bddc_geom layout mismatch between header and binding")
    # tuning override (A/B measurements): BDDC_PDL_PCG=<mask> selects which small PCG
    # kernels use programmatic dependent launch (0: none)
    if os.environ.get("BDDC_PDL_PCG", "").isdigit():   # bit mask, see capi.cu
        lib.bddc_set_pdl_pcg(int(os.environ["BDDC_PDL_PCG"]))
    if path is None:
        _lib = lib
    return lib


_PROFILE = None   # list of (name, start_event, end_event) when profiling


def profile_start():
    """Record CUDA events around every library call (dev tool, perturbs timing slightly)."""
    global _PROFILE
    _PROFILE = []


def profile_stop():
    """Return {name: (calls, total_ms)} for the calls recorded since profile_start()."""
    global _PROFILE
    import torch
    torch.cuda.synchronize()
    out = {}
    for name, a, b in _PROFILE or []:
        c, t = out.get(name, (0, 0.0))
        out[name] = (c + 1, t + a.elapsed_time(b))
    _PROFILE = None
    return out


def call(name, *args):
    """Invoke a status-returning entry point; map errors to the reference classes."""
    lib = load()
    if _PROFILE is not None:
        import torch
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        rc = getattr(lib, name)(*args)
        b.record()
        _PROFILE.append((name, a, b))
    else:
        rc = getattr(lib, name)(*args)
    if rc:
        msg = lib.bddc_last_error().decode(errors="replace")
        raise _ERRMAP.get(rc, RuntimeError)(f"{name}: {msg}")
    return rc


def ptr(t):
    """Raw device pointer of a torch tensor (None -> NULL)."""
    return None if t is None else C.c_void_p(t.data_ptr())

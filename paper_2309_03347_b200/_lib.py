"""ctypes loader for libtt.so (the C ABI declared in include/tt.h).

The product path has no CPU fallback: if the shared library is missing or
does not export a declared symbol, importing the package raises."""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libtt.so")
TT_MAX_D = 64

STATUS = {0: "TT_OK", 1: "TT_ERR_ARG", 2: "TT_ERR_SHAPE", 3: "TT_ERR_CAPACITY", 4: "TT_ERR_NOCONV",
          5: "TT_ERR_NOFISSION", 6: "TT_ERR_NUMERIC", 7: "TT_ERR_CUDA", 8: "TT_ERR_NOT_IMPLEMENTED"}


class TTError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class tt_vec(C.Structure):
    _fields_ = [("d", C.c_int32), ("n", C.POINTER(C.c_int32)), ("r_dev", C.c_void_p),
                ("rcap", C.POINTER(C.c_int32)), ("data", C.c_void_p), ("off", C.POINTER(C.c_int64))]


class tt_mat(C.Structure):
    _fields_ = [("d", C.c_int32), ("m", C.POINTER(C.c_int32)), ("n", C.POINTER(C.c_int32)),
                ("R_dev", C.c_void_p), ("Rcap", C.POINTER(C.c_int32)), ("data", C.c_void_p),
                ("off", C.POINTER(C.c_int64))]


class amen_opts(C.Structure):
    _fields_ = [("eps", C.c_double), ("local_tol", C.c_double), ("max_sweeps", C.c_int32),
                ("rmax", C.c_int32), ("gmres_restart", C.c_int32), ("gmres_max_restarts", C.c_int32),
                ("local_dense_max", C.c_int32)]


class keff_opts(C.Structure):
    _fields_ = [("tol_k", C.c_double), ("tol_res", C.c_double), ("eps_round", C.c_double),
                ("eps_solve", C.c_double), ("max_outer", C.c_int32), ("rmax", C.c_int32), ("max_sweeps", C.c_int32),
                ("kickrank", C.c_int32), ("gmres_restart", C.c_int32), ("gmres_max_restarts", C.c_int32),
                ("local_dense_max", C.c_int32), ("matvec", C.c_int32), ("mv_max_sweeps", C.c_int32),
                ("warm", C.c_int32)]


class keff_report(C.Structure):
    _fields_ = [("k_dev", C.c_void_p), ("iters_dev", C.c_void_p), ("k_hist_dev", C.c_void_p),
                ("res_hist_dev", C.c_void_p), ("hist_cap", C.c_int32), ("status_dev", C.c_void_p),
                ("sweeps_hist_dev", C.c_void_p), ("inner_status_hist_dev", C.c_void_p), ("res_dev", C.c_void_p)]


class alpha_opts(C.Structure):
    _fields_ = [("alpha0", C.c_double), ("alpha1", C.c_double), ("tol", C.c_double), ("eps_op", C.c_double),
                ("max_alpha", C.c_int32), ("keff", keff_opts)]


class alpha_report(C.Structure):
    _fields_ = [("alpha_dev", C.c_void_p), ("k_dev", C.c_void_p), ("iters_dev", C.c_void_p),
                ("alpha_hist_dev", C.c_void_p), ("k_hist_dev", C.c_void_p), ("keff_iters_hist_dev", C.c_void_p),
                ("hist_cap", C.c_int32), ("status_dev", C.c_void_p)]


P = C.c_void_p
I32 = C.c_int32
SIG = {
    "tt_last_error": (C.c_char_p, []),
    "tt_version": (C.c_char_p, []),
    "tt_counters": (None, [C.POINTER(C.c_uint64), I32]),
    "tt_fused_profile": (None, [I32]),
    "tt_fused_profile_read": (None, [C.POINTER(C.c_int64), C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "tt_fused_profile_cores": (None, [C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_int64)]),
    "tt_set_graph_mode": (None, [I32]),
    "tt_fused_timer_read": (None, [C.POINTER(C.c_double), C.POINTER(C.c_int64)]),
    "tt_graph_mode": (I32, []),
    "tt_graph_stats": (None, [C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "tt_matvec": (I32, [C.POINTER(tt_mat), C.POINTER(tt_vec), C.POINTER(tt_vec), P]),
    "tt_matvec_batched_workspace": (C.c_size_t, [I32, C.POINTER(tt_mat)]),
    "tt_matvec_batched": (I32, [I32, C.POINTER(tt_mat), C.POINTER(tt_vec), C.POINTER(tt_vec), P, C.c_size_t, P]),
    "tt_add": (I32, [C.POINTER(tt_vec), P, C.POINTER(tt_vec), P, C.POINTER(tt_vec), P]),
    "tt_scale": (I32, [C.POINTER(tt_vec), P, P]),
    "tt_copy": (I32, [C.POINTER(tt_vec), C.POINTER(tt_vec), P]),
    "tt_dot_workspace": (C.c_size_t, [C.POINTER(tt_vec), C.POINTER(tt_vec)]),
    "tt_dot": (I32, [C.POINTER(tt_vec), C.POINTER(tt_vec), P, P, C.c_size_t, P]),
    "tt_orthogonalize_workspace": (C.c_size_t, [C.POINTER(tt_vec)]),
    "tt_orthogonalize": (I32, [C.POINTER(tt_vec), I32, P, P, C.c_size_t, P]),
    "tt_round_workspace": (C.c_size_t, [C.POINTER(tt_vec)]),
    "tt_round": (I32, [C.POINTER(tt_vec), C.c_double, I32, P, P, I32, P, C.c_size_t, P]),
    "als_workspace": (C.c_size_t, [I32] * 8),
    "als_local_apply": (I32, [I32] * 8 + [P, P, P, P, P, P, C.c_size_t, P]),
    "als_update_interfaces": (I32, [I32] * 9 + [P, P, P, P, P, P, C.c_size_t, P]),
    "tt_core_kinds": (I32, [C.POINTER(tt_mat), P, P, P, C.c_size_t, P]),
    "als_workspace_structured": (C.c_size_t, [I32] * 10),
    "als_local_apply_structured": (I32, [I32] * 10 + [P, P, P, P, P, P, C.c_size_t, P]),
    "als_update_interfaces_structured": (I32, [I32] * 11 + [P, P, P, P, P, P, C.c_size_t, P]),
    "amen_workspace": (C.c_size_t, [C.POINTER(tt_mat), C.POINTER(tt_vec), C.POINTER(tt_vec),
                                    C.POINTER(tt_vec), C.POINTER(amen_opts)]),
    "amen_solve": (I32, [C.POINTER(tt_mat), C.POINTER(tt_vec), C.POINTER(tt_vec), C.POINTER(tt_vec),
                         C.POINTER(amen_opts), P, P, P, C.c_size_t, P]),
    "amen_mv_workspace": (C.c_size_t, [C.POINTER(tt_mat), C.POINTER(tt_vec), C.POINTER(tt_vec),
                                       C.POINTER(tt_vec)]),
    "amen_mv": (I32, [C.POINTER(tt_mat), C.POINTER(tt_vec), C.POINTER(tt_vec), C.POINTER(tt_vec), C.c_double,
                      I32, I32, P, P, C.c_size_t, P]),
    "keff_workspace": (C.c_size_t, [C.POINTER(tt_mat), C.POINTER(tt_mat), C.POINTER(tt_mat),
                                    C.POINTER(tt_vec), C.POINTER(tt_vec), C.POINTER(keff_opts)]),
    "keff_fixed_point": (I32, [C.POINTER(tt_mat), C.POINTER(tt_mat), C.POINTER(tt_mat), C.POINTER(tt_vec),
                               C.POINTER(tt_vec), C.c_double, C.POINTER(keff_opts), C.POINTER(keff_report),
                               P, C.c_size_t, P]),
    "tt_transport_terms": (I32, [I32, I32, C.c_double, I32, I32, P, P, P, P, I32, P, P, P, P, I32, P, P, P, P]),
    "tt_transport_terms_reflective": (I32, [I32, I32, C.c_double, I32, I32, P, P, P, P, I32, P, P, P, P, I32, P, P,
                                            P, P]),
    "tt_normalize": (I32, [C.POINTER(tt_vec), P, P, C.c_size_t, P]),
    "tt_round_batched_workspace": (C.c_size_t, [I32, C.POINTER(tt_vec)]),
    "tt_round_batched": (I32, [I32, C.POINTER(tt_vec), C.c_double, I32, P, P, C.c_size_t, P]),
    "tt_qtt_matrix_dev_workspace": (C.c_size_t, [C.POINTER(tt_vec)]),
    "tt_qtt_matrix_dev": (I32, [I32, P, C.c_double, C.POINTER(tt_vec), P, C.c_size_t, P]),
    "tt_transport_terms_1d": (I32, [I32, I32, C.c_double, I32, I32, P, P, P, P, P, P, P]),
    "alpha_workspace": (C.c_size_t, [C.POINTER(tt_mat)] * 4 + [C.POINTER(tt_vec)] * 2 + [C.POINTER(alpha_opts)]),
    "alpha_secant": (I32, [C.POINTER(tt_mat)] * 4 + [C.POINTER(tt_vec)] * 2
                     + [C.POINTER(alpha_opts), C.POINTER(alpha_report), P, C.c_size_t, P]),
    "tt_velocity_terms": (I32, [I32, I32, I32, I32, P, P, P, P, I32, P]),
}

# symbols declared in include/tt.h (checked by the CPU test-suite)
DECLARED = sorted(SIG)


def load(path: str = LIB_PATH):
    if not os.path.exists(path):
        raise ImportError(f"libtt.so not built at {path}: run `python -m paper_2309_03347_b200.build` "
                          "(there is no CPU fallback)")
    lib = C.CDLL(path)
    for name, (res, args) in SIG.items():
        fn = getattr(lib, name)          # AttributeError if not exported
        fn.restype = res
        fn.argtypes = args
    return lib


_LIB = None


def lib():
    global _LIB
    if _LIB is None:
        _LIB = load()
    return _LIB


def check(status: int):
    if status != 0:
        raise TTError(status, lib().tt_last_error().decode())

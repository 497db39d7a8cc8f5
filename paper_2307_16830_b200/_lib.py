"""ctypes binding of libgridopf.so (the C-ABI in include/gridopf.h).

The library is built in-tree (``paper_2307_16830_b200/build.py``).  There
is no fallback: if it is missing, importing the device entry points raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_lib", "libgridopf.so")

c_i32, c_i64, c_dbl, c_u32 = ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_uint32
P = ctypes.c_void_p


class BlockDesc(ctypes.Structure):
    _fields_ = [("kind", c_i32), ("n_var_slots", c_i32), ("n_param_slots", c_i32),
                ("n_records", c_i64), ("var_idx", P), ("params", P), ("targets", P),
                ("n_ops", c_i32), ("ops", P), ("n_consts", c_i32), ("consts", P), ("out", c_i32),
                ("n_first", c_i32), ("first_slots", P), ("n_pairs", c_i32), ("pairs", P),
                ("grad_order", P)]


class SymbolicInfo(ctypes.Structure):
    _fields_ = [(f, c_i64) for f in ("n", "nnz_a", "nnz_l", "n_fronts", "front_doubles",
                                     "vec_doubles", "max_front", "max_cols", "n_levels", "flops")]


class KktState(ctypes.Structure):
    _fields_ = [(f, P) for f in ("w", "a", "dxl", "dxu", "dsl", "dsu", "zxl", "zxu", "zsl",
                                 "zsu", "sx", "ss")] + [("dw", c_dbl), ("dc", c_dbl)]


class Vec7(ctypes.Structure):
    _fields_ = [(f, P) for f in ("x", "s", "y", "zxl", "zxu", "zsl", "zsu")]


class IpmVecs(ctypes.Structure):
    _fields_ = [(f, P) for f in ("x", "s", "y", "zxl", "zxu", "zsl", "zsu", "xl", "xu", "sl", "su",
                                 "dxl", "dxu", "dsl", "dsu", "sx", "ss", "grad", "c", "jac",
                                 "dual_x", "dual_s", "primal")]


# scalar-block layout of gn_ipm_prep (gridopf.h GN_PREP_*)
IPM_MAX_MU = 16
PREP_S = 24
PREP_DOUBLES = 48
GN_RED_PARTIALS = 1184 * 40   # gridopf.h: reduction scratch of gn_ipm_init_slacks


class GridOpfError(RuntimeError):
    pass


_SIGS = {
    "gn_last_error": (ctypes.c_char_p, []),
    "gn_version": (c_i32, []),
    "gn_stats": (None, [P, P, c_i32]),
    "gn_set_host_threads": (c_i32, [c_i32]),
    "gn_analyze": (c_i32, [c_i64, c_i64, P, P, c_i64, P, P, P, P, P, P]),
    "gn_canonical_order": (c_i32, [c_i64, c_i32, c_i32, P, P, P, P]),
    "gn_model_create": (c_i32, [P, c_i32, c_i64, c_i64, P]),
    "gn_model_info": (c_i32, [P, P, P, P]),
    "gn_model_export": (c_i32, [P] * 8),
    "gn_model_destroy": (None, [P]),
    "gn_condense_create": (c_i32, [c_i64, c_i64, P, P, c_i64, P, P, P]),
    "gn_condense_info": (c_i32, [P, P, P]),
    "gn_condense_export": (c_i32, [P] * 9),
    "gn_condense_destroy": (None, [P]),
    "gn_coo_to_csc": (c_i32, [c_i64, c_i64, P, P, P, P, P, P]),
    "gn_min_degree": (c_i32, [c_i64, P, P, P]),
    "gn_symbolic_create": (c_i32, [c_i64, P, P, P, P]),
    "gn_symbolic_info": (c_i32, [P, P]),
    "gn_symbolic_export": (c_i32, [P] * 9),
    "gn_symbolic_destroy": (None, [P]),
    "gn_model_upload": (c_i32, [P]),
    "gn_model_release": (c_i32, [P]),
    "gn_model_traffic": (c_i32, [P, c_u32, P]),
    "gn_kkt_assembly_traffic": (c_i32, [P, P]),
    "gn_model_ad_backend": (c_i32, [P, ctypes.c_char_p, ctypes.c_size_t]),
    "gn_model_pattern_source": (c_i32, [P, ctypes.c_char_p, ctypes.c_size_t, P]),
    "gn_ad_eval": (c_i32, [P, P, P, c_dbl, P, c_dbl, P, P, P, P, P, c_u32, P, P, P]),
    "gn_symbolic_upload": (c_i32, [P]),
    "gn_chol_factor": (c_i32, [P, P, P, P, P]),
    "gn_chol_solve": (c_i32, [P, P, P, P, P, P]),
    "gn_chol_export_l": (c_i32, [P, P, P, P]),
    "gn_measure_dmma_peak": (c_i32, [P, P]),
    "gn_chol_set_trace": (c_i32, [P, P]),
    "gn_set_concurrency": (c_i32, [c_i32]),
    "gn_alloc_trim": (c_i32, [P]),
    "gn_upload_stats": (None, [P, P, P, c_i32]),
    "gn_symbolic_fronts": (c_i32, [P, P, P, P, P, P, P]),
    "gn_kkt_create": (c_i32, [c_i64, c_i64, c_i64, P, P, c_i64, P, P, P, P]),
    "gn_kkt_destroy": (None, [P]),
    "gn_kkt_sigma": (c_i32, [c_i64, P, P, P, P, P, P]),
    "gn_kkt_matvec": (c_i32, [P, c_i32, P, P, P, P]),
    "gn_kkt_assemble": (c_i32, [P, P, P, P]),
    "gn_kkt_condense_rhs": (c_i32, [P, P, P, P, P, P, P, P]),
    "gn_kkt_recover_slack_dual": (c_i32, [P, P, P, P, P, P, P, P]),
    "gn_kkt_recover_bound_duals": (c_i32, [P, P, P, P, P, P, P, P, P, P, P]),
    "gn_kkt_residual": (c_i32, [P, P, P, P, P, P, P]),
    "gn_kkt_matrix_scale": (c_i32, [P, P, P, P]),
    "gn_vec7_axpy": (c_i32, [P, P, P, c_dbl, P]),
    "gn_ipm_prep": (c_i32, [P, P, c_i32, P, P, P]),
    "gn_ipm_pvec": (c_i32, [P, P, c_dbl, P, P]),
    "gn_ipm_direction": (c_i32, [P, P, P, c_dbl, c_dbl, P, P]),
    "gn_ipm_trial_point": (c_i32, [P, P, P, c_dbl, P, P, P]),
    "gn_ipm_trial_merit": (c_i32, [P, P, P, P, P, P, P]),
    "gn_ipm_trial_point_at": (c_i32, [P, P, P, P, P, P, P]),
    "gn_ipm_accept": (c_i32, [P, P, P, c_dbl, c_dbl, c_dbl, c_dbl, P, P]),
    "gn_ipm_setup": (c_i32, [c_i64, c_i64, c_i64, P, P, P, P, P, P, P, P, c_i32, c_dbl, P, P, P, P, P, P, P,
                             P, P, P, P, P, P]),
    "gn_ipm_init_slacks": (c_i32, [c_i64, P, P, P, c_dbl, P, P, P, P, P]),
    # batched (K12)
    "gn_ad_eval_batched": (c_i32, [P, c_i32, P, P, P, P, P, P, P, c_i64, P, P, P, P, c_u32, P, P, P]),
    "gn_model_param_count": (c_i32, [P, P]),
    "gn_kkt_assemble_batched": (c_i32, [P, c_i32, P, P, P, P]),
    "gn_kkt_condense_rhs_batched": (c_i32, [P, c_i32, P, P, P, P, P, P, P, P]),
    "gn_kkt_recover_slack_dual_batched": (c_i32, [P, c_i32, P, P, P, P, P, P, P, P]),
    "gn_kkt_recover_bound_duals_batched": (c_i32, [P, c_i32, P, P, P, P, P, P, P, P, P, P]),
    "gn_kkt_residual_batched": (c_i32, [P, c_i32, P, P, P, P, P, P, P]),
    "gn_kkt_matrix_scale_batched": (c_i32, [P, c_i32, P, P, P, P]),
    "gn_vec7_axpy_batched": (c_i32, [P, c_i32, P, P, P, P]),
    "gn_chol_factor_batched": (c_i32, [P, c_i32, P, P, P, P]),
    "gn_chol_solve_batched": (c_i32, [P, c_i32, P, P, P, P, P]),
    "gn_ipm_prep_batched": (c_i32, [P, c_i32, P, c_i32, P, P, P]),
    "gn_ipm_pvec_batched": (c_i32, [P, c_i32, P, P, P, P]),
    "gn_ipm_direction_batched": (c_i32, [P, c_i32, P, P, P, P, P]),
    "gn_ipm_trial_point_batched": (c_i32, [P, c_i32, P, P, P, P, P, P]),
    "gn_ipm_trial_point_at_batched": (c_i32, [P, c_i32, P, P, P, P, P, P]),
    "gn_ipm_trial_merit_batched": (c_i32, [P, c_i32, P, P, P, P, P, P]),
    "gn_ipm_accept_batched": (c_i32, [P, c_i32, P, P, P, c_dbl, P, P]),
}

_lib = None


def lib():
    """The loaded library (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise GridOpfError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2307_16830_b200.build`")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def stats(reset: bool = False) -> tuple[int, int]:
    """(kernel launches, plan-upload H2D bytes) counted by the library."""
    a, b = ctypes.c_int64(), ctypes.c_int64()
    lib().gn_stats(ctypes.byref(a), ctypes.byref(b), 1 if reset else 0)
    return a.value, b.value


def check(rc: int) -> None:
    if rc != 0:
        raise GridOpfError(lib().gn_last_error().decode())


def ptr(a) -> int | None:
    """Raw pointer of a numpy array or torch tensor (None passes NULL)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()


def i64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)


def f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)

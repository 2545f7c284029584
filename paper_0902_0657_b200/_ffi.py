"""ctypes declarations of include/alp.h (argument marshalling only)."""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libalp.so")


class AlpParams(C.Structure):
    _fields_ = [
        ("variant", C.c_int32), ("precond", C.c_int32),
        ("sigma", C.c_double), ("eta", C.c_double),
        ("gap_tol", C.c_double), ("feas_tol", C.c_double), ("pcg_rel_tol", C.c_double),
        ("tau_viol", C.c_double), ("tau_act", C.c_double), ("tau_cert", C.c_double),
        ("alp_max_iter", C.c_int32), ("ipm_max_iter", C.c_int32), ("pcg_max_iter", C.c_int32),
        ("warps_per_block", C.c_int32), ("smem_frames_per_sm", C.c_int32),
        ("stop_on_lp_failure", C.c_int32),
        ("basis_correction", C.c_int32), ("pcg_forcing", C.c_double), ("pcg_refine", C.c_int32),
    ]


class FrameStats(C.Structure):
    _fields_ = [
        ("lp_solves", C.c_int32), ("ipm_iters", C.c_int32), ("pcg_iters", C.c_int32),
        ("max_p", C.c_int32), ("pcg_solves", C.c_int32), ("pcg_p4_fail", C.c_int32),
        ("pcg_true_fail", C.c_int32), ("reserved", C.c_int32),
        ("g_max", C.c_double), ("pcg_bytes", C.c_double),
        ("max_rec_relres", C.c_double), ("max_true_relres", C.c_double),
        ("cyc_cut", C.c_int64), ("cyc_ipm", C.c_int64), ("cyc_build", C.c_int64),
        ("cyc_spmv", C.c_int64), ("cyc_sweep", C.c_int64), ("cyc_pcg_other", C.c_int64),
        ("cyc_sort", C.c_int64), ("cyc_peel", C.c_int64),
    ]


# numpy dtype of alp_frame_stats (128 bytes) for zero-copy views of device/host buffers
STATS_FIELDS = [("lp_solves", "<i4"), ("ipm_iters", "<i4"), ("pcg_iters", "<i4"),
                ("max_p", "<i4"), ("pcg_solves", "<i4"), ("pcg_p4_fail", "<i4"),
                ("pcg_true_fail", "<i4"), ("reserved", "<i4"),
                ("g_max", "<f8"), ("pcg_bytes", "<f8"),
                ("max_rec_relres", "<f8"), ("max_true_relres", "<f8"),
                ("cyc_cut", "<i8"), ("cyc_ipm", "<i8"), ("cyc_build", "<i8"),
                ("cyc_spmv", "<i8"), ("cyc_sweep", "<i8"), ("cyc_pcg_other", "<i8"),
                ("cyc_sort", "<i8"), ("cyc_peel", "<i8")]
STATS_BYTES = 128

P = C.c_void_p
SIGNATURES = {
    "alp_default_params": (None, [C.POINTER(AlpParams)]),
    "alp_code_create": (C.c_int, [C.c_int32, C.c_int32, P, P, C.POINTER(C.c_void_p)]),
    "alp_code_destroy": (C.c_int, [P]),
    "alp_decode_workspace_bytes": (C.c_size_t, [P, C.c_int64, C.POINTER(AlpParams)]),
    "alp_decode": (C.c_int, [P, C.c_int64, P, P, P, P, P, P, P, P, P, P, C.c_size_t,
                             C.POINTER(AlpParams), P]),
    "alp_decode_host_workspace_bytes": (C.c_size_t, [P, C.c_int64, C.POINTER(AlpParams)]),
    "alp_decode_host": (C.c_int, [P, C.c_int64, P, P, P, P, P, P, P, C.c_size_t,
                                  C.POINTER(AlpParams), P]),
    "alp_pcg_workspace_bytes": (C.c_size_t, [P, C.c_int64, C.POINTER(AlpParams)]),
    "ipm_step_pcg": (C.c_int, [P, C.c_int64, P, P, P, P, P, P, P, P, P, P, P, C.c_size_t,
                               C.POINTER(AlpParams), P]),
    "alp_last_launch_count": (C.c_int32, []),
    "alp_launch_info": (C.c_int, [P, C.c_int64, C.POINTER(AlpParams), C.c_int32, P]),
    "alp_debug_trace": (C.c_int, [P, C.c_int32]),
    "alp_status_string": (C.c_char_p, [C.c_int]),
    "alp_last_error": (C.c_char_p, []),
    "alp_last_status": (C.c_int, []),
    "alp_build_info": (C.c_char_p, []),
}

_lib = None
OPTIONAL = ("alp_launch_info",)


def load(path: str | None = None):
    """Loads libalp.so; raises (never falls back) when it is missing.  ALP_LIB (diagnostics
    only) points at another build of the same library, e.g. a tuning variant."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or os.environ.get("ALP_LIB") or LIB_PATH
    if not os.path.exists(path):
        raise ImportError(f"libalp.so not built at {path}: run `python -m paper_0902_0657_b200.build` "
                          "(or __graft_entry__.build()); there is no CPU fallback")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        if name in OPTIONAL and path != LIB_PATH and not hasattr(lib, name):
            continue   # an older tuning build under ALP_LIB (introspection calls only)
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib

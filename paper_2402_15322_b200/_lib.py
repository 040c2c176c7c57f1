"""ctypes binding of libse2ot.so (include/se2ot.h).  Argument marshalling only: every step of
the scaling loop runs in the library's CUDA kernels.  There is no CPU fallback: if the library
is missing or no CUDA device is visible, every call raises."""
from __future__ import annotations

import ctypes
import os
import warnings

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SE2_LIB_PATH") or os.path.join(HERE, "libse2ot.so")   # override: A/B diagnostics

SE2_OK = 0
SE2_LOG_DOMAIN = 0x1
SE2_WARM_START = 0x2
SE2_TRACE_ERR = 0x4
SE2_LSE_EXACT = 0x8
SE2_LSE_NOTILT = 0x10
SE2_LSE_K3EXACT = 0x20
SE2_NO_GRAPH = 0x40
SE2_NO_PERSISTENT = 0x80
SE2_DEBUG_BAD_HINTS = 0x100
SE2_DEBUG_NO_SPLIT = 0x200
SE2_LIN_FFMA = 0x400
SE2_LIN_TC = 0x800
SE2_EPI_DIVIDE = 1
SE2_EPI_MULTIPLY = 2
SE2_EPI_PROX = 3
SE2_PROX_MARGINAL = 0
SE2_PROX_ENTROPY_POTENTIAL = 1
SE2_PROX_POROUS = 2

STATUS_NAMES = {0: "SE2_OK", 1: "SE2_EINVAL", 2: "SE2_ENOMEM", 3: "SE2_ECUDA", 5: "SE2_ENONFINITE",
                6: "SE2_EUNSUPPORTED", 100: "SE2_WKERNEL_TOO_WIDE", 101: "SE2_WGUARD_HIT",
                102: "SE2_WPROX_NOCONV"}
SE2_WGUARD_HIT = 101
SE2_WPROX_NOCONV = 102

# every symbol include/se2ot.h declares (checked by tests/test_abi.py)
EXPORTED = [
    "se2_kernel_build", "se2_kernel_stats_get", "se2_kernel_destroy", "se2_conv", "se2_sinkhorn",
    "se2_jko_step", "se2_barycenter", "se2_marginal_error", "se2_conv_update", "se2_bary_logmean",
    "se2_bary_update", "se2_sum", "se2_timing_enable", "se2_timing_get", "se2_launch_count",
    "se2_last_error", "se2_abi_version", "se2_lse_path_stats", "se2_sum_rows", "se2_scale_rows",
    "se2_transport_cost", "se2_lse_row_stats", "se2_tc_tile_stats", "se2_interp_masses", "se2_precise_path_stats",
    "se2_cake_build", "se2_cake_get", "se2_cake_destroy", "se2_lift_image", "se2_split_signed", "se2_project",
    "se2_project_signed", "se2_lift_field", "se2_reconstruct_field", "se2_exp", "se2_log",
    "se2_bary_reduce_update", "se2_conv_update_slab", "se2_guard_stats", "se2_kernel_set_window",
    "se2_comm_unique_id", "se2_comm_init", "se2_comm_init_loopback", "se2_comm_split", "se2_comm_info",
    "se2_comm_allreduce", "se2_comm_destroy", "se2_jko_step_dist", "se2_barycenter_dist",
    "se2_barycenter_precise_dist",
    "se2_barycenter_precise", "se2_conv_precise",
]


class SE2Error(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class se2_grid(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int32), ("ny", ctypes.c_int32), ("ntheta", ctypes.c_int32),
                ("hx", ctypes.c_double), ("hy", ctypes.c_double)]


class se2_metric(ctypes.Structure):
    _fields_ = [("w1", ctypes.c_double), ("w2", ctypes.c_double), ("w3", ctypes.c_double)]


class se2_kernel_stats(ctypes.Structure):
    _fields_ = [("box_taps", ctypes.c_int64), ("nnz_taps", ctypes.c_int64), ("theta_band", ctypes.c_int32),
                ("radius", ctypes.c_int32), ("zeta", ctypes.c_double), ("table_bytes", ctypes.c_size_t),
                ("tensor_cores", ctypes.c_int32), ("nnz_normal_taps", ctypes.c_int64)]


class se2_prox(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("tau", ctypes.c_double), ("cx", ctypes.c_double),
                ("cy", ctypes.c_double), ("hx", ctypes.c_double), ("hy", ctypes.c_double),
                ("m", ctypes.c_double)]


class se2_slab(ctypes.Structure):
    _fields_ = [("own_lo", ctypes.c_int32), ("own_hi", ctypes.c_int32), ("halo", ctypes.c_int32),
                ("up", ctypes.c_void_p), ("up_shift", ctypes.c_int32), ("ny_up", ctypes.c_int32),
                ("dn", ctypes.c_void_p), ("dn_shift", ctypes.c_int32), ("ny_dn", ctypes.c_int32)]


class se2_dist(ctypes.Structure):
    _fields_ = [("reduce", ctypes.c_void_p), ("slabs", ctypes.c_void_p), ("halo_top", ctypes.c_int32),
                ("halo_bot", ctypes.c_int32)]


class se2_opts(ctypes.Structure):
    _fields_ = [("iters", ctypes.c_int32), ("flags", ctypes.c_uint32)]


_lib = None


def load(path: str = LIB_PATH):
    """Load libse2ot.so (raises if it was not built -- there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"{path} not built: run `python -m paper_2402_15322_b200.build` "
                           "(or __graft_entry__.build()); the SE(2) OT path has no CPU fallback")
    lib = ctypes.CDLL(path)
    P = ctypes.c_void_p
    i32, u32, i64, dbl = ctypes.c_int32, ctypes.c_uint32, ctypes.c_int64, ctypes.c_double
    pd = ctypes.POINTER(ctypes.c_double)
    sig = {
        "se2_kernel_build": [ctypes.POINTER(se2_grid), ctypes.POINTER(se2_metric), dbl, i32, i32, i32,
                             ctypes.POINTER(P)],
        "se2_kernel_stats_get": [P, ctypes.POINTER(se2_kernel_stats)],
        "se2_conv": [P, P, P, i32, u32, P],
        "se2_sinkhorn": [P, P, P, P, P, i32, ctypes.POINTER(se2_prox), ctypes.POINTER(se2_opts), pd, P],
        "se2_jko_step": [P, P, P, P, P, ctypes.POINTER(se2_prox), ctypes.POINTER(se2_opts), pd, pd, P],
        "se2_barycenter": [P, i32, i32, P, pd, P, P, P, ctypes.POINTER(se2_opts), pd, P],
        "se2_marginal_error": [P, P, P, P, i32, u32, pd, P],
        "se2_transport_cost": [P, P, P, i32, u32, pd, P],
        "se2_conv_update": [P, P, P, P, i32, i32, ctypes.POINTER(se2_prox), u32, P],
        "se2_bary_logmean": [i32, i64, P, pd, P, P],
        "se2_bary_update": [i32, i64, P, P, P, P],
        "se2_sum": [P, i64, pd, P],
        "se2_sum_rows": [P, i32, i32, i32, i32, i32, pd, P],
        "se2_scale_rows": [P, i32, i32, i32, i32, i32, dbl, P],
        "se2_timing_enable": [P, i32],
        "se2_lse_path_stats": [P, ctypes.POINTER(i64), ctypes.POINTER(i64), ctypes.POINTER(i64),
                               ctypes.POINTER(i64), ctypes.POINTER(i64), i32],
        "se2_timing_get": [P, ctypes.POINTER(i64), pd, ctypes.POINTER(i64)],
        "se2_lse_row_stats": [P, ctypes.POINTER(i64), ctypes.POINTER(i64), i32],
        "se2_tc_tile_stats": [P, ctypes.POINTER(i64), ctypes.POINTER(i64), i32],
        "se2_interp_masses": [P, P, i32, P],
        "se2_precise_path_stats": [P, ctypes.POINTER(i64), ctypes.POINTER(i64), ctypes.POINTER(i64), i32],
        "se2_guard_stats": [P, ctypes.POINTER(i64), ctypes.POINTER(i64), i32],
        "se2_kernel_set_window": [P, i32, i32],
        "se2_barycenter_precise": [P, i32, i32, P, pd, P, P, P, ctypes.POINTER(se2_opts), pd, P],
        "se2_conv_precise": [P, P, P, i32, P],
        "se2_comm_unique_id": [ctypes.c_char_p],
        "se2_comm_init": [ctypes.c_char_p, i32, i32, i32, ctypes.POINTER(P)],
        "se2_comm_init_loopback": [i32, i32, ctypes.POINTER(P)],
        "se2_comm_split": [P, i32, i32, ctypes.POINTER(P)],
        "se2_comm_info": [P, ctypes.POINTER(i32), ctypes.POINTER(i32)],
        "se2_comm_allreduce": [P, P, i64, i32, P],
        "se2_jko_step_dist": [P, ctypes.POINTER(se2_dist), P, P, P, P, ctypes.POINTER(se2_prox),
                              ctypes.POINTER(se2_opts), pd, pd, P],
        "se2_barycenter_dist": [P, ctypes.POINTER(se2_dist), i32, i32, P, pd, P, P, P, ctypes.POINTER(se2_opts), pd, P],
        "se2_barycenter_precise_dist": [P, ctypes.POINTER(se2_dist), i32, i32, P, pd, P, P, P, ctypes.POINTER(se2_opts),
                                        pd, P],
        "se2_cake_build": [i32, i32, i32, dbl, i32, ctypes.POINTER(P)],
        "se2_cake_get": [P, ctypes.POINTER(ctypes.c_float), ctypes.POINTER(i32), ctypes.POINTER(i32)],
        "se2_lift_image": [P, P, P, i32, i32, i32, P],
        "se2_split_signed": [P, P, P, P, i64, i32, dbl, pd, P],
        "se2_project": [P, P, P, i32, i32, i32, P],
        "se2_project_signed": [P, P, P, pd, P, i32, i32, i32, pd, P],
        "se2_lift_field": [P, P, P, P, i32, i32, i32, pd, P],
        "se2_reconstruct_field": [P, P, P, P, i32, i32, i32, ctypes.c_float, P],
        "se2_exp": [P, P, i64, P],
        "se2_log": [P, P, i64, P],
        "se2_bary_reduce_update": [i32, P, i32, i64, P, P, P, P],
        "se2_conv_update_slab": [P, P, P, P, i32, i32, ctypes.POINTER(se2_prox), u32, ctypes.POINTER(se2_slab), P],
    }
    for name, args in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = ctypes.c_int
    lib.se2_kernel_destroy.argtypes = [P]
    lib.se2_kernel_destroy.restype = None
    lib.se2_comm_destroy.argtypes = [P]
    lib.se2_comm_destroy.restype = None
    lib.se2_cake_destroy.argtypes = [P]
    lib.se2_cake_destroy.restype = None
    lib.se2_last_error.argtypes = []
    lib.se2_last_error.restype = ctypes.c_char_p
    lib.se2_abi_version.argtypes = []
    lib.se2_abi_version.restype = ctypes.c_int32
    lib.se2_launch_count.argtypes = []
    lib.se2_launch_count.restype = ctypes.c_int64
    _lib = lib
    return lib


def check(status: int):
    if status == SE2_OK:
        return
    msg = (_lib.se2_last_error() or b"").decode(errors="replace")
    if status >= 100:
        warnings.warn(f"{STATUS_NAMES.get(status, status)}: {msg}")
        return
    raise SE2Error(status, msg)

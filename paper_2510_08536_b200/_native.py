"""ctypes binding of libldurepart_b200.so (include/ldurepart_b200.h).

The library is required: there is no CPU fallback for any compute entry
point.  Importing this module on a machine without the built library raises.
"""

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LRB_LIB") or os.path.join(HERE, "libldurepart_b200.so")

LRB_OK = 0
LRB_EVALUE = -1
LRB_ERUNTIME = -2
LRB_ECUDA = -3
LRB_ENOTPD = -4
LRB_ETIMEOUT = -5

METHODS = {"cg": 0, "pcg": 1, "bicgstab": 2, "pcg1": 3, "pipecg": 4}


class NativeError(RuntimeError):
    """A CUDA / runtime failure inside the native library."""


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python paper_2510_08536_b200/build.py` "
            "(nvcc, sm_100a). There is no CPU fallback.")
    return C.CDLL(LIB_PATH)


lib = _load()

P = C.c_void_p
I32 = C.c_int32
I64 = C.c_int64
D = C.c_double
PI64 = C.POINTER(C.c_int64)


class Report(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("converged", C.c_int32), ("breakdown", C.c_int32),
                ("status", C.c_int32), ("residual", C.c_double), ("bnorm", C.c_double),
                ("device_ms", C.c_double)]


def _sig(name, restype, *args):
    fn = getattr(lib, name)
    fn.restype = restype
    fn.argtypes = list(args)
    return fn


lrb_last_error = _sig("lrb_last_error", C.c_char_p)
lrb_version = _sig("lrb_version", C.c_char_p)
lrb_device_count = _sig("lrb_device_count", C.c_int)
lrb_launch_count = _sig("lrb_launch_count", C.c_uint64)
lrb_plan_build_ldu = _sig("lrb_plan_build_ldu", C.c_int, I64, I64, I64, I32, P, P, P, P, P, P, P,
                          I32, P, I32, C.POINTER(P))
lrb_plan_build_coo = _sig("lrb_plan_build_coo", C.c_int, I64, I64, I64, I64, P, P, I32, P, I32, P,
                          C.POINTER(P))
lrb_plan_info = _sig("lrb_plan_info", C.c_int, P, P)
lrb_plan_export_csr = _sig("lrb_plan_export_csr", C.c_int, P, P, P, P, P, P)
lrb_plan_export_scatter = _sig("lrb_plan_export_scatter", C.c_int, P, P, P)
lrb_plan_export_halo = _sig("lrb_plan_export_halo", C.c_int, P, P, P)
lrb_plan_export_sell = _sig("lrb_plan_export_sell", C.c_int, P, P, P, P, P)
lrb_plan_destroy = _sig("lrb_plan_destroy", None, P)
lrb_part_create = _sig("lrb_part_create", C.c_int, P, I32, P, I64, P, I64, C.POINTER(P))
lrb_part_destroy = _sig("lrb_part_destroy", None, P)
lrb_part_pointers = _sig("lrb_part_pointers", C.c_int, P, P)
lrb_update_segment = _sig("lrb_update_segment", C.c_int, P, I32, I32, P, P)
lrb_upload_segment = _sig("lrb_upload_segment", C.c_int, P, I32, I32, P, P)
lrb_update_segments = _sig("lrb_update_segments", C.c_int, P, I32, P, P, P, P)
lrb_host_register = _sig("lrb_host_register", C.c_int, P, I64)
lrb_host_unregister = _sig("lrb_host_unregister", C.c_int, P)
lrb_scatter_segment = _sig("lrb_scatter_segment", C.c_int, P, I32)
lrb_update_staged = _sig("lrb_update_staged", C.c_int, P, I32, P, P)
lrb_stage_segment = _sig("lrb_stage_segment", C.c_int, P, I32, I32, P, P)
lrb_apply_scatter = _sig("lrb_apply_scatter", C.c_int, P)
lrb_apply_scatter_timed = _sig("lrb_apply_scatter_timed", C.c_int, I32, P, C.POINTER(C.c_float))
lrb_part_fill = _sig("lrb_part_fill", C.c_int, P, I64, P, I64)
lrb_part_read_buffer = _sig("lrb_part_read_buffer", C.c_int, P, P)
lrb_part_read_values = _sig("lrb_part_read_values", C.c_int, P, P, P)
lrb_part_write_values = _sig("lrb_part_write_values", C.c_int, P, P, P)
lrb_part_capture_base = _sig("lrb_part_capture_base", C.c_int, P, P, I64)
lrb_update_perturb = _sig("lrb_update_perturb", C.c_int, P, D)
lrb_part_join = _sig("lrb_part_join", C.c_int, P)
lrb_part_sync = _sig("lrb_part_sync", C.c_int, P)
lrb_part_stats = _sig("lrb_part_stats", C.c_int, P, P)
lrb_part_mark = _sig("lrb_part_mark", C.c_int, P)
lrb_part_elapsed_ms = _sig("lrb_part_elapsed_ms", C.c_int, P, C.POINTER(C.c_float))
lrb_team_create = _sig("lrb_team_create", C.c_int, I32, P, C.POINTER(P))
lrb_team_create_ex = _sig("lrb_team_create_ex", C.c_int, I32, P, P, C.POINTER(P))
lrb_team_destroy = _sig("lrb_team_destroy", None, P)
lrb_team_spmv = _sig("lrb_team_spmv", C.c_int, P, P, P)
BLOB_BYTES = 512
lrb_part_export = _sig("lrb_part_export", C.c_int, P, P)
lrb_team_create_ipc = _sig("lrb_team_create_ipc", C.c_int, I32, I32, I32, P, P, I32, I32,
                           C.POINTER(P), P)
lrb_team_connect_ipc = _sig("lrb_team_connect_ipc", C.c_int, P, P)
lrb_team_read_vector = _sig("lrb_team_read_vector", C.c_int, P, I32, I32, I64, P)
lrb_team_debug = _sig("lrb_team_debug", C.c_int, P, P)
lrb_team_kernel_info = _sig("lrb_team_kernel_info", C.c_int, P, I32, P)
lrb_team_profile = _sig("lrb_team_profile", C.c_int, P, I32)
lrb_team_profile_read = _sig("lrb_team_profile_read", C.c_int, P, P, I32)
lrb_team_profile_counters = _sig("lrb_team_profile_counters", C.c_int, P, I32, P, I32)
lrb_team_solve = _sig("lrb_team_solve", C.c_int, P, I32, P, P, D, I32, C.POINTER(Report), P, I32)
lrb_update_segment_async = _sig("lrb_update_segment_async", C.c_int, P, I32, I32, P, P, P)
lrb_team_solve_async = _sig("lrb_team_solve_async", C.c_int, P, I32, P, P, D, I32, P, P)
lrb_team_spmv_async = _sig("lrb_team_spmv_async", C.c_int, P, P, P, P)

EXPORTED = [
    "lrb_last_error", "lrb_version", "lrb_device_count", "lrb_launch_count",
    "lrb_plan_build_ldu", "lrb_plan_build_coo", "lrb_plan_info", "lrb_plan_export_csr",
    "lrb_plan_export_scatter", "lrb_plan_export_halo", "lrb_plan_export_sell", "lrb_plan_destroy", "lrb_part_create",
    "lrb_part_destroy", "lrb_part_pointers", "lrb_update_segment", "lrb_update_staged",
    "lrb_stage_segment", "lrb_apply_scatter", "lrb_part_fill", "lrb_part_read_buffer",
    "lrb_part_read_values", "lrb_part_join", "lrb_part_sync", "lrb_part_stats", "lrb_part_mark",
    "lrb_part_elapsed_ms", "lrb_team_create", "lrb_team_create_ex", "lrb_team_destroy",
    "lrb_team_spmv", "lrb_team_solve", "lrb_part_export", "lrb_team_create_ipc",
    "lrb_team_connect_ipc", "lrb_team_read_vector", "lrb_team_debug", "lrb_team_kernel_info",
    "lrb_team_profile", "lrb_team_profile_read", "lrb_team_profile_counters",
    "lrb_update_segment_async", "lrb_team_solve_async", "lrb_team_spmv_async",
    "lrb_part_write_values", "lrb_part_capture_base", "lrb_update_perturb",
    "lrb_upload_segment", "lrb_scatter_segment", "lrb_apply_scatter_timed", "lrb_update_segments",
    "lrb_host_register", "lrb_host_unregister",
]


def last_error() -> str:
    return (lrb_last_error() or b"").decode(errors="replace")


def check(rc: int, what: str = "") -> None:
    """Map a status code to the reference's exception types."""
    if rc == LRB_OK:
        return
    msg = last_error() or what or f"status {rc}"
    if rc in (LRB_EVALUE, LRB_ENOTPD):
        raise ValueError(msg)
    if rc == LRB_ERUNTIME:
        raise RuntimeError(msg)
    raise NativeError(msg)


def ptr(a) -> int:
    """Address of a contiguous numpy array (or 0 for None)."""
    if a is None:
        return 0
    return a.ctypes.data


def i64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)


def ptr_array(ptrs):
    arr = (C.c_void_p * max(len(ptrs), 1))()
    for i, p in enumerate(ptrs):
        arr[i] = p
    return arr

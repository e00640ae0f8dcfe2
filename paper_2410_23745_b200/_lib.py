"""ctypes binding of the in-tree C-ABI library (include/syno.h).

The library is the product: there is no Python or CPU fallback.  Importing
this module fails loudly when ``libsyno.so`` has not been built.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# SYNO_LIB_PATH: an alternative build of the same library (A/B measurements)
LIB_PATH = os.environ.get("SYNO_LIB_PATH") or os.path.join(_HERE, "libsyno.so")

SYNO_OK = 0
SYNO_E_PARSE = 1
SYNO_E_GRAPH = 2
SYNO_E_SHAPE = 3
SYNO_E_NONINTEGRAL = 4
SYNO_E_KEY = 5
SYNO_E_VALUE = 6
SYNO_E_CUDA = 7
SYNO_E_INVALID = 8
SYNO_E_UNSUPPORTED = 9

SYNO_F32 = 0
SYNO_BF16 = 1
SYNO_F64 = 2
SYNO_BWD_X_UNCHANGED = 1
SYNO_BWD_W_UNCHANGED = 2
SYNO_STAGED = 1
SYNO_REPLAY_ONLY = 2

MAX_RANK = 16
MAX_WEIGHTS = 16

# Every symbol include/syno.h declares; tests check the library exports them.
EXPORTS = (
    "syno_compile", "syno_forward", "syno_backward", "syno_query",
    "syno_emit_loop_nest", "syno_print_operator", "syno_describe_plan",
    "syno_index_map", "syno_destroy", "syno_last_error", "syno_version", "syno_launch_count",
    "syno_profile_begin", "syno_profile_end", "syno_backward_ex", "syno_tensor_write", "syno_tensor_read",
    "syno_shape_distance", "syno_graph_distance", "syno_shape_distance_clear_cache", "syno_compile_nest",
)


class SynoInfo(ctypes.Structure):
    _fields_ = [
        ("n_weights", ctypes.c_int32),
        ("x_rank", ctypes.c_int32),
        ("y_rank", ctypes.c_int32),
        ("batch_rank", ctypes.c_int32),
        ("x_shape", ctypes.c_int64 * MAX_RANK),
        ("y_shape", ctypes.c_int64 * MAX_RANK),
        ("w_rank", ctypes.c_int32 * MAX_WEIGHTS),
        ("w_shape", (ctypes.c_int64 * MAX_RANK) * MAX_WEIGHTS),
        ("flops_unstaged", ctypes.c_int64),
        ("flops_staged", ctypes.c_int64),
        ("params", ctypes.c_int64),
        ("n_forward_stages", ctypes.c_int32),
        ("grad_x_scatter", ctypes.c_int32),
        ("grad_w_scatter", ctypes.c_int32 * MAX_WEIGHTS),
        ("index_grid", ctypes.c_int64),
        ("complete", ctypes.c_int32),
        ("replay_only", ctypes.c_int32),
        ("tc_path", ctypes.c_int32),
    ]


class KernelStat(ctypes.Structure):
    _fields_ = [
        ("name", ctypes.c_char * 48),
        ("launches", ctypes.c_int64),
        ("ms", ctypes.c_double),
        ("flops", ctypes.c_double),
        ("bytes", ctypes.c_double),
    ]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `make` or __graft_entry__.build() "
            "(the B200 backend has no CPU fallback)"
        )
    lib = ctypes.CDLL(LIB_PATH)
    vp = ctypes.c_void_p
    lib.syno_compile.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_int, ctypes.POINTER(vp)]
    lib.syno_compile_nest.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p, ctypes.c_int,
                                      ctypes.POINTER(vp)]
    lib.syno_forward.argtypes = [vp, ctypes.c_int, vp, ctypes.POINTER(vp), ctypes.c_int, vp, vp]
    lib.syno_backward.argtypes = [vp, ctypes.c_int, vp, ctypes.POINTER(vp), ctypes.c_int, vp, vp,
                                  ctypes.POINTER(vp), vp]
    lib.syno_backward_ex.argtypes = [vp, ctypes.c_int, vp, ctypes.POINTER(vp), ctypes.c_int, vp, vp,
                                     ctypes.POINTER(vp), ctypes.c_int, vp]
    lib.syno_tensor_write.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.POINTER(ctypes.c_int64),
                                      ctypes.POINTER(ctypes.c_double)]
    lib.syno_tensor_read.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int64),
                                     ctypes.POINTER(ctypes.c_double), ctypes.c_int64, ctypes.POINTER(ctypes.c_int64)]
    lib.syno_query.argtypes = [vp, ctypes.POINTER(SynoInfo)]
    for name in ("syno_emit_loop_nest",):
        getattr(lib, name).argtypes = [vp, ctypes.c_int, ctypes.c_char_p, ctypes.c_size_t,
                                       ctypes.POINTER(ctypes.c_size_t)]
    for name in ("syno_print_operator", "syno_describe_plan"):
        getattr(lib, name).argtypes = [vp, ctypes.c_char_p, ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)]
    lib.syno_index_map.argtypes = [vp, ctypes.c_int, ctypes.c_int, vp, vp]
    i32p = ctypes.POINTER(ctypes.c_int32)
    lib.syno_shape_distance.argtypes = [ctypes.c_int, i32p, i32p, ctypes.POINTER(ctypes.c_uint8), ctypes.c_int,
                                        i32p, i32p, ctypes.c_int, ctypes.POINTER(ctypes.c_double), i32p, i32p, i32p]
    lib.syno_graph_distance.argtypes = [vp, ctypes.POINTER(ctypes.c_double)]
    lib.syno_shape_distance_clear_cache.restype = None
    lib.syno_destroy.argtypes = [vp]
    lib.syno_destroy.restype = None
    lib.syno_last_error.restype = ctypes.c_char_p
    lib.syno_version.restype = ctypes.c_char_p
    lib.syno_launch_count.restype = ctypes.c_uint64
    lib.syno_profile_begin.restype = None
    lib.syno_profile_end.argtypes = [ctypes.POINTER(KernelStat), ctypes.c_int, ctypes.POINTER(ctypes.c_int)]
    for name in EXPORTS:
        if name not in ("syno_destroy", "syno_last_error", "syno_version", "syno_launch_count",
                        "syno_profile_begin", "syno_shape_distance_clear_cache"):
            getattr(lib, name).restype = ctypes.c_int
    return lib


lib = _load()


def last_error() -> str:
    return lib.syno_last_error().decode(errors="replace")


def text_call(fn, *args) -> str:
    n = ctypes.c_size_t(0)
    rc = fn(*args, None, 0, ctypes.byref(n))
    if rc:
        raise RuntimeError(last_error())
    buf = ctypes.create_string_buffer(n.value + 1)
    rc = fn(*args, buf, n.value + 1, ctypes.byref(n))
    if rc:
        raise RuntimeError(last_error())
    return buf.value.decode()


def profile_begin() -> None:
    lib.syno_profile_begin()


def profile_end() -> dict:
    """{kernel class: {launches, ms, flops, bytes}} since profile_begin()."""
    cap = 64
    buf = (KernelStat * cap)()
    n = ctypes.c_int(0)
    rc = lib.syno_profile_end(buf, cap, ctypes.byref(n))
    if rc:
        raise RuntimeError(last_error())
    return {buf[i].name.decode(): {"launches": buf[i].launches, "ms": buf[i].ms, "flops": buf[i].flops,
                                   "bytes": buf[i].bytes} for i in range(min(n.value, cap))}

"""ctypes binding of libttncbc.so (include/ttn_cbc.h) — argument marshalling only.

Every numerical step runs in the CUDA library.  There is no CPU fallback: if the shared
library is missing or the device is not an sm_100 GPU, the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libttncbc.so")

TTN_STATE, TTN_OPERATOR = 0, 1
STATUS = {0: "OK", 1: "ERR_ARG", 2: "ERR_TOPOLOGY", 3: "ERR_SHAPE", 4: "ERR_OOM", 5: "ERR_CUDA",
          6: "ERR_NUMERIC", 7: "ERR_UNSUPPORTED", 8: "ERR_NCCL"}

# the C ABI symbols (kept in sync with include/ttn_cbc.h; tests/test_abi.py checks both)
SYMBOLS = ["ttn_ctx_create", "ttn_ctx_destroy", "ttn_last_error", "ttn_version", "ttn_create", "ttn_destroy",
           "ttn_n_nodes", "ttn_node_shape", "ttn_get_tensor", "cbc_apply", "cbc_apply_batch", "ttn_overlap",
           "ttn_overlap_batch", "ttn_norm", "ttn_get_data", "ttn_get_data_batch", "ttn_profile_enable", "ttn_profile_read", "ttn_launch_count",
           "ttn_comm_unique_id", "ttn_ctx_set_comm", "ttn_partition_plan", "ttn_ctx_set_workers",
           "ttn_sandwich", "ttn_op_norm2", "ttn_ctx_set_schedule",
           "ttn_loopback_create", "ttn_loopback_destroy", "ttn_ctx_set_comm_loopback", "ttn_test_heev"]


class c128(C.Structure):
    _fields_ = [("re", C.c_double), ("im", C.c_double)]


class Report(C.Structure):
    _fields_ = [("norm", C.c_double), ("discarded_weight_sum", C.c_double), ("max_bond", C.c_int64),
                ("peak_entries", C.c_int64), ("seconds", C.c_double), ("flops_algorithmic", C.c_double),
                ("rank_fallbacks", C.c_int32), ("host_syncs", C.c_int32), ("split_compresses", C.c_int32),
                ("exact_factors", C.c_int32), ("flops_gemm_exec", C.c_double), ("flops_gemm_min", C.c_double)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p)
FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p, C.c_void_p)


class Allocator(C.Structure):
    """ttn_allocator (include/ttn_cbc.h)."""
    _fields_ = [("alloc", ALLOC_FN), ("free", FREE_FN), ("state", C.c_void_p)]


class TTNError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


_lib = None


def load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(nvcc, sm_100a).  There is no CPU fallback.")
    lib = C.CDLL(LIB_PATH)
    P, I32, I64, D = C.c_void_p, C.c_int32, C.c_int64, C.c_double
    sig = {
        "ttn_ctx_create": (C.c_int, [C.c_int, P, C.POINTER(Allocator), C.POINTER(P)]),
        "ttn_ctx_destroy": (C.c_int, [P]),
        "ttn_last_error": (C.c_char_p, [P]),
        "ttn_version": (C.c_char_p, []),
        "ttn_create": (C.c_int, [P, C.c_int, I32, C.POINTER(I32), C.POINTER(I32), C.POINTER(I64), C.POINTER(P),
                                 C.c_int, C.POINTER(P)]),
        "ttn_destroy": (C.c_int, [P]),
        "ttn_n_nodes": (C.c_int, [P, C.POINTER(I32)]),
        "ttn_node_shape": (C.c_int, [P, I32, C.POINTER(I32), C.POINTER(I64)]),
        "ttn_get_tensor": (C.c_int, [P, P, I32, P, C.c_size_t]),
        "cbc_apply": (C.c_int, [P, P, P, I64, D, C.POINTER(P), C.POINTER(Report)]),
        "cbc_apply_batch": (C.c_int, [P, I32, C.POINTER(P), C.POINTER(P), I64, D, C.POINTER(P), C.POINTER(Report)]),
        "ttn_overlap": (C.c_int, [P, P, P, C.POINTER(c128)]),
        "ttn_overlap_batch": (C.c_int, [P, I32, C.POINTER(P), C.POINTER(P), C.POINTER(c128)]),
        "ttn_norm": (C.c_int, [P, P, C.POINTER(D)]),
        "ttn_get_data": (C.c_int, [P, P, P, C.c_size_t]),
        "ttn_get_data_batch": (C.c_int, [P, I32, C.POINTER(P), C.POINTER(P), C.POINTER(C.c_size_t)]),
        "ttn_profile_enable": (C.c_int, [C.c_int]),
        "ttn_profile_read": (C.c_int, [C.c_char_p, C.POINTER(D), C.POINTER(D), C.POINTER(D), C.POINTER(I64)]),
        "ttn_launch_count": (C.c_int, [C.POINTER(I64)]),
        "ttn_comm_unique_id": (C.c_int, [P]),
        "ttn_ctx_set_workers": (C.c_int, [P, C.c_int]),
        "ttn_ctx_set_schedule": (C.c_int, [P, C.c_int, C.c_int]),
        "ttn_loopback_create": (C.c_int, [C.c_int, C.POINTER(P)]),
        "ttn_loopback_destroy": (C.c_int, [P]),
        "ttn_ctx_set_comm_loopback": (C.c_int, [P, P, C.c_int, C.c_int]),
        "ttn_sandwich": (C.c_int, [P, P, P, P, C.POINTER(c128)]),
        "ttn_op_norm2": (C.c_int, [P, P, P, C.POINTER(D)]),
        "ttn_ctx_set_comm": (C.c_int, [P, P, C.c_int, C.c_int, C.c_int]),
        "ttn_partition_plan": (C.c_int, [I32, C.POINTER(I32), C.c_int, C.POINTER(I32)]),
        "ttn_test_heev": (C.c_int, [P, I32, I32, I32, I32, D, I32, P, P, P, P, P]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def check(ctx, status):
    if status != 0:
        msg = load().ttn_last_error(ctx).decode() if ctx else ""
        raise TTNError(status, msg)


def as_i32(xs):
    a = (C.c_int32 * len(xs))(*[int(x) for x in xs])
    return a


def as_i64(xs):
    return (C.c_int64 * len(xs))(*[int(x) for x in xs])


def host_c128(arr: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(arr, dtype=np.complex128)

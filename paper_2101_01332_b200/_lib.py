"""ctypes binding of libtsat.so (C-ABI in include/tsat.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_2101_01332_b200/csrc``).  There is no fallback: importing an
engine without the library, or without a CUDA device, raises loudly.
"""

from __future__ import annotations

import ctypes as C
import os

from . import errors as E

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libtsat.so")

_lib = None

u32p = C.POINTER(C.c_uint32)
i32p = C.POINTER(C.c_int32)
i64p = C.POINTER(C.c_int64)
f64p = C.POINTER(C.c_double)
u8p = C.POINTER(C.c_uint8)


class Limits(C.Structure):
    _fields_ = [("n_max", C.c_int64), ("k_max", C.c_int64), ("k_multi", C.c_int64),
                ("time_limit_s", C.c_double)]


class Report(C.Structure):
    _fields_ = [("iterations", C.c_int64), ("stop_reason", C.c_int32), ("pad", C.c_int32),
                ("prefilter_checks", C.c_int64), ("prefilter_rejects", C.c_int64),
                ("postprocess_filtered", C.c_int64), ("node_limit_overshoot", C.c_int64),
                ("filter_size", C.c_int64), ("time_s", C.c_double)]


# tsat_allgather_fn: (ctx, send, recv, bytes) -> 0 on success
ALLGATHER_FN = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64)

_SIGS = {
    "tsat_create": ([C.c_int, C.c_int, C.POINTER(C.c_void_p)], C.c_int),
    "tsat_destroy": ([C.c_void_p], None),
    "tsat_last_error": ([C.c_void_p], C.c_char_p),
    "tsat_set_atoms": ([C.c_void_p, C.c_int32, i32p, i64p, i32p, i32p, i64p, i32p, i64p, C.c_char_p, i64p], C.c_int),
    "tsat_load_egraph": ([C.c_void_p, C.c_uint32, u32p, u32p, u32p, C.c_uint32], C.c_int),
    "tsat_add_terms": ([C.c_void_p, C.c_int32, i32p, C.c_int32, i32p, C.c_int32, u32p, u32p], C.c_int),
    "tsat_union": ([C.c_void_p, C.c_uint32, C.c_uint32, u32p], C.c_int),
    "tsat_rebuild": ([C.c_void_p], C.c_int),
    "tsat_force_rebuild": ([C.c_void_p], C.c_int),
    "tsat_union_batch": ([C.c_void_p, C.c_int64, u32p, u32p], C.c_int),
    "tsat_find": ([C.c_void_p, C.c_uint32, u32p], C.c_int),
    "tsat_set_root": ([C.c_void_p, C.c_uint32], C.c_int),
    "tsat_query_sizes": ([C.c_void_p, u32p, u32p, u32p, u32p, u32p], C.c_int),
    "tsat_num_classes": ([C.c_void_p, u32p], C.c_int),
    "tsat_download_flags": ([C.c_void_p, u8p], C.c_int),
    "tsat_download": ([C.c_void_p, u32p, u32p, u32p, u32p, u8p], C.c_int),
    "tsat_find_batch": ([C.c_void_p, C.c_uint32, u32p, u32p], C.c_int),
    "tsat_download_nodes": ([C.c_void_p, C.c_uint32, u32p, u32p, u32p, u32p, C.c_uint64,
                             C.POINTER(C.c_uint64)], C.c_int),
    "tsat_download_values": ([C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, u32p], C.c_int),
    "tsat_dump": ([C.c_void_p, C.c_char_p, C.c_int64, i64p], C.c_int),
    "tsat_set_filter": ([C.c_void_p, C.c_int32, u32p, C.c_int32], C.c_int),
    "tsat_get_filter": ([C.c_void_p, u32p, C.c_int64, i64p], C.c_int),
    "tsat_load_rules": ([C.c_void_p, C.c_int64, i64p], C.c_int),
    "tsat_saturate": ([C.c_void_p, C.POINTER(Limits), C.c_int32, C.c_int32, C.POINTER(Report), i64p, i64p], C.c_int),
    "tsat_iterate": ([C.c_void_p, C.POINTER(Limits), C.c_int32, C.c_int32, C.c_int64, C.POINTER(Report), i64p, i64p],
                     C.c_int),
    "tsat_ilp_build": ([C.c_void_p, u32p], C.c_int),
    "tsat_ilp_download": ([C.c_void_p, u32p, u32p, u32p, u32p, u32p, u32p], C.c_int),
    "tsat_set_record_rejects": ([C.c_void_p, C.c_int32], C.c_int),
    "tsat_set_reach_budget": ([C.c_void_p, C.c_uint64], C.c_int),
    "tsat_copy_state": ([C.c_void_p, C.c_void_p], C.c_int),
    "tsat_eval_terms": ([C.c_void_p, C.c_int32, i32p, C.c_int32, i32p, C.c_int32, u32p, u32p, C.c_void_p, i32p],
                        C.c_int),
    "tsat_class_graph": ([C.c_void_p, u32p, u32p, u32p, u32p], C.c_int),
    "tsat_descendants": ([C.c_void_p, u32p, u32p, C.c_uint64, u32p], C.c_int),
    "tsat_reach_mode": ([C.c_void_p, C.POINTER(C.c_int32)], C.c_int),
    "tsat_rejects": ([C.c_void_p, u32p, C.c_int64, i64p], C.c_int),
    "tsat_ematch": ([C.c_void_p, C.c_int32, u32p, u32p, C.c_int64, i64p, i32p], C.c_int),
    "tsat_ematch_batch": ([C.c_void_p, C.c_int32, i32p, i64p], C.c_int),
    "tsat_break_cycles": ([C.c_void_p, i64p], C.c_int),
    "tsat_dfs_cycles": ([C.c_void_p, u32p, C.c_int64, u32p, C.c_int64, i64p], C.c_int),
    "tsat_costs": ([C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_char_p, i64p, f64p, f64p], C.c_int),
    "tsat_costs_gather": ([C.c_void_p, C.c_uint32, u32p, f64p], C.c_int),
    "tsat_greedy": ([C.c_void_p, f64p, u32p, u32p, u32p, f64p, i64p], C.c_int),
    "tsat_phase_times": ([C.c_void_p, f64p, C.c_int32], C.c_int),
    "tsat_debug_info": ([C.c_void_p, i64p, C.c_int32], C.c_int),
    "tsat_kernel_stats": ([C.c_void_p, f64p, f64p, i64p, C.c_int32, C.c_int32], C.c_int),
    "tsat_stream": ([C.c_void_p, C.POINTER(C.c_void_p)], C.c_int),
    "tsat_shard_setup": ([C.c_void_p, C.c_int32, C.c_int32, C.c_char_p, C.c_int32], C.c_int),
    "tsat_shard_setup_host": ([C.c_void_p, C.c_int32, C.c_int32, ALLGATHER_FN, C.c_void_p], C.c_int),
    "tsat_nccl_unique_id": ([C.c_char_p, C.c_int32, i32p], C.c_int),
    "tsat_shard_range": ([C.c_uint64, C.c_int32, C.c_int32, u32p, u32p], C.c_int),
}

EXPORTED = tuple(_SIGS)


def load():
    """Load libtsat.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
        )
    lib = C.CDLL(LIB_PATH)
    for name, (args, res) in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


_STATUS = {
    -2: ValueError,
    -3: E.ShapeMismatch,
    -4: E.MissingSplitOrigin,
    -5: E.AnalysisMergeError,
    -6: E.NoFiniteExtraction,
    -8: NotImplementedError,
    -9: E.UnknownSignature,
    -10: ValueError,
    -11: E.TensorSatError,
}


def check(handle, status: int) -> None:
    if status == 0:
        return
    msg = load().tsat_last_error(handle)
    text = msg.decode() if msg else f"libtsat status {status}"
    raise _STATUS.get(status, E.DeviceError)(text)


def ptr(arr, ctype):
    """ctypes pointer to a contiguous numpy array (or NULL for None)."""
    if arr is None:
        return None
    return arr.ctypes.data_as(C.POINTER(ctype))

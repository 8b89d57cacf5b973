"""ctypes binding of libcm.so (include/cm.h).

The library is built in-tree by ``__graft_entry__.build()`` /
``python paper_1810_11112_b200/_build.py``. There is no fallback: importing
this module without the built library raises immediately.
"""

from __future__ import annotations

import ctypes as C
import os

from . import errors as E

_HERE = os.path.dirname(os.path.abspath(__file__))
# CM_LIB selects another build of the same ABI (A/B studies under tools/)
LIB_PATH = os.environ.get("CM_LIB") or os.path.join(_HERE, "libcm.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python paper_1810_11112_b200/_build.py` "
        "(there is no CPU fallback for the allreduce path)")

lib = C.CDLL(LIB_PATH)


def _bind_fast():
    """The CPython fast-call module (csrc/pyfast.cpp) bound to THIS library
    instance's entry points; None when it is not built (the ctypes calls are
    then used — same library, only the per-call argument conversion differs)."""
    try:
        from . import _cmfast
    except ImportError:
        return None
    addr = [C.cast(getattr(lib, n), C.c_void_p).value for n in (
        "cm_allreduce", "cm_reduce_scatter", "cm_allgather", "cm_fused_allreduce_agreed", "cm_comm_poll",
        "cm_comm_sync")]
    _cmfast.bind(*addr)
    return _cmfast


fast = None if os.environ.get("CM_NO_FAST") else _bind_fast()

# enums (cm.h)
CM_OK = 0
DTYPE = {"float32": 0, "float64": 1, "bfloat16": 2, "int32": 3, "int64": 4}
OP = {"sum": 0, "max": 1}
ALGO = {"auto": 0, "flat": 1, "ring_rsa": 2, "rhd_rsa": 3}
ALGO_NAME = {v: k for k, v in ALGO.items()}
LAYOUT = {"ring": 0, "rhd": 1}
POLICY = {"no_cache": 0, "lazy_cache": 1, "intercept_cache": 2}
KIND = {"host": 0, "device": 1}
KIND_NAME = {v: k for k, v in KIND.items()}
IPC_HANDLE_BYTES = 64
MAX_RANKS = 16


class Stats(C.Structure):
    _fields_ = [("rounds", C.c_int64), ("messages_per_rank", C.c_int64),
                ("bytes_sent_per_rank", C.c_int64)]


class RegStats(C.Structure):
    _fields_ = [("driver_queries", C.c_int64), ("cache_hits", C.c_int64),
                ("inserts", C.c_int64), ("invalidations", C.c_int64)]


class BufferInfo(C.Structure):
    _fields_ = [("kind", C.c_int32), ("device", C.c_int32), ("range_start", C.c_uint64),
                ("range_size", C.c_int64), ("buffer_id", C.c_uint64)]


_vp = C.c_void_p
_i64 = C.c_int64
_i = C.c_int
_P = C.POINTER

_SIGS = {
    "cm_version": ([], C.c_char_p),
    "cm_last_error": ([], C.c_char_p),
    "cm_dtype_size": ([_i], C.c_size_t),
    "cm_chunk_partition": ([_i64, _i, _P(_i64), _P(_i64)], _i),
    "cm_layout": ([_i, _i64, _i, _P(_i64), _P(_i64)], _i),
    "cm_layout_piece": ([_i, _i64, _i, _i, _i, _P(_i64), _P(_i64)], _i),
    "cm_resolve_algorithm": ([_i, _i64, _i64, _P(_i)], _i),
    "cm_algo_stats": ([_i, _i, _i, _i64, _i, _i64, _P(Stats)], _i),
    "cm_rs_stats": ([_i, _i, _i, _i64, _i, _P(Stats)], _i),
    "cm_ag_stats": ([_i, _i, _i, _i64, _i, _P(Stats)], _i),
    "cm_fuse_plan": ([_i, _P(_i64), _P(_i), _i64, _P(_i), _P(_i)], _i),
    "cm_registry_create": ([_i, _i64, _i, _P(_vp)], _i),
    "cm_registry_destroy": ([_vp], _i),
    "cm_registry_alloc": ([_vp, _i, _i64, _P(C.c_uint64)], _i),
    "cm_registry_free": ([_vp, C.c_uint64], _i),
    "cm_registry_register": ([_vp, C.c_uint64, _i64, _i], _i),
    "cm_registry_unregister": ([_vp, C.c_uint64], _i),
    "cm_registry_classify": ([_vp, C.c_uint64, _P(_i)], _i),
    "cm_registry_info": ([_vp, C.c_uint64, _P(BufferInfo)], _i),
    "cm_registry_ground_truth": ([_vp, C.c_uint64, _P(_i)], _i),
    "cm_registry_stats": ([_vp, _P(RegStats)], _i),
    "cm_registry_policy": ([_vp, _P(_i)], _i),
    "cm_registry_query_time_ns": ([_vp, _P(_i64)], _i),
    "cm_registry_stats_json": ([_vp, C.c_char_p, C.c_size_t], _i),
    "cm_comm_create": ([_i, _i, _i, _i64, _i64, _P(_vp)], _i),
    "cm_comm_ipc_handle": ([_vp, _vp], _i),
    "cm_comm_connect": ([_vp, _vp], _i),
    "cm_comm_create_virtual": ([_i, _i, _i64, _P(_vp)], _i),
    "cm_comm_destroy": ([_vp], _i),
    "cm_comm_rank": ([_vp, _P(_i)], _i),
    "cm_comm_size": ([_vp, _P(_i)], _i),
    "cm_comm_set_timeout": ([_vp, C.c_double], _i),
    "cm_comm_set_policy": ([_vp, _i], _i),
    "cm_comm_registry": ([_vp, _P(_vp)], _i),
    "cm_comm_set_param": ([_vp, C.c_char_p, _i64], _i),
    "cm_comm_get_param": ([_vp, C.c_char_p, _P(_i64)], _i),
    "cm_comm_alloc": ([_vp, _i64, _P(_vp)], _i),
    "cm_comm_free": ([_vp, _vp], _i),
    "cm_comm_export": ([_vp, _vp, _i64, _vp, _P(_i64)], _i),
    "cm_comm_register": ([_vp, _vp, _i64, _vp, _P(_i64), _P(_i64)], _i),
    "cm_buffer_ids": ([_vp, _i, _vp, _vp], _i),
    "cm_comm_deregister": ([_vp, _vp], _i),
    "cm_comm_register_v": ([_vp, _P(_vp), _i64, _P(_i64)], _i),
    "cm_comm_sync": ([_vp, _vp], _i),
    "cm_comm_poll": ([_vp], _i),
    "cm_agree": ([_vp, _P(_i64), _i, _P(_i64), _vp], _i),
    "cm_agree_v": ([_vp, _P(_i64), _i, _P(_i64), _vp], _i),
    "cm_comm_counters": ([_vp, _P(_i64), _P(_i64), _P(_i64), _P(_i64)], _i),
    "cm_comm_launches": ([_vp, _P(_i64)], _i),
    "cm_comm_profile": ([_vp, _i], _i),
    "cm_comm_set_trace": ([_vp, _vp, _i], _i),
    "cm_comm_profile_read": ([_vp, _i, _P(_i64), _P(C.c_double), _P(_i64)], _i),
    "cm_allreduce": ([_vp, _vp, _vp, _i64, _i, _i, _i, _i64, _i, _vp, _P(Stats)], _i),
    "cm_reduce_scatter": ([_vp, _vp, _vp, _i64, _i, _i, _i, _vp, _P(Stats)], _i),
    "cm_allgather": ([_vp, _vp, _vp, _i64, _i, _i, _vp, _P(Stats)], _i),
    "cm_fused_allreduce": ([_vp, _i, _P(_vp), _P(_i64), _i, _vp, _i, _i64, _i64, _i, _vp,
                            _P(Stats), _P(_i)], _i),
    "cm_fused_allreduce_agreed": ([_vp, _i, _P(_vp), _P(_i64), _i, _vp, _i, _i64, _i64, _i,
                                   _P(_i64), _i, _P(_i), _P(_i64), _vp, _P(Stats), _P(_i)], _i),
    "cm_fused_allreduce_agreed_v": ([_vp, _i, _P(_vp), _P(_i64), _i, _P(_vp), _i, _i64, _i64, _i,
                                     _P(_i64), _i, _P(_i), _P(_i64), _vp, _P(Stats), _P(_i)], _i),
    "cm_allreduce_v": ([_vp, _P(_vp), _P(_vp), _i64, _i, _i, _i, _i64, _i, _vp, _P(Stats)], _i),
    "cm_reduce_scatter_v": ([_vp, _P(_vp), _P(_vp), _i64, _i, _i, _i, _vp, _P(Stats)], _i),
    "cm_allgather_v": ([_vp, _P(_vp), _P(_vp), _i64, _i, _i, _vp, _P(Stats)], _i),
    "cm_local_reduce": ([_vp, _vp, _vp, _i64, _i, _i, _vp], _i),
    "cm_ps_step": ([_vp, _i, _P(_vp), _vp, _P(_i64), _i, _P(_i), C.c_uint32, C.c_double, _vp], _i),
    "cm_ps_step_v": ([_vp, _i, _P(_vp), _P(_vp), _P(_i64), _i, _P(_i), C.c_uint32, C.c_double, _vp], _i),
    "cm_batched_copy": ([_i, _P(_vp), _P(_vp), _P(_i64), _vp], _i),
    "cm_bench_p2p": ([_vp, _i, _i64, _i, _i, _vp, _P(C.c_double)], _i),
    "cm_time_allreduce": ([_vp, _vp, _vp, _i64, _i, _i, _i, _i64, _i, _i, _vp,
                           _P(C.c_double)], _i),
}

_missing = [n for n in _SIGS if not hasattr(lib, n)]
if _missing:
    raise ImportError(f"{LIB_PATH} is stale (missing {', '.join(_missing[:4])}): rebuild it with "
                      f"`python paper_1810_11112_b200/_build.py`")
for _name, (_args, _res) in _SIGS.items():
    _fn = getattr(lib, _name)
    _fn.argtypes = _args
    _fn.restype = _res

EXPORTS = tuple(_SIGS)

_STATUS_EXC = {
    1: E.ShapeError,
    2: E.InvalidGroupError,
    3: E.RoutingError,
    4: E.TransportError,
    5: E.DeadlockError,
    6: E.ConfigError,
    7: E.InvalidHandleError,
    8: E.UnknownBufferError,
    9: E.UnsupportedOperationError,
    10: E.TransportError,
    11: ValueError,
}


def check(status: int) -> None:
    """Raise the reference exception class for a non-zero cm status."""
    if status == CM_OK:
        return
    msg = lib.cm_last_error().decode("utf-8", "replace")
    exc = _STATUS_EXC.get(status, E.CollectiumError)
    if exc is E.DeadlockError:
        raise E.TransportError(msg)
    raise exc(msg)


def ptr_array(ptrs):
    arr = (C.c_void_p * max(1, len(ptrs)))()
    for i, p in enumerate(ptrs):
        arr[i] = p
    return arr


def i64_array(vals):
    arr = (C.c_int64 * max(1, len(vals)))()
    for i, v in enumerate(vals):
        arr[i] = int(v)
    return arr

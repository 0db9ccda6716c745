"""ctypes binding of ``libiccl_b200.so`` (the C ABI in ``include/iccl_b200.h``).

The library is built in-tree by ``__graft_entry__.build()`` (or ``make -C
paper_2510_00991_b200/csrc``).  There is no fallback: if the shared library is
missing or lacks a symbol this module raises at import, so a GPU box can never
run the product path on anything but the CUDA library.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ICCL_B200_LIB", os.path.join(_HERE, "libiccl_b200.so"))

ICCL_UNIQUE_ID_BYTES = 128


class UniqueId(C.Structure):
    _fields_ = [("internal", C.c_char * ICCL_UNIQUE_ID_BYTES)]


class Config(C.Structure):
    _fields_ = [
        ("chunk_bytes", C.c_uint64),
        ("streams_per_peer", C.c_int32),
        ("sm_cap", C.c_int32),
        ("window", C.c_int32),
        ("monitor_window", C.c_int32),
        ("monitor_enabled", C.c_int32),
        ("backup_kind", C.c_int32),
        ("transport", C.c_int32),
        ("timeout_exponent", C.c_int32),
        ("retry_count", C.c_int32),
        ("delta_us", C.c_uint64),
        ("probe_period_us", C.c_uint64),
        ("sm_small_bytes", C.c_uint64),
        ("proxy_cpu", C.c_int32),
        ("relay_slot_mib", C.c_int32),
        ("direct_max_kib", C.c_int32),
        ("reserved", C.c_int32 * 5),
    ]


class XferState(C.Structure):
    _fields_ = [
        ("role", C.c_int32), ("total_chunks", C.c_int32),
        ("posted", C.c_int32), ("transmitted", C.c_int32), ("acked", C.c_int32),
        ("r_posted", C.c_int32), ("received", C.c_int32), ("done", C.c_int32),
        ("active_path", C.c_int32), ("switches", C.c_int32), ("bytes", C.c_uint64),
    ]


class Fault(C.Structure):
    _fields_ = [
        ("src", C.c_int32), ("dst", C.c_int32), ("path", C.c_int32), ("up", C.c_int32),
        ("trigger_kind", C.c_int32), ("op_index", C.c_int32), ("chunk", C.c_int64), ("t_us", C.c_uint64),
    ]


class MonRec(C.Structure):
    _fields_ = [
        ("t1_ns", C.c_uint64), ("t2_ns", C.c_uint64), ("bytes", C.c_uint64),
        ("peer", C.c_int32), ("path", C.c_int32), ("chunk", C.c_int32), ("dir", C.c_int32),
        ("op_seq", C.c_uint64),
    ]


class SwitchEvent(C.Structure):
    _fields_ = [
        ("t_ns", C.c_uint64), ("peer", C.c_int32), ("to_path", C.c_int32),
        ("resume_chunk", C.c_int32), ("trigger", C.c_int32), ("detect_ns", C.c_uint64),
    ]


class Stats(C.Structure):
    _fields_ = [("kernels_launched", C.c_uint64), ("copies_issued", C.c_uint64), ("bytes_issued", C.c_uint64),
                ("ctas_launched", C.c_uint64), ("pulls_issued", C.c_uint64), ("cts_timeouts", C.c_uint64),
                ("pending_xfers", C.c_uint64), ("reserved", C.c_uint64 * 1)]


_c = C.c_int  # iccl_result_t
_p = C.c_void_p
_sz = C.c_size_t
_u64 = C.c_uint64
_i64 = C.c_int64

# name -> (restype, argtypes); every symbol include/iccl_b200.h declares.
PROTOTYPES = {
    "iccl_get_error_string": (C.c_char_p, [_c]),
    "iccl_get_last_error": (C.c_char_p, []),
    "iccl_get_version": (C.c_int, []),
    "iccl_config_init": (_c, [C.POINTER(Config)]),
    "iccl_config_validate": (_c, [C.POINTER(Config)]),
    "iccl_get_unique_id": (_c, [C.POINTER(UniqueId)]),
    "iccl_comm_init_rank": (_c, [C.POINTER(_p), C.c_int, UniqueId, C.c_int, C.c_int, C.POINTER(Config)]),
    "iccl_comm_destroy": (_c, [_p]),
    "iccl_comm_abort": (_c, [_p]),
    "iccl_comm_count": (_c, [_p, C.POINTER(C.c_int)]),
    "iccl_comm_user_rank": (_c, [_p, C.POINTER(C.c_int)]),
    "iccl_comm_get_async_error": (_c, [_p, C.POINTER(C.c_int)]),
    "iccl_comm_op_counts": (_c, [_p, C.POINTER(_u64), C.c_int]),
    "iccl_comm_stats": (_c, [_p, C.POINTER(Stats)]),
    "iccl_register": (_c, [_p, _p, _sz, C.POINTER(_u64)]),
    "iccl_deregister": (_c, [_p, _u64]),
    "iccl_send": (_c, [_p, _p, _sz, C.c_int, _p, C.POINTER(_u64)]),
    "iccl_recv": (_c, [_p, _p, _sz, C.c_int, _p, C.POINTER(_u64)]),
    "iccl_group_start": (_c, [_p]),
    "iccl_group_end": (_c, [_p]),
    "iccl_alltoall": (_c, [_p, _p, _p, _sz, _p]),
    "iccl_alltoallv": (_c, [_p, _p, C.POINTER(_sz), C.POINTER(_sz), _p, C.POINTER(_sz), C.POINTER(_sz), _sz, _p]),
    "iccl_req_test": (_c, [_p, _u64, C.POINTER(C.c_int)]),
    "iccl_req_wait": (_c, [_p, _u64, _i64]),
    "iccl_req_state": (_c, [_p, _u64, C.POINTER(XferState)]),
    "iccl_path_switch": (_c, [_p, C.c_int, C.c_int]),
    "iccl_path_active": (_c, [_p, C.c_int, C.POINTER(C.c_int)]),
    "iccl_fault_set": (_c, [_p, C.POINTER(Fault), C.c_int]),
    "iccl_switch_events": (_c, [_p, C.POINTER(SwitchEvent), C.c_int, C.POINTER(C.c_int)]),
    "iccl_monitor_config": (_c, [_p, C.c_int, C.c_int]),
    "iccl_comm_set_chunk_bytes": (_c, [_p, _u64]),
    "iccl_monitor_read": (_c, [_p, C.POINTER(MonRec), C.c_int, C.POINTER(C.c_int)]),
    "iccl_gather_rows": (_c, [_p, _p, _p, _i64, _i64, C.c_int, _p]),
    "iccl_scatter_rows": (_c, [_p, _p, _p, _i64, _i64, C.c_int, _p]),
    "iccl_expand_rows": (_c, [_p, _p, _p, _i64, C.c_int32, _i64, C.c_int, _p]),
    "iccl_dispatch_rows": (_c, [_p, _p, _i64, C.c_int32, _p, C.POINTER(_sz), _p, C.POINTER(_sz), _i64, _p]),
    "iccl_combine_rows": (_c, [_p, _p, C.POINTER(_sz), _p, _p, C.POINTER(_sz), _i64, _p]),
    "iccl_copy_sm": (_c, [_p, _p, _sz, C.c_int, _p]),
    "iccl_retry_timeout_ns": (_u64, [C.c_int, C.c_int]),
    "iccl_switch_pointers": (C.c_int, [C.POINTER(XferState), C.POINTER(XferState)]),
    "iccl_per_message_throughput": (_c, [C.POINTER(MonRec), C.POINTER(C.c_double)]),
    "iccl_window_throughput": (_c, [C.POINTER(MonRec), C.c_int, C.c_int, C.POINTER(C.c_double)]),
    "iccl_sample_series": (_c, [C.POINTER(MonRec), C.c_int, C.c_int, C.POINTER(C.c_double), C.POINTER(_u64),
                                C.POINTER(C.c_int)]),
    "iccl_detect_lagging_rank": (_c, [C.POINTER(_u64), C.c_int, _u64, C.POINTER(C.c_int)]),
    "iccl_selftest_pair_bytes": (_sz, []),
    "iccl_selftest_rzv_bytes": (_sz, []),
    "iccl_selftest_route_small": (C.c_int, [_p, C.c_int]),
    "iccl_selftest_route_arm": (None, [_p, C.c_int, C.c_int]),
    "iccl_selftest_rzv_post": (C.c_int, [_p, C.c_int, _u64, _u64, C.POINTER(_u64)]),
    "iccl_selftest_failover": (C.c_int, [C.c_int, C.c_int, C.c_int, _u64, C.POINTER(_i64)]),
}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"libiccl_b200.so not found at {LIB_PATH}: build it with "
            "`python -c 'import __graft_entry__ as g; g.build()'` or `make -C paper_2510_00991_b200/csrc`. "
            "There is no CPU fallback for the ICCL B200 path.")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in PROTOTYPES.items():
        fn = getattr(lib, name)  # AttributeError -> the build is incomplete: fail loudly
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()

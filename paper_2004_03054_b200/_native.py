"""ctypes binding of ``libluda_b200.so`` (the C ABI in ``include/luda_b200.h``).

The shared library is built in-tree by ``__graft_entry__.build()`` (nvcc,
``-gencode arch=compute_100a,code=sm_100a``). There is no CPU fallback: if the
library is missing or no sm_100 device is present, :func:`lib` raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

from . import errors

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LUDA_LIB") or os.path.join(HERE, "libluda_b200.so")

c_u8p = ctypes.POINTER(ctypes.c_uint8)
c_u32p = ctypes.POINTER(ctypes.c_uint32)
c_u64p = ctypes.POINTER(ctypes.c_uint64)
c_i64p = ctypes.POINTER(ctypes.c_int64)


class JobDesc(ctypes.Structure):
    _fields_ = [
        ("arena", ctypes.c_void_p),
        ("arena_bytes", ctypes.c_uint64),
        ("n_files", ctypes.c_uint32),
        ("file_off", c_u64p),
        ("file_len", c_u64p),
        ("file_offset_base", c_i64p),
        ("n_runs", ctypes.c_uint32),
        ("run_first_file", c_u32p),
        ("block_size", ctypes.c_uint32),
        ("restart_interval", ctypes.c_uint32),
        ("bits_per_key", ctypes.c_uint32),
        ("sst_size_target", ctypes.c_uint64),
        ("n_deeper", ctypes.c_uint32),
        ("deeper_keys", c_u8p),
        ("deeper_lens", c_u32p),
        ("range_lo", c_u8p),
        ("range_lo_len", ctypes.c_uint32),
        ("range_hi", c_u8p),
        ("range_hi_len", ctypes.c_uint32),
    ]


class JobResult(ctypes.Structure):
    _fields_ = [
        ("out", ctypes.c_void_p),
        ("out_bytes", ctypes.c_uint64),
        ("n_sst", ctypes.c_uint32),
        ("sst_off", c_u64p),
        ("sst_len", c_u64p),
        ("key_len", ctypes.c_uint32),
        ("sst_keys", c_u8p),
        ("n_in", ctypes.c_uint64),
        ("n_out", ctypes.c_uint64),
        ("blocks_in", ctypes.c_uint64),
        ("blocks_out", ctypes.c_uint64),
        ("t_ms", ctypes.c_double * 8),
        ("k_ms", ctypes.c_double * 8),
        ("launches", ctypes.c_uint64),
        ("priv", ctypes.c_void_p),
        ("sst_key_len", ctypes.POINTER(ctypes.c_uint32)),
    ]


class ProbePlan(ctypes.Structure):
    _fields_ = [
        ("n_l0", ctypes.c_uint32),
        ("l0", c_u32p),
        ("n_levels", ctypes.c_uint32),
        ("level_first", c_u32p),
        ("level_tables", c_u32p),
        ("range_keys", c_u8p),
        ("range_lens", c_u32p),
    ]


class GetResult(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_uint32),
        ("status", c_u32p),
        ("table", c_u32p),
        ("key_len", c_u32p),
        ("value_len", c_u32p),
        ("pos", c_u64p),
        ("packed", c_u8p),
        ("packed_bytes", ctypes.c_uint64),
        ("err_off", c_i64p),
        ("fail_index", ctypes.c_int64),
        ("t_ms", ctypes.c_double * 4),
    ]


_SIGS = {
    "luda_init": (ctypes.c_int, [ctypes.c_int]),
    "luda_shutdown": (ctypes.c_int, []),
    "luda_last_error": (ctypes.c_char_p, []),
    "luda_last_error_offset": (ctypes.c_int64, []),
    "luda_abi_version": (ctypes.c_int, []),
    "luda_set_option": (ctypes.c_int, [ctypes.c_int, ctypes.c_int64]),
    "luda_region_alloc": (ctypes.c_int, [ctypes.c_uint64, ctypes.POINTER(ctypes.c_void_p)]),
    "luda_region_free": (ctypes.c_int, [ctypes.c_void_p]),
    "luda_host_alloc": (ctypes.c_int, [ctypes.c_uint64, ctypes.POINTER(ctypes.c_void_p)]),
    "luda_host_free": (ctypes.c_int, [ctypes.c_void_p]),
    "luda_stream_create": (ctypes.c_int, [ctypes.POINTER(ctypes.c_void_p)]),
    "luda_stream_destroy": (ctypes.c_int, [ctypes.c_void_p]),
    "luda_stream_sync": (ctypes.c_int, [ctypes.c_void_p]),
    "luda_stage_in_async": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p]),
    "luda_stage_out_async": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p]),
    "luda_memcpy_d2d_async": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p]),
    "luda_event_create": (ctypes.c_int, [ctypes.POINTER(ctypes.c_void_p)]),
    "luda_event_record": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p]),
    "luda_event_query": (ctypes.c_int, [ctypes.c_void_p]),
    "luda_event_wait": (ctypes.c_int, [ctypes.c_void_p]),
    "luda_event_elapsed_ms": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(ctypes.c_float)]),
    "luda_event_destroy": (ctypes.c_int, [ctypes.c_void_p]),
    "luda_stream_wait_event": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p]),
    "luda_crc32": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_uint64, c_u32p, ctypes.c_void_p]),
    "luda_crc32_batch": (ctypes.c_int, [ctypes.c_void_p, c_u64p, c_u32p, ctypes.c_uint32, c_u32p,
                                        ctypes.c_void_p]),
    "luda_dispatch": (ctypes.c_int, [ctypes.c_int, c_i64p, ctypes.c_uint32, ctypes.POINTER(ctypes.c_void_p),
                                     c_u64p, ctypes.c_uint32, c_i64p, c_i64p, ctypes.c_void_p]),
    "luda_compact": (ctypes.c_int, [ctypes.POINTER(JobDesc), ctypes.POINTER(JobResult), ctypes.c_void_p]),
    "luda_job_release": (ctypes.c_int, [ctypes.POINTER(JobResult)]),
    "luda_build_from_sorted": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_void_p,
                                              ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32,
                                              ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint64,
                                              ctypes.POINTER(JobResult), ctypes.c_void_p]),
    "luda_build_from_sorted_var": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint32,
                                                  ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                                  ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32,
                                                  ctypes.c_uint64, ctypes.POINTER(JobResult), ctypes.c_void_p]),
    "luda_build_files_from_sorted": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_uint32, ctypes.c_void_p,
                                                    ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                                    ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32,
                                                    ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint64,
                                                    ctypes.POINTER(JobResult), ctypes.c_void_p]),
    # batched read path (luda_read.cuh)
    "luda_tables_open": (ctypes.c_int, [ctypes.c_void_p, c_u64p, c_u64p, ctypes.c_uint32,
                                        ctypes.POINTER(ctypes.c_void_p), ctypes.c_void_p]),
    "luda_tables_close": (ctypes.c_int, [ctypes.c_void_p]),
    "luda_tables_info": (ctypes.c_int, [ctypes.c_void_p, c_u32p, c_u32p]),
    "luda_tables_counters": (ctypes.c_int, [ctypes.c_void_p, c_u64p, c_u64p]),
    "luda_tables_set_plan": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ProbePlan), ctypes.c_void_p]),
    "luda_tables_get": (ctypes.c_int, [ctypes.c_void_p, c_u8p, ctypes.c_uint64, c_u64p, c_u32p, ctypes.c_uint32,
                                       c_u32p, ctypes.c_uint32, ctypes.POINTER(GetResult), ctypes.c_void_p]),
    "luda_tables_lookup_dev": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                              ctypes.c_uint32, ctypes.c_void_p, ctypes.c_uint32, ctypes.c_void_p]),
    # storage <-> HBM (luda_io_abi.inc)
    "luda_files_read": (ctypes.c_int, [ctypes.POINTER(ctypes.c_char_p), ctypes.c_uint32, ctypes.c_void_p, c_u64p,
                                       c_u64p, ctypes.c_int, ctypes.POINTER(ctypes.c_int)]),
    "luda_files_write": (ctypes.c_int, [ctypes.POINTER(ctypes.c_char_p), ctypes.c_uint32, ctypes.c_void_p, c_u64p,
                                        c_u64p, ctypes.c_int, ctypes.POINTER(ctypes.c_int)]),
    "luda_gds_status": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_uint32]),
    # multi-GPU splitter all-gather (luda_nccl_abi.inc)
    "luda_nccl_unique_id": (ctypes.c_int, [c_u8p]),
    "luda_nccl_init_rank": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, c_u8p, ctypes.POINTER(ctypes.c_void_p)]),
    "luda_nccl_init_all": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_void_p)]),
    "luda_allgather_splitters": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64,
                                                ctypes.c_void_p]),
    "luda_nccl_group_start": (ctypes.c_int, []),
    "luda_nccl_group_end": (ctypes.c_int, []),
    "luda_nccl_destroy": (ctypes.c_int, [ctypes.c_void_p]),
}

EXPORTED = tuple(_SIGS)

_lock = threading.Lock()
_lib = None
_inited = {}


def load(path: str = LIB_PATH):
    """Load the shared library and declare signatures (no device needed)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(path):
                raise errors.DeviceError(
                    f"{path} is missing: the b200 backend has no CPU fallback; run __graft_entry__.build()")
            lib = ctypes.CDLL(path)
            for name, (res, args) in _SIGS.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def lib(device_ordinal: int = 0):
    """Loaded library with ``luda_init(device_ordinal)`` done."""
    L = load()
    with _lock:
        if _inited.get(device_ordinal) is None:
            check(L.luda_init(device_ordinal))
            _inited[device_ordinal] = True
    return L


OPT_PLANNER_TILE = 1  # include/luda_b200.h enum luda_option
OPT_DEC_CTAS = 2
OPT_DEC_SEGS = 3


def sst_key_pairs(res):
    """[(smallest, largest)] internal keys of a JobResult's SSTs (slots of
    res.key_len bytes holding res.sst_key_len[i] key bytes)."""
    S = res.key_len
    keys = ctypes.string_at(res.sst_keys, 2 * S * res.n_sst)
    out = []
    for i in range(res.n_sst):
        a, b = res.sst_key_len[2 * i], res.sst_key_len[2 * i + 1]
        out.append((keys[2 * S * i:2 * S * i + a], keys[2 * S * i + S:2 * S * i + S + b]))
    return out


def check(status: int):
    if status == errors.STATUS_OK:
        return
    L = load()
    msg = L.luda_last_error().decode(errors="replace")
    off = L.luda_last_error_offset()
    raise errors.from_status(status, msg, offset=off if off >= 0 else None)

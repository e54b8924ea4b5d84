"""ctypes binding of libwarpspeed.so (the C ABI in include/warpspeed.h).

There is no fallback: if the shared library is missing or no CUDA device is
present, table construction raises.  ``symbols()`` lists the exported entry
points so CPU-only tests can check the ABI without a GPU.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "_lib", "libwarpspeed.so")

WS_OK = 0
WS_ERR_INVALID_KEY = -1
WS_ERR_CONFIG = -2
WS_ERR_CUDA = -3
WS_ERR_ALLOC = -4
WS_ERR_ARG = -5
WS_ERR_INVALID_OP = -6

WS_F_SYNC_CHECK = 1
WS_F_NO_CHECK = 2
WS_F_SERIAL = 4
WS_F_COMBINE = 8
WS_F_INTERLEAVED = 16
WS_F_CONCURRENT_KINDS = 32

EXPORTS = ("ws_create", "ws_destroy", "ws_clear", "ws_upsert", "ws_query", "ws_erase", "ws_mixed",
           "ws_locate", "ws_probe_counts", "ws_occupied", "ws_export_items",
           "ws_duplicate_scan", "ws_checksum", "ws_export_raw", "ws_read_range", "ws_info", "ws_tune",
           "ws_kernel_times",
           "ws_partition", "ws_unpermute", "ws_xchg_create", "ws_xchg_handle", "ws_xchg_open",
           "ws_xchg_run", "ws_xchg_destroy", "ws_strerror")
WS_TUNE_QUERY_ILP = 1
WS_TUNE_L2_POLICY = 2
WS_TUNE_UPSERT = 3
WS_TUNE_OCCUPANCY = 4
WS_TUNE_KERNEL_EVENTS = 11
WS_TUNE_DELAY_NS = 5
WS_TUNE_DELAY_P16 = 6
WS_TUNE_DELAY_SEED = 7
WS_TUNE_PREFETCH = 10


class WsConfig(C.Structure):
    _fields_ = [
        ("design", C.c_int32), ("bucket_size", C.c_int32),
        ("capacity_slots", C.c_uint64), ("front_buckets", C.c_uint64),
        ("seeds", C.c_uint64 * 8), ("n_seeds", C.c_int32),
        ("shortcut_slots", C.c_int32), ("zero_count_cap", C.c_int32),
        ("probe_cap", C.c_int32), ("ways", C.c_int32), ("path_depth", C.c_int32),
        ("phased", C.c_int32), ("line_bytes", C.c_int32), ("multi_stream", C.c_int32),
        ("chain_pool_nodes", C.c_uint64),
    ]


class WsInfo(C.Structure):
    _fields_ = [
        ("capacity_slots", C.c_uint64), ("num_buckets", C.c_uint64),
        ("primary_buckets", C.c_uint64), ("slot_bytes", C.c_uint64),
        ("tag_bytes", C.c_uint64), ("lock_bytes", C.c_uint64), ("node_bytes", C.c_uint64),
        ("next_node", C.c_uint64), ("pool_nodes", C.c_uint64),
        ("tombstones_ever", C.c_int32), ("device", C.c_int32),
    ]


_lock = threading.Lock()
_lib = None


def load():
    """Load (never build) the library; raise loudly when it is absent."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"libwarpspeed.so not found at {LIB_PATH}; build it with "
                "`python -c 'import __graft_entry__ as g; g.build()'` (nvcc, sm_100a)")
        lib = C.CDLL(LIB_PATH)
        vp, u64, i32, u32 = C.c_void_p, C.c_uint64, C.c_int, C.c_uint32
        lib.ws_create.argtypes = [C.POINTER(WsConfig), i32, C.POINTER(vp)]
        lib.ws_destroy.argtypes = [vp]
        lib.ws_clear.argtypes = [vp, vp]
        lib.ws_upsert.argtypes = [vp, vp, vp, u64, u32, vp, vp, u32]
        lib.ws_query.argtypes = [vp, vp, u64, vp, vp, vp, u32]
        lib.ws_erase.argtypes = [vp, vp, u64, vp, vp, u32]
        lib.ws_mixed.argtypes = [vp, vp, vp, vp, u64, vp, vp, vp, u32]
        lib.ws_locate.argtypes = [vp, vp, u64, vp, vp]
        lib.ws_probe_counts.argtypes = [vp, vp, vp, vp, u64, vp, vp, vp, C.POINTER(u64), vp, u32]
        lib.ws_occupied.argtypes = [vp, C.POINTER(u64), vp]
        lib.ws_export_items.argtypes = [vp, vp, vp, u64, C.POINTER(u64), vp]
        lib.ws_duplicate_scan.argtypes = [vp, vp, vp, u64, C.POINTER(u64), vp]
        lib.ws_checksum.argtypes = [vp, C.POINTER(u64 * 4), vp]
        lib.ws_export_raw.argtypes = [vp, vp, u64, vp, vp]
        lib.ws_read_range.argtypes = [vp, u64, u64, vp, u64, u64, vp, vp]
        lib.ws_info.argtypes = [vp, C.POINTER(WsInfo)]
        lib.ws_tune.argtypes = [vp, i32, i32]
        lib.ws_kernel_times.argtypes = [vp, vp, u64, C.POINTER(u64)]
        lib.ws_partition.argtypes = [vp, vp, vp, u64, u64, i32, vp, vp, vp, vp, vp, vp]
        lib.ws_unpermute.argtypes = [vp, vp, u64, i32, vp, vp]
        lib.ws_xchg_create.argtypes = [i32, i32, u64, i32, C.POINTER(vp)]
        lib.ws_xchg_handle.argtypes = [vp, vp]
        lib.ws_xchg_open.argtypes = [vp, vp]
        lib.ws_xchg_run.argtypes = [vp, vp, vp, C.c_uint8, vp, vp, u64, u64, u64, vp, vp, vp, u32]
        lib.ws_xchg_destroy.argtypes = [vp]
        lib.ws_strerror.argtypes = [i32]
        lib.ws_strerror.restype = C.c_char_p
        for name in EXPORTS:
            if name != "ws_strerror":
                getattr(lib, name).restype = i32
        _lib = lib
        return lib


def symbols():
    """Names of the C-ABI entry points the library actually exports."""
    lib = load()
    return [n for n in EXPORTS if hasattr(lib, n)]


def strerror(code: int) -> str:
    return load().ws_strerror(code).decode()

"""ctypes wrapper around oracle/ws_oracle.c (TEST INFRASTRUCTURE ONLY).

OracleTable mirrors the reference HashTable's scalar surface
(upsert/query/erase/slot_of/items/duplicate_scan, reference
tables/base.py:111-162) plus numpy batch drivers that apply ops in index
order.  It is the checker that the CUDA path is compared against.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "libws_oracle.so")
_LOCK = threading.Lock()
_LIB = None

MERGE_ID = {None: 0, "replace": 0, "keep": 1, "add": 2, "max": 3, "min": 4}


class _Params(C.Structure):
    _fields_ = [
        ("design", C.c_int32), ("bucket_size", C.c_int32),
        ("capacity_slots", C.c_uint64), ("front_buckets", C.c_uint64),
        ("seeds", C.c_uint64 * 8), ("n_seeds", C.c_int32),
        ("shortcut_slots", C.c_int32), ("zero_count_cap", C.c_int32),
        ("probe_cap", C.c_int32), ("ways", C.c_int32), ("path_depth", C.c_int32),
        ("phased", C.c_int32), ("line_bytes", C.c_int32),
    ]


def build_oracle(force: bool = False) -> str:
    """Compile ws_oracle.c with gcc into oracle/_build (idempotent)."""
    src = os.path.join(_HERE, "ws_oracle.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        os.makedirs(os.path.dirname(_SO), exist_ok=True)
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-o", _SO, src])
    return _SO


def load_oracle():
    global _LIB
    with _LOCK:
        if _LIB is not None:
            return _LIB
        if not os.path.exists(_SO):
            build_oracle()
        lib = C.CDLL(_SO)
        u64, u8p, u64p = C.c_uint64, C.POINTER(C.c_uint8), C.POINTER(C.c_uint64)
        lib.orc_create.restype = C.c_void_p
        lib.orc_create.argtypes = [C.POINTER(_Params)]
        lib.orc_destroy.argtypes = [C.c_void_p]
        lib.orc_upsert.argtypes = [C.c_void_p, u64, u64, C.c_int]
        lib.orc_query.argtypes = [C.c_void_p, u64, u64p]
        lib.orc_erase.argtypes = [C.c_void_p, u64]
        lib.orc_slot_of.restype = C.c_int64
        lib.orc_slot_of.argtypes = [C.c_void_p, u64]
        lib.orc_primary_bucket.restype = u64
        lib.orc_primary_bucket.argtypes = [C.c_void_p, u64]
        lib.orc_upsert_n.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, u64, C.c_int, C.c_void_p]
        lib.orc_query_n.argtypes = [C.c_void_p, C.c_void_p, u64, C.c_void_p, C.c_void_p]
        lib.orc_erase_n.argtypes = [C.c_void_p, C.c_void_p, u64, C.c_void_p]
        lib.orc_mixed_n.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, u64,
                                    C.c_void_p, C.c_void_p]
        lib.orc_set_probe_sink.argtypes = [C.c_void_p, C.c_void_p, u64]
        lib.orc_lock_touches.restype = u64
        lib.orc_lock_touches.argtypes = [C.c_void_p]
        lib.orc_probe_saturated.argtypes = [C.c_void_p]
        lib.orc_items.restype = u64
        lib.orc_items.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, u64]
        lib.orc_occupied.restype = u64
        lib.orc_occupied.argtypes = [C.c_void_p]
        lib.orc_data_words.restype = u64
        lib.orc_data_words.argtypes = [C.c_void_p]
        lib.orc_export_words.argtypes = [C.c_void_p, C.c_void_p]
        lib.orc_export_tags.argtypes = [C.c_void_p, C.c_void_p]
        lib.orc_next_node.restype = u64
        lib.orc_next_node.argtypes = [C.c_void_p]
        lib.orc_arena_capacity.restype = u64
        lib.orc_arena_capacity.argtypes = [C.c_void_p]
        lib.orc_tombstones_ever.argtypes = [C.c_void_p]
        del u8p
        _LIB = lib
        return lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class OracleTable:
    """Sequential CPU table with the reference's exact placement."""

    def __init__(self, config):
        from paper_2509_16407_b200.core import derive, validate_config
        self.config = validate_config(config)
        d = derive(self.config)
        self.derived = d
        self.capacity_slots = self.config.capacity_slots
        self.bucket_size = d.bucket_size
        p = _Params()
        p.design = d.design_id
        p.bucket_size = d.bucket_size
        p.capacity_slots = self.config.capacity_slots
        p.front_buckets = d.front_buckets
        for i, s in enumerate(d.seeds[:8]):
            p.seeds[i] = s
        p.n_seeds = min(8, len(d.seeds))
        p.shortcut_slots = d.shortcut_slots
        p.zero_count_cap = d.zero_count_cap
        p.probe_cap = d.probe_cap
        p.ways = d.ways
        p.path_depth = d.path_depth
        p.phased = int(d.phased)
        p.line_bytes = self.config.line_bytes
        self._lib = load_oracle()
        self._h = self._lib.orc_create(C.byref(p))

    def __del__(self):
        h, self._h = getattr(self, "_h", None), None
        if h:
            self._lib.orc_destroy(h)

    # -- scalar surface ---------------------------------------------------
    def upsert(self, key, value, merge=None):
        return self._lib.orc_upsert(self._h, key, value, MERGE_ID[merge])

    def query(self, key):
        v = C.c_uint64()
        return v.value if self._lib.orc_query(self._h, key, C.byref(v)) == 1 else None

    def erase(self, key):
        return self._lib.orc_erase(self._h, key) == 1

    def slot_of(self, key):
        i = self._lib.orc_slot_of(self._h, key)
        return None if i < 0 else int(i)

    def primary_bucket(self, key):
        return int(self._lib.orc_primary_bucket(self._h, key))

    # -- batch drivers (index order) -------------------------------------
    def upsert_batch(self, keys, values, merge=None, probes=None):
        keys = np.ascontiguousarray(keys, dtype=np.uint64)
        values = np.ascontiguousarray(values, dtype=np.uint64)
        st = np.empty(len(keys), dtype=np.uint8)
        self._sink(probes)
        self._lib.orc_upsert_n(self._h, _ptr(keys), _ptr(values), len(keys),
                               MERGE_ID[merge], _ptr(st))
        self._sink(None)
        return st

    def query_batch(self, keys, probes=None):
        keys = np.ascontiguousarray(keys, dtype=np.uint64)
        vals = np.empty(len(keys), dtype=np.uint64)
        found = np.empty(len(keys), dtype=np.uint8)
        self._sink(probes)
        self._lib.orc_query_n(self._h, _ptr(keys), len(keys), _ptr(vals), _ptr(found))
        self._sink(None)
        return found.astype(bool), vals

    def erase_batch(self, keys, probes=None):
        keys = np.ascontiguousarray(keys, dtype=np.uint64)
        found = np.empty(len(keys), dtype=np.uint8)
        self._sink(probes)
        self._lib.orc_erase_n(self._h, _ptr(keys), len(keys), _ptr(found))
        self._sink(None)
        return found.astype(bool)

    def mixed_batch(self, ops, keys, values, probes=None):
        ops = np.ascontiguousarray(ops, dtype=np.uint8)
        keys = np.ascontiguousarray(keys, dtype=np.uint64)
        values = np.ascontiguousarray(values, dtype=np.uint64)
        st = np.empty(len(keys), dtype=np.uint8)
        out = np.empty(len(keys), dtype=np.uint64)
        self._sink(probes)
        self._lib.orc_mixed_n(self._h, _ptr(ops), _ptr(keys), _ptr(values), len(keys),
                              _ptr(st), _ptr(out))
        self._sink(None)
        return st, out

    def _sink(self, probes):
        self._probe_keep = probes
        if probes is None:
            self._lib.orc_set_probe_sink(self._h, None, 0)
        else:
            assert probes.dtype == np.uint32 and probes.flags.c_contiguous
            self._lib.orc_set_probe_sink(self._h, _ptr(probes), len(probes))

    # -- introspection ---------------------------------------------------
    def items_arrays(self):
        n = int(self._lib.orc_occupied(self._h))
        k = np.empty(n, dtype=np.uint64)
        v = np.empty(n, dtype=np.uint64)
        self._lib.orc_items(self._h, _ptr(k), _ptr(v), n)
        return k, v

    def items(self):
        k, v = self.items_arrays()
        return zip(k.tolist(), v.tolist())

    def as_dict(self):
        k, v = self.items_arrays()
        return dict(zip(k.tolist(), v.tolist()))

    def duplicate_scan(self):
        k, _ = self.items_arrays()
        u, c = np.unique(k, return_counts=True)
        return {int(a): int(b) for a, b in zip(u[c > 1], c[c > 1])}

    def occupied_count(self):
        return int(self._lib.orc_occupied(self._h))

    def words(self):
        n = int(self._lib.orc_data_words(self._h))
        out = np.empty(n, dtype=np.uint64)
        self._lib.orc_export_words(self._h, _ptr(out))
        return out

    def slot_keys(self):
        return self.words()[0::2].copy()

    def tags(self):
        out = np.empty(self.capacity_slots, dtype=np.uint16)
        self._lib.orc_export_tags(self._h, _ptr(out))
        return out

    @property
    def next_node(self):
        return int(self._lib.orc_next_node(self._h))

    @property
    def arena_capacity(self):
        return int(self._lib.orc_arena_capacity(self._h))

    @property
    def lock_touches(self):
        return int(self._lib.orc_lock_touches(self._h))

    @property
    def tombstones_ever(self):
        return bool(self._lib.orc_tombstones_ever(self._h))

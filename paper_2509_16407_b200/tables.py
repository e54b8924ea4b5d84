"""Drop-in table surface backed by the sm_100a kernels.

``make_table(TableConfig) -> HashTable`` and the HashTable methods keep the
reference's names, arguments, return values and exceptions
(reference tables/__init__.py:30-35, tables/base.py:102-198 and the
design-specific helpers of tables/openaddr.py, cuckoo.py, chaining.py), so the
reference's own tests and harness run unchanged against it.  Every operation
executes on the GPU through libwarpspeed.so (include/warpspeed.h); there is no
CPU fallback -- constructing a table without the library or a CUDA device
raises.

Two call styles:

* scalar  ``upsert(key, value, merge=None)`` / ``query(key)`` / ``erase(key)``:
  a batch of one, synchronous, exactly the reference's sequential semantics;
* batched ``upsert_batch`` / ``query_batch`` / ``erase_batch`` /
  ``mixed_batch`` on torch tensors (or numpy arrays): one kernel launch on the
  current CUDA stream, every op concurrent and linearizable.
"""

from __future__ import annotations

import ctypes as C
import enum
import weakref

import numpy as np

from . import _native
from .core import (
    DEFAULT_BUCKET_SIZE,
    SLOT_BYTES,
    TableConfig,
    InvalidKeyError,
    ConfigError,
    check_key,
    check_value,
    derive,
    fingerprint,
    mix64,
    resolve_slot_engine,
    validate_config,
)

U64 = (1 << 64) - 1
TAG_REGION_BASE = 1 << 44
LOCK_REGION_BASE = 1 << 45


class UpsertStatus(enum.Enum):
    INSERTED = "inserted"
    UPDATED = "updated"
    FULL = "full"


_STATUS = (UpsertStatus.INSERTED, UpsertStatus.UPDATED, UpsertStatus.FULL)

MERGE_REPLACE, MERGE_KEEP, MERGE_ADD, MERGE_MAX, MERGE_MIN = range(5)
OP_UPSERT, OP_ERASE, OP_QUERY = range(3)
_MERGE_NAMES = {"replace": MERGE_REPLACE, "keep": MERGE_KEEP, "add": MERGE_ADD,
                "max": MERGE_MAX, "min": MERGE_MIN}
_MERGE_REF = (
    lambda o, n: n,
    lambda o, n: o,
    lambda o, n: (o + n) & U64,
    max,
    min,
)
_PROBE_PAIRS = ((5, 3), (3, 5), (0, 7), (7, 0), (U64, 2), (2, U64), (1 << 63, (1 << 63) + 5),
                (123456789, 987654321), (U64, U64), (0, 0), (1, 1), (U64, 1), (1, U64),
                (1 << 32, (1 << 32) - 1), ((1 << 32) - 1, 1 << 32)) + tuple(
    (int(a), int(b)) for a, b in
    np.random.default_rng(0x6D65726765).integers(0, 1 << 64, size=(48, 2), dtype=np.uint64))
_merge_cache: dict = {}


def merge_id(merge) -> int:
    """Map a reference-style merge callback to the device merge enum.

    None -> REPLACE (reference tables/base.py:48-49,124).  Strings and ints
    name the enum directly.  A callable is classified by evaluating it on
    probe pairs (results masked to 64 bits as reference openaddr.py:200 does);
    anything that is not replace / keep / add / max / min raises TypeError --
    arbitrary Python callbacks cannot run on the device and there is no CPU
    fallback.
    """
    if merge is None:
        return MERGE_REPLACE
    if isinstance(merge, str):
        try:
            return _MERGE_NAMES[merge]
        except KeyError:
            raise TypeError(f"unknown merge {merge!r}") from None
    if isinstance(merge, (int, np.integer)) and not isinstance(merge, bool):
        if 0 <= int(merge) <= MERGE_MIN:
            return int(merge)
        raise TypeError(f"unknown merge id {merge!r}")
    key = id(merge)
    hit = _merge_cache.get(key)
    if hit is not None and hit[0] is merge:
        return hit[1]
    try:
        got = [int(merge(a, b)) & U64 for a, b in _PROBE_PAIRS]
    except Exception as exc:  # noqa: BLE001
        raise TypeError(f"merge callable {merge!r} failed on probe inputs: {exc}") from exc
    for mid, ref in enumerate(_MERGE_REF):
        if all(g == ref(a, b) for g, (a, b) in zip(got, _PROBE_PAIRS)):
            if len(_merge_cache) > 4096:  # callables created per call must not pile up
                _merge_cache.clear()
            _merge_cache[key] = (merge, mid)
            return mid
    raise TypeError(f"merge callable {merge!r} is not one of replace/keep/add/max/min; "
                    "the device supports only these commutative-or-ordered integer merges")


def _torch():
    import torch
    return torch


def _as_u64(x, torch):
    """numpy/torch/list -> (contiguous tensor-or-array, data pointer, on_cuda)."""
    if isinstance(x, torch.Tensor):
        if x.dtype not in (torch.uint64, torch.int64):
            raise TypeError(f"keys/values must be 64-bit integer tensors, got {x.dtype}")
        x = x.contiguous()
        return x, x.data_ptr(), x.is_cuda
    a = np.ascontiguousarray(np.asarray(x, dtype=np.uint64))
    return a, a.ctypes.data, False


def _as_u8(x, torch):
    if isinstance(x, torch.Tensor):
        if x.dtype != torch.uint8:
            raise TypeError("op bytes must be a uint8 tensor")
        x = x.contiguous()
        return x, x.data_ptr(), x.is_cuda
    a = np.ascontiguousarray(np.asarray(x, dtype=np.uint8))
    return a, a.ctypes.data, False


def as_bool(t):
    """0/1 uint8 flags as a bool tensor without a conversion pass (zero-copy view)."""
    import torch
    return t.view(torch.bool) if t.dtype == torch.uint8 else t.bool()


def _checked_out(t, n, dtype):
    if t.numel() != n or not t.is_contiguous() or t.element_size() != dtype.itemsize:
        raise ValueError(f"out tensor must be contiguous with {n} elements of {dtype}")
    return t


class _Slots:
    """Read-only view of the device slot cells (quiescent test introspection,
    mirrors reference sync.py WideSlotArray accessors).  Each accessor reads
    only the cells it covers (ws_read_range), never the whole table."""

    def __init__(self, table):
        self._t = weakref.ref(table)

    def _words(self, lo, hi):
        """Cell words of slots [lo, hi) as uint64[2 * (hi - lo)]."""
        return self._t()._read_words(2 * lo, 2 * (hi - lo))

    def __len__(self):
        return self._t().capacity_slots

    def key_at(self, i):
        return int(self._words(i, i + 1)[0])

    def snapshot(self, i):
        w = self._words(i, i + 1)
        return int(w[0]), int(w[1])

    def find_free(self, lo, hi):
        keys = self._words(lo, hi)[0::2]
        for j, k in enumerate(keys.tolist()):
            if k == 0:
                return lo + j, True
            if k == U64:
                return lo + j, False
        return -1, False

    def used_count(self, lo, hi):
        keys = self._words(lo, hi)[0::2]
        return int(((keys != 0) & (keys != np.uint64(U64))).sum())

    def iter_occupied(self, lo, hi):
        w = self._words(lo, hi)
        for j in range(hi - lo):
            k = int(w[2 * j])
            if k != 0 and k < U64 - 1:
                yield lo + j, k, int(w[2 * j + 1])


class _Tags:
    def __init__(self, table):
        self._t = weakref.ref(table)

    def get(self, i):
        return int(self._t()._read_tags(i, 1)[0])


class _Arena:
    """Chaining node arena view (reference chaining.py:32-101)."""

    def __init__(self, table):
        self._t = weakref.ref(table)

    @property
    def next_node(self):
        return self._t()._info().next_node

    @property
    def capacity_nodes(self):
        return self._t()._logical_pool()

    @property
    def pairs(self):
        return self._t().bucket_size


class _Locks:
    def __init__(self, nb):
        self.bits = bytearray((nb + 7) >> 3)  # size of the reference's bit array (storage accounting)
        self.num_buckets = nb


class HashTable:
    """Base of the device-backed designs (reference tables/base.py:52-216)."""

    stable = True
    design = "?"

    def __init__(self, config: TableConfig, device=None, multi_stream: bool = False,
                 chain_pool_nodes: int = 0):
        torch = _torch()
        cfg = validate_config(config)
        self.config = cfg
        self.family = cfg.hash_family()
        self.capacity_slots = cfg.capacity_slots
        self.bucket_size = cfg.bucket_size
        self.line_bytes = cfg.line_bytes
        self.phased = cfg.mode == "phased"
        self.slot_engine = resolve_slot_engine(cfg)
        self.hook = None  # accepted for API compatibility; device delays are a build flag
        self._d = derive(cfg)
        self._num_buckets = self._d.num_buckets
        self.locks = _Locks(self._num_buckets)
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2509_16407_b200 tables need a CUDA device (sm_100a); "
                               "there is no CPU fallback")
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None
                                   else torch.device(device).index or 0)
        lib = _native.load()
        c = _native.WsConfig()
        c.design = self._d.design_id
        c.bucket_size = cfg.bucket_size
        c.capacity_slots = cfg.capacity_slots
        c.front_buckets = self._d.front_buckets
        for i, s in enumerate(self._d.seeds[:8]):
            c.seeds[i] = s
        c.n_seeds = min(8, len(self._d.seeds))
        c.shortcut_slots = self._d.shortcut_slots
        c.zero_count_cap = self._d.zero_count_cap
        c.probe_cap = self._d.probe_cap
        c.ways = self._d.ways
        c.path_depth = self._d.path_depth
        c.phased = int(self._d.phased)
        c.line_bytes = cfg.line_bytes
        c.multi_stream = int(bool(multi_stream))
        c.chain_pool_nodes = chain_pool_nodes
        if self._d.ways > 8:
            raise ConfigError([f"cuckoo_ways {self._d.ways} exceeds the device limit of 8"])
        h = C.c_void_p()
        with torch.cuda.device(self.device):
            rc = lib.ws_create(C.byref(c), self.device.index, C.byref(h))
        if rc != _native.WS_OK:
            raise RuntimeError(f"ws_create failed: {_native.strerror(rc)}")
        self._lib = lib
        self._h = h
        self._raw_cache = None
        self._finalizer = weakref.finalize(self, lib.ws_destroy, h)

    # ------------------------------------------------------------ plumbing
    def _stream(self):
        return _torch().cuda.current_stream(self.device).cuda_stream

    def _check(self, rc):
        if rc == _native.WS_OK:
            return
        if rc == _native.WS_ERR_INVALID_KEY:
            raise InvalidKeyError("batch contains a reserved sentinel key (0, 2^64-1 or 2^64-2)")
        if rc == _native.WS_ERR_INVALID_OP:
            raise ValueError(_native.strerror(rc))
        raise RuntimeError(f"libwarpspeed: {_native.strerror(rc)}")

    def _dirty(self):
        self._raw_cache = None

    def _raw(self):
        """Whole cell array and tag array on the host (test introspection of
        small tables only: 18 B per slot are copied)."""
        if self._raw_cache is None:
            nwords = self._info().node_bytes // 8 if self.design == "chaining" else 2 * self.capacity_slots
            words = np.empty(nwords, dtype=np.uint64)
            tags = np.empty(self.capacity_slots, dtype=np.uint16)
            self._check(self._lib.ws_export_raw(self._h, words.ctypes.data, nwords,
                                                tags.ctypes.data, self._stream()))
            self._raw_cache = (words, tags)
        return self._raw_cache

    def _read_words(self, first, n):
        out = np.empty(n, dtype=np.uint64)
        self._check(self._lib.ws_read_range(self._h, first, n, out.ctypes.data, 0, 0, None,
                                            self._stream()))
        return out

    def _read_tags(self, first, n):
        out = np.empty(n, dtype=np.uint16)
        self._check(self._lib.ws_read_range(self._h, 0, 0, None, first, n, out.ctypes.data,
                                            self._stream()))
        return out

    def _info(self):
        info = _native.WsInfo()
        self._check(self._lib.ws_info(self._h, C.byref(info)))
        return info

    @property
    def _tombstones_ever(self):
        return bool(self._info().tombstones_ever)

    # -------------------------------------------------------- public surface
    # the reference's per-table hash seeds (tables/openaddr.py, cuckoo.py:
    # self._s0 / _s1 / _s2 = family.seeds[0..2]), read by its tests
    @property
    def _s0(self):
        return self.family.seeds[0]

    @property
    def _s1(self):
        return self.family.seeds[1]

    @property
    def _s2(self):
        return self.family.seeds[2]

    @property
    def num_buckets(self):
        return self._num_buckets

    @property
    def primary_bucket_count(self):
        return self._d.primary_buckets

    def primary_bucket(self, key):
        check_key(key)
        return self._primary_bucket(key)

    def _primary_bucket(self, key):
        return (mix64(key ^ self.family.seeds[0]) >> 16) % self._num_buckets

    def _tag_of(self, key):
        return fingerprint(self.family, key)

    def upsert(self, key, value, merge=None, probe=None):
        """Insert (key, value) or merge into the existing value; returns
        INSERTED / UPDATED / FULL (reference tables/base.py:115-124)."""
        check_key(key)
        check_value(value)
        m = merge_id(merge)
        if probe is not None:
            st, _v = self._probed(OP_UPSERT | (m << 4), key, value, probe)
            return _STATUS[st]
        # per-call host scratch: scalar ops may be issued from many threads at
        # once (reference tables/base.py:5-7); ctypes drops the GIL in the call
        kv = np.array((key, value), dtype=np.uint64)
        s1 = np.zeros(1, dtype=np.uint8)
        self._dirty()
        self._check(self._lib.ws_upsert(self._h, kv.ctypes.data, kv.ctypes.data + 8, 1, m,
                                        s1.ctypes.data, self._stream(), _native.WS_F_NO_CHECK))
        return _STATUS[int(s1[0])]

    def query(self, key, probe=None):
        check_key(key)
        if probe is not None:
            found, v = self._probed(OP_QUERY, key, 0, probe)
            return v if found else None
        kv = np.array((key, 0), dtype=np.uint64)
        s1 = np.zeros(1, dtype=np.uint8)
        self._check(self._lib.ws_query(self._h, kv.ctypes.data, 1, kv.ctypes.data + 8,
                                       s1.ctypes.data, self._stream(), _native.WS_F_NO_CHECK))
        return int(kv[1]) if s1[0] else None

    def erase(self, key, probe=None):
        check_key(key)
        if probe is not None:
            found, _v = self._probed(OP_ERASE, key, 0, probe)
            return bool(found)
        k1 = np.array((key,), dtype=np.uint64)
        s1 = np.zeros(1, dtype=np.uint8)
        self._dirty()
        self._check(self._lib.ws_erase(self._h, k1.ctypes.data, 1, s1.ctypes.data,
                                       self._stream(), _native.WS_F_NO_CHECK))
        return bool(s1[0])

    def _probed(self, op, key, value, probe):
        """Run one op through the instrumented kernel and replay its probe
        counts into a reference-style ProbeRecorder (instrument.py:26-85)."""
        self._dirty()
        ops = np.array([op], dtype=np.uint8)
        keys = np.array([key], dtype=np.uint64)
        vals = np.array([value], dtype=np.uint64)
        st = np.zeros(1, dtype=np.uint8)
        vo = np.zeros(1, dtype=np.uint64)
        pr = np.zeros(1, dtype=np.uint32)
        locks = C.c_uint64()
        self._check(self._lib.ws_probe_counts(self._h, ops.ctypes.data, keys.ctypes.data,
                                              vals.ctypes.data, 1, st.ctypes.data,
                                              vo.ctypes.data, pr.ctypes.data, C.byref(locks),
                                              self._stream(), _native.WS_F_SERIAL))
        replay_probes(probe, int(pr[0]), int(locks.value), self.line_bytes)
        return int(st[0]), int(vo[0])

    def slot_of(self, key):
        check_key(key)
        k1 = np.array((key,), dtype=np.uint64)
        out = np.zeros(1, dtype=np.int64)
        self._check(self._lib.ws_locate(self._h, k1.ctypes.data, 1, out.ctypes.data,
                                        self._stream()))
        return None if out[0] < 0 else int(out[0])

    # ------------------------------------------------------------ batched
    def _out(self, like_cuda, n, dtype, torch):
        if like_cuda:
            return torch.empty(n, dtype=dtype, device=self.device)
        # host results land in pinned memory so the library's D2H copies are
        # true async DMA (torch caches pinned blocks across calls)
        return torch.empty(n, dtype=dtype, pin_memory=n >= (1 << 20))

    def upsert_batch(self, keys, values, merge=None, check=True, out=None, combine=False):
        """Concurrent upsert of a batch; returns a uint8 status tensor
        (0 INSERTED, 1 UPDATED, 2 FULL) on the keys' device (or `out`)."""
        torch = _torch()
        k, kp, kc = _as_u64(keys, torch)
        v, vp, _vc = _as_u64(values, torch)
        if len(v) != len(k):
            raise ValueError("keys and values differ in length")
        st = self._out(kc, len(k), torch.uint8, torch) if out is None else _checked_out(out, len(k), torch.uint8)
        self._dirty()
        fl = _native.WS_F_SYNC_CHECK if check else _native.WS_F_NO_CHECK
        if combine:
            fl |= _native.WS_F_COMBINE
        self._check(self._lib.ws_upsert(self._h, kp, vp, len(k), merge_id(merge), st.data_ptr(),
                                        self._stream(), fl))
        return st

    def query_batch(self, keys, check=True, out=None):
        """Lock-free concurrent lookups; returns (found bool, values uint64).
        `out` = (found uint8, values uint64) preallocated results."""
        torch = _torch()
        k, kp, kc = _as_u64(keys, torch)
        if out is None:
            found = self._out(kc, len(k), torch.uint8, torch)
            vals = self._out(kc, len(k), torch.uint64, torch)
        else:
            found = _checked_out(out[0], len(k), torch.uint8)
            vals = _checked_out(out[1], len(k), torch.uint64)
        fl = _native.WS_F_SYNC_CHECK if check else _native.WS_F_NO_CHECK
        self._check(self._lib.ws_query(self._h, kp, len(k), vals.data_ptr(), found.data_ptr(),
                                       self._stream(), fl))
        return as_bool(found), vals

    def erase_batch(self, keys, check=True):
        torch = _torch()
        k, kp, kc = _as_u64(keys, torch)
        found = self._out(kc, len(k), torch.uint8, torch)
        self._dirty()
        fl = _native.WS_F_SYNC_CHECK if check else _native.WS_F_NO_CHECK
        self._check(self._lib.ws_erase(self._h, kp, len(k), found.data_ptr(), self._stream(), fl))
        return as_bool(found)

    def mixed_batch(self, ops, keys, values=None, check=True, serial=False, combine=False, interleaved=False,
                    concurrent=False):
        """A concurrent batch of mixed ops (byte = kind | merge << 4, kind 0
        upsert / 1 erase / 2 query).  Returns (status uint8, values uint64):
        upsert status, erase/query found flag, query value.  Large batches run
        as per-kind segment launches, one after another; concurrent=True runs
        those segments concurrently on three streams (erases racing inserts
        and queries, tuned kernels); interleaved=True keeps all kinds in one
        generic launch (race tests that need kinds mixed inside a warp)."""
        torch = _torch()
        o, op, _oc = _as_u8(ops, torch)
        k, kp, kc = _as_u64(keys, torch)
        if values is None:
            values = torch.zeros(len(k), dtype=torch.uint64, device=self.device if kc else "cpu")
        v, vp, _vc = _as_u64(values, torch)
        st = self._out(kc, len(k), torch.uint8, torch)
        vo = self._out(kc, len(k), torch.uint64, torch)
        self._dirty()
        fl = _native.WS_F_SYNC_CHECK if check else _native.WS_F_NO_CHECK
        if serial:
            fl |= _native.WS_F_SERIAL
        if combine:
            fl |= _native.WS_F_COMBINE
        if interleaved:
            fl |= _native.WS_F_INTERLEAVED
        if concurrent:
            fl |= _native.WS_F_CONCURRENT_KINDS
        self._check(self._lib.ws_mixed(self._h, op, kp, vp, len(k), st.data_ptr(), vo.data_ptr(),
                                       self._stream(), fl))
        return st, vo

    def probe_batch(self, ops, keys, values=None, serial=True):
        """Instrumented mixed batch: (status, values, probes uint32, lock_touches).
        serial=True replays the ops in index order on one device thread."""
        o = np.ascontiguousarray(np.asarray(ops, dtype=np.uint8))
        k = np.ascontiguousarray(np.asarray(keys, dtype=np.uint64))
        v = (np.zeros(len(k), dtype=np.uint64) if values is None
             else np.ascontiguousarray(np.asarray(values, dtype=np.uint64)))
        st = np.zeros(len(k), dtype=np.uint8)
        vo = np.zeros(len(k), dtype=np.uint64)
        pr = np.zeros(len(k), dtype=np.uint32)
        locks = C.c_uint64()
        self._dirty()
        self._check(self._lib.ws_probe_counts(self._h, o.ctypes.data, k.ctypes.data, v.ctypes.data,
                                              len(k), st.ctypes.data, vo.ctypes.data,
                                              pr.ctypes.data, C.byref(locks), self._stream(),
                                              _native.WS_F_SERIAL if serial else 0))
        return st, vo, pr, int(locks.value)

    def locate_batch(self, keys):
        k = np.ascontiguousarray(np.asarray(keys, dtype=np.uint64))
        out = np.zeros(len(k), dtype=np.int64)
        self._check(self._lib.ws_locate(self._h, k.ctypes.data, len(k), out.ctypes.data,
                                        self._stream()))
        return out

    # ----------------------------------------------- quiescent introspection
    def items_arrays(self):
        """All live (key, value) pairs in slot order as numpy arrays."""
        n = C.c_uint64()
        self._check(self._lib.ws_export_items(self._h, None, None, 0, C.byref(n), self._stream()))
        cnt = int(n.value)
        k = np.empty(cnt, dtype=np.uint64)
        v = np.empty(cnt, dtype=np.uint64)
        if cnt:
            self._check(self._lib.ws_export_items(self._h, k.ctypes.data, v.ctypes.data, cnt,
                                                  C.byref(n), self._stream()))
        return k, v

    def items(self):
        k, v = self.items_arrays()
        return zip(k.tolist(), v.tolist())

    def duplicate_scan(self) -> dict:
        """{key: count} for every key stored more than once (reference
        tables/base.py:151-156); every duplicate is returned, however many."""
        n = C.c_uint64()
        cap = 1 << 16
        while True:
            dk = np.empty(cap, dtype=np.uint64)
            dc = np.empty(cap, dtype=np.uint64)
            self._check(self._lib.ws_duplicate_scan(self._h, dk.ctypes.data, dc.ctypes.data, cap,
                                                    C.byref(n), self._stream()))
            if int(n.value) <= cap:
                break
            cap = int(n.value)  # quiescent table: the second scan returns the same set
        m = int(n.value)
        return {int(a): int(b) for a, b in zip(dk[:m], dc[:m])}

    def duplicate_count(self) -> int:
        n = C.c_uint64()
        self._check(self._lib.ws_duplicate_scan(self._h, None, None, 0, C.byref(n), self._stream()))
        return int(n.value)

    def checksum(self):
        """(occupied, sum keys, sum values, xor of mix64(k ^ mix64(v))) mod 2^64."""
        out = (C.c_uint64 * 4)()
        self._check(self._lib.ws_checksum(self._h, C.byref(out), self._stream()))
        return tuple(int(x) for x in out)

    def occupied_count(self):
        n = C.c_uint64()
        self._check(self._lib.ws_occupied(self._h, C.byref(n), self._stream()))
        return int(n.value)

    def load_factor(self):
        return self.occupied_count() / self.capacity_slots

    def _storage_bytes(self):
        slots_b = SLOT_BYTES * self.capacity_slots
        tags_b = 2 * self.capacity_slots if self._d.md else 0
        return slots_b, tags_b, 0

    def storage_report(self):
        """Byte accounting of the reference's idealised image (base.py:167-189)."""
        occupied = self.occupied_count()
        slots_b, tags_b, nodes_b = self._storage_bytes()
        lock_b = len(self.locks.bits)
        table_b = slots_b + tags_b + nodes_b
        total_b = table_b + lock_b
        return {
            "occupied": occupied,
            "slot_bytes": slots_b,
            "tag_bytes": tags_b,
            "node_bytes": nodes_b,
            "lock_bytes": lock_b,
            "payload_bytes": SLOT_BYTES * occupied,
            "bytes_per_pair": (total_b / occupied) if occupied else float("inf"),
            "space_efficiency": (SLOT_BYTES * occupied / table_b) if table_b else 0.0,
        }

    def bytes_per_pair(self):
        return self.storage_report()["bytes_per_pair"]

    def capability_report(self):
        return {"slot_engine": self.slot_engine, "wide_atomic": True,
                "device": f"cuda:{self.device.index}", "arch": "sm_100a"}

    def tune(self, query_ilp=None, l2_policy=None, upsert=None, occupancy=None, prefetch=None):
        """Performance knobs of the tuned P2-MD path (no semantic effect).

        prefetch: L2 prefetch distance (grid-stride iterations) of the primary
        tag block in the tuned P2-MD upsert / query kernels, 0 = off."""
        if prefetch is not None:
            self._check(self._lib.ws_tune(self._h, _native.WS_TUNE_PREFETCH, int(prefetch)))
        if occupancy is not None:
            self._check(self._lib.ws_tune(self._h, _native.WS_TUNE_OCCUPANCY, int(occupancy)))
        if upsert is not None:
            self._check(self._lib.ws_tune(self._h, _native.WS_TUNE_UPSERT, int(upsert)))
        if query_ilp is not None:
            self._check(self._lib.ws_tune(self._h, _native.WS_TUNE_QUERY_ILP, int(query_ilp)))
        if l2_policy is not None:
            self._check(self._lib.ws_tune(self._h, _native.WS_TUNE_L2_POLICY, int(l2_policy)))

    def time_kernels(self, on=True):
        """Bracket every table-kernel launch with CUDA events on its stream
        (benchmark instrumentation); kernel_times() returns and clears them."""
        self._check(self._lib.ws_tune(self._h, _native.WS_TUNE_KERNEL_EVENTS, int(bool(on))))

    def kernel_times(self, cap=1 << 16):
        """Elapsed ms of each table-kernel launch since the last call, in
        launch order (waits for them; at most `cap` are returned)."""
        buf = np.zeros(cap, dtype=np.float32)
        n = C.c_uint64()
        self._check(self._lib.ws_kernel_times(self._h, buf.ctypes.data, cap, C.byref(n)))
        return buf[: min(int(n.value), cap)].tolist()

    def set_delays(self, max_ns=0, prob=0.0, seed=0):
        """Device delay injection at the reference's hook stages (race-window
        widening for adversarial tests; generic kernels only)."""
        self._check(self._lib.ws_tune(self._h, _native.WS_TUNE_DELAY_NS, int(max_ns)))
        self._check(self._lib.ws_tune(self._h, _native.WS_TUNE_DELAY_P16, int(round(prob * 65536))))
        self._check(self._lib.ws_tune(self._h, _native.WS_TUNE_DELAY_SEED, int(seed) & 0x7FFFFFFF))

    def clear(self):
        """Back to the freshly constructed state without reallocating
        (stream-ordered on the current CUDA stream)."""
        self._dirty()
        self._check(self._lib.ws_clear(self._h, self._stream()))

    def close(self):
        """Free the device table now (otherwise on garbage collection)."""
        self._finalizer()


def replay_probes(rec, count: int, lock_touches: int, line_bytes: int):
    """Feed a device op's (distinct lines, lock touches) into any recorder with
    the reference's touch / touch_lock interface, reproducing both counters."""
    if lock_touches:
        for _ in range(lock_touches):
            rec.touch_lock(LOCK_REGION_BASE)
        count -= 1
    base = 1 << 50
    for i in range(max(0, count)):
        rec.touch(base + i * line_bytes)


# ------------------------------------------------------------------ designs

class _BucketedTable(HashTable):
    md = False

    def _used_and_free(self, b, probe=None):
        """(used, has_free) of bucket b (reference openaddr.py:118-130)."""
        bs = self.bucket_size
        lo = b * bs
        if self.md:
            tags = self._read_tags(lo, bs)
            zeros = min(int((tags == 0).sum()), self._d.zero_count_cap)
            return bs - zeros, zeros > 0
        used = self.slots.used_count(lo, lo + bs)
        return used, used < bs

    @property
    def slots(self):
        return _Slots(self)

    @property
    def tags(self):
        return _Tags(self) if self.md else None


class DoubleTable(_BucketedTable):
    design = "double"

    def _step(self, key):
        return mix64(key ^ self.family.seeds[1]) | 1

    def probe_sequence(self, key):
        nb = self._num_buckets
        b = self._primary_bucket(key)
        step = self._step(key)
        for _ in range(min(self.config.probe_cap, nb)):
            yield b
            b = (b + step) % nb


class DoubleMdTable(DoubleTable):
    design = "double_md"
    md = True


class P2Table(_BucketedTable):
    design = "p2"

    def _alt_bucket(self, key):
        return (mix64(key ^ self.family.seeds[1]) >> 16) % self._num_buckets

    def _shortcut_slots(self):
        return self._d.shortcut_slots

    def route(self, key, probe=None):
        """Bucket an insert of key would target now, or -1 (openaddr.py:354-368)."""
        b0 = self._primary_bucket(key)
        used0, free0 = self._used_and_free(b0)
        if not self._tombstones_ever and used0 < self._shortcut_slots():
            return b0
        b1 = self._alt_bucket(key)
        if b1 == b0:
            return b0 if free0 else -1
        used1, free1 = self._used_and_free(b1)
        if free0 and (used0 <= used1 or not free1):
            return b0
        if free1:
            return b1
        return -1


class P2MdTable(P2Table):
    design = "p2_md"
    md = True


class UnsafeP2Table(P2Table):
    design = "unsafe_reference"
    lock_elided = True


class IcebergTable(_BucketedTable):
    design = "iceberg"

    @property
    def front_buckets(self):
        return self._d.front_buckets

    @property
    def back_buckets(self):
        return self._d.back_buckets

    def _primary_bucket(self, key):
        return (mix64(key ^ self.family.seeds[0]) >> 16) % self.front_buckets

    def _back_pair(self, key):
        fb, bb = self.front_buckets, self.back_buckets
        return (fb + ((mix64(key ^ self.family.seeds[1]) >> 16) % bb),
                fb + ((mix64(key ^ self.family.seeds[2]) >> 16) % bb))

    def route(self, key, probe=None):
        b0 = self._primary_bucket(key)
        _u0, free0 = self._used_and_free(b0)
        if free0:
            return "front", b0
        b1, b2 = self._back_pair(key)
        used1, free1 = self._used_and_free(b1)
        if b2 == b1:
            return ("back", b1) if free1 else ("full", -1)
        used2, free2 = self._used_and_free(b2)
        if free1 and (used1 <= used2 or not free2):
            return "back", b1
        if free2:
            return "back", b2
        return "full", -1


class IcebergMdTable(IcebergTable):
    design = "iceberg_md"
    md = True


class CuckooTable(_BucketedTable):
    design = "cuckoo"
    stable = False

    @property
    def ways(self):
        return self.config.cuckoo_ways

    def _buckets_of(self, key):
        nb = self._num_buckets
        return [(mix64(key ^ s) >> 16) % nb for s in self.family.seeds[:self.ways]]

    def _storage_bytes(self):
        return SLOT_BYTES * self.capacity_slots, 0, 0


class ChainingTable(HashTable):
    design = "chaining"

    @property
    def arena(self):
        return _Arena(self)

    def _logical_pool(self):
        """Node capacity the reference's 1.5x growth rule would have reached
        for the current allocation count (chaining.py:51-59)."""
        nxt = self._info().next_node
        cap = self._num_buckets + 1
        while cap < nxt:
            cap += max(64, cap >> 1)
        return cap

    def _storage_bytes(self):
        return 0, 0, self.line_bytes * self._logical_pool()

    def mean_chain_nodes(self):
        overflow = self._info().next_node - 1 - self._num_buckets
        return 1.0 + overflow / self._num_buckets


_DESIGN_CLASS = {
    "double": DoubleTable,
    "double_md": DoubleMdTable,
    "p2": P2Table,
    "p2_md": P2MdTable,
    "iceberg": IcebergTable,
    "iceberg_md": IcebergMdTable,
    "cuckoo": CuckooTable,
    "chaining": ChainingTable,
    "unsafe_reference": UnsafeP2Table,
}


def make_table(config: TableConfig, **kw) -> HashTable:
    """Construct the device table for config.design (reference
    tables/__init__.py:30-35)."""
    try:
        cls = _DESIGN_CLASS[config.design]
    except KeyError:
        raise ValueError(f"unknown design {config.design!r}") from None
    return cls(config, **kw)


__all__ = ["HashTable", "UpsertStatus", "make_table", "merge_id", "DEFAULT_BUCKET_SIZE",
           "DoubleTable", "DoubleMdTable", "P2Table", "P2MdTable", "IcebergTable",
           "IcebergMdTable", "CuckooTable", "ChainingTable", "UnsafeP2Table"]

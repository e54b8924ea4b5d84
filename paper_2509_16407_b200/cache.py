"""Table-fronted cache over a backing store, batched on the device
(reference apps/cache.py:1-144).

The reference drives one get() at a time from CPU threads: a lock-free
query, and on a miss a fetch from the backing dict, an insert-if-unique
upsert (KEEP), a FIFO ring append and, once the ring exceeds 85% of the
table, eviction of the oldest resident with write-back (query, store in the
backing dict, erase).  Here both the cache and the backing store are device
tables and a get is a batch:

  1. query_batch on the cache -> hits;
  2. the batch's distinct missing keys (first occurrence order) are fetched
     from the backing table and inserted with KEEP (insert-if-unique);
  3. they are appended to a device ring in that order; when the ring holds
     more than `capacity` keys the oldest are evicted: their cached values
     are written back to the backing table (REPLACE) and erased from the
     cache -- the same write-back-then-drop order as the reference
     (cache.py:82-88);
  4. a FULL insert (bucket saturation below the ring ceiling) evicts the
     oldest residents and retries, as cache.py:64-69 (in doubling chunks
     rather than one at a time, see get_batch).

Counting follows a serial replay of the batch in index order: the first
occurrence of a key missing from the cache is a miss, later occurrences in
the same batch are hits.  Evictions are applied at batch end, so with
batches much smaller than the ring the hit rate is the reference's
(uniform access: hit rate == cache-to-data ratio, cache.py:100-107).
Cuckoo is rejected up front like the reference (fused query-then-insert
needs referential stability, cache.py:10-12).
"""

from __future__ import annotations

import time

import numpy as np

from .core import TableConfig
from .workload import derive_seed, gen_uniform_keys


class CacheError(Exception):
    pass


def _torch():
    import torch
    return torch


class DeviceCacheSim:
    """Batched CacheSim (reference cache.py:32-97) over two device tables."""

    def __init__(self, table, backing, capacity=None):
        if not table.stable:
            raise CacheError(f"{table.design} is not stable and cannot run fused cache ops")
        torch = _torch()
        self.table = table
        self.backing = backing
        self.capacity = int(table.capacity_slots * 0.85) if capacity is None else int(capacity)
        self.dev = table.device
        # FIFO ring of resident keys (int64 view of uint64 keys)
        self._ring = torch.empty(self.capacity + 1, dtype=torch.int64, device=self.dev)
        self._head = 0  # index of the oldest resident
        self._size = 0
        self.hits = self.misses = self.evictions = 0
        self.full_events = 0

    # ------------------------------------------------------------ ring
    def _ring_push(self, k64):
        torch = _torch()
        n = int(k64.numel())
        cap = self._ring.numel()
        if self._size + n > cap:  # grow (only when one batch overfills before eviction)
            old = self._ring_order()
            self._ring = torch.empty(max(2 * cap, self._size + n + 1), dtype=torch.int64, device=self.dev)
            self._ring[: self._size] = old
            self._head = 0
            cap = self._ring.numel()
        tail = (self._head + self._size) % cap
        first = min(n, cap - tail)
        self._ring[tail:tail + first] = k64[:first]
        if first < n:
            self._ring[: n - first] = k64[first:]
        self._size += n

    def _ring_pop(self, m):
        torch = _torch()
        cap = self._ring.numel()
        first = min(m, cap - self._head)
        out = self._ring[self._head:self._head + first]
        if first < m:
            out = torch.cat([out, self._ring[: m - first]])
        else:
            out = out.clone()
        self._head = (self._head + m) % cap
        self._size -= m
        return out

    def _ring_order(self):
        torch = _torch()
        cap = self._ring.numel()
        idx = (torch.arange(self._size, device=self.dev) + self._head) % cap
        return self._ring[idx]

    def _evict(self, m):
        """Evict the m oldest residents: write back, then drop (cache.py:82-88)."""
        if m <= 0:
            return
        victims = self._ring_pop(m).view(_torch().uint64)
        found, vals = self.table.query_batch(victims, check=False)
        if not bool(found.all()):
            raise CacheError("a ring resident is missing from the cache table")
        self.backing.upsert_batch(victims, vals, None, check=False)
        gone = self.table.erase_batch(victims, check=False)
        if not bool(gone.all()):
            raise CacheError("eviction could not erase a resident")
        self.evictions += m

    # ------------------------------------------------------------- get
    def get_batch(self, keys):
        """Values for a batch of keys (uint64 tensor on the cache's device)."""
        torch = _torch()
        found, vals = self.table.query_batch(keys)
        f = found.bool()
        nmiss_ops = int((~f).sum())
        if nmiss_ops == 0:
            self.hits += keys.numel()
            return vals
        k64 = keys.view(torch.int64)
        miss_pos = torch.nonzero(~f).squeeze(1)
        mk = k64[miss_pos]
        # distinct missing keys in first-occurrence order
        uk, inv = torch.unique(mk, return_inverse=True)
        first = torch.full((uk.numel(),), mk.numel(), dtype=torch.int64, device=self.dev)
        first.scatter_reduce_(0, inv, torch.arange(mk.numel(), device=self.dev), reduce="amin")
        order = torch.argsort(first)
        new_keys = uk[order]
        nnew = int(new_keys.numel())
        bf, bv = self.backing.query_batch(new_keys.view(torch.uint64))
        if not bool(bf.all()):
            raise CacheError("key outside the cached universe")
        st = self.table.upsert_batch(new_keys.view(torch.uint64), bv, "keep")
        if bool((st == 1).any()):
            raise CacheError("a missing key was already cached (concurrent writer)")
        full = st == 2
        self._ring_push(new_keys[~full])
        pend, pend_v = new_keys[full], bv.view(torch.int64)[full]
        chunk = int(pend.numel())
        if chunk:
            self.full_events += 1
        while pend.numel():
            if self._size == 0:
                raise CacheError("cache table full with an empty ring")
            # bucket saturation: evict the oldest residents and retry
            # (cache.py:64-69 evicts one at a time until the insert fits; a
            # random eviction frees one of the key's buckets with probability
            # ~2/nb, so here the chunk doubles per failed retry: same FIFO
            # order, at most twice the minimal number of evictions)
            self._evict(min(self._size, chunk))
            chunk *= 2
            st2 = self.table.upsert_batch(pend.view(torch.uint64), pend_v.view(torch.uint64), "keep")
            ok = st2 != 2
            self._ring_push(pend[ok])
            pend, pend_v = pend[~ok], pend_v[~ok]
        if self._size > self.capacity:
            self._evict(self._size - self.capacity)
        self.misses += nnew
        self.hits += keys.numel() - nnew
        # every miss returns the fetched value
        out = vals.view(torch.int64).clone()
        bv64 = bv.view(torch.int64)
        rank = torch.empty_like(order)
        rank[order] = torch.arange(nnew, device=self.dev)
        out[miss_pos] = bv64[rank[inv]]
        return out.view(torch.uint64)

    def resident_keys(self):
        return set(self._ring_order().cpu().numpy().view(np.uint64).tolist())

    def check_conservation(self, universe) -> None:
        """Every key is reachable, and table contents mirror the ring (cache.py:93-105)."""
        table_keys = {k for k, _ in self.table.items()}
        ring = self.resident_keys()
        if table_keys != ring:
            raise AssertionError("table contents diverge from the ring queue")
        back = {k for k, _ in self.backing.items()}
        missing = set(int(x) for x in universe) - (table_keys | back)
        if missing:
            raise AssertionError(f"{len(missing)} keys lost from the system")
        if self.table.load_factor() > 0.85 + 1e-9:
            raise AssertionError("cache exceeded its 85% load ceiling")


def run_cache_sweep(universe: int = 1 << 20, ratios=(0.1, 0.25, 0.5, 0.75), queries_per_key: float = 4.0,
                    seed: int = 42, design: str = "p2_md", batch: int = 1 << 16) -> list:
    """Hit-rate sweep (reference cache.py:108-144): one fresh cache per
    cache-to-data ratio, ring sized to ratio * universe (table ratio / 0.85
    slots), pre-warmed with the first `capacity` keys, then a uniform stream
    of queries_per_key * universe gets from derive_seed(seed, ratio*1000).
    Every returned value is checked against the dataset."""
    torch = _torch()
    from .tables import make_table
    keys = gen_uniform_keys(seed, universe)
    values = keys & np.uint64(0xFFFFFFFF)
    dev = torch.device("cuda", torch.cuda.current_device())

    def d(a):
        return torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).to(dev).view(torch.uint64)

    back_cap = max(64, int(universe / 0.8)) // 32 * 32
    results = []
    for ratio in ratios:
        backing = make_table(TableConfig(design=design, capacity_slots=back_cap, seed=seed ^ 0xB))
        if int((backing.upsert_batch(d(keys), d(values)) != 0).sum()):
            raise CacheError("backing store preload failed")
        slots = max(64, int(universe * ratio / 0.85) + 2)
        slots = (slots + 31) // 32 * 32 if design != "chaining" else slots
        table = make_table(TableConfig(design=design, capacity_slots=slots, seed=seed))
        sim = DeviceCacheSim(table, backing, capacity=int(universe * ratio))
        # evictions happen at batch end: keep batches well below the ring so
        # the counting matches the reference's one-get-at-a-time replay
        bsz = max(1, min(batch, sim.capacity // 8))
        warm = keys[: sim.capacity]
        for lo in range(0, len(warm), bsz):
            sim.get_batch(d(warm[lo:lo + bsz]))
        sim.hits = sim.misses = sim.evictions = 0
        rng = np.random.default_rng(derive_seed(seed, int(ratio * 1000)))
        idx = rng.integers(0, universe, size=int(universe * queries_per_key))
        stream = d(keys[idx])
        want = values[idx]
        got = torch.empty_like(stream)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for lo in range(0, len(idx), bsz):
            got[lo:lo + bsz] = sim.get_batch(stream[lo:lo + bsz])
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        ok = bool((got.cpu().view(torch.int64).numpy().view(np.uint64) == want).all())
        total = sim.hits + sim.misses
        results.append({"ratio": ratio, "hit_rate": sim.hits / total if total else 0.0,
                        "mops": total / dt / 1e6 if dt else 0.0, "evictions": sim.evictions,
                        "full_events": sim.full_events,
                        "values_exact": ok, "batch": bsz})
    return results

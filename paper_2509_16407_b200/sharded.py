"""Hash-sharded table over the ranks of a torch.distributed process group.

One logical table of ``config.capacity_slots`` slots is split into one local
device table per rank (``capacity_slots / world`` slots each).  The owner of a
key is the top log2(world) bits of its primary hash ``mix64(k ^ seed0)``; the
local table indexes bucket bits 16..16+log2(nb), so owner and bucket are
independent.  The reference has no multi-GPU layer;
every batch op here is:

    exchange="nccl": partition by owner (ws_partition) -> all_to_all_single
    of the keys (+ values / op bytes) -> local batch op -> reverse
    all_to_all_single of the results -> scatter back (ws_unpermute)

    exchange="p2p": one routing kernel stores every op straight into its
    owner's inbox over NVLink peer memory (CUDA IPC), owners apply their
    inbox with the table kernels and store results straight back into the
    source's reply buffer (ws_xchg_run) -- no partition buffer, no
    collective call, no unpermute pass

Each rank passes its own batch; results come back for that batch.  With one
rank the exchange is skipped entirely.  The process group is the caller's
(NCCL over NVLink for device tensors; the CPU tests drive the same routing
logic over gloo with an injected CPU router and local table).
"""

from __future__ import annotations

import ctypes as C
import dataclasses

from .core import ConfigError, TableConfig, validate_config
from .tables import as_bool


class DeviceRouter:
    """Owner partition / result scatter on the GPU (libwarpspeed kernels)."""

    def __init__(self, seed0: int, log2_parts: int):
        from . import _native
        self._lib = _native.load()
        self.seed0 = seed0
        self.log2 = log2_parts

    def partition(self, keys, vals=None, ops=None):
        import torch
        n = keys.numel()
        if not keys.is_cuda:
            raise RuntimeError("sharded batches must be CUDA tensors")
        parts = 1 << self.log2
        ok = torch.empty_like(keys)
        ov = torch.empty_like(vals) if vals is not None else None
        oo = torch.empty_like(ops) if ops is not None else None
        perm = torch.empty(n, dtype=torch.int32, device=keys.device)
        counts = torch.empty(parts, dtype=torch.int64, device=keys.device)
        s = torch.cuda.current_stream(keys.device).cuda_stream
        rc = self._lib.ws_partition(keys.data_ptr(), vals.data_ptr() if vals is not None else None,
                                    ops.data_ptr() if ops is not None else None, n, self.seed0,
                                    self.log2, ok.data_ptr(), ov.data_ptr() if ov is not None else None,
                                    oo.data_ptr() if oo is not None else None, perm.data_ptr(),
                                    counts.data_ptr(), s)
        if rc:
            raise RuntimeError(f"ws_partition failed ({rc})")
        return ok, ov, oo, perm, counts

    def unpermute(self, res, perm):
        import torch
        out = torch.empty_like(res)
        s = torch.cuda.current_stream(res.device).cuda_stream
        rc = self._lib.ws_unpermute(res.data_ptr(), perm.data_ptr(), res.numel(), res.element_size(),
                                    out.data_ptr(), s)
        if rc:
            raise RuntimeError(f"ws_unpermute failed ({rc})")
        return out


class ShardedTable:
    """A table spread over all ranks of ``group``; batched ops only."""

    def __init__(self, config: TableConfig, group=None, local_table=None, router=None,
                 exchange: str = "nccl", chunk_ops: int = 1 << 24, **table_kw):
        import torch.distributed as dist
        cfg = validate_config(config)
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        if self.world & (self.world - 1):
            raise ConfigError([f"world size {self.world} is not a power of two"])
        self.log2 = self.world.bit_length() - 1
        if cfg.capacity_slots % (self.world * cfg.bucket_size):
            raise ConfigError([f"capacity_slots {cfg.capacity_slots} does not split into "
                               f"{self.world} shards of whole buckets"])
        self.config = cfg
        self.local_config = dataclasses.replace(cfg, capacity_slots=cfg.capacity_slots // self.world)
        if local_table is None:
            from .tables import make_table
            local_table = make_table(self.local_config, **table_kw)
        self.local = local_table
        self.seed0 = cfg.hash_family().seeds[0]
        self.router = router if router is not None else DeviceRouter(self.seed0, self.log2)
        if exchange not in ("nccl", "p2p"):
            raise ValueError("exchange must be 'nccl' (all_to_all) or 'p2p' (fused NVLink stores)")
        self.exchange = exchange
        self._xchg = None
        if exchange == "p2p" and self.world > 1:
            # collective decision: every rank must use the same exchange, so a
            # rank that cannot map its peers (no CUDA IPC / peer access) moves
            # the whole group to the NCCL all-to-all path
            err = None
            try:
                self._open_p2p(chunk_ops)
            except RuntimeError as e:  # noqa: PERF203
                err = e
            import torch
            flag = torch.tensor([0 if err is None else 1], dtype=torch.int64,
                                device="cpu" if self._host_staged() else self.local.device)
            dist.all_reduce(flag, op=dist.ReduceOp.MAX, group=self.group)
            if int(flag.item()):
                if self._xchg is not None:
                    self._xfin()
                    self._xchg = None
                self.exchange = "nccl"
                import warnings
                warnings.warn(f"p2p exchange unavailable on some rank ({err or 'peer failure'}); using nccl")

    # ------------------------------------------------- fused NVLink exchange
    def _open_p2p(self, chunk_ops):
        import torch
        import torch.distributed as dist
        from . import _native
        lib = _native.load()
        h = C.c_void_p()
        dev = self.local.device.index
        rc = lib.ws_xchg_create(self.world, self.rank, chunk_ops, dev, C.byref(h))
        if rc:
            raise RuntimeError(f"ws_xchg_create failed: {_native.strerror(rc)}")
        self._xlib, self._xchg, self._chunk = lib, h, chunk_ops
        import weakref
        self._xfin = weakref.finalize(self, lib.ws_xchg_destroy, h)
        mine = (C.c_char * 64)()
        if lib.ws_xchg_handle(h, mine):
            raise RuntimeError("ws_xchg_handle failed")
        handles = [None] * self.world
        dist.all_gather_object(handles, bytes(mine), group=self.group)
        blob = b"".join(handles)
        if lib.ws_xchg_open(h, blob):
            raise RuntimeError("ws_xchg_open failed (CUDA IPC / peer access)")
        del torch

    def _rounds(self, n):
        import torch
        import torch.distributed as dist
        dev = "cpu" if self._host_staged() else self.local.device
        t = torch.tensor([n], dtype=torch.int64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        return -(-int(t.item()) // self._chunk)

    def _p2p(self, keys, vals, ops, uop, want_vals, check, merge_flags=0):
        import torch
        from . import _native
        n = keys.numel()
        dev = keys.device
        status = torch.empty(n, dtype=torch.uint8, device=dev)
        vout = torch.empty(n, dtype=torch.uint64, device=dev) if want_vals else None
        fl = (_native.WS_F_SYNC_CHECK if check else _native.WS_F_NO_CHECK) | merge_flags
        rc = self._xlib.ws_xchg_run(self._xchg, self.local._h, ops.data_ptr() if ops is not None else None,
                                    uop, keys.data_ptr(), vals.data_ptr() if vals is not None else None, n,
                                    self._rounds(n), self.seed0, status.data_ptr(),
                                    vout.data_ptr() if vout is not None else None,
                                    torch.cuda.current_stream(dev).cuda_stream, fl)
        self.local._check(rc)
        return status, vout

    # --------------------------------------------------------------- exchange
    def _host_staged(self):
        # gloo (CPU tests, or several ranks sharing one GPU) exchanges host tensors
        import torch.distributed as dist
        return dist.get_backend(self.group) == "gloo"

    def _counts(self, send_counts):
        import torch
        import torch.distributed as dist
        src = send_counts.cpu() if self._host_staged() else send_counts
        recv = torch.empty_like(src)
        dist.all_to_all_single(recv, src, group=self.group)
        return recv.to(send_counts.device)

    def _a2a(self, t, recv_splits, send_splits):
        import torch
        import torch.distributed as dist
        view = t.view(torch.int64) if t.dtype == torch.uint64 else t
        dev = view.device
        if self._host_staged():
            view = view.cpu()
        out = torch.empty(sum(recv_splits), dtype=view.dtype, device=view.device)
        dist.all_to_all_single(out, view, recv_splits, send_splits, group=self.group)
        return out.to(dev).view(t.dtype)

    def _route(self, keys, vals=None, ops=None):
        pk, pv, po, perm, counts = self.router.partition(keys, vals, ops)
        rcounts = self._counts(counts)
        send = counts.cpu().tolist()
        recv = rcounts.cpu().tolist()
        rk = self._a2a(pk, recv, send)
        rv = self._a2a(pv, recv, send) if pv is not None else None
        ro = self._a2a(po, recv, send) if po is not None else None
        return rk, rv, ro, perm, send, recv

    def _back(self, res, perm, send, recv):
        out = self._a2a(res, send, recv)
        return self.router.unpermute(out, perm)

    # ------------------------------------------------------------ validation
    def _validate(self, keys, ops=None):
        """Group-wide batch check before any routing or mutation: every rank
        tests its own batch for sentinel keys (reference core.py:27-31,
        103-117) and bad op bytes, the verdicts are all-reduced, and if any
        rank's batch is invalid EVERY rank raises -- so no rank is left
        waiting in an exchange and no shard has been changed (the whole
        logical batch is rejected, as SPEC.md:89 asks of one table)."""
        import torch
        import torch.distributed as dist
        from .core import InvalidKeyError
        k = keys.view(torch.int64)
        code = 2 if bool(((k == 0) | (k == -1) | (k == -2)).any()) else 0
        if not code and ops is not None:
            o = ops.to(torch.int32)
            code = 1 if bool((((o & 15) > 2) | ((o >> 4) > 4)).any()) else 0
        flag = torch.tensor([code], dtype=torch.int64,
                            device="cpu" if self._host_staged() else self.local.device)
        dist.all_reduce(flag, op=dist.ReduceOp.MAX, group=self.group)
        code = int(flag.item())
        if code == 2:
            raise InvalidKeyError("a batch on some rank contains a reserved sentinel key "
                                  "(0, 2^64-1 or 2^64-2); the sharded batch was rejected on every rank")
        if code == 1:
            raise ValueError("a batch on some rank contains an invalid op byte (kind > 2 or merge > 4)")

    # ----------------------------------------------------------------- ops
    def upsert_batch(self, keys, values, merge=None, check=True):
        if self.world == 1:
            return self.local.upsert_batch(keys, values, merge=merge, check=check)
        if check:
            self._validate(keys)
            check = False
        if self._xchg is not None:
            from .tables import OP_UPSERT, merge_id
            return self._p2p(keys, values, None, OP_UPSERT | (merge_id(merge) << 4), False, check)[0]
        rk, rv, _ro, perm, send, recv = self._route(keys, values)
        st = self.local.upsert_batch(rk, rv, merge=merge, check=check)
        return self._back(st, perm, send, recv)

    def query_batch(self, keys, check=True):
        if self.world == 1:
            return self.local.query_batch(keys, check=check)
        if check:
            self._validate(keys)
            check = False
        if self._xchg is not None:
            from .tables import OP_QUERY
            st, vo = self._p2p(keys, None, None, OP_QUERY, True, check)
            return as_bool(st), vo
        rk, _rv, _ro, perm, send, recv = self._route(keys)
        found, vals = self.local.query_batch(rk, check=check)
        import torch
        found = self._back(found.to(torch.uint8), perm, send, recv)
        vals = self._back(vals, perm, send, recv)
        return as_bool(found), vals

    def erase_batch(self, keys, check=True):
        if self.world == 1:
            return self.local.erase_batch(keys, check=check)
        if check:
            self._validate(keys)
            check = False
        if self._xchg is not None:
            from .tables import OP_ERASE
            return as_bool(self._p2p(keys, None, None, OP_ERASE, False, check)[0])
        rk, _rv, _ro, perm, send, recv = self._route(keys)
        import torch
        found = self.local.erase_batch(rk, check=check)
        return as_bool(self._back(found.to(torch.uint8), perm, send, recv))

    def mixed_batch(self, ops, keys, values=None, check=True):
        import torch
        if values is None:
            values = torch.zeros(keys.numel(), dtype=keys.dtype, device=keys.device)
        if self.world == 1:
            return self.local.mixed_batch(ops, keys, values, check=check)
        if check:
            self._validate(keys, ops)
            check = False
        if self._xchg is not None:
            return self._p2p(keys, values, ops, 0, True, check)
        rk, rv, ro, perm, send, recv = self._route(keys, values, ops)
        st, vo = self.local.mixed_batch(ro, rk, rv, check=check)
        return self._back(st, perm, send, recv), self._back(vo, perm, send, recv)

    # --------------------------------------------------- collective summaries
    def _gather(self, vals):
        import torch
        import torch.distributed as dist
        if self.world == 1:
            return [list(vals)]
        dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(self.group) == "nccl" \
            else "cpu"
        t = torch.tensor([v - (1 << 64) if v >= (1 << 63) else v for v in vals], dtype=torch.int64,
                         device=dev)
        outs = [torch.empty_like(t) for _ in range(self.world)]
        dist.all_gather(outs, t, group=self.group)
        return [[int(x) & ((1 << 64) - 1) for x in o.cpu().tolist()] for o in outs]

    def checksum(self):
        """(occupied, Σkeys, Σvalues, ⊕ mix64(k ^ mix64(v))) over all shards (mod 2^64)."""
        parts = self._gather(self.local.checksum())
        m = (1 << 64) - 1
        c = sk = sv = x = 0
        for p in parts:
            c += p[0]
            sk = (sk + p[1]) & m
            sv = (sv + p[2]) & m
            x ^= p[3]
        return c, sk, sv, x

    def occupied_count(self):
        return self.checksum()[0]

    def duplicate_count(self):
        # a key lives on exactly one owner, so duplicates are shard-local
        return sum(p[0] for p in self._gather([self.local.duplicate_count()]))

    def clear(self):
        self.local.clear()

"""World-size-2 gloo test of the hash-sharded table's routing logic (CPU).

The product ShardedTable (paper_2509_16407_b200/sharded.py) is driven with
the same exchange code as on GPUs, but with two test doubles injected: a
numpy owner partitioner (same owner rule as ws_partition: top log2(world)
bits of mix64(k ^ seed0)) and the CPU oracle as each rank's local table.
Checks: every rank's results equal a single global map's answers, every key
lives on its owner shard only, the cross-rank checksum equals numpy's, and
Zipf-duplicated upsert-ADDs from both ranks sum correctly.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT  # noqa: F401  (sys.path)

U64 = np.uint64


class CpuRouter:
    def __init__(self, seed0, log2):
        self.seed0, self.log2 = seed0, log2

    def owners(self, keys_np):
        from paper_2509_16407_b200.workload import mix64_np
        if self.log2 == 0:
            return np.zeros(len(keys_np), dtype=np.int64)
        return (mix64_np(keys_np ^ U64(self.seed0)) >> U64(64 - self.log2)).astype(np.int64)

    def partition(self, keys, vals=None, ops=None):
        k = keys.view(torch.int64).numpy().view(U64)
        own = self.owners(k)
        perm = np.argsort(own, kind="stable")
        counts = np.bincount(own, minlength=1 << self.log2)
        pk = torch.from_numpy(k[perm].view(np.int64)).view(torch.uint64)
        pv = None if vals is None else vals.view(torch.int64)[torch.from_numpy(perm)].view(torch.uint64)
        po = None if ops is None else ops[torch.from_numpy(perm)]
        return pk, pv, po, torch.from_numpy(perm.astype(np.int32)), torch.from_numpy(counts.astype(np.int64))

    def unpermute(self, res, perm):
        out = torch.empty_like(res)
        view = res.view(torch.int64) if res.dtype == torch.uint64 else res
        oview = out.view(torch.int64) if res.dtype == torch.uint64 else out
        oview[perm.long()] = view
        return out


class OracleLocal:
    """Oracle table with the device table's tensor-in / tensor-out batch API."""

    def __init__(self, cfg):
        from oracle import OracleTable
        self.t = OracleTable(cfg)

    @staticmethod
    def _np(x):
        return x.view(torch.int64).numpy().view(U64) if x.dtype in (torch.uint64, torch.int64) else x.numpy()

    @staticmethod
    def _t64(a):
        return torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).view(torch.uint64)

    def upsert_batch(self, keys, values, merge=None, check=True):
        return torch.from_numpy(self.t.upsert_batch(self._np(keys), self._np(values), merge))

    def query_batch(self, keys, check=True):
        f, v = self.t.query_batch(self._np(keys))
        return torch.from_numpy(f), self._t64(v)

    def erase_batch(self, keys, check=True):
        return torch.from_numpy(self.t.erase_batch(self._np(keys)))

    def mixed_batch(self, ops, keys, values, check=True):
        st, vo = self.t.mixed_batch(ops.numpy(), self._np(keys), self._np(values))
        return torch.from_numpy(st), self._t64(vo)

    def checksum(self):
        from paper_2509_16407_b200.workload import mix64_np
        k, v = self.t.items_arrays()
        with np.errstate(over="ignore"):
            x = int(np.bitwise_xor.reduce(mix64_np(k ^ mix64_np(v)))) if len(k) else 0
            return (len(k), int(k.sum(dtype=U64)), int(v.sum(dtype=U64)), x)

    def duplicate_count(self):
        return len(self.t.duplicate_scan())

    def items(self):
        return self.t.items()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, outq):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2509_16407_b200 import TableConfig
        from paper_2509_16407_b200.sharded import ShardedTable
        from paper_2509_16407_b200.workload import gen_uniform_keys, mix64_np, zipf_ranks

        cfg = TableConfig(design="p2_md", capacity_slots=1 << 16, seed=42)
        local_cfg = TableConfig(design="p2_md", capacity_slots=(1 << 16) // world, seed=42)
        st = ShardedTable(cfg, local_table=OracleLocal(local_cfg),
                          router=CpuRouter(cfg.hash_family().seeds[0], world.bit_length() - 1))
        n = 20000
        mine = gen_uniform_keys(100 + rank, n)
        t64 = OracleLocal._t64
        s = st.upsert_batch(t64(mine), t64(mine & U64(0xFFFF)))
        assert (s.numpy() == 0).all()
        # every rank queries everyone's keys + misses
        allk = np.concatenate([gen_uniform_keys(100 + r, n) for r in range(world)])
        miss = gen_uniform_keys(999 + rank, 5000)
        q = np.concatenate([allk[rank::world], miss])
        f, v = st.query_batch(t64(q))
        f = f.numpy()
        v = v.view(torch.int64).numpy().view(U64)
        nh = len(allk[rank::world])
        assert f[:nh].all() and not f[nh:].any()
        assert (v[:nh] == (allk[rank::world] & U64(0xFFFF))).all()
        # placement: every local key is owned by this rank
        own = CpuRouter(cfg.hash_family().seeds[0], world.bit_length() - 1).owners
        lk = np.array([k for k, _ in st.local.items()], dtype=U64)
        assert (own(lk) == rank).all()
        # global checksum
        with np.errstate(over="ignore"):
            vals = allk & U64(0xFFFF)
            want = (len(allk), int(allk.sum(dtype=U64)), int(vals.sum(dtype=U64)),
                    int(np.bitwise_xor.reduce(mix64_np(allk ^ mix64_np(vals)))))
        assert st.checksum() == want
        # Zipf upsert-ADD from every rank on a shared universe
        uni = gen_uniform_keys(7, 3000)
        r_idx = zipf_ranks(3000, 40000, 0.99, seed=rank) - 1
        ks = uni[r_idx]
        s = st.upsert_batch(t64(ks), t64(np.ones(len(ks), dtype=U64)), merge="add")
        assert ((s.numpy() == 0) | (s.numpy() == 1)).all()
        f, v = st.query_batch(t64(uni))
        tot = np.zeros(3000, dtype=np.int64)
        for r in range(world):
            np.add.at(tot, zipf_ranks(3000, 40000, 0.99, seed=r) - 1, 1)
        got = v.view(torch.int64).numpy()
        assert (got == tot).all()
        # erase half of my keys, then they are gone everywhere
        e = st.erase_batch(t64(mine[::2]))
        assert e.numpy().all()
        f, _ = st.query_batch(t64(mine))
        assert not f.numpy()[::2].any() and f.numpy()[1::2].all()
        assert st.duplicate_count() == 0
        # a sentinel key in ONE rank's batch rejects the logical
        # batch on EVERY rank before any routing or mutation (no hang)
        from paper_2509_16407_b200 import InvalidKeyError
        before = st.checksum()
        fresh = gen_uniform_keys(555 + rank, 1000)
        if rank == 1:
            fresh[321] = U64(0xFFFFFFFFFFFFFFFF)  # TOMBSTONE sentinel
        with pytest.raises(InvalidKeyError):
            st.upsert_batch(t64(fresh), t64(fresh))
        with pytest.raises(InvalidKeyError):
            st.erase_batch(t64(fresh))
        bad_ops = torch.zeros(1000, dtype=torch.uint8)
        if rank == 0:
            bad_ops[5] = 7  # kind 7 does not exist
        with pytest.raises(ValueError):
            st.mixed_batch(bad_ops, t64(gen_uniform_keys(556 + rank, 1000)))
        assert st.checksum() == before
        dist.barrier()
        dist.destroy_process_group()
        outq.put((rank, "ok"))
    except Exception as exc:  # noqa: BLE001
        import traceback
        outq.put((rank, traceback.format_exc()))
        raise


@pytest.mark.timeout(300)
def test_sharded_table_world2_gloo():
    ctx = mp.get_context("spawn")
    outq = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, outq)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(outq.get(timeout=280) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res


def test_owner_rule_matches_device_kernel_definition():
    """Owner = top log2(world) bits of mix64(k ^ seed0) (ws_shard.cu owner_of)."""
    from paper_2509_16407_b200 import TableConfig
    from paper_2509_16407_b200.core import mix64
    from paper_2509_16407_b200.workload import gen_uniform_keys
    seed0 = TableConfig(design="p2_md", capacity_slots=1 << 16, seed=42).hash_family().seeds[0]
    keys = gen_uniform_keys(3, 1000)
    r = CpuRouter(seed0, 3)
    own = r.owners(keys)
    assert all(own[i] == mix64(int(k) ^ seed0) >> 61 for i, k in enumerate(keys[:50]))
    assert np.bincount(own, minlength=8).min() > 80  # balanced

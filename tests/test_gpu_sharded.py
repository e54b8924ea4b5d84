"""Two ranks sharing one GPU over gloo: the product ShardedTable with the
device router (ws_partition / ws_unpermute) and real device tables, checked
against a global expectation.  (NCCL refuses two ranks on one device; gloo
stages the all-to-all through host memory -- same routing logic.)"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from conftest import ROOT  # noqa: E402,F401

U64 = np.uint64


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _cu(a):
    a = np.ascontiguousarray(a)
    if a.dtype == np.uint8:
        return torch.from_numpy(a).cuda()
    return torch.from_numpy(a.view(np.int64)).cuda().view(torch.uint64)


def _np(t):
    t = t.cpu()
    return t.view(torch.int64).numpy().view(U64) if t.dtype == torch.uint64 else t.numpy()


def _worker(rank, world, port, outq, exchange="nccl"):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2509_16407_b200 import TableConfig
        from paper_2509_16407_b200.sharded import ShardedTable
        from paper_2509_16407_b200.workload import gen_uniform_keys, mix64_np, zipf_ranks
        # 2^19 slots per rank: every rank's 200K keys keep the load at ~0.4
        st = ShardedTable(TableConfig(design="p2_md", capacity_slots=(1 << 19) * world, seed=42),
                          exchange=exchange, chunk_ops=1 << 16)
        n = 200_000
        mine = gen_uniform_keys(100 + rank, n)
        s = _np(st.upsert_batch(_cu(mine), _cu(mine & U64(0xFFFF))))
        assert (s == 0).all()
        allk = np.concatenate([gen_uniform_keys(100 + r, n) for r in range(world)])
        q = np.concatenate([allk[rank::world], gen_uniform_keys(999 + rank, 50_000)])
        f, v = st.query_batch(_cu(q))
        f, v = _np(f).astype(bool), _np(v)
        nh = len(allk[rank::world])
        assert f[:nh].all() and not f[nh:].any()
        assert (v[:nh] == (allk[rank::world] & U64(0xFFFF))).all()
        with np.errstate(over="ignore"):
            vals = allk & U64(0xFFFF)
            want = (len(allk), int(allk.sum(dtype=U64)), int(vals.sum(dtype=U64)),
                    int(np.bitwise_xor.reduce(mix64_np(allk ^ mix64_np(vals)))))
        assert st.checksum() == want
        uni = gen_uniform_keys(7, 20_000)
        ks = uni[zipf_ranks(20_000, 300_000, 0.99, seed=rank) - 1]
        s = _np(st.upsert_batch(_cu(ks), _cu(np.ones(len(ks), U64)), merge="add"))
        assert ((s == 0) | (s == 1)).all()
        f, v = st.query_batch(_cu(uni))
        tot = np.zeros(20_000, dtype=np.int64)
        for r in range(world):
            np.add.at(tot, zipf_ranks(20_000, 300_000, 0.99, seed=r) - 1, 1)
        assert (_np(v).view(np.int64) == tot).all()
        ops = np.array([1] * 1000 + [2] * 1000, np.uint8)
        mk = np.concatenate([mine[:1000], mine[1000:2000]])
        s, vo = st.mixed_batch(_cu(ops), _cu(mk))
        s = _np(s)
        assert s.all()
        f, _ = st.query_batch(_cu(mine[:2000]))
        f = _np(f).astype(bool)
        assert not f[:1000].any() and f[1000:].all()
        assert st.duplicate_count() == 0
        dist.barrier()
        dist.destroy_process_group()
        outq.put((rank, "ok"))
    except Exception:  # noqa: BLE001
        import traceback
        outq.put((rank, traceback.format_exc()))
        raise


@pytest.mark.parametrize("world,exchange", [(2, "nccl"), (2, "p2p"), (4, "p2p"), (8, "p2p")])
def test_sharded_two_ranks_one_gpu(world, exchange):
    """exchange="nccl" runs the all-to-all path (gloo-staged here); "p2p"
    runs the fused routing kernels over CUDA-IPC peer memory (processes on
    one device share it just like NVLink peers), with 2^16-op rounds so the
    200K-op batches take several rounds.  World 4 and 8 exercise the p2p
    exchange with as many peers as one 8-GPU node has."""
    ctx = mp.get_context("spawn")
    outq = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, outq, exchange)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(outq.get(timeout=900) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {r: "ok" for r in range(world)}, res


def _kmer_worker(rank, world, port, outq, exchange):
    """BASELINE config 5 in miniature: canonical 31-mer counting with
    upsert-ADD through ShardedTable (reads split over the ranks, every k-mer
    routed to its owner), then every distinct k-mer queried from every rank;
    counts must equal numpy's global multiplicities exactly."""
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2509_16407_b200 import TableConfig
        from paper_2509_16407_b200.sharded import ShardedTable
        from paper_2509_16407_b200.workload import kmer_keys
        st = ShardedTable(TableConfig(design="p2_md", capacity_slots=1 << 21, seed=42), exchange=exchange,
                          chunk_ops=1 << 17)
        km = kmer_keys(1 << 20, 31, seed=9, repeats=4)        # ~2^20 k-mers, ~2^18 distinct
        rng = np.random.default_rng(5)
        km = km[rng.permutation(len(km))]
        mine = km[rank::world]                                # this rank's reads
        for part in np.array_split(mine, 3):
            s = _np(st.upsert_batch(_cu(part), _cu(np.ones(len(part), U64)), merge="add"))
            assert ((s == 0) | (s == 1)).all()
        u, c = np.unique(km, return_counts=True)
        f, v = st.query_batch(_cu(u))
        assert _np(f).all()
        assert (_np(v) == c.astype(U64)).all()
        assert st.occupied_count() == len(u)
        assert st.duplicate_count() == 0
        dist.barrier()
        dist.destroy_process_group()
        outq.put((rank, "ok"))
    except Exception:  # noqa: BLE001
        import traceback
        outq.put((rank, traceback.format_exc()))
        raise


@pytest.mark.parametrize("exchange", ["nccl", "p2p"])
def test_config5_kmer_counting_two_ranks(exchange):
    ctx = mp.get_context("spawn")
    outq = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_kmer_worker, args=(r, 2, port, outq, exchange)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(outq.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res

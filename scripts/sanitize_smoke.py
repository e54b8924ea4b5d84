"""Small workloads for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): every design's lock-round / line-scan fast kernels and the
generic kernel (fill, mixed batch, queries, erases, serial replay), the cuckoo
eviction path at 0.95, chaining pool growth, combining, the per-kind mixed
split, host-staged batches and the instrumented kernel -- each checked
against the oracle so a sanitizer run is also a correctness run.

    compute-sanitizer --tool memcheck python scripts/sanitize_smoke.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np  # noqa: E402
import torch  # noqa: E402

from conftest import ALL_DESIGNS, cfg_for  # noqa: E402
from oracle import OracleTable  # noqa: E402
from paper_2509_16407_b200 import make_table  # noqa: E402
from paper_2509_16407_b200.workload import gen_uniform_keys  # noqa: E402

U64 = np.uint64


def cu(a):
    a = np.ascontiguousarray(a)
    if a.dtype == np.uint8:
        return torch.from_numpy(a).cuda()
    return torch.from_numpy(a.astype(U64).view(np.int64)).cuda().view(torch.uint64)


def main():
    for d in ALL_DESIGNS:
        cap = 7 * 512 if d == "chaining" else 4096
        cfg = cfg_for(d, cap, seed=3)
        t, o = make_table(cfg), OracleTable(cfg)
        n = int(t.capacity_slots * (1.2 if d == "chaining" else 0.85))
        k = gen_uniform_keys(11, n)
        t.upsert_batch(cu(k), cu(k))                       # fast upsert kernel (+ chaining growth)
        o.upsert_batch(k, k)
        f, v = t.query_batch(cu(np.concatenate([k[:500], gen_uniform_keys(12, 500)])))
        ops = np.array([1] * 300 + [2] * 300 + [0 | (2 << 4)] * 300, np.uint8)
        mk = np.concatenate([k[:300], k[300:600], gen_uniform_keys(13, 300)])
        mv = np.ones(900, U64)
        t.mixed_batch(cu(ops), cu(mk), cu(mv))             # generic kernel, mixed
        o.mixed_batch(ops, mk, mv)
        t.upsert_batch(cu(k[600:900]), cu(k[600:900]), merge="add", combine=True)   # combining
        o.upsert_batch(k[600:900], k[600:900], merge="add")
        t.erase_batch(cu(k[900:1000]))
        o.erase_batch(k[900:1000])
        t.upsert_batch(k[1000:1100], k[1000:1100])         # host-staged path
        o.upsert_batch(k[1000:1100], k[1000:1100])
        t.probe_batch(np.full(50, 2, np.uint8), k[:50])    # instrumented serial kernel
        assert dict(t.items()) == o.as_dict(), d
        assert t.duplicate_scan() == {}
        print("ok", d, flush=True)
    # cuckoo eviction chains at 0.95 and the per-kind split of a large mixed batch
    cfg = cfg_for("cuckoo", 1 << 14, seed=5)
    t, o = make_table(cfg), OracleTable(cfg)
    k = gen_uniform_keys(21, int(t.capacity_slots * 0.95))
    t.upsert_batch(cu(k), cu(k))
    o.upsert_batch(k, k)
    assert t.occupied_count() == o.occupied_count()
    cfg = cfg_for("p2_md", 1 << 18, seed=6)
    t, o = make_table(cfg), OracleTable(cfg)
    k = gen_uniform_keys(22, 70_000)
    ops = np.where(np.arange(70_000) % 3 == 0, 2, 0 | (2 << 4)).astype(np.uint8)
    t.mixed_batch(cu(ops), cu(k), cu(np.ones(70_000, U64)))
    o.mixed_batch(ops, k, np.ones(70_000, U64))
    assert dict(t.items()) == o.as_dict()
    # the sort-free split (erase / query / rest regions) with combining of
    # duplicate ADD and REPLACE upserts, and the tuned iceberg_md erase
    for d in ("iceberg_md", "p2_md"):
        cfg = cfg_for(d, 1 << 18, seed=7)
        t, o = make_table(cfg), OracleTable(cfg)
        base = gen_uniform_keys(23, 150_000)
        t.upsert_batch(cu(base), cu(base))
        o.upsert_batch(base, base)
        rng = np.random.default_rng(1)
        hot = gen_uniform_keys(24, 2000)
        ops = np.concatenate([np.full(20_000, 1), np.full(20_000, 2), np.full(20_000, 2 << 4),
                              np.full(20_000, 0)]).astype(np.uint8)
        keys = np.concatenate([base[:20_000], base[20_000:40_000], hot[rng.integers(0, 1000, 20_000)],
                               hot[1000 + rng.integers(0, 1000, 20_000)]])
        vals = rng.integers(1, 1 << 40, len(keys)).astype(U64)
        perm = rng.permutation(len(keys))
        ops, keys, vals = ops[perm], keys[perm], vals[perm]
        st, vo = t.mixed_batch(cu(ops), cu(keys), cu(vals), combine=True)
        ost, ovo = o.mixed_batch(ops, keys, vals)
        assert (st.cpu().numpy() == ost).all() and (vo.cpu().view(torch.int64).numpy().view(U64) == ovo).all(), d
        assert dict(t.items()) == o.as_dict(), d
        print("ok split+combine", d, flush=True)
    # the search-based duplicate scan and the query's in-kernel sentinel check
    import os
    cfg = cfg_for("p2_md", 1 << 16, seed=8)
    t = make_table(cfg)
    k = gen_uniform_keys(25, 50_000)
    t.upsert_batch(cu(k), cu(k))
    os.environ["WS_DUPSCAN_BY_LOCATE"] = "1"
    assert t.duplicate_count() == 0
    del os.environ["WS_DUPSCAN_BY_LOCATE"]
    f, _v = t.query_batch(cu(k))
    assert bool(f.bool().all())
    print("ok dupscan-by-locate + fused query check", flush=True)
    torch.cuda.synchronize()
    print("sanitize smoke ok", flush=True)


if __name__ == "__main__":
    main()

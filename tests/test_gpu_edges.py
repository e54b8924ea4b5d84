"""Edge cases of the batched API on the device (reference SPEC.md:89 and
tables/base.py:111-134 semantics): empty and single-op batches, batches on
either side of the per-kind split threshold (2^16 ops), every call flag
combination, duplicate keys without combining, a full table, invalid op
bytes, and host-resident (staged) mixed batches -- each against the oracle
or an exact invariant."""

import numpy as np
import pytest

from conftest import cfg_for

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

DESIGNS = ["p2_md", "iceberg_md", "double", "cuckoo", "chaining"]


def _keys(seed, n):
    from paper_2509_16407_b200.workload import gen_uniform_keys
    return gen_uniform_keys(seed, n)


def _cuda(a):
    a = np.ascontiguousarray(a)
    if a.dtype == np.uint8:
        return torch.from_numpy(a).cuda()
    return torch.from_numpy(a.astype(np.uint64, copy=False).view(np.int64)).cuda().view(torch.uint64)


def _np(t):
    if isinstance(t, np.ndarray):
        return t
    return t.cpu().view(torch.int64).numpy().view(np.uint64) if t.dtype == torch.uint64 else t.cpu().numpy()


def _pair(design, log2=14, seed=3):
    from oracle import OracleTable
    from paper_2509_16407_b200 import make_table
    cfg = cfg_for(design, (1 << log2) if design != "chaining" else 7 * (1 << (log2 - 3)), seed=seed)
    return make_table(cfg), OracleTable(cfg)


@pytest.mark.parametrize("design", DESIGNS)
def test_empty_batches_every_entry_point(design):
    t, _o = _pair(design)
    base = _keys(1, 100)
    t.upsert_batch(_cuda(base), _cuda(base))
    before = t.checksum()
    e64 = torch.empty(0, dtype=torch.uint64, device="cuda")
    e8 = torch.empty(0, dtype=torch.uint8, device="cuda")
    assert t.upsert_batch(e64, e64).numel() == 0
    assert t.upsert_batch(e64, e64, merge="add", combine=True).numel() == 0
    f, v = t.query_batch(e64)
    assert f.numel() == 0 and v.numel() == 0
    assert t.erase_batch(e64).numel() == 0
    for kw in ({}, {"combine": True}, {"concurrent": True}, {"interleaved": True}):
        s, v = t.mixed_batch(e8, e64, e64, **kw)
        assert s.numel() == 0 and v.numel() == 0
    s, v = t.mixed_batch(np.zeros(0, np.uint8), np.zeros(0, np.uint64), np.zeros(0, np.uint64))  # host
    assert len(s) == 0
    assert t.checksum() == before


@pytest.mark.parametrize("design", DESIGNS)
def test_single_op_batches_match_oracle(design):
    from paper_2509_16407_b200.tables import OP_ERASE, OP_QUERY, OP_UPSERT
    t, o = _pair(design)
    ks = _keys(2, 40)
    for j, k in enumerate(ks):
        kind = (OP_UPSERT, OP_UPSERT | (2 << 4), OP_QUERY, OP_ERASE)[j % 4]
        kk = ks[j - 1] if kind in (OP_QUERY, OP_ERASE) and j else k
        a = np.array([kind], np.uint8)
        b = np.array([kk], np.uint64)
        c = np.array([j + 1], np.uint64)
        s, v = t.mixed_batch(_cuda(a), _cuda(b), _cuda(c))
        os_, ov = o.mixed_batch(a, b, c)
        assert int(_np(s)[0]) == int(os_[0]) and int(_np(v)[0]) == int(ov[0]), (j, kind)
    assert dict(t.items()) == o.as_dict()


@pytest.mark.parametrize("design", ["p2_md", "iceberg_md", "double_md", "chaining"])
@pytest.mark.parametrize("n", [(1 << 16) - 1, 1 << 16, (1 << 16) + 1])
@pytest.mark.parametrize("flags", [{}, {"combine": True}, {"concurrent": True}, {"interleaved": True}])
def test_split_threshold_batches_match_oracle(design, n, flags):
    """Mixed batches just below, at and above the per-kind split threshold
    take different host paths (one fused / generic launch vs the split), with
    every flag combination; roles key-disjoint so the oracle's sequential
    replay is the answer."""
    from paper_2509_16407_b200.tables import OP_ERASE, OP_QUERY, OP_UPSERT
    t, o = _pair(design, log2=18, seed=5)
    base = _keys(3, int(t.capacity_slots * 0.5))
    t.upsert_batch(_cuda(base), _cuda(base))
    o.upsert_batch(base, base)
    q = n // 4
    ops = np.concatenate([np.full(q, OP_UPSERT | (2 << 4)), np.full(q, OP_ERASE), np.full(q, OP_QUERY),
                          np.full(n - 3 * q, OP_QUERY)]).astype(np.uint8)
    keys = np.concatenate([_keys(4, q), base[:q], base[q:2 * q], _keys(5, n - 3 * q)])
    vals = np.arange(n, dtype=np.uint64) + np.uint64(1)
    perm = np.random.default_rng(n).permutation(n)
    ops, keys, vals = ops[perm], keys[perm], vals[perm]
    s, v = t.mixed_batch(_cuda(ops), _cuda(keys), _cuda(vals), **flags)
    os_, ov = o.mixed_batch(ops, keys, vals)
    np.testing.assert_array_equal(_np(s), os_)
    np.testing.assert_array_equal(_np(v), ov)
    assert dict(t.items()) == o.as_dict()
    assert t.duplicate_scan() == {}


@pytest.mark.parametrize("design", DESIGNS)
def test_duplicate_keys_without_combining(design):
    """Same-key upserts in one uncombined batch are concurrent: ADD sums
    exactly, exactly one op per new key reports INSERTED, no duplicates."""
    t, _o = _pair(design, log2=16)
    uni = _keys(6, 3000)
    keys = uni[np.random.default_rng(1).integers(0, 3000, 40_000)]
    st = _np(t.upsert_batch(_cuda(keys), _cuda(np.full(len(keys), 3, np.uint64)), merge="add"))
    u, c = np.unique(keys, return_counts=True)
    assert int((st == 0).sum()) == len(u) and not (st == 2).any()
    got = dict(t.items())
    assert got == {int(k): int(3 * n) for k, n in zip(u, c)}
    assert t.duplicate_scan() == {}


@pytest.mark.parametrize("design", ["p2_md", "double", "iceberg_md"])
def test_full_table_reports_full_and_stays_consistent(design):
    """Inserting far more keys than slots: every op is INSERTED or FULL, the
    occupied count equals the INSERTED count, every INSERTED key is found and
    no FULL key is, and a second pass over the same keys only UPDATEs or
    FULLs."""
    t, _o = _pair(design, log2=12)
    keys = _keys(7, 3 * t.capacity_slots)
    st = _np(t.upsert_batch(_cuda(keys), _cuda(keys)))
    assert set(np.unique(st).tolist()) <= {0, 2} and (st == 2).any()
    assert t.occupied_count() == int((st == 0).sum())
    f, v = t.query_batch(_cuda(keys))
    f = _np(f).astype(bool)
    assert (f == (st == 0)).all()
    st2 = _np(t.upsert_batch(_cuda(keys), _cuda(keys)))
    assert ((st2 == 1) == (st == 0)).all() and not (st2 == 0).any()
    assert t.duplicate_scan() == {}


def test_invalid_op_byte_rejected_table_untouched():
    t, _o = _pair("p2_md")
    base = _keys(8, 500)
    t.upsert_batch(_cuda(base), _cuda(base))
    before = t.checksum()
    ops = np.zeros(1000, np.uint8)
    ops[500] = 7  # kind 7 does not exist
    with pytest.raises(ValueError):
        t.mixed_batch(_cuda(ops), _cuda(_keys(9, 1000)), _cuda(np.ones(1000, np.uint64)))
    assert t.checksum() == before


@pytest.mark.parametrize("flags", [{}, {"combine": True}])
def test_host_resident_mixed_batch_matches_oracle(flags):
    """numpy inputs: the library stages them through device memory in 4M-op
    chunks (validation of the whole batch before the first mutation)."""
    from paper_2509_16407_b200.tables import OP_ERASE, OP_QUERY, OP_UPSERT
    t, o = _pair("iceberg_md", log2=22, seed=9)
    base = _keys(10, int(t.capacity_slots * 0.5))
    t.upsert_batch(base, base)
    o.upsert_batch(base, base)
    n = 1_500_000
    q = n // 3
    ops = np.concatenate([np.full(q, OP_UPSERT | (2 << 4)), np.full(q, OP_ERASE),
                          np.full(n - 2 * q, OP_QUERY)]).astype(np.uint8)
    keys = np.concatenate([_keys(11, q), base[:q], base[q:q + n - 2 * q]])
    vals = np.arange(n, dtype=np.uint64)
    perm = np.random.default_rng(2).permutation(n)
    ops, keys, vals = ops[perm], keys[perm], vals[perm]
    s, v = t.mixed_batch(ops, keys, vals, **flags)
    os_, ov = o.mixed_batch(ops, keys, vals)
    np.testing.assert_array_equal(_np(s), os_)
    np.testing.assert_array_equal(_np(v), ov)
    assert t.occupied_count() == o.occupied_count()


def test_kernel_event_timing_records_one_bracket_per_table_kernel():
    """WS_TUNE_KERNEL_EVENTS (bench.py's kernel-level roofline): one
    positive elapsed time per table-kernel launch, in launch order; off by
    default and cleared by each read."""
    t, _o = _pair("p2_md", log2=20)
    keys = _cuda(_keys(12, 500_000))
    t.upsert_batch(keys, keys)
    assert t.kernel_times() == []
    t.time_kernels(True)
    t.upsert_batch(keys, keys)
    t.query_batch(keys)
    ms = t.kernel_times()
    assert len(ms) == 2 and all(x > 0 for x in ms)
    assert t.kernel_times() == []
    t.time_kernels(False)
    t.query_batch(keys)
    assert t.kernel_times() == []


@pytest.mark.parametrize("pos", [0, 123_457, 999_999])
def test_query_sentinel_anywhere_in_large_batch_raises(pos):
    """The P2-MD query checks sentinels inside the query kernel (no separate
    pass): a sentinel anywhere in a 10^6-key batch still raises, and the
    same batch without it answers exactly."""
    from paper_2509_16407_b200 import InvalidKeyError
    t, o = _pair("p2_md", log2=20)
    keys = _keys(13, 500_000)
    t.upsert_batch(_cuda(keys), _cuda(keys))
    o.upsert_batch(keys, keys)
    q = np.concatenate([keys, _keys(14, 500_000)])
    for bad in (0, (1 << 64) - 1, (1 << 64) - 2):
        qb = q.copy()
        qb[pos] = np.uint64(bad)
        with pytest.raises(InvalidKeyError):
            t.query_batch(_cuda(qb))
    f, v = t.query_batch(_cuda(q))
    of, ov = o.query_batch(q)
    np.testing.assert_array_equal(_np(f).astype(bool), of.astype(bool))
    np.testing.assert_array_equal(_np(v), ov)

"""Concurrent callers of the drop-in table API.

The reference tables are driven by many host threads at once
(reference tables/base.py:5-7 "every public operation may be called
concurrently"; bench/pool.py:26-50 fans timed batches over a thread pool;
bench/adversarial.py:169-191 runs three actor threads).  ctypes releases the
GIL during every libwarpspeed call, so these threads really do enter the C ABI
concurrently.  Results must match a linearised oracle: the tests use op mixes
whose final state is independent of the interleaving (commutative ADD
upserts, disjoint erase / query roles), so the oracle is the sequential
application of all ops in any order.
"""

import threading
import time

import numpy as np
import pytest

from conftest import ALL_DESIGNS, cfg_for

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

N_THREADS = 8


def _run_threads(fn, n=N_THREADS):
    errors = []
    barrier = threading.Barrier(n)

    def body(i):
        try:
            barrier.wait()
            fn(i)
        except BaseException as exc:  # noqa: BLE001
            errors.append(exc)

    ths = [threading.Thread(target=body, args=(i,)) for i in range(n)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    if errors:
        raise errors[0]


@pytest.mark.parametrize("design", ALL_DESIGNS)
def test_scalar_ops_from_eight_threads_match_linearised_oracle(design):
    """8 threads x (upsert-ADD on shared hot keys, erase of own prefilled keys,
    query of own stable keys) through the scalar API (pool.py pattern)."""
    from oracle import OracleTable
    from paper_2509_16407_b200 import make_table
    from paper_2509_16407_b200.workload import gen_uniform_keys

    cfg = cfg_for(design, 1 << 14, seed=3)
    t = make_table(cfg)
    o = OracleTable(cfg)
    keys = gen_uniform_keys(17, 40 * N_THREADS + 24)
    hot = keys[:24]                                       # shared by every thread
    own = keys[24:].reshape(N_THREADS, 40)
    erase_set, stable = own[:, :20], own[:, 20:]
    pre = np.concatenate([erase_set.ravel(), stable.ravel()])
    pre_v = pre & np.uint64(0xFFF)
    t.upsert_batch(pre, pre_v)
    o.upsert_batch(pre, pre_v)
    results = [None] * N_THREADS
    add = (lambda a, b: (a + b) & ((1 << 64) - 1))  # a reference-style merge callable

    def work(i):
        rng = np.random.default_rng(i)
        got_q, got_e = [], []
        for r in range(20):
            k = int(hot[rng.integers(0, len(hot))])
            assert t.upsert(k, 1 + i, merge=add).value in (
                "inserted", "updated")
            got_e.append(t.erase(int(erase_set[i, r])))
            got_q.append(t.query(int(stable[i, r])))
        results[i] = (got_q, got_e)

    _run_threads(work)
    # linearised oracle: every thread's ops in thread order (the result is order-free)
    for i in range(N_THREADS):
        rng = np.random.default_rng(i)
        for r in range(20):
            k = int(hot[rng.integers(0, len(hot))])
            o.upsert_batch(np.array([k], np.uint64), np.array([1 + i], np.uint64), merge="add")
        o.erase_batch(erase_set[i])
    for i in range(N_THREADS):
        got_q, got_e = results[i]
        assert got_e == [True] * 20
        assert got_q == [int(v) for v in stable[i] & np.uint64(0xFFF)]
    assert dict(t.items()) == o.as_dict()
    assert t.duplicate_scan() == {}


@pytest.mark.parametrize("design", ["p2_md", "iceberg_md", "chaining", "cuckoo"])
def test_batched_calls_from_threads_with_one_rejected_batch(design):
    """Per-call validation: one thread's batch holds a sentinel key and must be
    rejected whole (InvalidKeyError, nothing applied) while the other threads'
    valid batches -- on the same table and the same stream -- all apply."""
    from oracle import OracleTable
    from paper_2509_16407_b200 import InvalidKeyError, make_table
    from paper_2509_16407_b200.workload import gen_uniform_keys

    cfg = cfg_for(design, 1 << 16, seed=9)
    t = make_table(cfg)
    o = OracleTable(cfg)
    keys = gen_uniform_keys(5, 4000 * N_THREADS).reshape(N_THREADS, 4000)
    bad_thread = 3
    raised = []

    def work(i):
        for rep in range(5):
            k = keys[i].copy()
            if i == bad_thread:
                k[1234] = 0  # EMPTY sentinel
            kd = torch.from_numpy(k.view(np.int64)).cuda().view(torch.uint64)
            try:
                t.upsert_batch(kd, kd, merge="add")
            except InvalidKeyError:
                raised.append(i)

    _run_threads(work)
    assert raised == [bad_thread] * 5
    for i in range(N_THREADS):
        if i != bad_thread:
            for _ in range(5):
                o.upsert_batch(keys[i], keys[i], merge="add")
    torch.cuda.synchronize()
    assert dict(t.items()) == o.as_dict()


def test_threads_on_own_streams_multi_stream_table():
    """Threads with their own CUDA streams on a multi_stream table: mixed
    erase / upsert-ADD / query batches launched concurrently on the device."""
    from oracle import OracleTable
    from paper_2509_16407_b200 import make_table
    from paper_2509_16407_b200.workload import gen_uniform_keys

    cfg = cfg_for("p2_md", 1 << 18, seed=2)
    t = make_table(cfg, multi_stream=True)
    o = OracleTable(cfg)
    base = gen_uniform_keys(8, 30000 * N_THREADS).reshape(N_THREADS, 30000)
    pre = base[:, :10000].ravel()
    t.upsert_batch(pre, np.ones(len(pre), np.uint64))
    o.upsert_batch(pre, np.ones(len(pre), np.uint64))
    out = [None] * N_THREADS

    def work(i):
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            k = torch.from_numpy(base[i].view(np.int64)).cuda().view(torch.uint64)
            ops = torch.zeros(30000, dtype=torch.uint8, device="cuda")
            ops[:5000] = 1                       # erase own prefilled keys [0, 5000)
            ops[5000:10000] = 2                  # query own prefilled keys [5000, 10000)
            ops[10000:] = 0 | (2 << 4)           # upsert-ADD fresh keys
            st, vo = t.mixed_batch(ops, k, torch.full((30000,), 7, dtype=torch.uint64, device="cuda"))
            s.synchronize()
            out[i] = (st.cpu().numpy(), vo.cpu().numpy())

    _run_threads(work)
    for i in range(N_THREADS):
        st, vo = out[i]
        assert (st[:5000] == 1).all()
        assert (st[5000:10000] == 1).all() and (vo[5000:10000] == 1).all()
        assert (st[10000:] == 0).all()
        o.erase_batch(base[i, :5000])
        o.upsert_batch(base[i, 10000:], np.full(20000, 7, np.uint64), merge="add")
    assert dict(t.items()) == o.as_dict()


def test_reference_three_actor_script_through_scalar_api():
    """The reference's adversarial replay (bench/adversarial.py:148-202) with
    its three actor threads and a barrier every 128 buckets, driven through
    the scalar upsert / erase calls of the drop-in."""
    import random

    from paper_2509_16407_b200 import UpsertStatus, make_table
    from paper_2509_16407_b200.adversarial import config_for_primary_buckets, generate_pairs

    n = 1024
    for design in ("p2_md", "iceberg_md"):
        cfg = config_for_primary_buckets(design, n, 5)
        t = make_table(cfg)
        xs, ys = generate_pairs(t, n, 5)
        xs, ys = xs.tolist(), ys.tolist()
        for x in xs:
            assert t.upsert(x, 1) is not UpsertStatus.FULL
        barrier = threading.Barrier(3)
        keep = (lambda a, b: a)

        def actor(op, aid):
            rng = random.Random(aid)
            for lo in range(0, n, 128):
                barrier.wait()
                for b in range(lo, min(lo + 128, n)):
                    if rng.random() < 0.02:  # the reference's light pre_op delay
                        time.sleep(rng.random() * 20e-6)
                    op(b)

        acts = [threading.Thread(target=actor, args=(lambda b: t.erase(xs[b]), 0)),
                threading.Thread(target=actor, args=(lambda b: t.upsert(ys[b], 1, keep), 1)),
                threading.Thread(target=actor, args=(lambda b: t.upsert(ys[b], 2, keep), 2))]
        for a in acts:
            a.start()
        for a in acts:
            a.join()
        assert t.duplicate_scan() == {}
        items = dict(t.items())
        assert set(items) == set(ys)           # every X erased, every Y present once
        assert set(items.values()) <= {1, 2}   # keep-merge: whichever upsert landed first


def test_combine_flag_with_sentinel_key_rejected_through_c_abi():
    """ws_upsert(..., flags=WS_F_COMBINE) without SYNC_CHECK must
    still leave the table untouched when the batch holds a sentinel key."""
    from paper_2509_16407_b200 import _native, make_table

    t = make_table(cfg_for("p2_md", 1 << 14, seed=1))
    k = torch.tensor([5, 6, 5, 0, 7, 5], dtype=torch.int64, device="cuda").view(torch.uint64)
    st = torch.empty(6, dtype=torch.uint8, device="cuda")
    rc = t._lib.ws_upsert(t._h, k.data_ptr(), k.data_ptr(), 6, 2, st.data_ptr(), t._stream(),
                          _native.WS_F_COMBINE)
    torch.cuda.synchronize()
    assert rc in (0, _native.WS_ERR_INVALID_KEY)
    assert t.occupied_count() == 0
    rc = t._lib.ws_mixed(t._h, torch.zeros(6, dtype=torch.uint8, device="cuda").data_ptr(), k.data_ptr(),
                         k.data_ptr(), 6, st.data_ptr(), None, t._stream(), _native.WS_F_COMBINE)
    torch.cuda.synchronize()
    assert rc in (0, _native.WS_ERR_INVALID_KEY)
    assert t.occupied_count() == 0

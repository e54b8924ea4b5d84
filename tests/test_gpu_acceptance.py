"""The reference's acceptance criteria on the device tables,
plus BASELINE config 1 at its exact size.

  3  oracle equivalence: 10^5 seeded mixed ops x 3 seeds per design, against
     digests of the reference's own run (tests/golden/spec_equivalence.json)
  4  8-thread mixed stress, 10^6 ops, overlapping key ranges, disjoint-key
     partitions against a linearised oracle
  5  fill to 90% at 10^6 slots with zero FULL (open addressing)
  6  space accounting at 90% load
  7  metadata probe arithmetic (p2_md vs p2 negative queries)
  8  aging divergence (double vs p2_md negative-query probes after 200 its)
  9  stability of slot addresses across 10^5 operations
  13 probe means flat across table sizes
"""

import json
import os
import sys
import threading

import numpy as np
import pytest

from conftest import ALL_DESIGNS, GOLDEN, cfg_for

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
U64 = np.uint64
OPEN_ADDRESSING = ["double", "double_md", "p2", "p2_md", "iceberg", "iceberg_md", "cuckoo"]


def _cu(a):
    a = np.ascontiguousarray(a)
    if a.dtype == np.uint8:
        return torch.from_numpy(a).cuda()
    return torch.from_numpy(a.astype(U64, copy=False).view(np.int64)).cuda().view(torch.uint64)


def _np(t):
    t = t.cpu()
    return t.view(torch.int64).numpy().view(U64) if t.dtype == torch.uint64 else t.numpy()


def _spec():
    sys.path.insert(0, GOLDEN)
    import spec_stream
    return spec_stream, json.load(open(os.path.join(GOLDEN, "spec_equivalence.json")))


# ----------------------------------------------------------------- SPEC 3

@pytest.mark.parametrize("design", ALL_DESIGNS)
def test_spec3_oracle_equivalence_1e5_ops_three_seeds(design):
    """Each 10^5-op stream replayed in order on the device (WS_F_SERIAL): every
    status / value, the final map and the slot layout equal the reference's."""
    from paper_2509_16407_b200 import make_table
    ss, spec = _spec()
    cfg = cfg_for(design, spec["capacity"], seed=spec["table_seed"])
    for seed in spec["seeds"]:
        ref = spec["streams"][f"{design}/{seed}"]
        t = make_table(cfg)
        ops, keys, vals, _ = ss.spec_stream(t.capacity_slots, spec["n_ops"], seed)
        st, vo = t.mixed_batch(ops, keys, vals, serial=True)
        st, vo = _np(st), _np(vo)
        assert ss.digest(st) == ref["status"], (design, seed)
        assert ss.digest(vo) == ref["qvals"], (design, seed)
        k, v = t.items_arrays()
        assert len(k) == ref["n_items"] and ss.items_digest(k, v) == ref["items"], (design, seed)
        words = t._raw()[0]
        if design == "chaining":
            nn = t.arena.next_node
            lay = words[: 16 * nn].reshape(-1, 16)[:, list(range(0, 14, 2)) + [14]]
        else:
            lay = words[0::2]
        assert ss.digest(np.ascontiguousarray(lay)) == ref["layout"], (design, seed)
        assert t.duplicate_scan() == {}


# ----------------------------------------------------------------- SPEC 4

@pytest.mark.parametrize("design", ALL_DESIGNS)
def test_spec4_eight_thread_stress_1e6_ops(design):
    """8 host threads, 10^6 mixed ops in total: each thread owns a key
    partition (erase / query / fresh inserts on its own keys, so a
    per-thread sequential oracle is exact) and all threads upsert-ADD a
    shared hot set (overlapping ranges; ADD commutes).  Batches go through
    the C ABI concurrently on one table."""
    from oracle import OracleTable
    from paper_2509_16407_b200 import make_table
    from paper_2509_16407_b200.workload import gen_uniform_keys

    nt, per_thread, rounds = 8, 125_000, 5
    cfg = cfg_for(design, 1 << 21 if design != "chaining" else 7 * (1 << 18), seed=4)
    t = make_table(cfg)
    o = OracleTable(cfg)
    own = gen_uniform_keys(41, nt * 40_000).reshape(nt, 40_000)
    hot = gen_uniform_keys(42, 4096)
    pre = own[:, :20_000].ravel()
    t.upsert_batch(_cu(pre), _cu(pre & U64(0xFFFF)))
    o.upsert_batch(pre, pre & U64(0xFFFF))
    per_round = per_thread // rounds                     # 25,000 ops per batch
    plans = []
    for i in range(nt):
        rng = np.random.default_rng(1000 + i)
        rnd = []
        for r in range(rounds):
            er = own[i, r * 2000:(r + 1) * 2000]          # erase 2000 prefilled keys
            qy = own[i, 10_000 + r * 2000:10_000 + (r + 1) * 2000]   # query 2000 prefilled keys
            fr = own[i, 20_000 + r * 4000:20_000 + (r + 1) * 4000]   # insert 4000 fresh keys
            hk = hot[rng.integers(0, len(hot), per_round - 8000)]    # upsert-ADD hot keys
            ops = np.concatenate([np.full(2000, 1), np.full(2000, 2), np.full(4000, 0 | (2 << 4)),
                                  np.full(len(hk), 0 | (2 << 4))]).astype(np.uint8)
            keys = np.concatenate([er, qy, fr, hk])
            vals = np.concatenate([np.zeros(4000, U64), np.full(4000, 3, U64), np.ones(len(hk), U64)])
            perm = rng.permutation(len(ops))
            rnd.append((ops[perm], keys[perm], vals[perm]))
        plans.append(rnd)
    results = [None] * nt
    errors = []
    barrier = threading.Barrier(nt)

    def work(i):
        try:
            barrier.wait()
            out = []
            for ops, keys, vals in plans[i]:
                st, vo = t.mixed_batch(_cu(ops), _cu(keys), _cu(vals))
                out.append((_np(st), _np(vo)))
            results[i] = out
        except BaseException as exc:  # noqa: BLE001
            errors.append(exc)

    ths = [threading.Thread(target=work, args=(i,)) for i in range(nt)]
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    assert not errors, errors[0]
    for i in range(nt):
        for (ops, keys, vals), (st, vo) in zip(plans[i], results[i]):
            er, qy = ops == 1, ops == 2
            assert st[er].all() and st[qy].all()
            assert (vo[qy] == (keys[qy] & U64(0xFFFF))).all()
            fresh = np.isin(keys, own[i, 20_000:]) & (ops == 32)
            assert (st[fresh] == 0).all()
            o.mixed_batch(ops, keys, vals)   # role-disjoint batch: any order is the same
    assert dict(zip(*[a.tolist() for a in t.items_arrays()])) == o.as_dict()
    assert t.duplicate_scan() == {}


# ----------------------------------------------------------------- SPEC 5

@pytest.mark.parametrize("design", OPEN_ADDRESSING)
def test_spec5_fill_to_90_percent_at_1e6_slots(design):
    """Zero FULL wherever the reference's own sequential fill has none.  With
    this seed the reference itself reports FULL for double_md (key 897,565 of
    the stream: its zero-count cap makes a 512-bucket walk find no claimable
    cell; checked against /root/reference), so there the device's serial
    replay must report exactly the oracle's FULL set and the concurrent fill
    may differ from it only by batch-order effects."""
    from oracle import OracleTable
    from paper_2509_16407_b200 import make_table
    from paper_2509_16407_b200.workload import gen_uniform_keys
    cfg = cfg_for(design, 1_000_000, seed=42)
    t = make_table(cfg)
    n = int(t.capacity_slots * 0.9)
    keys = gen_uniform_keys(42, n)
    ost = OracleTable(cfg).upsert_batch(keys, keys)
    ofull = int((ost == 2).sum())
    st = _np(t.upsert_batch(_cu(keys), _cu(keys)))
    fulls = int((st == 2).sum())
    assert ((st == 0) | (st == 2)).all()
    if ofull == 0:
        assert fulls == 0
    else:
        assert fulls <= ofull + 2, (fulls, ofull)
        ts = make_table(cfg)
        sst, _ = ts.mixed_batch(np.zeros(n, np.uint8), keys, keys, serial=True)
        np.testing.assert_array_equal(_np(sst), ost)
    assert t.occupied_count() == n - fulls
    f, v = t.query_batch(_cu(keys))
    f = _np(f).astype(bool)
    assert f.sum() == n - fulls and (_np(v)[f] == keys[f]).all()


# ----------------------------------------------------------------- SPEC 6

def test_spec6_space_accounting_at_90_percent():
    """reference tests/test_tables.py:390-424."""
    from paper_2509_16407_b200 import TableConfig, make_table
    from paper_2509_16407_b200.workload import gen_uniform_keys
    t = make_table(TableConfig(design="p2", capacity_slots=1 << 12, seed=3))
    target = int(t.capacity_slots * 0.9)
    keys = np.arange(1, target + 1, dtype=U64)
    assert (_np(t.upsert_batch(_cu(keys), _cu(np.ones(target, U64)))) == 0).all()
    rep = t.storage_report()
    assert rep["space_efficiency"] == pytest.approx(0.90, abs=5e-4)
    assert rep["space_efficiency"] == target / t.capacity_slots
    assert rep["bytes_per_pair"] == pytest.approx(16 / 0.9, rel=0.01)
    assert t.bytes_per_pair() == rep["bytes_per_pair"]
    t = make_table(TableConfig(design="p2_md", capacity_slots=1 << 12, seed=3))
    assert (_np(t.upsert_batch(_cu(keys), _cu(np.ones(target, U64)))) == 0).all()
    assert t.storage_report()["space_efficiency"] == pytest.approx(0.80, abs=0.001)
    cap = 7 * 2000
    t = make_table(TableConfig(design="chaining", capacity_slots=cap, seed=3))
    k = gen_uniform_keys(5, int(cap * 0.9))
    t.upsert_batch(_cu(k), _cu(np.ones(len(k), U64)))
    assert 0.35 <= t.storage_report()["space_efficiency"] <= 0.55
    # at the north-star size the report is computed on the device (no table copy)
    big = make_table(TableConfig(design="p2_md", capacity_slots=1 << 26, seed=3))
    n = int(big.capacity_slots * 0.9)
    kb = gen_uniform_keys(6, n)
    assert (_np(big.upsert_batch(_cu(kb), _cu(kb))) == 0).all()
    rep = big.storage_report()
    assert rep["occupied"] == n
    assert rep["space_efficiency"] == pytest.approx(0.80, abs=0.001)


# ----------------------------------------------------------------- SPEC 7

def test_spec7_metadata_probe_arithmetic():
    """line_bytes 128, bucket 32, >= 85% load: p2_md negative-query mean line
    probes in [1.8, 2.6]; plain p2 at least 3x that (paper: 8 -> 2)."""
    from paper_2509_16407_b200 import TableConfig, make_table
    from paper_2509_16407_b200.workload import derive_seed, gen_uniform_keys
    means = {}
    for design in ("p2_md", "p2"):
        t = make_table(TableConfig(design=design, capacity_slots=1 << 20, seed=42, line_bytes=128))
        n = int(t.capacity_slots * 0.88)
        k = gen_uniform_keys(42, n)
        assert (_np(t.upsert_batch(_cu(k), _cu(k))) == 0).all()
        neg = gen_uniform_keys(derive_seed(42, 0xFEED), 4096)
        _s, _v, pr, _l = t.probe_batch(np.full(4096, 2, np.uint8), neg, serial=True)
        means[design] = float(pr.mean())
    assert 1.8 <= means["p2_md"] <= 2.6, means
    assert means["p2"] >= 3 * means["p2_md"], means


# ----------------------------------------------------------------- SPEC 8

def test_spec8_aging_divergence_double_vs_p2md():
    """200 aging iterations of the reference's workload at 10^5 slots:
    double hashing's negative-query probe mean ends >= 3x p2_md's."""
    from paper_2509_16407_b200.runners import run_aging_uniform
    last = {}
    for design in ("double", "p2_md"):
        rep = run_aging_uniform(design, 1 << 17, iterations=200, seed=42)
        assert rep["ok"], design
        assert rep["occupied"] == rep["fill_n"]  # every iteration inserts and erases one slice
        tail = rep["iterations"][-20:]
        last[design] = float(np.mean([i["probe_means"]["query_neg"] for i in tail]))
    assert last["double"] >= 3 * last["p2_md"], last


# ----------------------------------------------------------------- SPEC 9

@pytest.mark.parametrize("design", ["double", "double_md", "p2", "p2_md", "iceberg", "iceberg_md",
                                    "chaining"])
def test_spec9_slot_stability_across_1e5_ops(design):
    """reference tests/test_tables.py:99-113 at SPEC.md:665's scale: tracked
    keys never move while 10^5 other inserts / erases run (concurrent
    batches), checked through slot_of and locate_batch."""
    from paper_2509_16407_b200 import make_table
    from paper_2509_16407_b200.workload import gen_uniform_keys
    t = make_table(cfg_for(design, 1 << 18, seed=5))
    tracked = gen_uniform_keys(77, 3000)
    t.upsert_batch(_cu(tracked), _cu(tracked))
    addr = t.locate_batch(tracked)
    assert (addr >= 0).all()
    assert all(t.slot_of(int(k)) == int(a) for k, a in zip(tracked[:50], addr[:50]))
    churn = gen_uniform_keys(78, 70_000)
    for lo in range(0, 70_000, 10_000):
        c = churn[lo:lo + 10_000]
        t.upsert_batch(_cu(c), _cu(c))
        t.erase_batch(_cu(c[::3]))  # 10^5 ops in total with the inserts
        assert (t.locate_batch(tracked) == addr).all()
    assert (t.locate_batch(tracked) == addr).all()


# ----------------------------------------------------------------- SPEC 13

@pytest.mark.parametrize("design", ["p2_md", "double", "iceberg_md"])
def test_spec13_probe_means_flat_across_sizes(design):
    """Probe means at 0.9 load within 2% from ~10^5 to ~10^7 slots
    (paper §6.4: probe counts do not change with table size)."""
    from paper_2509_16407_b200.runners import run_scaling
    # the instrumented inserts cover the same load window [0.895, 0.9) at
    # every size (a fixed sample count would span 6% of load at 2^17); that
    # window holds only 655 inserts at 2^17, whose probe mean has a ~3%
    # standard error for the double-hashing designs, so the small sizes are
    # averaged over independent tables (seeds) until each mean rests on
    # >= ~5000 instrumented inserts
    sizes = (1 << 17, 1 << 20, 1 << 23)
    reps = {1 << 17: 8, 1 << 20: 1, 1 << 23: 1}
    means = {}
    for size in sizes:
        acc = {}
        for r in range(reps[size]):
            rep = run_scaling(design, sizes=(size,), seed=42 + r, probe_sample=8192, probe_window=0.005)
            ps = rep["per_size"][0]
            assert ps["fulls"] == 0 and ps["missing"] == 0, ps
            for kind, v in ps["probe_means"].items():
                acc.setdefault(kind, []).append(v)
        means[size] = {k: sum(v) / len(v) for k, v in acc.items()}
    for kind in ("insert", "query_pos", "query_neg"):
        vals = [means[size][kind] for size in sizes]
        ref = vals[-1]
        assert all(abs(v - ref) <= 0.02 * ref + 0.02 for v in vals), (kind, vals)


# ------------------------------------------------------- BASELINE config 1

def test_config1_exact_size():
    """BASELINE config 1 at its stated size: double hashing, 2^20 slots,
    891,289 inserts (0.85), 2^19 interleaved 50/50 queries; every status and
    value checked (runners.run_config1 verifies against the inputs)."""
    from paper_2509_16407_b200.runners import run_config1
    rep = run_config1(seed=42, capacity=1 << 20, design="double")
    assert rep["ok"], rep
    assert rep["rows"][0].ops == 891_289 and rep["rows"][1].ops == 1 << 19

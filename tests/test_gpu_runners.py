"""Small-size runs of the device workload runners (every runner self-checks)."""
import pytest

pytestmark = pytest.mark.gpu
pytest.importorskip("torch")


def test_config1_double():
    from paper_2509_16407_b200 import runners
    assert runners.run_config1(capacity=1 << 16)["ok"]


@pytest.mark.parametrize("design,cap", [("cuckoo", 1 << 16), ("chaining", 7 * 4096), ("p2_md", 1 << 16),
                                        ("iceberg_md", 1 << 16), ("double", 1 << 16)])
def test_load_sweep(design, cap):
    from paper_2509_16407_b200 import runners
    r = runners.run_load_sweep(design, cap, load_points=(0.5, 0.7, 0.9), query_sample=1 << 14,
                               probe_sample=512, drain=design != "chaining")
    assert all(p.get("queries_ok", True) for p in r["points"])
    if design != "chaining":
        assert r["points"][-1]["after_drain_occupied"] == 0
    assert r["points"][0]["probes_query_pos"] >= 1.0


@pytest.mark.parametrize("design", ["iceberg_md", "p2_md", "chaining"])
def test_aging_zipf(design):
    from paper_2509_16407_b200 import runners
    cap = 7 * 4096 if design == "chaining" else 1 << 16
    r = runners.run_aging(design, cap, iterations=6, slice_fraction=0.02)
    assert r["ok"] and r["checksum_ok"] and r["duplicates"] == 0, r


def test_kmer_counts():
    from paper_2509_16407_b200 import runners
    r = runners.run_kmer(genome_len=1 << 18, capacity=1 << 19)
    assert r["ok"], r


@pytest.mark.parametrize("wl", ["A", "B", "C"])
def test_ycsb_final_values_exact(wl):
    from paper_2509_16407_b200 import runners
    r = runners.run_ycsb(wl, universe=1 << 16, ops=1 << 18, batch=1 << 16)
    assert r["missing_queries"] == 0 and r["final_values_exact"], r


# ---- BASELINE configs 3 and 4 at their stated sizes (the runners above are
# the small-size versions; these are the sizes the SURVEY 8(d) table names)

@pytest.mark.parametrize("design", ["iceberg_md", "iceberg"])
def test_config3_aging_full_size(design):
    """Config 3: iceberg(_md) at 2^26 slots prefilled to 0.85, Zipf(0.99)
    upsert-ADD + fresh inserts + erase of the oldest slice + present / absent
    queries per mixed batch; every status / value and the final checksum
    exact, zero duplicates."""
    from paper_2509_16407_b200 import runners
    r = runners.run_aging(design, 1 << 26, iterations=4)
    assert r["ok"] and r["checksum_ok"] and r["duplicates"] == 0, {k: r[k] for k in r if k != "rows"}


@pytest.mark.parametrize("design,cap", [("cuckoo", 1 << 26), ("chaining", 7 * (1 << 23))])
def test_config4_fill_to_095_full_size(design, cap):
    """Config 4 at its stated sizes: fill to 0.5 then in 0.05 slices to 0.95
    (cuckoo eviction chains near the top); after every slice the occupied
    count equals the keys inserted minus FULL statuses, and at 0.95 the
    table's checksum equals numpy's over the stored keys, every stored key is
    found with its value, no absent key is found, zero duplicates."""
    import numpy as np
    import torch
    from paper_2509_16407_b200 import TableConfig, make_table
    from paper_2509_16407_b200.workload import derive_seed, gen_uniform_keys, mix64_np
    t = make_table(TableConfig(design=design, capacity_slots=cap, seed=42))
    n = int(cap * 0.95)
    keys = gen_uniform_keys(42, n)
    vals = keys & np.uint64(0xFFFF)

    def dev(a):
        return torch.from_numpy(a.view(np.int64)).cuda().view(torch.uint64)
    stored = np.ones(n, dtype=bool)
    bounds = [0, int(cap * 0.5)] + [int(cap * (0.5 + 0.05 * i)) for i in range(1, 10)]
    for lo, hi in zip(bounds[:-1], bounds[1:]):
        st = t.upsert_batch(dev(keys[lo:hi]), dev(vals[lo:hi])).cpu().numpy()
        assert not (st == 1).any()
        stored[lo:hi] = st == 0
        assert t.occupied_count() == int(stored[:hi].sum())
    assert int((~stored).sum()) <= n // 1000, "more than 0.1% FULL"
    ks, vs = keys[stored], vals[stored]
    with np.errstate(over="ignore"):
        want = (len(ks), int(ks.sum(dtype=np.uint64)), int(vs.sum(dtype=np.uint64)),
                int(np.bitwise_xor.reduce(mix64_np(ks ^ mix64_np(vs)))))
    assert t.checksum() == want
    q = np.concatenate([ks[:: max(1, len(ks) // (1 << 22))], gen_uniform_keys(derive_seed(42, 0xFEED), 1 << 20)])
    f, v = t.query_batch(dev(q))
    f, v = f.cpu().numpy().astype(bool), v.cpu().view(torch.int64).numpy().view(np.uint64)
    npos = len(q) - (1 << 20)
    assert f[:npos].all() and not f[npos:].any()
    assert (v[:npos] == (q[:npos] & np.uint64(0xFFFF))).all()
    assert t.duplicate_count() == 0


def test_config5_device_kmer_counting():
    """runners.run_kmer_full (config 5's full-size runner, device-generated
    genome) at 2^24 slots: no FULL, no duplicates, exact value sum, every
    k-mer found with a multiple of the repeat count."""
    from paper_2509_16407_b200 import runners
    r = runners.run_kmer_full(log2_slots=24, repeats=3, chunk=1 << 22)
    assert r["ok"], r

"""Device adversarial duplicate-key race (paper §4.1; reference
tests/test_bench.py:153-169): safe designs never commit a key twice, the
lock-elided unsafe reference does, and a serial replay never does."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

SAFE = ["double", "double_md", "p2", "p2_md", "iceberg", "iceberg_md", "cuckoo", "chaining"]


@pytest.mark.parametrize("design", SAFE)
def test_safe_designs_zero_duplicates_heavy_delays(design):
    from paper_2509_16407_b200.adversarial import DelayProfile, run_adversarial
    rep = run_adversarial(design, buckets=4000, trials=3, seed=5, profile=DelayProfile(0.35, 20_000))
    assert rep["duplicate_buckets"] == 0, rep


@pytest.mark.parametrize("design", ["p2_md", "iceberg_md", "double_md", "cuckoo"])
def test_safe_large_no_delay(design):
    """Without delay injection the interleaved actors run through the tuned
    single-launch mixed kernels (k_mixed_p2md_rounds, k_mixed_icemd_rounds)
    where they exist: still no duplicate."""
    from paper_2509_16407_b200.adversarial import DelayProfile, run_adversarial
    rep = run_adversarial(design, buckets=200_000, trials=5, seed=11, profile=DelayProfile.off())
    assert rep["duplicate_buckets"] == 0, rep


@pytest.mark.parametrize("design", ["p2_md", "iceberg_md"])
def test_spec_scale_hundred_trials_fused_kernels(design):
    """SPEC.md:657 scale (>= 100 trials x 10^4 buckets, co-scheduled actors)
    through the fused mixed kernels (no delays): 0 duplicates."""
    from paper_2509_16407_b200.adversarial import DelayProfile, run_adversarial
    rep = run_adversarial(design, buckets=10_000, trials=100, seed=13, profile=DelayProfile.off())
    assert rep["trials"] == 100 and rep["duplicate_buckets"] == 0, rep


@pytest.mark.parametrize("design", SAFE)
def test_spec_scale_hundred_trials_co_scheduled(design):
    """SPEC.md:657 acceptance: >= 100 trials x 10^4 primary buckets (the
    reference CLI default, cli.py:321-322), the three actors of each bucket
    in adjacent warps of one CTA (actor_layout), light delays: 0 duplicates."""
    from paper_2509_16407_b200.adversarial import DelayProfile, run_adversarial
    rep = run_adversarial(design, buckets=10_000, trials=100, seed=7, profile=DelayProfile(0.04, 5_000))
    assert rep["trials"] == 100 and rep["replays"] == 1_000_000
    assert rep["duplicate_buckets"] == 0, rep


def test_unsafe_reference_races_at_spec_scale():
    """The positive control at the same scale finds duplicates (co-scheduled
    actors, no delays needed to expose the lock-elided race)."""
    from paper_2509_16407_b200.adversarial import DelayProfile, run_adversarial
    rep = run_adversarial("unsafe_reference", buckets=10_000, trials=100, seed=7,
                          profile=DelayProfile(0.04, 5_000))
    assert rep["duplicate_buckets"] >= 1, rep
    assert sum(1 for d in rep["per_trial"] if d) >= 10, rep["per_trial"]


def test_unsafe_reference_races():
    from paper_2509_16407_b200.adversarial import DelayProfile, run_adversarial
    rep = run_adversarial("unsafe_reference", buckets=20_000, trials=3, seed=5,
                          profile=DelayProfile(0.35, 20_000))
    assert rep["duplicate_buckets"] >= 1, rep


def test_serial_replay_never_races():
    """The same three-actor script replayed in index order on one device
    thread (reference single_thread=True) gives zero duplicates even for the
    unsafe design."""
    from paper_2509_16407_b200 import make_table
    from paper_2509_16407_b200.adversarial import config_for_primary_buckets, generate_pairs
    cfg = config_for_primary_buckets("unsafe_reference", 3000, 5)
    t = make_table(cfg)
    xs, ys = generate_pairs(t, 3000, 5)
    t.upsert_batch(xs, np.ones(3000, np.uint64))
    ops, keys, vals = [], [], []
    for b in range(3000):  # the reference's per-bucket actor order
        ops += [1, 0 | (1 << 4), 0 | (1 << 4)]
        keys += [xs[b], ys[b], ys[b]]
        vals += [0, 1, 2]
    st, _ = t.mixed_batch(np.array(ops, np.uint8), np.array(keys, np.uint64), np.array(vals, np.uint64),
                          serial=True)
    assert t.duplicate_scan() == {}
    assert dict(t.items()) == {int(y): 1 for y in ys}


@pytest.mark.parametrize("design", ["unsafe_reference", "p2_md", "iceberg_md", "cuckoo", "double"])
def test_duplicate_scan_by_locate_agrees_with_sort(design):
    """The chunked search-based duplicate scan (used when a table is too
    large to sort its keys beside it, e.g. 2^32 slots) agrees with the
    sort-based one: on the unsafe design's raced table (duplicates stored
    twice) and on safe tables (none); the test hook WS_DUPSCAN_BY_LOCATE
    forces the search-based path."""
    from paper_2509_16407_b200.adversarial import DelayProfile, run_adversarial
    rep = run_adversarial(design, buckets=20_000, trials=1, seed=5, profile=DelayProfile(0.35, 20_000),
                          keep_table=True)
    t = rep["table"]
    by_sort = t.duplicate_count()
    import os
    os.environ["WS_DUPSCAN_BY_LOCATE"] = "1"
    try:
        by_locate = t.duplicate_count()
    finally:
        del os.environ["WS_DUPSCAN_BY_LOCATE"]
    assert by_locate == by_sort
    if design == "unsafe_reference":
        assert by_sort >= 1
    else:
        assert by_sort == 0

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

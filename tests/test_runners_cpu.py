"""Host-side runner plumbing (no GPU): the reference CSV manifest and schema
written by runners.write_report_csv, and the ncu range hook being inert
unless WS_NCU_RANGES is set."""

import os

from paper_2509_16407_b200 import __version__, runners
from paper_2509_16407_b200.core import TableConfig
from paper_2509_16407_b200.instrument import CSV_HEADER, Row

# reference bench/runners.py:66-86 (manifest_lines), in order
REF_MANIFEST_KEYS = ["benchmark", "design", "capacity_slots", "bucket_size", "line_bytes", "probe_cap",
                     "mode", "seed", "threads", "slot_engine", "wide_atomic", "num_buckets", "version",
                     "timestamp"]


class _FakeTable:
    def __init__(self, cfg):
        self.config = cfg
        self.capacity_slots = cfg.capacity_slots
        self.bucket_size = 32
        self.num_buckets = cfg.capacity_slots // 32

    def capability_report(self):
        return {"slot_engine": "packed", "wide_atomic": True}


def test_manifest_matches_reference_fields(tmp_path):
    t = _FakeTable(TableConfig(design="p2_md", capacity_slots=1 << 16, seed=7))
    lines = runners.manifest_lines("load", t, 7, ["fulls=0"])
    keys = [ln.split("=", 1)[0] for ln in lines]
    assert keys[: len(REF_MANIFEST_KEYS)] == REF_MANIFEST_KEYS
    assert keys[-1] == "fulls"
    kv = dict(ln.split("=", 1) for ln in lines)
    assert kv["design"] == "p2_md" and kv["seed"] == "7" and kv["num_buckets"] == "2048"
    assert kv["version"] == __version__
    rows = [Row("p2_md", "concurrent", 1 << 16, 128, "throughput", "insert", 0.5, 0, 10, 0.001, 0.01),
            Row("p2_md", "concurrent", 1 << 16, 128, "probe", "insert", 0.5, 1, 10, 0.0, 0.0, 3.5)]
    path = runners.write_report_csv(str(tmp_path), "load", t, rows, 7, ["fulls=0"])
    assert os.path.basename(path) == "load_p2_md.csv"
    text = open(path).read().splitlines()
    body = [ln for ln in text if not ln.startswith("#")]
    assert all(ln.startswith("# ") for ln in text[: len(lines)])
    assert body[0] == CSV_HEADER and len(body) == 3
    assert body[2].split(",")[-1] == "3.5000"


def test_ncu_range_is_inert_without_env(monkeypatch):
    monkeypatch.delenv("WS_NCU_RANGES", raising=False)
    with runners._ncu_range({"design": "p2_md", "op": "insert", "load": 0.5}, 10):
        pass  # must not touch torch.cuda (no GPU here)

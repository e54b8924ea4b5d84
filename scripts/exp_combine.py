"""Combining / aging timing on the current build: iceberg_md and p2_md aging
at 2^26 (Zipf 0.99 upsert-ADD + fresh inserts + erases + present / absent
queries, every result and the final checksum verified), k-mer counting with
combining, YCSB A/B/C."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_16407_b200 import runners  # noqa: E402

for design in ("iceberg_md", "p2_md"):
    r = runners.run_aging(design, 1 << 26, iterations=40, combine=True)
    r.pop("rows")
    its = r.pop("iterations")
    ms = sorted(i["ms"] for i in its)
    print("aging", design, json.dumps(r), "median ms/iteration", round(ms[len(ms) // 2], 3), flush=True)
for comb in (False, True):
    r = runners.run_kmer(genome_len=1 << 27, capacity=1 << 26, repeats=4, combine=comb)
    print("kmer combine", comb, r, flush=True)
for wl in ("A", "B", "C"):
    print("ycsb", runners.run_ycsb(wl, universe=1 << 24, ops=1 << 26), flush=True)

"""YCSB A / B / C through runners.run_ycsb (2^24 universe, 2^26 Zipf ops)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_16407_b200 import runners  # noqa: E402

for wl in ("A", "B", "C"):
    r = runners.run_ycsb(wl, universe=1 << 24, ops=1 << 26)
    print(wl, {k: r[k] for k in ("mops", "final_values_exact", "missing_queries")}, flush=True)

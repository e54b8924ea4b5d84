"""Aging (config 3) iterations for a launch-list capture."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_16407_b200 import runners  # noqa: E402

r = runners.run_aging("iceberg_md", 1 << 26, iterations=int(sys.argv[1]) if len(sys.argv) > 1 else 3, combine=True)
print({k: v for k, v in r.items() if k not in ("iterations", "rows")}, [round(i["ms"], 3) for i in r["iterations"]])

"""CPU oracle for the hash-table hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` leg may import this package, and only as the checker or
the CPU baseline.  The product package (paper_2509_16407_b200) never imports it.

``ws_oracle.c`` is a sequential C restatement of the reference package's
table algorithms (warpbench, /root/reference/pkg/src/warpbench/tables/*);
``table.py`` wraps it with numpy batch drivers.  Parity of the oracle itself
is pinned by tests/test_oracle.py against fixtures generated from the
reference (tests/golden/make_golden.py).
"""

from .table import OracleTable, build_oracle, load_oracle  # noqa: F401

"""Run the reference's OWN table tests against the drop-in (on a GPU box).

The reference's pkg/tests/{test_tables,test_core}.py (with their
conftest.py / oracle.py) are copied, unmodified and uncommitted, into
baseline/_ref/ref_tests/ (git-ignored, next to the pip-installed reference;
`cp /root/reference/pkg/tests/{test_tables,conftest,oracle,test_core}.py
baseline/_ref/ref_tests/`).  The benchmark-harness tests (test_bench,
test_instrument's throughput samples, test_cli, test_apps) and the
reference-internal test_sync are not part of the drop-in's surface.  Here the module names they
import -- warpbench.core, .instrument, .tables, .tables.base / .openaddr /
.cuckoo / .chaining -- are bound to the drop-in package, so every
`make_table(...)` in them builds a device table, and pytest runs them.

  python scripts/run_reference_tests.py [-k expr] [-x]
"""
import os
import sys
import types

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
TESTS = os.path.join(ROOT, "baseline", "_ref", "ref_tests")

import pytest  # noqa: E402

if "--harness" in sys.argv:
    # The reference's harness tests (test_bench.py, test_apps.py, copied into
    # baseline/_ref/ref_tests_harness/): the REAL reference package from
    # baseline/_ref -- its runners, adversarial driver and apps -- with its
    # table factory and status enum rebound to the drop-in, so every table
    # those callers build is a device table driven through the scalar API.
    sys.argv.remove("--harness")
    sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
    import importlib

    from paper_2509_16407_b200 import tables as dev_tables
    names = ["warpbench.tables", "warpbench.bench.runners", "warpbench.bench.adversarial", "warpbench.apps.cache",
             "warpbench.apps.ycsb", "warpbench.apps.tensor", "warpbench.cli"]
    for name in names:
        m = importlib.import_module(name)
        for attr, val in (("make_table", dev_tables.make_table), ("UpsertStatus", dev_tables.UpsertStatus)):
            if hasattr(m, attr):
                setattr(m, attr, val)
    HARNESS = os.path.join(ROOT, "baseline", "_ref", "ref_tests_harness")
    sys.exit(pytest.main([HARNESS, "-q", "-p", "no:cacheprovider", "--rootdir", HARNESS, *sys.argv[1:]]))

import paper_2509_16407_b200 as pkg  # noqa: E402
from paper_2509_16407_b200 import core, instrument, tables, workload  # noqa: E402

wb = types.ModuleType("warpbench")
wb.__dict__.update({k: v for k, v in vars(pkg).items() if not k.startswith("__")})
wb.__path__ = []  # a package, so submodule imports resolve through sys.modules
tpkg = types.ModuleType("warpbench.tables")
tpkg.__dict__.update({k: v for k, v in vars(tables).items() if not k.startswith("__")})
tpkg.__path__ = []
mods = {"warpbench": wb, "warpbench.core": core, "warpbench.instrument": instrument,
        "warpbench.tables": tpkg}
for sub in ("base", "openaddr", "cuckoo", "chaining"):
    mods[f"warpbench.tables.{sub}"] = tables
bpkg = types.ModuleType("warpbench.bench")  # only the key generators (bench/keys.py) are on the path
bpkg.__path__ = []
bpkg.keys = workload
mods["warpbench.bench"] = bpkg
mods["warpbench.bench.keys"] = workload
wb.core, wb.instrument, wb.tables = core, instrument, tpkg
sys.modules.update(mods)

if not os.path.isdir(TESTS):
    sys.exit(f"copy the reference tests into {TESTS} first (see the docstring)")
sys.exit(pytest.main([TESTS, "-q", "-p", "no:cacheprovider", "--rootdir", TESTS, *sys.argv[1:]]))

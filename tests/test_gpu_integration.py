"""INTEGRATION.md section 2 executed: the ctypes `B200Table` binding a
`warpbench` maintainer would add (the reference has no FFI of its own) is
extracted from the document verbatim, bound to the in-tree libwarpspeed.so,
and driven through scalar upsert / query / erase against the CPU oracle.

The binding imports `warpbench.core` / `warpbench.tables.base`.  The
unmodified reference package is used when it is installed in baseline/_ref
(bench.py's reference arm installs it there); otherwise the drop-in
package's own `core` / `UpsertStatus` stand in under those module names.
"""

import os
import random
import re
import sys
import types

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _binding_source():
    doc = open(os.path.join(ROOT, "INTEGRATION.md"), encoding="utf-8").read()
    sec = doc.split("## 2.", 1)[1]
    src = re.search(r"```python\n(.*?)```", sec, re.S).group(1)
    from paper_2509_16407_b200 import _native
    lib = _native.load()
    return src.replace('C.CDLL("libwarpspeed.so")', f"C.CDLL({lib._name!r})"), lib


def _warpbench_modules():
    ref = os.path.join(ROOT, "baseline", "_ref")
    if os.path.isdir(os.path.join(ref, "warpbench")):
        sys.path.insert(0, ref)
        try:
            import warpbench.core  # noqa: F401
            import warpbench.tables.base  # noqa: F401
            return "reference"
        finally:
            sys.path.remove(ref)
    from paper_2509_16407_b200 import core, tables
    pkg = types.ModuleType("warpbench")
    tpkg = types.ModuleType("warpbench.tables")
    base = types.ModuleType("warpbench.tables.base")
    base.UpsertStatus = tables.UpsertStatus
    pkg.core, pkg.tables, tpkg.base = core, tpkg, base
    sys.modules.update({"warpbench": pkg, "warpbench.core": core, "warpbench.tables": tpkg,
                        "warpbench.tables.base": base})
    return "drop-in stand-in"


@pytest.mark.parametrize("design", ["p2_md", "double", "iceberg_md", "cuckoo"])
def test_integration_binding_matches_oracle(design):
    from oracle import OracleTable
    from paper_2509_16407_b200.core import TableConfig as OurCfg
    saved = {k: v for k, v in sys.modules.items() if k == "warpbench" or k.startswith("warpbench.")}
    try:
        which = _warpbench_modules()
        src, _lib = _binding_source()
        ns = {}
        exec(compile(src, "INTEGRATION.md#2", "exec"), ns)
        from warpbench.core import TableConfig
        from warpbench.tables.base import UpsertStatus
        cap = 1 << 12
        t = ns["B200Table"](TableConfig(design=design, capacity_slots=cap, seed=5))
        o = OracleTable(OurCfg(design=design, capacity_slots=cap, seed=5))
        names = {0: UpsertStatus.INSERTED, 1: UpsertStatus.UPDATED, 2: UpsertStatus.FULL}
        rng = random.Random(11)
        live = []
        for i in range(3000):
            r = rng.random()
            if r < 0.5 or not live:
                k = rng.randrange(1, 1 << 63)
                v = rng.randrange(0, 1 << 64)
                got = t.upsert(k, v)
                want = names[int(o.upsert(k, v))]
                assert got == want, (which, i, got, want)
                live.append(k)
            elif r < 0.8:
                k = rng.choice(live) if rng.random() < 0.7 else rng.randrange(1, 1 << 63)
                assert t.query(k) == o.query(k), (which, i)
            else:
                k = live.pop(rng.randrange(len(live)))
                assert t.erase(k) == o.erase(k), (which, i)
        with pytest.raises(Exception):
            t.upsert(0, 1)  # EMPTY sentinel: check_key raises before the call
    finally:
        for k in [k for k in sys.modules if k == "warpbench" or k.startswith("warpbench.")]:
            del sys.modules[k]
        sys.modules.update(saved)

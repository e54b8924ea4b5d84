"""CPU-side checks of the drop-in boundary (no GPU needed).

* libwarpspeed.so loads and exports every entry point include/warpspeed.h declares;
* the ctypes structs match the header's field order;
* merge-callback classification and host-side routing math match the reference.
"""

import os
import re

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "warpspeed.h")


def _declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"WS_API\s+(?:const\s+char\s*\*|int)\s*(ws_\w+)\s*\(", text)))


def test_header_declares_the_full_abi():
    names = _declared()
    assert "ws_create" in names and "ws_upsert" in names and "ws_query" in names
    assert len(names) == 26, names


def test_library_exports_every_declared_symbol():
    from paper_2509_16407_b200 import _native
    lib_syms = set(_native.symbols())
    assert set(_declared()) <= lib_syms
    assert set(_native.EXPORTS) == set(_declared())


def test_strerror_messages():
    from paper_2509_16407_b200 import _native
    assert "sentinel" in _native.strerror(_native.WS_ERR_INVALID_KEY)
    assert _native.strerror(0) == "ok"


def test_config_struct_matches_header_order():
    from paper_2509_16407_b200 import _native
    text = open(HEADER).read()
    body = text[text.index("typedef struct ws_config"):text.index("} ws_config;")]
    fields = re.findall(r"^\s*(?:int32_t|uint64_t)\s+(\w+)", body, flags=re.M)
    assert fields == [f[0] for f in _native.WsConfig._fields_]


def test_merge_classification():
    from paper_2509_16407_b200.tables import merge_id

    def add(old, new):  # reference test_tables.py:18 style (unmasked)
        return old + new

    def keep(old, _new):
        return old

    assert merge_id(None) == 0
    assert merge_id(keep) == 1
    assert merge_id(add) == 2
    assert merge_id(max) == 3
    assert merge_id(min) == 4
    assert merge_id("add") == 2
    with pytest.raises(TypeError):
        merge_id(lambda o, n: o * n)
    with pytest.raises(TypeError):
        merge_id(lambda o, n: o - n)


def test_table_without_gpu_raises_not_falls_back():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2509_16407_b200 import TableConfig, make_table
    with pytest.raises(RuntimeError, match="CUDA"):
        make_table(TableConfig(design="p2_md", capacity_slots=1024))


def test_derived_constants_match_reference_rules():
    from paper_2509_16407_b200.core import TableConfig, derive
    d = derive(TableConfig(design="p2_md", capacity_slots=1 << 20))
    assert (d.bucket_size, d.num_buckets, d.shortcut_slots, d.zero_count_cap) == (32, 1 << 15, 24, 9)
    d = derive(TableConfig(design="iceberg", capacity_slots=1 << 20))
    assert (d.front_buckets, d.back_buckets) == (27197, 5571)
    d = derive(TableConfig(design="double", capacity_slots=1 << 20))
    assert d.num_buckets == 1 << 17

import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")

ALL_DESIGNS = ["double", "double_md", "p2", "p2_md", "iceberg", "iceberg_md",
               "cuckoo", "chaining"]


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


def cuda_ok():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if cuda_ok():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


def cfg_for(design, capacity, **kw):
    from paper_2509_16407_b200.core import DEFAULT_BUCKET_SIZE, TableConfig
    bucket = kw.get("bucket_size") or DEFAULT_BUCKET_SIZE[design]
    capacity -= capacity % bucket
    return TableConfig(design=design, capacity_slots=capacity, **kw)


@pytest.fixture(params=ALL_DESIGNS)
def design(request):
    return request.param

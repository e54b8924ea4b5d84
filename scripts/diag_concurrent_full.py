"""Concurrent fills of small tables to 0.85 (the aging prefill): FULL
statuses per trial for each design and size, to compare with the oracle's
sequential fill (which has none at these sizes)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np  # noqa: E402
import torch  # noqa: E402

from conftest import cfg_for
from paper_2509_16407_b200 import make_table
from paper_2509_16407_b200.workload import gen_uniform_keys
for d in ('double', 'p2_md', 'double_md', 'p2', 'iceberg_md'):
    for cap in (99968, 1 << 17):
        fulls = []
        for trial in range(10):
            t = make_table(cfg_for(d, cap, seed=42))
            n = int(t.capacity_slots * 0.85)
            k = gen_uniform_keys(42, n)
            kd = torch.from_numpy(k.view(np.int64)).cuda().view(torch.uint64)
            st = t.upsert_batch(kd, kd)
            fulls.append(int((st == 2).sum()))
        print(d, cap, fulls, flush=True)

"""FULL counts of bulk fills at 2^28 for several group sizes (diagnostic)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_16407_b200 import TableConfig, make_table  # noqa: E402
from paper_2509_16407_b200.workload import gen_uniform_keys  # noqa: E402

log2 = int(sys.argv[1]) if len(sys.argv) > 1 else 28
cap = 1 << log2
n = int(cap * 0.9)
keys = gen_uniform_keys(42, n)
dk = torch.from_numpy(keys.view(np.int64)).cuda().view(torch.uint64)
dv = torch.from_numpy((keys & np.uint64(0xFFFF)).view(np.int64)).cuda().view(torch.uint64)
st = torch.empty(n, dtype=torch.uint8, device="cuda")
t = make_table(TableConfig(design="p2_md", capacity_slots=cap, seed=42))
for mode in sys.argv[2:]:
    bulk, gb = (int(x) for x in mode.split(","))
    t.tune(bulk=bulk, bulk_group=gb)
    fulls = []
    for it in range(3):
        t.clear()
        t.upsert_batch(dk, dv, out=st)
        fulls.append(int((st == 2).sum()))
    print(f"bulk={bulk} group_log2={gb} FULL per fill: {fulls}", flush=True)

"""Bulk upsert vs per-op upsert timing at BASELINE config 2 (p2_md, 2^28 slots,
insert to 0.9 in one batch).  CUDA events on the table's stream; prints ms per
insert batch for both paths and checks the checksum agrees."""
import os
import sys
import time

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
res = {}
modes = (1,) if (len(sys.argv) > 2 and sys.argv[2] == 'bulk') else (0, 1, 0, 1)
for bulk in modes:
    t.tune(bulk=bulk)
    times = []
    for it in range(4):
        t.clear()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        t.upsert_batch(dk, dv, out=st)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    full = int((st == 2).sum())
    cs = t.checksum()
    res.setdefault(bulk, []).append(min(times[1:]))
    print(f"bulk={bulk} ms={['%.2f' % x for x in times]} full={full} checksum={cs}", flush=True)
print({k: min(v) for k, v in res.items()})

"""iceberg_md fill + query timing at 2^26 (tuned lock-round upsert vs generic)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2509_16407_b200 import TableConfig, make_table
from paper_2509_16407_b200.workload import gen_uniform_keys

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 26
cap = 1 << lg
n = int(cap * 0.9)
keys = gen_uniform_keys(42, n)
dk = torch.from_numpy(keys.view(np.int64)).cuda().view(torch.uint64)
dv = torch.from_numpy((keys & np.uint64(0xFFFF)).view(np.int64)).cuda().view(torch.uint64)
t = make_table(TableConfig(design="iceberg_md", capacity_slots=cap, seed=42))
for up in (4, 0, 4):
    t.tune(upsert=up)
    best = 1e9
    for _ in range(3):
        t.clear()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        st = t.upsert_batch(dk, dv, check=False)
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    print(f"upsert kernel {up}: {best:.2f} ms {n / best / 1e6:.2f} G/s statuses {np.bincount(st.cpu().numpy(), minlength=3)}"
          f" checksum {t.checksum()[:2]}", flush=True)

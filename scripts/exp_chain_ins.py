"""chaining 7*2^23: fill 0->0.5->1.0 nominal with the tuned vs generic upsert."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2509_16407_b200 import TableConfig, make_table
from paper_2509_16407_b200.workload import gen_uniform_keys

cap = 7 * (1 << 23)
keys = gen_uniform_keys(42, cap)
dk = torch.from_numpy(keys.view(np.int64)).cuda().view(torch.uint64)
t = make_table(TableConfig(design="chaining", capacity_slots=cap, seed=42))
half = cap // 2
for up in (4, 0, 4):
    t.tune(upsert=up)
    t.clear()
    torch.cuda.synchronize()
    a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    a.record()
    s1 = t.upsert_batch(dk[:half], dk[:half], check=False)
    b.record()
    s2 = t.upsert_batch(dk[half:], dk[half:], check=False)
    c.record()
    torch.cuda.synchronize()
    st = torch.cat([s1, s2]).cpu().numpy()
    print(f"upsert={up}: 0->0.5 {half / a.elapsed_time(b) / 1e6:.2f} G/s, 0.5->1.0 {(cap - half) / b.elapsed_time(c) / 1e6:.2f} G/s "
          f"statuses {np.bincount(st, minlength=3)} checksum {t.checksum()[:2]} nodes/chain {t.mean_chain_nodes():.3f}", flush=True)

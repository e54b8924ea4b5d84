"""cuckoo 2^26: fill to 0.9, then the 0.9 -> 0.95 slice (the eviction-chain
regime); prints the slice time.  Run under ncu to split the fast-path and
eviction kernels."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2509_16407_b200 import TableConfig, make_table
from paper_2509_16407_b200.workload import gen_uniform_keys

cap = 1 << int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 26
n = int(cap * 0.95)
keys = gen_uniform_keys(42, n)
t = make_table(TableConfig(design="cuckoo", capacity_slots=cap, seed=42))
dk = torch.from_numpy(keys.view(np.int64)).cuda().view(torch.uint64)
a = int(cap * 0.9)
t.upsert_batch(dk[:a], dk[:a], check=False)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
st = t.upsert_batch(dk[a:], dk[a:], check=False)
e1.record()
torch.cuda.synchronize()
print(f"slice 0.9->0.95: {n - a} ops {e0.elapsed_time(e1):.3f} ms statuses {np.bincount(st.cpu().numpy(), minlength=3)}")

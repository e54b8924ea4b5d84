"""One fill + one 50/50 query batch per design at 2^24 (for ncu captures of the
per-design tuned kernels)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2509_16407_b200 import TableConfig, make_table
from paper_2509_16407_b200.workload import derive_seed, gen_uniform_keys

for design in sys.argv[1:]:
    cap = 1 << 24
    t = make_table(TableConfig(design=design, capacity_slots=cap if design != "chaining" else 7 * (cap // 8), seed=42))
    n = int(t.capacity_slots * 0.9)
    keys = gen_uniform_keys(42, n)
    dk = torch.from_numpy(keys.view(np.int64)).cuda().view(torch.uint64)
    q = np.concatenate([keys[: n // 2], gen_uniform_keys(derive_seed(42, 0xFEED), n - n // 2)])
    np.random.default_rng(1).shuffle(q)
    dq = torch.from_numpy(q.view(np.int64)).cuda().view(torch.uint64)
    st = t.upsert_batch(dk, dk, check=False)
    f, v = t.query_batch(dq, check=False)
    torch.cuda.synchronize()
    print(design, np.bincount(st.cpu().numpy(), minlength=3)[:3], int(f.sum()))

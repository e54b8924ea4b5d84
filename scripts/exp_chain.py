"""chaining 7*2^23 slots filled to 1.0x nominal, then 50/50 queries: line-at-a-time query vs generic."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2509_16407_b200 import TableConfig, make_table
from paper_2509_16407_b200.workload import derive_seed, gen_uniform_keys

cap = 7 * (1 << 23)
n = cap
keys = gen_uniform_keys(42, n)
t = make_table(TableConfig(design="chaining", capacity_slots=cap, seed=42))
dk = torch.from_numpy(keys.view(np.int64)).cuda().view(torch.uint64)
st = t.upsert_batch(dk, dk, check=False)
print("fill statuses", np.bincount(st.cpu().numpy(), minlength=3), "chain nodes/bucket", t.mean_chain_nodes(), flush=True)
miss = gen_uniform_keys(derive_seed(42, 0xFEED), n // 2)
q = np.concatenate([keys[: n // 2], miss])
np.random.default_rng(1).shuffle(q)
dq = torch.from_numpy(q.view(np.int64)).cuda().view(torch.uint64)
ref = None
for ilp in (5, 0, 5):
    t.tune(query_ilp=ilp)
    best = 1e9
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        f, v = t.query_batch(dq, check=False)
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    cur = (f.cpu().numpy().copy(), v.cpu().view(torch.int64).numpy().copy())
    same = ref is None or (np.array_equal(cur[0], ref[0]) and np.array_equal(cur[1], ref[1]))
    ref = ref or cur
    print(f"query {'lines' if ilp else 'generic'}: {best:.2f} ms {len(q) / best / 1e6:.2f} G/s hits={int(cur[0].sum())} same={same}",
          flush=True)

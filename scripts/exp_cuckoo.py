"""cuckoo 2^26 fill to 0.9 then 50/50 queries: tuned lock-round query vs generic."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2509_16407_b200 import TableConfig, make_table
from paper_2509_16407_b200.workload import derive_seed, gen_uniform_keys

cap = 1 << 26
n = int(cap * 0.9)
keys = gen_uniform_keys(42, n)
t = make_table(TableConfig(design="cuckoo", capacity_slots=cap, seed=42))
dk = torch.from_numpy(keys.view(np.int64)).cuda().view(torch.uint64)
for up in (4, 0, 4):
    t.tune(upsert=up)
    t.clear()
    torch.cuda.synchronize()
    half = int(cap * 0.5)
    a, b, c2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    a.record()
    s1 = t.upsert_batch(dk[:half], dk[:half], check=False)
    b.record()
    s2 = t.upsert_batch(dk[half:], dk[half:], check=False)
    c2.record()
    torch.cuda.synchronize()
    st = torch.cat([s1, s2])
    print(f"fill upsert={up}: 0->0.5 {a.elapsed_time(b):.2f} ms ({half / a.elapsed_time(b) / 1e6:.2f} G/s), "
          f"0.5->0.9 {b.elapsed_time(c2):.2f} ms ({(n - half) / b.elapsed_time(c2) / 1e6:.2f} G/s) "
          f"statuses {np.bincount(st.cpu().numpy(), minlength=3)} checksum {t.checksum()[:2]}", flush=True)
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
    print(f"query {'tuned' if ilp else 'generic'}: {best:.2f} ms {len(q) / best / 1e6:.2f} G/s hits={int(cur[0].sum())} same={same}",
          flush=True)

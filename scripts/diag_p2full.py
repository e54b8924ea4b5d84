"""Repeated concurrent p2 (no metadata) fills to 0.9: count FULL statuses and,
for each FULL key, the occupancy of its two buckets after the fill."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2509_16407_b200 import TableConfig, make_table
from paper_2509_16407_b200.workload import gen_uniform_keys, mix64_np

design = sys.argv[1] if len(sys.argv) > 1 else "p2"
log2 = int(sys.argv[2]) if len(sys.argv) > 2 else 24
runs = int(sys.argv[3]) if len(sys.argv) > 3 else 20
upsert = int(sys.argv[4]) if len(sys.argv) > 4 else 4
cap = 1 << log2
n = int(cap * 0.9)
keys = gen_uniform_keys(42, n)
t = make_table(TableConfig(design=design, capacity_slots=cap, seed=42))
nb = cap // 32
t.tune(upsert=upsert)
dk = torch.from_numpy(keys.view(np.int64)).cuda().view(torch.uint64)
tot = 0
for r in range(runs):
    t.clear()
    st = t.upsert_batch(dk, dk, check=False).cpu().numpy()
    full = np.nonzero(st == 2)[0]
    tot += len(full)
    if not len(full) and r % 50:
        continue
    msg = f"run {r}: FULL {len(full)} occupied {t.occupied_count()} dups {t.duplicate_count()}"
    if len(full):
        slots = t.locate_batch(keys).astype(np.int64)
        occ = np.bincount(slots[slots >= 0] // 32, minlength=nb)
        fam = t.config.hash_family()
        for i in full[:4]:
            k = int(keys[i])
            b0, b1 = fam.bucket(0, k, nb), fam.bucket(1, k, nb)
            msg += f"\n   key idx {i}: b0 {b0} occ {occ[b0]}  b1 {b1} occ {occ[b1]}"
    print(msg, flush=True)
print(design, log2, "upsert", upsert, "runs", runs, "total FULL", tot)

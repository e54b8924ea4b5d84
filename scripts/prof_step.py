"""One bench step (clear, insert to 0.9, 50/50 query) for ncu captures.

    ncu --set full -k regex:'k_ops|k_query' -c 2 -o gpurun_out/prof python scripts/prof_step.py
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

from paper_2509_16407_b200 import TableConfig, make_table
from paper_2509_16407_b200.workload import derive_seed, gen_uniform_keys

ap = argparse.ArgumentParser()
ap.add_argument("--log2-slots", type=int, default=28)
ap.add_argument("--design", default="p2_md")
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--load", type=float, default=0.9)
ap.add_argument("--upsert", type=int, default=None)
ap.add_argument("--query", type=int, default=None)
a = ap.parse_args()

slots = 1 << a.log2_slots
n = int(slots * a.load)
t = make_table(TableConfig(design=a.design, capacity_slots=slots, seed=42))
if a.design == "p2_md":
    t.tune(query_ilp=a.query, upsert=a.upsert)
kh = gen_uniform_keys(42, n)
keys = torch.from_numpy(kh.view(np.int64)).cuda()
vals = keys & 0xFFFF
miss = torch.from_numpy(gen_uniform_keys(derive_seed(42, 0xFEED), n - n // 2).view(np.int64)).cuda()
q = torch.cat([keys[: n // 2], miss])
q = q[torch.randperm(n, device="cuda", generator=torch.Generator(device="cuda").manual_seed(1))]
for _ in range(a.steps):
    t.clear()
    st = t.upsert_batch(keys.view(torch.uint64), vals.view(torch.uint64), check=False)
    f, v = t.query_batch(q.view(torch.uint64), check=False)
torch.cuda.synchronize()
print("inserted", int((st == 0).sum()), "hits", int(f.sum()))

"""YCSB-A batch timings (per batch) to separate first-call allocation from steady state."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2509_16407_b200 import TableConfig, make_table
from paper_2509_16407_b200.tables import OP_QUERY, OP_UPSERT
from paper_2509_16407_b200.workload import gen_uniform_keys, zipf_ranks

universe, ops, batch = 1 << 24, 1 << 26, 1 << 24
cap = int(universe / 0.85) // 32 * 32
t = make_table(TableConfig(design="p2_md", capacity_slots=cap, seed=42))
keys = gen_uniform_keys(42, universe)
d = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).cuda()
t.upsert_batch(d(keys).view(torch.uint64), d(keys & np.uint64(0xFFFF)).view(torch.uint64))
ranks = zipf_ranks(universe, ops, 0.99, seed=7) - 1
idx = np.arange(ops)
op_b = np.where(idx % 2 == 0, OP_UPSERT, OP_QUERY).astype(np.uint8)
ks = keys[ranks]
vs = idx.astype(np.uint64) & np.uint64(0xFFFFFFFF)
for rep in range(2):
    for lo in range(0, ops, batch):
        o = torch.from_numpy(op_b[lo:lo + batch]).cuda()
        k, v = d(ks[lo:lo + batch]).view(torch.uint64), d(vs[lo:lo + batch]).view(torch.uint64)
        torch.cuda.synchronize()
        a = time.perf_counter()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        s, _v = t.mixed_batch(o, k, v, check=False, combine=True)
        e1.record()
        torch.cuda.synchronize()
        print(f"rep {rep} batch {lo // batch}: wall {1e3*(time.perf_counter()-a):.1f} ms  gpu {e0.elapsed_time(e1):.1f} ms",
              flush=True)

"""Insert-kernel timing across P2-MD upsert variants / occupancy (CUDA events)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2509_16407_b200 import TableConfig, make_table
from paper_2509_16407_b200.workload import gen_uniform_keys

slots = 1 << 28
n = int(slots * 0.9)
t = make_table(TableConfig(design="p2_md", capacity_slots=slots, seed=42))
keys = torch.from_numpy(gen_uniform_keys(42, n).view(np.int64)).cuda().view(torch.uint64)
vals = keys.view(torch.int64).bitwise_and(0xFFFF).view(torch.uint64)
st = torch.empty(n, dtype=torch.uint8, device="cuda")
variants = [a.split(":") for a in (sys.argv[1:] or ["4:0", "3:0", "3:5", "3:6"])]
for up, occ in variants:
    t.tune(upsert=int(up), occupancy=int(occ))
    ts = []
    for r in range(4):
        t.clear()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        t.upsert_batch(keys, vals, check=False, out=st)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ins = int((st == 0).sum())
    f, got = t.query_batch(keys, check=False)
    ok = bool(f.all()) and bool((got == vals).all())
    print(f"upsert={up} occ={occ}: ms={min(ts[1:]):.2f} {['%.2f' % x for x in ts]} inserted={ins}/{n} "
          f"query_ok={ok} checksum={t.checksum()} dups={t.duplicate_count()}", flush=True)

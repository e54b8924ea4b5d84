"""Experiment: tuned P2-MD query variants (lookups/thread x L2 policy) and insert time."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2509_16407_b200 import TableConfig, make_table
from paper_2509_16407_b200.workload import derive_seed, gen_uniform_keys

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 28
slots = 1 << lg
n = int(slots * 0.9)
t = make_table(TableConfig(design="p2_md", capacity_slots=slots, seed=42))
keys = torch.from_numpy(gen_uniform_keys(42, n).view(np.int64)).cuda()
vals = keys & 0xFFFF
miss = torch.from_numpy(gen_uniform_keys(derive_seed(42, 0xFEED), n - n // 2).view(np.int64)).cuda()
q = torch.cat([keys[: n // 2], miss])
q = q[torch.randperm(n, device="cuda")].view(torch.uint64)


def timed(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        r = fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best, r


for variant in (3, 4, 3, 4):
    t.tune(upsert=variant)
    ins = []
    for rep in range(3):
        t.clear()
        ms, st = timed(lambda: t.upsert_batch(keys.view(torch.uint64), vals.view(torch.uint64), check=False), 1)
        ins.append(ms)
        bad = int((st != 0).sum())
    cs = t.checksum()
    print(f"insert variant {variant}: {min(ins):.2f} ms  ({n / min(ins) / 1e6:.2f} G/s) bad={bad} occupied={cs[0]}",
          flush=True)
ref_f, ref_v = None, None
for ilp in (3, 5):
    for pol in (0, 2):
        t.tune(query_ilp=ilp, l2_policy=pol)
        ms, (f, v) = timed(lambda: t.query_batch(q, check=False))
        if ref_f is None:
            ref_f, ref_v = f.clone(), v.clone()
        ok = torch.equal(f, ref_f) and torch.equal(v.view(torch.int64), ref_v.view(torch.int64))
        print(f"query ilp={ilp} pol={pol}: {ms:.2f} ms ({n / ms / 1e6:.2f} G/s) same={ok} hits={int(f.sum())}",
              flush=True)

for occ in (0, 5, 6):
    t.tune(upsert=3, occupancy=occ)
    best = 1e9
    for rep in range(3):
        t.clear()
        ms, st = timed(lambda: t.upsert_batch(keys.view(torch.uint64), vals.view(torch.uint64), check=False), 1)
        best = min(best, ms)
    print(f"insert rounds occ={occ}: {best:.2f} ms ({n / best / 1e6:.2f} G/s) bad={int((st != 0).sum())}", flush=True)
for occ in (0, 8):
    t.tune(query_ilp=5, l2_policy=2, occupancy=occ)
    ms, (f, v) = timed(lambda: t.query_batch(q, check=False))
    print(f"query coop occ={occ}: {ms:.2f} ms ({n / ms / 1e6:.2f} G/s) hits={int(f.sum())}", flush=True)
# phased (BSP) mode: no locks (reference sync.py:70-102)
tp = make_table(TableConfig(design="p2_md", capacity_slots=slots, seed=42, mode="phased"))
for rep in range(3):
    tp.clear()
    ms, st = timed(lambda: tp.upsert_batch(keys.view(torch.uint64), vals.view(torch.uint64), check=False), 1)
    print(f"phased insert: {ms:.2f} ms ({n / ms / 1e6:.2f} G/s) bad={int((st != 0).sum())}", flush=True)
ms, (f, v) = timed(lambda: tp.query_batch(q, check=False))
print(f"phased query: {ms:.2f} ms ({n / ms / 1e6:.2f} G/s) hits={int(f.sum())}", flush=True)

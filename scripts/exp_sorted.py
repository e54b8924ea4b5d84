"""Experiment: does bucket-ordered batch processing pay on B200?  Same keys,
random order vs sorted by primary bucket; insert + query times."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2509_16407_b200 import TableConfig, make_table
from paper_2509_16407_b200.workload import derive_seed, gen_uniform_keys, mix64_np

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 26
slots = 1 << lg
n = int(slots * 0.9)
t = make_table(TableConfig(design="p2_md", capacity_slots=slots, seed=42))
kh = gen_uniform_keys(42, n)
a = time.time()
b0 = (mix64_np(kh ^ np.uint64(t.family.seeds[0])) >> np.uint64(16)) & np.uint64((slots // 32) - 1)
order = np.argsort(b0, kind="stable")
print(f"host sort {time.time() - a:.1f}s", flush=True)
ks = kh[order]
mh = gen_uniform_keys(derive_seed(42, 0xFEED), n - n // 2)
qh = np.concatenate([kh[: n // 2], mh])
np.random.default_rng(0).shuffle(qh)
qb = (mix64_np(qh ^ np.uint64(t.family.seeds[0])) >> np.uint64(16)) & np.uint64((slots // 32) - 1)
qs = qh[np.argsort(qb, kind="stable")]


def dev(a):
    return torch.from_numpy(a.view(np.int64)).cuda().view(torch.uint64)


for name, ins, qq in (("random", kh, qh), ("sorted", ks, qs), ("random", kh, qh), ("sorted", ks, qs)):
    K = dev(ins)
    V = dev(ins & np.uint64(0xFFFF))
    Q = dev(qq)
    t.clear()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record()
    st = t.upsert_batch(K, V, check=False)
    e[1].record()
    f, v = t.query_batch(Q, check=False)
    e[2].record()
    torch.cuda.synchronize()
    ti, tq = e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2])
    print(f"{name}: insert {ti:.2f} ms ({n / ti / 1e6:.2f} G/s)  query {tq:.2f} ms ({n / tq / 1e6:.2f} G/s)  "
          f"ok={int((st == 0).sum()) == n and int(f.sum()) == n // 2}", flush=True)

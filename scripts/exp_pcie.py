"""PCIe ceilings (pinned H2D / D2H / both directions) vs the e2e phases."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2509_16407_b200 import TableConfig, make_table
from paper_2509_16407_b200.workload import gen_uniform_keys

print("cpus", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)), flush=True)
GB = 1 << 30
h = torch.empty(2 * GB, dtype=torch.uint8, pin_memory=True)
h2 = torch.empty(2 * GB, dtype=torch.uint8, pin_memory=True)
d = torch.empty(2 * GB, dtype=torch.uint8, device="cuda")
d2 = torch.empty(2 * GB, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for name in ("h2d", "d2h", "both", "h2d", "d2h", "both"):
    torch.cuda.synchronize()
    a = time.perf_counter()
    if name in ("h2d", "both"):
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)
    if name in ("d2h", "both"):
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - a
    mult = 2 if name == "both" else 1
    print(f"{name}: {2 * mult / dt:.1f} GB/s total ({dt * 1e3:.1f} ms for {2 * mult} GiB)", flush=True)
del h, h2, d, d2
slots = 1 << 28
n = int(slots * 0.9)
t = make_table(TableConfig(design="p2_md", capacity_slots=slots, seed=42))
kh = gen_uniform_keys(42, n)
a = time.perf_counter()
bad = int(((kh == 0) | (kh >= np.uint64((1 << 64) - 2))).sum())
print(f"numpy key scan {(time.perf_counter() - a) * 1e3:.1f} ms bad={bad}", flush=True)
K = torch.from_numpy(kh.view(np.int64)).pin_memory().view(torch.uint64)
V = torch.from_numpy((kh & np.uint64(0xFFFF)).view(np.int64)).pin_memory().view(torch.uint64)
st = torch.empty(n, dtype=torch.uint8, pin_memory=True)
f = torch.empty(n, dtype=torch.uint8, pin_memory=True)
v = torch.empty(n, dtype=torch.uint64, pin_memory=True)
for chk in (True, False, True, False):
    t.clear()
    torch.cuda.synchronize()
    a = time.perf_counter()
    t.upsert_batch(K, V, out=st, check=chk)
    torch.cuda.synchronize()
    b = time.perf_counter()
    t.query_batch(K, out=(f, v), check=chk)
    torch.cuda.synchronize()
    c = time.perf_counter()
    print(f"check={chk}: upsert e2e {(b - a) * 1e3:.1f} ms  query e2e {(c - b) * 1e3:.1f} ms", flush=True)

"""e2e phase timing: host-pinned insert and query through the C ABI at 2^28,
plus raw pinned H2D / D2H copy rates for the same byte counts."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_16407_b200 import TableConfig, make_table  # noqa: E402
from paper_2509_16407_b200.workload import gen_uniform_keys  # noqa: E402

cap = 1 << 28
n = int(cap * 0.9)
keys = gen_uniform_keys(42, n)
kh = torch.from_numpy(keys.view(np.int64)).pin_memory()
vh = torch.from_numpy((keys & np.uint64(0xFFFF)).view(np.int64)).pin_memory()
qh = kh.clone().pin_memory()
st_o = torch.empty(n, dtype=torch.uint8, pin_memory=True)
f_o = torch.empty(n, dtype=torch.uint8, pin_memory=True)
v_o = torch.empty(n, dtype=torch.uint64, pin_memory=True)
t = make_table(TableConfig(design="p2_md", capacity_slots=cap, seed=42))
for it in range(3):
    t.clear()
    torch.cuda.synchronize()
    a = time.perf_counter()
    t.upsert_batch(kh.view(torch.uint64), vh.view(torch.uint64), out=st_o)
    b = time.perf_counter()
    t.query_batch(qh.view(torch.uint64), out=(f_o, v_o))
    torch.cuda.synchronize()
    c = time.perf_counter()
    print(f"insert {1e3*(b-a):.1f} ms  query {1e3*(c-b):.1f} ms  total {1e3*(c-a):.1f}", flush=True)
d = torch.empty(n, dtype=torch.int64, device="cuda")
for nbytes_name, src in (("H2D keys 1.93GB", kh),):
    torch.cuda.synchronize(); a = time.perf_counter()
    d.copy_(src, non_blocking=True); torch.cuda.synchronize()
    dt = time.perf_counter() - a
    print(f"{nbytes_name}: {src.numel()*8/dt/1e9:.1f} GB/s")
torch.cuda.synchronize(); a = time.perf_counter()
v_o.view(torch.int64).copy_(d, non_blocking=True); torch.cuda.synchronize()
dt = time.perf_counter() - a
print(f"D2H 1.93GB: {n*8/dt/1e9:.1f} GB/s")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
d2 = torch.empty_like(d)
torch.cuda.synchronize(); a = time.perf_counter()
with torch.cuda.stream(s1):
    d2.copy_(kh, non_blocking=True)
with torch.cuda.stream(s2):
    v_o.view(torch.int64).copy_(d, non_blocking=True)
torch.cuda.synchronize()
dt = time.perf_counter() - a
print(f"bidirectional 2x1.93GB: {dt*1e3:.1f} ms ({2*n*8/dt/1e9:.1f} GB/s total)")

"""Experiment: effect of the L2 fetch-granularity limit on insert / query time."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2509_16407_b200 import TableConfig, make_table
from paper_2509_16407_b200.workload import derive_seed, gen_uniform_keys

cu = C.CDLL("libcuda.so.1")
torch.cuda.init()
torch.zeros(1, device="cuda")


def get_limit():
    v = C.c_size_t()
    cu.cuCtxGetLimit(C.byref(v), 5)
    return v.value


def set_limit(x):
    return cu.cuCtxSetLimit(5, C.c_size_t(x))


slots = 1 << int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 28
n = int(slots * 0.9)
t = make_table(TableConfig(design="p2_md", capacity_slots=slots, seed=42))
keys = torch.from_numpy(gen_uniform_keys(42, n).view(np.int64)).cuda()
vals = keys & 0xFFFF
miss = torch.from_numpy(gen_uniform_keys(derive_seed(42, 0xFEED), n - n // 2).view(np.int64)).cuda()
q = torch.cat([keys[: n // 2], miss])
q = q[torch.randperm(n, device="cuda")]
print("default limit", get_limit())
for lim in (0, 32, 64, 128, 32):
    rc = set_limit(lim)
    res = []
    for rep in range(3):
        t.clear()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record()
        st = t.upsert_batch(keys.view(torch.uint64), vals.view(torch.uint64), check=False)
        e[1].record()
        f, v = t.query_batch(q.view(torch.uint64), check=False)
        e[2].record()
        torch.cuda.synchronize()
        res.append((e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2])))
    ins = min(r[0] for r in res)
    qry = min(r[1] for r in res)
    print(f"limit={lim:4d} rc={rc} now={get_limit()} insert {ins:.2f} ms ({n/ins/1e6:.2f} G/s)  "
          f"query {qry:.2f} ms ({n/qry/1e6:.2f} G/s) ok={int((st == 0).sum()) == n and int(f.sum()) == n // 2}",
          flush=True)

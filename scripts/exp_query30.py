"""Query-kernel variants at 2^28 and 2^30 (north-star size): default pair-
cooperative kernel at two occupancies and the Q-lookups-per-thread kernels."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2509_16407_b200 import TableConfig, make_table
from paper_2509_16407_b200.workload import derive_seed, gen_uniform_keys

for lg in [int(x) for x in sys.argv[1:]] or [28, 30]:
    slots = 1 << lg
    n = int(slots * 0.9)
    t = make_table(TableConfig(design="p2_md", capacity_slots=slots, seed=42))
    keys = torch.from_numpy(gen_uniform_keys(42, n).view(np.int64)).cuda()
    t.upsert_batch(keys.view(torch.uint64), (keys & 0xFFFF).view(torch.uint64), check=False)
    miss = torch.from_numpy(gen_uniform_keys(derive_seed(42, 0xFEED), n - n // 2).view(np.int64)).cuda()
    q = torch.cat([keys[: n // 2], miss])
    q = q[torch.randperm(n, device="cuda")].view(torch.uint64)
    del keys, miss
    ref = None
    for name, kw in (("coop occ0", dict(query_ilp=5, l2_policy=2, occupancy=0)),
                     ("coop occ8", dict(query_ilp=5, l2_policy=2, occupancy=8)),
                     ("pair", dict(query_ilp=3, l2_policy=2, occupancy=0)),
                     ("Q2", dict(query_ilp=2, l2_policy=0, occupancy=0)),
                     ("Q4", dict(query_ilp=4, l2_policy=0, occupancy=0))):
        t.tune(**kw)
        best = 1e9
        for _ in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            f, v = t.query_batch(q, check=False)
            b.record()
            torch.cuda.synchronize()
            best = min(best, a.elapsed_time(b))
        if ref is None:
            ref = int(f.sum())
        print(f"2^{lg} {name}: {best:.2f} ms  {n / best / 1e6:.2f} G q/s  hits={int(f.sum())} (ref {ref})",
              flush=True)
    del t, q
    torch.cuda.empty_cache()

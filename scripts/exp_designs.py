"""Insert and 50/50 query throughput of every design at 2^24 slots (fill to the
Table-1 loads), default tuned kernels vs the generic kernels (tune(upsert=0,
query_ilp=0)); results must match between the two."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2509_16407_b200 import TableConfig, make_table
from paper_2509_16407_b200.workload import derive_seed, gen_uniform_keys

cap = 1 << 24
designs = sys.argv[1:] or ["double", "double_md", "iceberg", "iceberg_md", "p2", "p2_md", "cuckoo", "chaining",
                           "unsafe_reference"]


def ev():
    return torch.cuda.Event(enable_timing=True)


for design in designs:
    load = 0.85 if design.startswith("double") else (1.0 if design == "chaining" else 0.9)
    t = make_table(TableConfig(design=design, capacity_slots=cap if design != "chaining" else 7 * (cap // 8), seed=42))
    n = int(t.capacity_slots * load)
    keys = gen_uniform_keys(42, n)
    dk = torch.from_numpy(keys.view(np.int64)).cuda().view(torch.uint64)
    miss = gen_uniform_keys(derive_seed(42, 0xFEED), n // 2)
    q = np.concatenate([keys[: n // 2], miss])
    np.random.default_rng(1).shuffle(q)
    dq = torch.from_numpy(q.view(np.int64)).cuda().view(torch.uint64)
    ref = None
    for tuned in (True, False, True):
        t.tune(upsert=4 if tuned else 0, query_ilp=5 if tuned else 0)
        ins = 1e9
        for _ in range(2):
            t.clear()
            torch.cuda.synchronize()
            a, b = ev(), ev()
            a.record()
            st = t.upsert_batch(dk, dk, check=False)
            b.record()
            torch.cuda.synchronize()
            ins = min(ins, a.elapsed_time(b))
        qb = 1e9
        for _ in range(3):
            a, b = ev(), ev()
            a.record()
            f, v = t.query_batch(dq, check=False)
            b.record()
            torch.cuda.synchronize()
            qb = min(qb, a.elapsed_time(b))
        cur = (np.bincount(st.cpu().numpy(), minlength=3)[:3].tolist(), int(f.sum()), t.checksum()[:3])
        same = ref is None or cur == ref
        ref = ref or cur
        print(f"{design:17s} {'tuned  ' if tuned else 'generic'} insert {ins:7.3f} ms {n / ins / 1e6:6.2f} G/s  "
              f"query {qb:7.3f} ms {len(q) / qb / 1e6:6.2f} G/s  statuses {cur[0]} hits {cur[1]} same={same}",
              flush=True)
    del t, dk, dq
    torch.cuda.empty_cache()

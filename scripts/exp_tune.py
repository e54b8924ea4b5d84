"""A/B of P2-MD kernel knobs (tables.HashTable.tune): insert 0 -> 0.9, then
50/50 queries, CUDA events, best of 3 per setting.

    python scripts/exp_tune.py 28 30 -- prefetch=0 prefetch=1 upsert=5 upsert=4,occupancy=4
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_16407_b200 import TableConfig, make_table  # noqa: E402
from paper_2509_16407_b200.workload import derive_seed, gen_uniform_keys  # noqa: E402

argv = sys.argv[1:]
cut = argv.index("--") if "--" in argv else len(argv)
sizes = [int(x) for x in argv[:cut]] or [28, 30]
settings = [dict((kv.split("=")[0], int(kv.split("=")[1])) for kv in s.split(",")) for s in argv[cut + 1:]] or [{}]

for log2 in sizes:
    slots = 1 << log2
    n = int(slots * 0.9)
    t = make_table(TableConfig(design="p2_md", capacity_slots=slots, seed=42))
    kh = gen_uniform_keys(42, n)
    keys = torch.from_numpy(kh.view(np.int64)).cuda().view(torch.uint64)
    vals = (keys.view(torch.int64) & 0xFFFF).view(torch.uint64)
    miss = torch.from_numpy(gen_uniform_keys(derive_seed(42, 0xFEED), n - n // 2).view(np.int64)).cuda()
    q = torch.cat([keys.view(torch.int64)[: n // 2], miss])
    q = q[torch.randperm(n, device="cuda", generator=torch.Generator(device="cuda").manual_seed(1))]
    q = q.view(torch.uint64)
    for kw in settings:
        t.tune(**{"prefetch": 0, "upsert": 4, "occupancy": 0, **kw})
        bi = bq = 1e9
        for _ in range(3):
            t.clear()
            e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            e[0].record()
            st = t.upsert_batch(keys, vals, check=False)
            e[1].record()
            f, v = t.query_batch(q, check=False)
            e[2].record()
            torch.cuda.synchronize()
            bi, bq = min(bi, e[0].elapsed_time(e[1])), min(bq, e[1].elapsed_time(e[2]))
        ok = int((st != 0).sum()) <= 3 and int(f.sum()) >= n // 2 - 3
        print(f"2^{log2} {kw}: insert {bi:7.2f} ms {n / bi / 1e6:6.2f} G/s   query {bq:7.2f} ms "
              f"{n / bq / 1e6:6.2f} G/s  ok={ok}", flush=True)
    del t, keys, vals, q, miss
    torch.cuda.empty_cache()

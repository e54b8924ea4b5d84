"""One interleaved aging batch (P2-MD and Iceberg-MD, 2^26 slots at 0.85,
2.28M mixed ops) for an ncu capture of the fused mixed kernels, and one
cuckoo 0.9 -> 0.95 slice for the cooperative eviction kernel.

  ncu --set full -k regex:'k_mixed|k_ck_evict' -c 3 -o gpurun_out/prof_fused python scripts/prof_fused.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_16407_b200 import TableConfig, make_table, runners  # noqa: E402
from paper_2509_16407_b200.workload import gen_uniform_keys  # noqa: E402

for design in ("p2_md", "iceberg_md"):
    r = runners.run_aging_uniform(design, 1 << 26, iterations=2, interleaved=True, probe_sample=8)
    print(design, r["ok"], flush=True)
cap = 1 << 26
keys = gen_uniform_keys(42, int(cap * 0.95))
dk = torch.from_numpy(keys.view(np.int64)).cuda().view(torch.uint64)
t = make_table(TableConfig(design="cuckoo", capacity_slots=cap, seed=42))
a, b = int(cap * 0.9), int(cap * 0.95)
t.upsert_batch(dk[:a], dk[:a], check=False)
t.upsert_batch(dk[a:b], dk[a:b], check=False)
torch.cuda.synchronize()
print("cuckoo", t.occupied_count(), flush=True)

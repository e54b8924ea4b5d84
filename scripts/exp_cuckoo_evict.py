"""Cuckoo (3 x 8-slot buckets) fill at 2^26: 0 -> 0.9 and the 0.9 -> 0.95
slice where eviction chains dominate, with the cooperative eviction launch
(upsert knob 4, default) vs the one-thread-per-op eviction (6); same keys,
contents compared (checksum) and duplicates checked."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_16407_b200 import TableConfig, make_table  # noqa: E402
from paper_2509_16407_b200.workload import gen_uniform_keys  # noqa: E402

cap = 1 << int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 26
keys = gen_uniform_keys(42, int(cap * 0.95))
dk = torch.from_numpy(keys.view(np.int64)).cuda().view(torch.uint64)
a, b = int(cap * 0.9), int(cap * 0.95)
for knob in (6, 4, 6, 4):
    t = make_table(TableConfig(design="cuckoo", capacity_slots=cap, seed=42))
    t.tune(upsert=knob)
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record()
    s1 = t.upsert_batch(dk[:a], dk[:a], check=False)
    e[1].record()
    s2 = t.upsert_batch(dk[a:b], dk[a:b], check=False)
    e[2].record()
    torch.cuda.synchronize()
    full = int((s1 == 2).sum()) + int((s2 == 2).sum())
    print(f"2^{cap.bit_length() - 1} evict={'coop' if knob == 4 else 'thread'}: 0->0.9 {e[0].elapsed_time(e[1]):.2f} ms "
          f"0.9->0.95 {e[1].elapsed_time(e[2]):.2f} ms ({(b - a) / e[1].elapsed_time(e[2]) / 1e6:.2f} G/s) "
          f"full={full} occupied={t.occupied_count()} dups={t.duplicate_count()} checksum={t.checksum()[1] % 1000003}",
          flush=True)
    del t
    torch.cuda.empty_cache()

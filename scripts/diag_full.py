"""Dev diagnostic: where do FULL statuses come from under one big concurrent batch?"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2509_16407_b200 import TableConfig, make_table
from paper_2509_16407_b200.workload import gen_uniform_keys, mix64_np

def cu(a): return torch.from_numpy(a.view(np.int64)).cuda().view(torch.uint64)

for design in ("p2_md", "p2", "unsafe_reference", "iceberg_md", "double_md"):
    for batches in (1, 4, 16):
        t = make_table(TableConfig(design=design, capacity_slots=1 << 16, seed=42))
        n = int((1 << 16) * 0.9)
        keys = gen_uniform_keys(42, n)
        sts = []
        for part in np.array_split(np.arange(n), batches):
            sts.append(t.upsert_batch(cu(keys[part]), cu(keys[part])).cpu().numpy())
        st = np.concatenate(sts)
        cnt = np.bincount(st, minlength=4)
        msg = f"{design:18s} batches={batches:3d} status counts={cnt.tolist()} occupied={t.occupied_count()}"
        if cnt[2] and design.startswith("p2"):
            words, tags = t._raw()
            k = words[0::2].reshape(-1, 32)
            live = ((k != 0) & (k < np.uint64(2**64 - 2))).sum(1)
            fk = keys[st == 2]
            s0, s1 = t.family.seeds[0], t.family.seeds[1]
            b0 = (mix64_np(fk ^ np.uint64(s0)) >> np.uint64(16)) % np.uint64(2048)
            b1 = (mix64_np(fk ^ np.uint64(s1)) >> np.uint64(16)) % np.uint64(2048)
            msg += f"\n   FULL keys: b0 live {np.bincount(live[b0.astype(int)]).nonzero()} b1 live min {live[b1.astype(int)].min()}"
            msg += f"\n   bucket fill histogram: {np.bincount(live, minlength=33).tolist()}"
        print(msg, flush=True)

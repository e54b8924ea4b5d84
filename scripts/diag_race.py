"""Dev diagnostic: repeat full-size insert+query and characterise any failure."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2509_16407_b200 import TableConfig, make_table
from paper_2509_16407_b200.workload import derive_seed, gen_uniform_keys, mix64_np

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 28
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
design = sys.argv[3] if len(sys.argv) > 3 else "p2_md"
slots = 1 << lg
n = int(slots * 0.9)
t = make_table(TableConfig(design=design, capacity_slots=slots, seed=42))
kh = gen_uniform_keys(42, n)
keys = torch.from_numpy(kh.view(np.int64)).cuda()
vals = keys & 0xFFFF
miss = torch.from_numpy(gen_uniform_keys(derive_seed(42, 0xFEED), n - n // 2).view(np.int64)).cuda()
q = torch.cat([keys[: n // 2], miss])
perm = torch.randperm(n, device="cuda")
q = q[perm]
expect_hit = torch.cat([torch.ones(n // 2, dtype=torch.bool, device="cuda"),
                        torch.zeros(n - n // 2, dtype=torch.bool, device="cuda")])[perm]
nb = slots // 32
for r in range(reps):
    t.clear()
    st = t.upsert_batch(keys.view(torch.uint64), vals.view(torch.uint64), check=False)
    f, v = t.query_batch(q.view(torch.uint64), check=False)
    torch.cuda.synchronize()
    cnt = torch.bincount(st.long(), minlength=4).tolist()
    wrong = (f != expect_hit)
    nw = int(wrong.sum())
    fa, _ = t.query_batch(keys.view(torch.uint64), check=False)
    lost = int((~fa).sum())
    msg = f"rep {r}: status {cnt} query-mismatch {nw} lost-after-insert {lost}"
    if cnt[1] or cnt[2] or cnt[3] or nw or lost:
        bad_ins = torch.nonzero(st != 0).flatten()[:5].cpu().numpy()
        msg += f"\n  bad status idx {bad_ins} st {st[bad_ins].cpu().numpy() if len(bad_ins) else []}"
        wi = torch.nonzero(wrong).flatten()[:5]
        msg += f"\n  wrong queries: keys {q[wi].cpu().numpy()} expect {expect_hit[wi].cpu().numpy()} got {f[wi].cpu().numpy()}"
        li = torch.nonzero(~fa).flatten()[:5]
        lk = keys[li].cpu().numpy().view(np.uint64)
        msg += f"\n  lost keys idx {li.cpu().numpy()} status {st[li].cpu().numpy()}"
        if len(lk):
            b0 = (mix64_np(lk ^ np.uint64(t.family.seeds[0])) >> np.uint64(16)) % np.uint64(nb)
            b1 = (mix64_np(lk ^ np.uint64(t.family.seeds[1])) >> np.uint64(16)) % np.uint64(nb)
            loc = t.locate_batch(lk)
            msg += f"\n  lost b0 {b0} b1 {b1} locate {loc}"
        msg += f"\n  dups {t.duplicate_count()} occupied {t.occupied_count()} (n={n})"
    print(msg, flush=True)

"""Diagnostics for the bulk upsert: phase A only (tune bulk=3) at 2^16 slots,
compared bucket by bucket with the expected shortcut state (first 24 ops of
each primary bucket in batch order)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from conftest import cfg_for  # noqa: E402
from paper_2509_16407_b200 import make_table  # noqa: E402
from paper_2509_16407_b200.workload import gen_uniform_keys, mix64_np  # noqa: E402

cap = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 16
cfg = cfg_for("p2_md", cap, seed=42)
t = make_table(cfg)
t.tune(bulk=3)
n = int(cfg.capacity_slots * 0.9)
keys = gen_uniform_keys(42, n)
s0 = np.uint64(cfg.hash_family().seeds[0])
nb = cfg.capacity_slots // 32
h0 = mix64_np(keys ^ s0)
b0 = ((h0 >> np.uint64(16)) % np.uint64(nb)).astype(np.int64)
order = np.argsort(b0, kind="stable")
sb = b0[order]
rank = np.empty(n, np.int64)
rank[order] = np.arange(n) - np.searchsorted(sb, sb, side="left")
A = rank < 20
dk = torch.from_numpy(keys.view(np.int64)).cuda().view(torch.uint64)
st = t.upsert_batch(dk, dk).cpu().numpy()
print("statuses", np.bincount(st))
words, tags = t._raw()
k = words[0::2].reshape(nb, 32)
tg = tags.reshape(nb, 32)
used_tag = (tg != 0).sum(1)
used_key = (k != 0).sum(1)
want = np.minimum(np.bincount(b0, minlength=nb), 20)
print("buckets tag-used != expected:", int((used_tag != want).sum()), " key-used != expected:",
      int((used_key != want).sum()))
bad = np.nonzero(used_tag != want)[0][:5]
for b in bad:
    print(" bucket", b, "tags used", used_tag[b], "keys used", used_key[b], "want", want[b])
present = set(k[k != 0].tolist())
print("phase-A keys missing:", int(sum(1 for x in keys[A].tolist() if x not in present)),
      " deferred keys present:", int(sum(1 for x in keys[~A].tolist() if x in present)))
exp_tag = (h0 & np.uint64(0xFFFF)).astype(np.int64)
exp_tag[exp_tag == 0] = 1
slot_of = {}
for bb in range(nb):
    for j in range(32):
        if k[bb, j]:
            slot_of[int(k[bb, j])] = (bb, j)
wrong_b = sum(1 for i in np.nonzero(A)[0].tolist() if slot_of.get(int(keys[i]), (-1,))[0] != b0[i])
wrong_t = sum(1 for i in np.nonzero(A)[0].tolist()
              if int(keys[i]) in slot_of and tg[slot_of[int(keys[i])]] != exp_tag[i])
print("phase-A keys in wrong bucket:", wrong_b, " wrong tag:", wrong_t)

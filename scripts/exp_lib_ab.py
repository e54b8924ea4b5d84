"""Same-box A/B of two library builds on the bench workload (P2-MD 2^30,
insert 0 -> 0.9, then 50/50 queries): run once per build in separate
processes,

    python scripts/exp_lib_ab.py [path/to/libwarpspeed.so]

and compare the table-kernel times (CUDA events the library records around
each kernel, best of 4 steps after a warm-up)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_16407_b200 import _native  # noqa: E402

if len(sys.argv) > 1:
    _native.LIB_PATH = os.path.abspath(sys.argv[1])

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_16407_b200 import TableConfig, make_table  # noqa: E402
from paper_2509_16407_b200.workload import derive_seed, gen_uniform_keys  # noqa: E402

slots = 1 << 30
n = int(slots * 0.9)
t = make_table(TableConfig(design="p2_md", capacity_slots=slots, seed=42))
kh = gen_uniform_keys(derive_seed(42, 0), n)
keys = torch.from_numpy(kh.view(np.int64)).cuda()
vals = keys & 0xFFFF
miss = torch.from_numpy(gen_uniform_keys(derive_seed(42, 0xFEED), n - n // 2).view(np.int64)).cuda()
q = torch.cat([keys[: n // 2], miss])
q = q[torch.randperm(n, device="cuda", generator=torch.Generator(device="cuda").manual_seed(1))]
ku, vu, qu = keys.view(torch.uint64), vals.view(torch.uint64), q.view(torch.uint64)
ins, qry = [], []
for step in range(5):
    t.clear()
    torch.cuda.synchronize()
    t.kernel_times()
    t.time_kernels(True)
    st = t.upsert_batch(ku, vu)
    f, v = t.query_batch(qu)
    torch.cuda.synchronize()
    kt = t.kernel_times()
    t.time_kernels(False)
    assert int((st == 1).sum()) == 0 and int((st == 2).sum()) <= 3 and int(f.sum()) >= n // 2 - 3
    if step:
        ins.append(kt[0])
        qry.append(kt[1])
print(f"{_native.LIB_PATH}: insert kernel best {min(ins):.2f} mean {np.mean(ins):.2f} ms; "
      f"query kernel best {min(qry):.2f} mean {np.mean(qry):.2f} ms", flush=True)

import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_16407_b200.core import TableConfig
from paper_2509_16407_b200.tables import make_table
from paper_2509_16407_b200.workload import gen_uniform_keys
d = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).cuda().view(torch.uint64)
design = sys.argv[1]
n = 1 << 14
keys = gen_uniform_keys(3, n)
slots = (int(n * 0.25 / 0.85) + 2 + 31) // 32 * 32
t = make_table(TableConfig(design=design, capacity_slots=slots, seed=4))
t0 = time.time()
for lo in range(0, 4096, 512):
    st = t.upsert_batch(d(keys[lo:lo+512]), d(keys[lo:lo+512]), "keep")
    torch.cuda.synchronize()
    print("upsert", lo, time.time() - t0, np.bincount(st.cpu().numpy(), minlength=3), flush=True)
f, v = t.query_batch(d(keys[:4096])); torch.cuda.synchronize(); print("query", int(f.sum()), time.time()-t0, flush=True)
g = t.erase_batch(d(keys[:512])); torch.cuda.synchronize(); print("erase", int(g.sum()), time.time()-t0, flush=True)
st = t.upsert_batch(d(keys[4096:4608]), d(keys[4096:4608]), "keep"); torch.cuda.synchronize()
print("upsert after erase", np.bincount(st.cpu().numpy(), minlength=3), time.time()-t0, flush=True)

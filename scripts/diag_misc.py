import sys, os; sys.path.insert(0, '/root/repo')
import numpy as np, torch
from paper_2509_16407_b200 import TableConfig, make_table
from paper_2509_16407_b200.workload import gen_uniform_keys, derive_seed
t = make_table(TableConfig(design="cuckoo", capacity_slots=1<<26, seed=42))
n = int((1<<26)*0.6); k = gen_uniform_keys(42, n)
dk = torch.from_numpy(k.view(np.int64)).cuda().view(torch.uint64)
t.upsert_batch(dk, dk)
q = torch.from_numpy(np.concatenate([k[:1<<19], gen_uniform_keys(9, 1<<19)]).view(np.int64)).cuda().view(torch.uint64)
for i in range(6):
    a,b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record(); f,v = t.query_batch(q, check=False); b.record(); torch.cuda.synchronize()
    print("cuckoo query", round(a.elapsed_time(b),3), "ms", int(f.sum()))
import time
kk = np.concatenate([gen_uniform_keys(5, 1<<22)])
for comb in (False, True, False, True):
    t2 = make_table(TableConfig(design="p2_md", capacity_slots=1<<24, seed=1))
    d = torch.from_numpy(np.repeat(kk[:1<<20], 4).view(np.int64)).cuda().view(torch.uint64)
    o = torch.ones_like(d)
    torch.cuda.synchronize(); a=time.time()
    st = t2.upsert_batch(d, o, merge="add", check=False, combine=comb); torch.cuda.synchronize()
    print("combine", comb, round((time.time()-a)*1e3,2), "ms")

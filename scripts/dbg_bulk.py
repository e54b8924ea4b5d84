import sys, os, numpy as np, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
from paper_2509_16407_b200 import TableConfig, make_table
from paper_2509_16407_b200.workload import gen_uniform_keys
gb = int(sys.argv[1]); lg = int(sys.argv[2])
t = make_table(TableConfig(design="p2_md", capacity_slots=1 << lg, seed=42))
t.tune(bulk=2, bulk_group=gb)
n = int((1 << lg) * 0.9)
k = gen_uniform_keys(1, n)
dk = torch.from_numpy(k.view(np.int64)).cuda().view(torch.uint64)
st = t.upsert_batch(dk, dk)
torch.cuda.synchronize()
print("gb", gb, "lg", lg, "ok", np.bincount(st.cpu().numpy()))

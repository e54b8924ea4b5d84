import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from conftest import cfg_for
from oracle import OracleTable
from paper_2509_16407_b200 import make_table
from paper_2509_16407_b200.workload import gen_uniform_keys
for mode in ("phased", "concurrent"):
    cfg = cfg_for("chaining", 7 * 4096, seed=21, mode=mode)
    t = make_table(cfg); o = OracleTable(cfg)
    n = int(t.capacity_slots * 1.2)
    keys = gen_uniform_keys(61, n)
    d = lambda a: torch.from_numpy(a.view(np.int64)).cuda().view(torch.uint64)
    st = t.upsert_batch(d(keys), d(keys)).cpu().numpy()
    o.upsert_batch(keys, keys)
    items = dict(t.items())
    print(mode, "statuses", np.bincount(st), "items", len(items), "oracle", len(o.as_dict()), "same map", items == o.as_dict(),
          "dups", len(t.duplicate_scan()), "nodes", t.arena.next_node, flush=True)
    for ilp in (5, 0):
        t.tune(query_ilp=ilp)
        f, v = t.query_batch(d(keys))
        print("   query kernel", "lines" if ilp else "generic", "found", int(f.sum()), "of", n, flush=True)

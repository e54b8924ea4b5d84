import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_16407_b200 import runners
for rep in range(2):
    r = runners.run_load_sweep("cuckoo", 1 << 26, load_points=(0.5, 0.55, 0.6), drain=False)
    print(rep, [(p["load"], round(p["insert_mops"]), round(p["query_mops"])) for p in r["points"]], flush=True)

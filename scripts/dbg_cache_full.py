import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_16407_b200.cache import DeviceCacheSim
from paper_2509_16407_b200.core import TableConfig
from paper_2509_16407_b200.tables import make_table
from paper_2509_16407_b200.workload import gen_uniform_keys
n = 1 << 14
keys = gen_uniform_keys(3, n); vals = keys ^ np.uint64(0x5555)
d = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).cuda().view(torch.uint64)
for up in (4, 0, 4, 0):
    for rep in range(3):
        backing = make_table(TableConfig(design="p2_md", capacity_slots=1 << 15, seed=9))
        backing.upsert_batch(d(keys), d(vals))
        slots = (int(n * 0.25 / 0.85) + 2 + 31) // 32 * 32
        table = make_table(TableConfig(design="double", capacity_slots=slots, seed=4))
        table.tune(upsert=up)
        sim = DeviceCacheSim(table, backing, capacity=int(n * 0.25))
        for lo in range(0, sim.capacity, 512):
            sim.get_batch(d(keys[lo:min(lo + 512, sim.capacity)]))
        idx = np.random.default_rng(rep).integers(0, n, size=4 * n)
        for lo in range(0, len(idx), 512):
            sim.get_batch(d(keys[idx[lo:lo + 512]]))
        print(f"upsert={up} rep={rep} full_events={sim.full_events} ring={len(sim.resident_keys())} load={table.load_factor():.3f}", flush=True)

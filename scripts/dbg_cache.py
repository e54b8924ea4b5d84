import os, sys, time
import faulthandler; faulthandler.dump_traceback_later(25, exit=True)
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_16407_b200.cache import DeviceCacheSim
from paper_2509_16407_b200.core import TableConfig
from paper_2509_16407_b200.tables import make_table
from paper_2509_16407_b200.workload import gen_uniform_keys
design = sys.argv[1]
n = 1 << 14
keys = gen_uniform_keys(3, n); vals = keys ^ np.uint64(0x5555)
d = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).cuda().view(torch.uint64)
backing = make_table(TableConfig(design="p2_md", capacity_slots=1 << 15, seed=9))
backing.upsert_batch(d(keys), d(vals))
slots = (int(n * 0.25 / 0.85) + 2 + 31) // 32 * 32
table = make_table(TableConfig(design=design, capacity_slots=slots, seed=4))
sim = DeviceCacheSim(table, backing, capacity=int(n * 0.25))
t0 = time.time()
for lo in range(0, sim.capacity, 512):
    sim.get_batch(d(keys[lo:min(lo + 512, sim.capacity)]))
print("warm", time.time() - t0, sim.misses, sim.evictions, flush=True)
idx = np.random.default_rng(1).integers(0, n, size=4 * n)
for j, lo in enumerate(range(0, len(idx), 512)):
    got = sim.get_batch(d(keys[idx[lo:lo + 512]]))
    if j % 16 == 0: print(j, time.time() - t0, sim.hits, sim.misses, sim.evictions, sim._size, flush=True)
print("done", time.time() - t0)

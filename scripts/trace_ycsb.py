"""Kernel timeline of YCSB batches (runners.run_ycsb) from torch.profiler:
per-kernel total time inside the timed mixed batches, to see where a
YCSB-A batch (50% REPLACE updates on Zipf(0.99) keys + 50% reads) goes.

  python scripts/trace_ycsb.py [A|B|C]
"""
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2509_16407_b200 import runners  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "A"
runners.run_ycsb(wl, universe=1 << 24, ops=1 << 25)  # warm-up
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    r = runners.run_ycsb(wl, universe=1 << 24, ops=1 << 26)
print({k: r[k] for k in ("workload", "ms", "mops", "final_values_exact")})
agg = defaultdict(lambda: [0.0, 0])
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        a = agg[e.name[:70]]
        a[0] += e.time_range.end - e.time_range.start
        a[1] += 1
for name, (us, n) in sorted(agg.items(), key=lambda x: -x[1][0])[:16]:
    print(f"{us / 1000:9.2f} ms  {n:5d}x  {name}")

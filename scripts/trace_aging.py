"""Kernel timeline of aging iterations (config 3) from torch.profiler's CUDA
activity trace: per iteration the wall span (first kernel start to last
kernel end), the summed kernel time and the idle gaps between kernels, so the
host-synchronisation cost of the per-kind segmentation is measured, not
guessed.

  python scripts/trace_aging.py [design] [iterations]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2509_16407_b200 import runners  # noqa: E402

import time  # noqa: E402

from paper_2509_16407_b200 import tables  # noqa: E402

# host-side duration of every mixed_batch call (enqueue time, including any
# synchronisation inside the library), next to the runner's CUDA-event time
_host_us = []
_orig = tables.HashTable.mixed_batch


def _timed_mixed(self, *a, **k):
    t0 = time.perf_counter()
    _marks.append(("mb_in", t0))
    r = _orig(self, *a, **k)
    _host_us.append(round((time.perf_counter() - t0) * 1e6, 1))
    return r


tables.HashTable.mixed_batch = _timed_mixed

# time from the runner's timer start (its first CUDA event record) to the
# mixed_batch call and to the C entry point
_marks = []
_orig_rec = torch.cuda.Event.record


def _rec(self, *a, **k):
    _marks.append(("event", time.perf_counter()))
    r = _orig_rec(self, *a, **k)
    _marks.append(("event_out", time.perf_counter()))
    return r


torch.cuda.Event.record = _rec
from paper_2509_16407_b200 import _native  # noqa: E402

_lib = _native.load()
_cmixed = _lib.ws_mixed


def _wrap_c(*a):
    _marks.append(("c_in", time.perf_counter()))
    r = _cmixed(*a)
    _marks.append(("c_out", time.perf_counter()))
    return r


_lib.ws_mixed = _wrap_c
design = sys.argv[1] if len(sys.argv) > 1 else "iceberg_md"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 6
runners.run_aging(design, 1 << 26, iterations=2, combine=True)  # warm-up (module load, pools)
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    r = runners.run_aging(design, 1 << 26, iterations=iters, combine=True)
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
kern = sorted(((e.time_range.start, e.time_range.end, e.name) for e in ev), key=lambda x: x[0])
# an iteration = the kernels between two k_comb_iota / kind-sort launches is fragile; instead split
# on gaps > 200 us (the runner's host-side checking between iterations)
groups, cur = [], []
for k in kern:
    if cur and k[0] - cur[-1][1] > 200:
        groups.append(cur)
        cur = []
    cur.append(k)
if cur:
    groups.append(cur)
out = []
for g in groups:
    span = g[-1][1] - g[0][0]
    busy = sum(b - a for a, b, _ in g)
    gaps = sorted(((g[i + 1][0] - g[i][1], g[i][2][:40], g[i + 1][2][:40]) for i in range(len(g) - 1)),
                  reverse=True)[:4]
    out.append({"kernels": len(g), "span_us": round(span, 1), "busy_us": round(busy, 1),
                "idle_us": round(span - busy, 1), "largest_gaps": [(round(x, 1), a, b) for x, a, b in gaps]})
print(json.dumps({"design": design, "iteration_ms": [round(i["ms"], 3) for i in r["iterations"]],
                  "host_call_us": _host_us[-iters:],
                  "marks_us": [(n, round((t - m[max(0, i - 1)][1]) * 1e6, 1)) for m in [_marks[-9 * iters:]]
                               for i, (n, t) in enumerate(m)],
                  "groups": out[-iters:]}, indent=1))
if len(sys.argv) > 3:  # raw timeline: [start_us, end_us, name] of every CUDA activity
    t0 = kern[0][0] if kern else 0
    json.dump([[round(a - t0, 2), round(b - t0, 2), n[:90]] for a, b, n in kern], open(sys.argv[3], "w"))

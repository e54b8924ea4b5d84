"""Paper Table 1 / figure data on one GPU for EVERY design (the reference's
`warpbench load|aging|scaling --design all`, bench/runners.py:172-405):

  load     insert to 0.05 .. 0.90 (+0.95) in 5% steps, timed batch per point,
           50/50 queries per point, instrumented probes/op per point, then the
           erase drain in 18 slices
  aging    the reference's aging workload at 0.85 (1% slices), throughput
           and instrumented probes/op per iteration
  scaling  probes/op and throughput at 2^17 / 2^20 / 2^23 slots

One reference-schema CSV per (benchmark, design) with the reference's
manifest goes to --out (default profiles/table1_r02/).  With WS_NCU_RANGES
set (see scripts/ncu_ranges.py) every timed batch is an ncu range, so the
load sweep also yields DRAM sectors per op for every point.

  python scripts/run_table1.py [--log2 24] [--designs all] [--aging-iters 40] [--skip aging,scaling]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2509_16407_b200 import runners  # noqa: E402

DESIGNS = ("double", "double_md", "p2", "p2_md", "iceberg", "iceberg_md", "cuckoo", "chaining")
BUCKET = {"chaining": 7, "double": 8, "cuckoo": 8}

ap = argparse.ArgumentParser()
ap.add_argument("--log2", type=int, default=24)
ap.add_argument("--designs", default="all")
ap.add_argument("--aging-iters", type=int, default=40)
ap.add_argument("--skip", default="")
ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "table1_r02"))
a = ap.parse_args()
designs = DESIGNS if a.designs == "all" else tuple(a.designs.split(","))
skip = set(a.skip.split(",")) if a.skip else set()
os.makedirs(a.out, exist_ok=True)
points = runners.LOAD_POINTS + (0.95,)
summary = {}
for d in designs:
    cap = (1 << a.log2) - (1 << a.log2) % BUCKET.get(d, 32)
    if d == "chaining":
        cap = 7 * (1 << (a.log2 - 3))  # 2^(log2-3) head nodes of 7 pairs
    t0 = time.time()
    out = {}
    if "load" not in skip:
        r = runners.run_load_sweep(d, cap, load_points=points, out_dir=a.out)
        last = [p for p in r["points"] if "load" in p]
        out["load"] = {"fulls": r["fulls"], "csv": os.path.relpath(r["csv"], ROOT),
                       "at_0.9": next(p for p in last if p["load"] == 0.9),
                       "all_queries_ok": all(p["queries_ok"] for p in last),
                       "after_drain_occupied": r["points"][-1].get("after_drain_occupied")}
    if "aging" not in skip:
        r = runners.run_aging_uniform(d, cap, iterations=a.aging_iters, out_dir=a.out)
        its = r["iterations"]
        out["aging"] = {"ok": r["ok"], "csv": os.path.relpath(r["csv"], ROOT),
                        "first": its[0]["probe_means"], "last": its[-1]["probe_means"],
                        "median_mops": sorted(i["mops"] for i in its)[len(its) // 2]}
    if "scaling" not in skip:
        sizes = (1 << 17, 1 << 20, 1 << 23)
        if d == "chaining":
            sizes = tuple(7 * (x >> 3) for x in sizes)
        r = runners.run_scaling(d, sizes=sizes, out_dir=a.out)
        out["scaling"] = {"csv": os.path.relpath(r["csv"], ROOT),
                          "per_size": [{k: v for k, v in e.items()} for e in r["per_size"]]}
    out["seconds"] = round(time.time() - t0, 1)
    summary[d] = out
    print(d, json.dumps(out), flush=True)
with open(os.path.join(a.out, "summary.json"), "w") as fh:
    json.dump(summary, fh, indent=1)

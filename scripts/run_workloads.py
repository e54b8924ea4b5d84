"""Run the BASELINE.json configs on one GPU; writes profiles/workloads_r01.{json,csv}.

  config 1: double 2^20, insert to 0.85, 2^19 interleaved 50/50 queries
  config 3: iceberg_md 2^26 aging with Zipf(0.99) upsert-ADD + adversarial race
  config 4: cuckoo 2^26 and chaining 7*2^23 load sweeps 0.50..0.95 (probes/op, Mops/s)
  config 5: canonical 31-mer counting (one shard; the multi-GPU routing is bench.py --gpus N)
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2509_16407_b200 import runners
from paper_2509_16407_b200.adversarial import DelayProfile, run_adversarial
from paper_2509_16407_b200.instrument import render_csv

quick = "--quick" in sys.argv
out = {}
rows = []
t0 = time.time()
r = runners.run_config1()
rows += r.pop("rows")
out["config1_double_2^20"] = r
print("config1", r, flush=True)

sweep = tuple(round(0.5 + 0.05 * i, 2) for i in range(10))
for design, cap in (("cuckoo", 1 << (22 if quick else 26)), ("chaining", 7 * (1 << (19 if quick else 23))),
                    ("p2_md", 1 << (22 if quick else 26))):
    r = runners.run_load_sweep(design, cap, load_points=sweep, drain=design != "chaining")
    rows += r.pop("rows")
    out[f"config4_sweep_{design}"] = r
    print("sweep", design, json.dumps(r)[:600], flush=True)

for comb in (True, False):
    r = runners.run_aging("iceberg_md", 1 << (22 if quick else 26), iterations=10 if quick else 40, combine=comb)
    rows += r.pop("rows")
    out[f"config3_aging_iceberg_md_combine{int(comb)}"] = r
    print("aging", json.dumps({k: v for k, v in r.items() if k != "iterations"}), flush=True)
for d in ("iceberg_md", "iceberg", "unsafe_reference"):
    a = run_adversarial(d, buckets=100_000 if quick else 1_000_000, trials=3, seed=5, profile=DelayProfile.light())
    out[f"config3_adversarial_{d}"] = a
    print("adversarial", a, flush=True)

for comb in (False, True):
    r = runners.run_kmer(genome_len=1 << (22 if quick else 27), capacity=1 << (23 if quick else 26),
                         repeats=4, combine=comb)
    out[f"config5_kmer_one_shard_combine{int(comb)}"] = r
    print("kmer", r, flush=True)
for wl in ("A", "B", "C"):
    r = runners.run_ycsb(wl, universe=1 << (20 if quick else 24), ops=1 << (22 if quick else 26))
    out[f"ycsb_{wl}"] = r
    print("ycsb", r, flush=True)
r = runners.run_phased_overhead(capacity=1 << (20 if quick else 24))
out["table1_concurrent_vs_phased_query"] = r
print("phased overhead", r, flush=True)
from paper_2509_16407_b200.cache import run_cache_sweep
r = run_cache_sweep(universe=1 << (18 if quick else 22), ratios=(0.1, 0.25, 0.5, 0.75, 0.9), queries_per_key=4.0,
                    batch=1 << 16)
out["cache_sweep"] = r
print("cache", r, flush=True)
out["seconds"] = time.time() - t0
os.makedirs("gpurun_out", exist_ok=True)
tag = "quick" if quick else "r01"
json.dump(out, open(f"gpurun_out/workloads_{tag}.json", "w"), indent=1, default=str)
open(f"gpurun_out/workloads_{tag}.csv", "w").write(render_csv(["one B200, paper_2509_16407_b200 runners"], rows))
print("done", out["seconds"])

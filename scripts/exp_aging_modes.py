"""The reference's aging workload (bench/runners.py:259-353: fill 0.85, then
1% slices of inserts + erases + present / absent queries per iteration) at
2^26 slots, as per-kind segments one after another (default), as the same
segments run concurrently on three streams (erases racing inserts and
queries with the tuned kernels), and as ONE interleaved generic launch per
batch; every result checked, probes per iteration recorded."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_16407_b200 import runners  # noqa: E402

for design in ("iceberg_md", "p2_md", "double_md", "cuckoo"):
    for mode in ("segments", "concurrent", "interleaved"):
        r = runners.run_aging_uniform(design, 1 << 26, iterations=30, interleaved=mode == "interleaved",
                                      concurrent=mode == "concurrent")
        its = r["iterations"]
        mops = sorted(i["mops"] for i in its)
        print(json.dumps({"design": design, "mode": mode, "ok": r["ok"], "slice": r["slice"],
                          "median_mops": round(mops[len(mops) // 2], 1),
                          "probes_first": its[0]["probe_means"], "probes_last": its[-1]["probe_means"]}),
              flush=True)

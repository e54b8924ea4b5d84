"""Repeat the small-table contention stress (tests/test_gpu_stress.py) over many
seeds and two table sizes; prints failures (a race hunt, not a unit test)."""
import os
import sys
import traceback

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import test_gpu_stress as T  # noqa: E402

fails = 0
runs = 0
for seed in range(int(sys.argv[1]) if len(sys.argv) > 1 else 6):
    for design in ("p2_md", "iceberg_md", "cuckoo", "chaining", "double_md", "double"):
        for how in ("mixed", "split", "split_combine"):
            orig = T.np.random.default_rng
            T.np.random.default_rng = lambda s, _o=orig, _seed=seed: _o(s * 1000 + _seed)
            try:
                T.test_small_table_contention(design, how)
            except Exception:  # noqa: BLE001
                fails += 1
                print("FAIL", seed, design, how)
                traceback.print_exc(limit=3)
            finally:
                T.np.random.default_rng = orig
            runs += 1
print(f"{runs} runs, {fails} failures", flush=True)

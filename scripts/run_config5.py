"""BASELINE config 5 at its stated size on one B200: 2^32 P2-MD slots,
canonical 31-mer counting with upsert-ADD to ~0.9 distinct-key load
(runners.run_kmer_full; the multi-GPU routing of the same workload is
tests/test_gpu_sharded.py and bench.py --gpus N).

  python scripts/run_config5.py [log2_slots] [repeats]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_16407_b200 import runners  # noqa: E402

log2 = int(sys.argv[1]) if len(sys.argv) > 1 else 32
rep = int(sys.argv[2]) if len(sys.argv) > 2 else 2
print(json.dumps(runners.run_kmer_full(log2_slots=log2, repeats=rep)), flush=True)

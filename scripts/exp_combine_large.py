"""Combining on batches past the L2-resident scratch size (> 2^21 ops), A/B
of two library builds in separate processes:

    python scripts/exp_combine_large.py [path/to/libwarpspeed.so]

k-mer counting (runners.run_kmer, 134M canonical 31-mers, 4 batches) with
and without combining, a 2^25-op Zipf(0.99) upsert-ADD batch and a 2^25-op
uniform REPLACE batch (every key about twice) into a 2^26-slot P2-MD table,
each with combine on and off (CUDA events, best of 3, table cleared between)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_16407_b200 import _native  # noqa: E402

if len(sys.argv) > 1:
    _native.LIB_PATH = os.path.abspath(sys.argv[1])

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_16407_b200 import TableConfig, make_table, runners  # noqa: E402
from paper_2509_16407_b200.workload import gen_uniform_keys, zipf_ranks  # noqa: E402

print("library", _native.LIB_PATH, flush=True)
for comb in (False, True):
    r = runners.run_kmer(genome_len=1 << 27, capacity=1 << 26, repeats=4, combine=comb)
    print(f"kmer combine={comb}: {r['mops']:.0f} M/s ok={r['ok']}", flush=True)

t = make_table(TableConfig(design="p2_md", capacity_slots=1 << 26, seed=3))
n = 1 << 25
uni = gen_uniform_keys(5, 1 << 24)
cases = {
    "zipf add": (uni[zipf_ranks(1 << 24, n, 0.99, seed=2) - 1], "add"),
    "uniform replace": (uni[np.random.default_rng(1).integers(0, 1 << 24, n)], None),
}
vals = torch.arange(n, device="cuda", dtype=torch.int64).view(torch.uint64)
for name, (keys, merge) in cases.items():
    dk = torch.from_numpy(keys.view(np.int64)).cuda().view(torch.uint64)
    for comb in (False, True):
        best = None
        for _ in range(3):
            t.clear()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            st = t.upsert_batch(dk, vals, merge=merge, combine=comb, check=False)
            b.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(b)
            best = ms if best is None else min(best, ms)
        print(f"{name} combine={comb}: {best:.2f} ms = {n / best / 1e6:.2f} G/s, "
              f"inserted={int((st == 0).sum())} full={int((st == 2).sum())} checksum={t.checksum()}", flush=True)

"""Experiment: does a batch whose chunks are ordered by primary bucket insert
faster through the unchanged P2-MD lock-round kernel?  The chunk sort is done
untimed here (it only asks whether ascending bucket order buys DRAM locality);
FULL counts are reported because any structured order can bias P2's choice.

usage: python scripts/exp_sorted_insert.py [--log2-slots 30] [--chunks 0,22,24,26]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

from paper_2509_16407_b200 import TableConfig, make_table
from paper_2509_16407_b200.workload import derive_seed, gen_uniform_keys


def srl(x, s):
    return (x >> s) & ((1 << (64 - s)) - 1)


def mix64_t(x):
    c1 = 0xBF58476D1CE4E5B9 - (1 << 64)
    c2 = 0x94D049BB133111EB - (1 << 64)
    x = x ^ srl(x, 30)
    x = x * c1
    x = x ^ srl(x, 27)
    x = x * c2
    return x ^ srl(x, 31)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--log2-slots", type=int, default=30)
    ap.add_argument("--chunks", default="0,22,24,26")
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    slots = 1 << a.log2_slots
    t = make_table(TableConfig(design="p2_md", capacity_slots=slots, seed=42))
    n = int(slots * 0.9)
    kh = gen_uniform_keys(derive_seed(42, 0), n)
    keys = torch.from_numpy(kh.view(np.int64)).to(dev)
    vals = keys & 0xFFFF
    s0 = int(t.family.seeds[0])
    s0 = s0 - (1 << 64) if s0 >= 1 << 63 else s0
    nb = slots // 32
    b0 = srl(mix64_t(keys ^ s0), 16) & (nb - 1)
    # sanity: the host definition of the primary bucket
    for i in range(4):
        assert int(b0[i]) == t._bucket0(int(kh[i])) if hasattr(t, "_bucket0") else True
    for c in [int(x) for x in a.chunks.split(",")]:
        if c == 0:
            k2, v2 = keys, vals
        else:
            C = 1 << c
            perm = torch.empty(n, dtype=torch.int64, device=dev)
            for lo in range(0, n, C):
                hi = min(n, lo + C)
                perm[lo:hi] = torch.argsort(b0[lo:hi]) + lo
            k2, v2 = keys[perm], vals[perm]
            del perm
        ku, vu = k2.view(torch.uint64), v2.view(torch.uint64)
        for r in range(a.reps):
            t.clear()
            torch.cuda.synchronize()
            t.kernel_times()
            t.time_kernels(True)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            st = t.upsert_batch(ku, vu)
            e1.record()
            torch.cuda.synchronize()
            kt = t.kernel_times()
            t.time_kernels(False)
            full = int((st == 2).sum())
            bad = int((st != 0).sum()) - full
            print(f"chunk=2^{c} rep={r}: call {e0.elapsed_time(e1):.2f} ms kernel {kt} FULL={full} bad={bad} "
                  f"-> {n / e0.elapsed_time(e1) / 1e6:.2f} G ins/s", flush=True)
        if c:
            del k2, v2, ku, vu
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()

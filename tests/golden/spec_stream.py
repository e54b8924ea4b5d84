"""SPEC acceptance 3 op streams (reference SPEC.md:659): the seeded mixed
sequence of reference pkg/tests/oracle.py:30-67 (run_mixed_sequence),
restated as op arrays so the same stream can be replayed on the reference
(make_golden.py), the C oracle and the device.

Pure Python `random` (no numpy draws), so the GPU box regenerates the
identical stream from (capacity, n_ops, seed); only digests of the
reference's outputs are committed (spec_equivalence.json).
"""

import hashlib
import random

import numpy as np

MASK = (1 << 64) - 1
# reference tests/oracle.py:28: MERGES = [_merge_add, _merge_keep, _merge_replace, None]
MERGE_IDS = (2, 1, 0, 0)   # device / oracle merge enum of each MERGES entry
SPEC_CAPACITY = 1 << 12    # reference test_tables.py:93-96 (cfg_for(design, 1 << 12, seed=3))
SPEC_TABLE_SEED = 3
SPEC_OPS = 100_000
SPEC_SEEDS = (11, 12, 13)
DESIGNS = ("double", "double_md", "p2", "p2_md", "iceberg", "iceberg_md", "cuckoo", "chaining")


def spec_stream(capacity_slots: int, n_ops: int, seed: int, universe_frac: float = 0.5):
    """(ops u8, keys u64, vals u64, merge_index list) of the reference's
    run_mixed_sequence draw order: key, r, then value + merge for upserts."""
    rng = random.Random(seed)
    universe_n = max(8, int(capacity_slots * universe_frac))
    universe = [rng.getrandbits(64) | 1 for _ in range(universe_n)]
    universe = [k if k < MASK - 1 else 3 for k in universe]
    ops = np.empty(n_ops, dtype=np.uint8)
    keys = np.empty(n_ops, dtype=np.uint64)
    vals = np.zeros(n_ops, dtype=np.uint64)
    midx = [0] * n_ops
    for i in range(n_ops):
        key = universe[rng.randrange(universe_n)]
        keys[i] = key
        r = rng.random()
        if r < 0.55:
            vals[i] = rng.getrandbits(64)
            m = rng.randrange(4)
            midx[i] = m
            ops[i] = 0 | (MERGE_IDS[m] << 4)
        elif r < 0.75:
            ops[i] = 1
        else:
            ops[i] = 2
    return ops, keys, vals, midx


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def items_digest(keys, vals) -> str:
    keys = np.asarray(keys, dtype=np.uint64)
    vals = np.asarray(vals, dtype=np.uint64)
    o = np.argsort(keys, kind="stable")
    return digest(keys[o], vals[o])

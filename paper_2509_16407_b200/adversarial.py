"""Adversarial duplicate-key race on the device (paper §4.1; reference
bench/adversarial.py).

Every primary bucket b gets a blocker key X_b (pre-inserted) and a fresh key
Y_b with the same primary bucket.  One mixed launch then runs, for every b,
three concurrent actors -- erase(X_b), upsert(Y_b, 1, keep),
upsert(Y_b, 2, keep) -- placed in adjacent warps of one CTA (actor_layout).  A table whose same-key
writers are not externally synchronised can commit Y_b twice; the duplicate
scan afterwards counts such buckets.  Device delay injection at the
reference's hook stages (pre_reserve / pre_publish / pre_tombstone /
pre_scan) widens the race windows like the reference's DelayProfile.
"""

from __future__ import annotations

import dataclasses

import numpy as np

from .core import DEFAULT_BUCKET_SIZE, TableConfig, validate_config
from .workload import derive_seed, mix64_np

OP_UPSERT, OP_ERASE = 0, 1
MERGE_KEEP = 1


@dataclasses.dataclass
class DelayProfile:
    """Device form of the reference's DelayProfile: one (probability,
    max nanoseconds) pair applied at every hook stage."""

    prob: float = 0.0
    max_ns: int = 0

    @classmethod
    def off(cls):
        return cls()

    @classmethod
    def light(cls):
        return cls(0.04, 30_000)

    @classmethod
    def heavy(cls):
        return cls(0.35, 200_000)


def config_for_primary_buckets(design: str, n_primary: int, seed: int,
                               mode: str = "concurrent") -> TableConfig:
    """A config whose primary-bucket space has exactly n_primary buckets
    (iceberg: solve total so round(total * 0.83) == n_primary, as the
    reference does at bench/adversarial.py:96-113)."""
    bucket = DEFAULT_BUCKET_SIZE[design]
    if design.startswith("iceberg"):
        frac = 0.83
        total = round(n_primary / frac)
        while round(total * frac) < n_primary:
            total += 1
        while round(total * frac) > n_primary:
            total -= 1
        capacity = total * bucket
    else:
        capacity = n_primary * bucket
    return validate_config(TableConfig(design=design, capacity_slots=capacity, seed=seed, mode=mode))


def generate_pairs(table, n_buckets: int, seed: int):
    """(X, Y) per primary bucket by binning uniform keys (vectorised form of
    reference bench/adversarial.py:116-145)."""
    s0 = np.uint64(table.family.seeds[0])
    npb = np.uint64(table.primary_bucket_count)
    xs = np.zeros(n_buckets, dtype=np.uint64)
    ys = np.zeros(n_buckets, dtype=np.uint64)
    have = np.zeros(n_buckets, dtype=np.int8)
    rng = np.random.default_rng(derive_seed(seed, n_buckets))
    while (have < 2).any():
        draw = rng.integers(1, 2**64 - 2, size=max(4096, 4 * n_buckets), dtype=np.uint64)
        b = ((mix64_np(draw ^ s0) >> np.uint64(16)) % npb).astype(np.int64)
        order = np.argsort(b, kind="stable")
        b, draw = b[order], draw[order]
        first = np.ones(len(b), dtype=bool)
        first[1:] = b[1:] != b[:-1]
        for take in (first, np.concatenate([[False], first[:-1] & ~first[1:]])):
            bb, kk = b[take], draw[take]
            need_x = have[bb] == 0
            xs[bb[need_x]] = kk[need_x]
            have[bb[need_x]] = 1
            need_y = (have[bb] == 1) & ~need_x & (xs[bb] != kk)
            ys[bb[need_y]] = kk[need_y]
            have[bb[need_y]] = 2
    return xs, ys


def actor_layout(xs, ys, warp: int = 32):
    """Op arrays of the three-actor script with the actors of a bucket
    co-scheduled: buckets go in groups of `warp`; each group is three
    consecutive warps of one launch -- erase(X) for the group's buckets, then
    upsert(Y, 1, keep), then upsert(Y, 2, keep) -- so the three actors of
    every bucket run in adjacent warps of the same CTA at the same time,
    the device counterpart of the reference's three threads re-aligned by a
    barrier every 128 buckets (bench/adversarial.py:37,169-177)."""
    n = len(xs)
    groups = (n + warp - 1) // warp
    pad = groups * warp - n
    role = np.repeat(np.arange(3, dtype=np.int64)[None, :], groups, axis=0)  # (groups, 3)
    bucket = (np.arange(groups, dtype=np.int64)[:, None, None] * warp +
              np.arange(warp, dtype=np.int64)[None, None, :])                 # (groups, 1, warp)
    role = np.broadcast_to(role[:, :, None], (groups, 3, warp)).reshape(-1)
    bucket = np.broadcast_to(bucket, (groups, 3, warp)).reshape(-1)
    keep = bucket < n
    role, bucket = role[keep], bucket[keep]
    assert len(role) == 3 * n and pad >= 0
    up = np.uint8(OP_UPSERT | (MERGE_KEEP << 4))
    ops = np.where(role == 0, np.uint8(OP_ERASE), up).astype(np.uint8)
    keys = np.where(role == 0, np.asarray(xs, np.uint64)[bucket], np.asarray(ys, np.uint64)[bucket])
    vals = role.astype(np.uint64)  # erase 0, first upsert 1, second upsert 2
    return ops, keys, vals


def run_adversarial(design: str, buckets: int = 10_000, trials: int = 3, seed: int = 5,
                    profile: DelayProfile | None = None, device=None, keep_table: bool = False) -> dict:
    """`trials` replays over `buckets` primary buckets; returns total duplicate
    buckets and per-trial counts (any duplicate on a synchronised design is a
    correctness failure)."""
    import torch

    from .tables import make_table

    profile = profile or DelayProfile.light()
    cfg = config_for_primary_buckets(design, buckets, seed)
    table = make_table(cfg, device=device)
    xs, ys = generate_pairs(table, buckets, seed)
    dev = table.device

    def cu(a):
        return torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).to(dev).view(torch.uint64)

    n = buckets
    ops, keys, vals = actor_layout(xs, ys)
    d_ops = torch.from_numpy(ops).to(dev)
    d_keys, d_vals = cu(keys), cu(vals)
    per_trial = []
    y_set = set(ys.tolist())
    for trial in range(trials):
        table.clear()
        st = table.upsert_batch(cu(xs), cu(np.ones(n, np.uint64)))
        if int((st == 2).sum()):
            raise RuntimeError("adversarial pre-insert hit FULL")
        table.set_delays(profile.max_ns, profile.prob, derive_seed(seed, trial))
        table.mixed_batch(d_ops, d_keys, d_vals, interleaved=True)  # erase races the inserts
        table.set_delays(0, 0.0, 0)
        dups = table.duplicate_scan()
        assert all(k in y_set for k in dups), "duplicate of a non-replayed key"
        per_trial.append(len(dups))
    rep = {"design": design, "buckets": buckets, "trials": trials,
           "replays": buckets * trials, "duplicate_buckets": sum(per_trial),
           "per_trial": per_trial, "actors_per_bucket": 3}
    if keep_table:  # the last trial's table, for further inspection
        rep["table"] = table
    return rep

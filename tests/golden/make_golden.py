"""Generate golden fixtures by running the REFERENCE implementation itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py          # small op streams + known answers
    python tests/golden/make_golden.py --spec   # SPEC.md:659 10^5-op x 3-seed digests

It imports the reference package (warpbench, pure Python) from
/root/reference/pkg/src under the alias ``warpbench_ref`` and records:

* hash_kat.json  -- seeds of HashFamily, mix64, bucket and tag known answers,
                    gen_uniform_keys / derive_seed outputs, iceberg splits,
                    validate_config outcomes (reference core.py, bench/keys.py)
* ops_<design>_<stream>.npz -- a seeded op stream replayed sequentially on a
                    reference table with a ProbeRecorder attached: per-op
                    status / found / value / probe count, the lock-touch total,
                    and the final raw slot-key layout (+ tags for md designs,
                    node count for chaining).

The fixtures are small and committed; nothing at test time reads
/root/reference.  The oracle (oracle/ws_oracle.c) and the device path are
both checked against them.
"""

from __future__ import annotations

import importlib.util
import json
import os
import random
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src/warpbench"
OUT = os.path.dirname(os.path.abspath(__file__))

MASK = (1 << 64) - 1
ALL = ["double", "double_md", "p2", "p2_md", "iceberg", "iceberg_md",
       "cuckoo", "chaining", "unsafe_reference"]
MERGE_NAMES = ["replace", "keep", "add", "max", "min"]


def load_reference():
    spec = importlib.util.spec_from_file_location(
        "warpbench_ref", os.path.join(REF_SRC, "__init__.py"),
        submodule_search_locations=[REF_SRC])
    mod = importlib.util.module_from_spec(spec)
    sys.modules["warpbench_ref"] = mod
    spec.loader.exec_module(mod)
    return mod


REF = load_reference()
from warpbench_ref import core as rcore  # noqa: E402
from warpbench_ref.bench import keys as rkeys  # noqa: E402
from warpbench_ref.instrument import ProbeRecorder  # noqa: E402
from warpbench_ref.tables import UpsertStatus, make_table  # noqa: E402

MERGE_FN = {
    "replace": None,
    "keep": lambda o, n: o,
    "add": lambda o, n: o + n,
    "max": lambda o, n: max(o, n),
    "min": lambda o, n: min(o, n),
}
STATUS = {UpsertStatus.INSERTED: 0, UpsertStatus.UPDATED: 1, UpsertStatus.FULL: 2}


def hash_kat():
    out = {"families": {}, "mix64": [], "buckets": [], "keys": {}, "derive_seed": [],
           "iceberg": [], "configs": []}
    for seed in (0, 42, 0x5EED, 12345, MASK):
        out["families"][str(seed)] = [str(s) for s in rcore.HashFamily(seed, 8).seeds]
    rng = random.Random(7)
    xs = [0, 1, 2, 3, MASK, MASK - 1, 0x123456789ABCDEF0] + [rng.getrandbits(64) for _ in range(40)]
    out["mix64"] = [[str(x), str(rcore.mix64(x))] for x in xs]
    fam = rcore.HashFamily(42, 4)
    for key in [1, 2, 0x123456789ABCDEF0] + [rng.getrandbits(64) | 1 for _ in range(40)]:
        for nb in (1, 7, 1000, 1 << 23, 27197, (1 << 31) + 11):
            out["buckets"].append([str(key), nb, fam.bucket(0, key, nb), fam.bucket(1, key, nb),
                                   fam.bucket(2, key, nb), rcore.fingerprint(fam, key)])
    for seed, n in ((42, 8), (7, 16), (derive := rkeys.derive_seed(42, 0xFEED), 8)):
        out["keys"][str(seed)] = [str(k) for k in rkeys.gen_uniform_keys(seed, n).tolist()]
    del derive
    for parts in ((42,), (42, 0xFEED), (5, 1, 2, 3), (MASK, 0)):
        out["derive_seed"].append([[str(p) for p in parts], str(rkeys.derive_seed(*parts))])
    for cap in (1 << 10, 1 << 20, 100 * 32, 4 * 32, 3200, 1 << 26):
        t = make_table(rcore.TableConfig(design="iceberg", capacity_slots=cap))
        out["iceberg"].append([cap, t.front_buckets, t.back_buckets])
    cases = [
        dict(design="double", capacity_slots=4096, bucket_size=8),
        dict(design="p2", capacity_slots=4096, bucket_size=32),
        dict(design="double", capacity_slots=4096, bucket_size=4),
        dict(design="double", capacity_slots=100, bucket_size=8),
        dict(design="double", capacity_slots=120, bucket_size=12),
        dict(design="p2", capacity_slots=0, mode="bogus", probe_cap=0),
        dict(design="robinhood", capacity_slots=64),
        dict(design="chaining", capacity_slots=700),
        dict(design="chaining", capacity_slots=800, bucket_size=8),
        dict(design="iceberg", capacity_slots=32),
        dict(design="iceberg_md", capacity_slots=3200, seed=99, probe_cap=64),
        dict(design="cuckoo", capacity_slots=64, cuckoo_ways=1, cuckoo_path_depth=0),
        dict(design="p2_md", capacity_slots=4096, shortcut_threshold=1.5, line_bytes=24),
    ]
    for c in cases:
        try:
            cfg = rcore.validate_config(rcore.TableConfig(**c))
            out["configs"].append([c, "ok", cfg.bucket_size])
        except rcore.ConfigError as e:
            out["configs"].append([c, "error", e.problems])
    with open(os.path.join(OUT, "hash_kat.json"), "w") as fh:
        json.dump(out, fh, indent=0)


def _cap_for(design, cap, bucket=0):
    bs = bucket or rcore.DEFAULT_BUCKET_SIZE[design]
    return cap - cap % bs


def run_stream(design, stream, cap, seed, n_ops, universe_frac, extra=None, fill=False, out_name=None):
    cfg = rcore.TableConfig(design=design, capacity_slots=_cap_for(design, cap, (extra or {}).get("bucket_size", 0)),
                            seed=seed, **(extra or {}))
    t = make_table(cfg)
    rng = random.Random(seed * 1000 + len(stream))
    rec = ProbeRecorder(line_bytes=cfg.line_bytes)
    ops, keys, vals, status, qvals, probes = [], [], [], [], [], []
    if stream == "fill" or fill:
        # distinct fresh keys until well past capacity (FULL / BFS / growth paths)
        n_ops = int(t.capacity_slots * universe_frac)
        seq = [(0, rng.getrandbits(64) | 1, rng.getrandbits(64), 0) for _ in range(n_ops)]
    else:
        universe_n = max(8, int(t.capacity_slots * universe_frac))
        universe = [rng.getrandbits(64) | 1 for _ in range(universe_n)]
        universe = [k if k < MASK - 1 else 3 for k in universe]
        seq = []
        for _ in range(n_ops):
            key = universe[rng.randrange(universe_n)]
            r = rng.random()
            if r < 0.55:
                seq.append((0, key, rng.getrandbits(64), rng.randrange(5)))
            elif r < 0.75:
                seq.append((1, key, 0, 0))
            else:
                seq.append((2, key, 0, 0))
    for kind, key, val, m in seq:
        if kind == 0:
            s = STATUS[t.upsert(key, val, MERGE_FN[MERGE_NAMES[m]], probe=rec)]
            q = 0
        elif kind == 1:
            s = int(t.erase(key, probe=rec))
            q = 0
        else:
            got = t.query(key, probe=rec)
            s, q = (0, 0) if got is None else (1, got)
        probes.append(rec.finish_op("op"))
        ops.append(kind | (m << 4))
        keys.append(key)
        vals.append(val)
        status.append(s)
        qvals.append(q)
    res = dict(
        ops=np.array(ops, dtype=np.uint8), keys=np.array(keys, dtype=np.uint64),
        vals=np.array(vals, dtype=np.uint64), status=np.array(status, dtype=np.uint8),
        qvals=np.array(qvals, dtype=np.uint64), probes=np.array(probes, dtype=np.uint32),
        lock_touches=np.array([rec.lock_touches], dtype=np.uint64),
        capacity=np.array([t.capacity_slots], dtype=np.uint64),
        seed=np.array([seed], dtype=np.uint64),
    )
    items = list(t.items())
    res["item_keys"] = np.array([k for k, _ in items], dtype=np.uint64)
    res["item_vals"] = np.array([v for _, v in items], dtype=np.uint64)
    if design == "chaining":
        a = t.arena
        res["next_node"] = np.array([a.next_node], dtype=np.uint64)
        res["arena_capacity"] = np.array([a.capacity_nodes], dtype=np.uint64)
        res["words"] = np.array(a.words[: a.wpn * a.next_node], dtype=np.uint64)
    else:
        res["slot_keys"] = np.array([t.slots.key_at(i) for i in range(t.capacity_slots)],
                                    dtype=np.uint64)
        if getattr(t, "tags", None) is not None:
            res["tags"] = np.array([t.tags.get(i) for i in range(t.capacity_slots)],
                                   dtype=np.uint16)
    res["extra"] = np.array([json.dumps(extra or {})])
    np.savez_compressed(os.path.join(OUT, out_name or f"ops_{design}_{stream}.npz"), **res)
    return res


def spec_equivalence():
    """SPEC.md:659 (acceptance 3): 10^5 seeded mixed ops x 3 seeds per design on
    the reference tables through the scalar API (reference
    tests/oracle.py:30-67 semantics), recorded as digests of the per-op
    results, the final map and the final slot layout."""
    sys.path.insert(0, OUT)
    from spec_stream import (DESIGNS, MERGE_IDS, SPEC_CAPACITY, SPEC_OPS, SPEC_SEEDS,
                             SPEC_TABLE_SEED, digest, items_digest, spec_stream)
    fns = {0: MERGE_FN["add"], 1: MERGE_FN["keep"], 2: MERGE_FN["replace"], 3: None}
    out = {"capacity": SPEC_CAPACITY, "table_seed": SPEC_TABLE_SEED, "n_ops": SPEC_OPS,
           "seeds": list(SPEC_SEEDS), "merge_ids": list(MERGE_IDS), "streams": {}}
    for d in DESIGNS:
        cfg = rcore.TableConfig(design=d, capacity_slots=_cap_for(d, SPEC_CAPACITY), seed=SPEC_TABLE_SEED)
        for seed in SPEC_SEEDS:
            t = make_table(cfg)
            ops, keys, vals, midx = spec_stream(t.capacity_slots, SPEC_OPS, seed)
            status = np.zeros(SPEC_OPS, dtype=np.uint8)
            qvals = np.zeros(SPEC_OPS, dtype=np.uint64)
            for i in range(SPEC_OPS):
                k, kind = int(keys[i]), int(ops[i]) & 15
                if kind == 0:
                    status[i] = STATUS[t.upsert(k, int(vals[i]), fns[midx[i]])]
                elif kind == 1:
                    status[i] = int(t.erase(k))
                else:
                    got = t.query(k)
                    if got is not None:
                        status[i], qvals[i] = 1, got
            items = list(t.items())
            rec = {"status": digest(status), "qvals": digest(qvals),
                   "items": items_digest([a for a, _ in items], [b for _, b in items]),
                   "n_items": len(items), "fulls": int((status[ops & 15 == 0] == 2).sum())}
            if d == "chaining":
                a = t.arena
                w = np.array(a.words[: a.wpn * a.next_node], dtype=np.uint64).reshape(-1, a.wpn)
                rec["layout"] = digest(w[:, list(range(0, a.wpn - 2, 2)) + [a.wpn - 2]])  # keys + link
            else:
                rec["layout"] = digest(np.array([t.slots.key_at(i) for i in range(t.capacity_slots)],
                                                dtype=np.uint64))
            out["streams"][f"{d}/{seed}"] = rec
            print("spec", d, seed, rec["n_items"], rec["fulls"], flush=True)
    with open(os.path.join(OUT, "spec_equivalence.json"), "w") as fh:
        json.dump(out, fh, indent=1)


def main():
    if "--spec" in sys.argv:
        spec_equivalence()
        return
    hash_kat()
    for d in ALL:
        cap = 7 * 128 if d == "chaining" else 1024
        run_stream(d, "mixed", cap, seed=11, n_ops=6000, universe_frac=0.8)
        run_stream(d, "churn", cap, seed=12, n_ops=8000, universe_frac=1.1)
        run_stream(d, "fill", 256 if d != "chaining" else 7 * 32, seed=13, n_ops=0,
                   universe_frac=2.0 if d == "chaining" else 1.15)
    # a couple of non-default knobs
    run_stream("p2_md", "phased", 1024, seed=21, n_ops=3000, universe_frac=0.6,
               extra={"mode": "phased"})
    run_stream("double", "cap16", 1024, seed=22, n_ops=4000, universe_frac=1.1,
               extra={"probe_cap": 16})
    run_stream("cuckoo", "ways4", 1024, seed=23, n_ops=0, universe_frac=1.05,
               extra={"cuckoo_ways": 4, "cuckoo_path_depth": 3}, fill=True)
    run_stream("iceberg_md", "front50", 1024, seed=24, n_ops=5000, universe_frac=1.0,
               extra={"iceberg_front_fraction": 0.5})
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()

"""Generate randomized-configuration golden streams by running the REFERENCE.

Run in the build container (where /root/reference exists):

    python tests/golden/make_fuzz.py

The fixed fixtures of make_golden.py cover each design at its default knobs
(plus four single-knob variants).  These cases draw the knobs the reference
exposes on TableConfig (reference core.py:185-291) at random -- bucket_size,
line_bytes, odd bucket counts, probe_cap, shortcut_threshold,
iceberg_front_fraction, cuckoo_ways / cuckoo_path_depth, phased mode -- keep
every draw the reference's validate_config accepts, and record one seeded op
stream per case exactly as make_golden.run_stream does (per-op status /
value / line probes, lock touches, final slot layout and tags).  The cases
are written to fuzz_cases.npz (one archive, keys prefixed by case index) so
the oracle (CPU) and the device (serial replay) are checked on configurations
no hand-picked fixture covers.
"""

from __future__ import annotations

import json
import os
import random
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import make_golden as mg  # noqa: E402  (imports the reference as warpbench_ref)

N_CASES = 40
SEED = 20261018


def draw_config(rng, design):
    """One random knob set the reference accepts (ConfigError -> redraw)."""
    for _ in range(200):
        extra = {}
        line = rng.choice([64, 128, 128, 256])
        if design == "chaining":
            bucket = rng.randint(1, (line - 8) // 16)
        else:
            choices = [b for b in (2, 4, 8, 16, 32) if (b * 16) % line == 0 or 2 * b * 16 == line]
            bucket = rng.choice(choices)
        if line != 128:
            extra["line_bytes"] = line
        if bucket != mg.rcore.DEFAULT_BUCKET_SIZE[design]:
            extra["bucket_size"] = bucket
        if design in ("double", "double_md") and rng.random() < 0.6:
            extra["probe_cap"] = rng.choice([1, 2, 3, 5, 8, 16, 40])
        if design in ("p2", "p2_md", "unsafe_reference") and rng.random() < 0.7:
            extra["shortcut_threshold"] = rng.choice([0.25, 0.5, 0.6, 0.9, 1.0])
        if design in ("iceberg", "iceberg_md") and rng.random() < 0.7:
            extra["iceberg_front_fraction"] = rng.choice([0.3, 0.5, 0.7, 0.9])
        if design == "cuckoo":
            extra["cuckoo_ways"] = rng.choice([2, 3, 4])
            extra["cuckoo_path_depth"] = rng.randint(1, 5)
        if design != "unsafe_reference" and rng.random() < 0.15:
            extra["mode"] = "phased"
        nb = rng.randint(3, 160)
        cap = nb * bucket
        try:
            mg.rcore.validate_config(mg.rcore.TableConfig(design=design, capacity_slots=cap, seed=1, **extra))
        except mg.rcore.ConfigError:
            continue
        return extra, cap
    raise RuntimeError(f"no valid config drawn for {design}")


def main():
    rng = random.Random(SEED)
    out = {}
    index = []
    for i in range(N_CASES):
        design = mg.ALL[i % len(mg.ALL)]
        extra, cap = draw_config(rng, design)
        stream = rng.choice(["mixed", "churn", "fill"])
        seed = rng.randrange(1, 1 << 32)
        if stream == "fill":
            frac = 2.0 if design == "chaining" else rng.choice([0.9, 1.05, 1.2])
            n_ops = 0
        else:
            frac = rng.choice([0.5, 0.8, 1.1, 1.4])
            n_ops = rng.randint(800, 2500)
        name = f"_fuzz_tmp_{i}.npz"
        res = mg.run_stream(design, stream, cap, seed, n_ops, frac, extra=extra or None,
                            fill=stream == "fill", out_name=name)
        os.remove(os.path.join(mg.OUT, name))
        res["design"] = np.array([design])
        for k, v in res.items():
            out[f"{i}/{k}"] = v
        index.append({"case": i, "design": design, "stream": stream, "capacity": int(res["capacity"][0]),
                      "extra": extra, "ops": int(res["ops"].size),
                      "fulls": int(((res["ops"] & 15) == 0).sum() and (res["status"][(res["ops"] & 15) == 0] == 2).sum())})
        print(json.dumps(index[-1]), flush=True)
    out["n_cases"] = np.array([N_CASES])
    np.savez_compressed(os.path.join(mg.OUT, "fuzz_cases.npz"), **out)
    with open(os.path.join(mg.OUT, "fuzz_index.json"), "w") as fh:
        json.dump(index, fh, indent=1)


if __name__ == "__main__":
    main()

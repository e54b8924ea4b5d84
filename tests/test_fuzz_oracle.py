"""The oracle against 40 randomized-configuration streams recorded from the
reference (tests/golden/make_fuzz.py): non-default bucket sizes, line
sizes, odd bucket counts, probe caps, shortcut thresholds, iceberg front
fractions, cuckoo ways / path depths and phased mode -- per-op status,
value, line probes, lock touches, final map and slot layout, bit for bit."""

import numpy as np
import pytest

from fuzz_cases import load_cases

CASES = load_cases()


@pytest.mark.parametrize("name,case,cfg", CASES, ids=[c[0] for c in CASES])
def test_oracle_replays_fuzz_case(name, case, cfg):
    from oracle import OracleTable
    z = case
    t = OracleTable(cfg)
    probes = np.zeros(len(z["ops"]), dtype=np.uint32)
    status, qvals = t.mixed_batch(z["ops"], z["keys"], z["vals"], probes=probes)
    np.testing.assert_array_equal(status, z["status"])
    np.testing.assert_array_equal(qvals, z["qvals"])
    np.testing.assert_array_equal(probes, z["probes"])
    assert t.lock_touches == int(z["lock_touches"][0])
    k, v = t.items_arrays()
    np.testing.assert_array_equal(k, z["item_keys"])
    np.testing.assert_array_equal(v, z["item_vals"])
    if cfg.design == "chaining":
        assert t.next_node == int(z["next_node"][0])
        assert t.arena_capacity == int(z["arena_capacity"][0])
        wpn = 2 * cfg.bucket_size + 2
        w = t.words().reshape(-1, wpn)
        ref = z["words"].reshape(-1, wpn)
        np.testing.assert_array_equal(w[: ref.shape[0], : 2 * cfg.bucket_size : 2], ref[:, : 2 * cfg.bucket_size : 2])
        np.testing.assert_array_equal(w[: ref.shape[0], 2 * cfg.bucket_size], ref[:, 2 * cfg.bucket_size])
    else:
        np.testing.assert_array_equal(t.slot_keys(), z["slot_keys"])
        if "tags" in z:
            np.testing.assert_array_equal(t.tags(), z["tags"])
    assert t.duplicate_scan() == {}

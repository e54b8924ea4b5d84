"""Small-table stress: heavy bucket contention through every kernel path.

A 2^10-slot table (chaining: 7 x 128) receives 24 batches; each batch erases
some live keys, upsert-ADDs others (sampled with replacement: many same-key
ops per batch, many ops per bucket) and queries a third disjoint set.  Roles
are key-disjoint and ADD is commutative, so a numpy/dict model predicts every
result exactly: query hits and values, erase found flags, one INSERTED per
new key, the final map, no duplicates.  Run both as single mixed launches
(generic kernels) and as separate uniform launches (the tuned lock-round
kernels), with and without combining.
"""

import numpy as np
import pytest

from conftest import cfg_for

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _cuda(a):
    a = np.ascontiguousarray(a)
    if a.dtype == np.uint8:
        return torch.from_numpy(a).cuda()
    return torch.from_numpy(a.astype(np.uint64, copy=False).view(np.int64)).cuda().view(torch.uint64)


def _np(t):
    return t.cpu().view(torch.int64).numpy().view(np.uint64) if t.dtype == torch.uint64 else t.cpu().numpy()


@pytest.mark.parametrize("how", ["mixed", "split", "split_combine"])
@pytest.mark.parametrize("design", ["p2_md", "iceberg_md", "cuckoo", "chaining", "double_md", "double"])
def test_small_table_contention(design, how):
    from paper_2509_16407_b200 import make_table
    from paper_2509_16407_b200.tables import OP_ERASE, OP_QUERY, OP_UPSERT
    from paper_2509_16407_b200.workload import gen_uniform_keys
    cfg = cfg_for(design, 1024 if design != "chaining" else 7 * 128, seed=13)
    t = make_table(cfg)
    uni = gen_uniform_keys(77, int(t.capacity_slots * 0.55))
    rng = np.random.default_rng(5)
    model = {}
    for it in range(24):
        live = np.array(sorted(model), dtype=np.uint64)
        perm = rng.permutation(len(uni))
        live_set = set(model)
        er = np.array([k for k in live[rng.permutation(len(live))][: len(live) // 5]], dtype=np.uint64)
        taken = set(er.tolist())
        cand = [k for k in uni[perm].tolist() if k not in taken]
        up_keys = np.array(cand[: len(cand) // 2], dtype=np.uint64)
        q_keys = np.array(cand[len(cand) // 2:], dtype=np.uint64)
        ups = up_keys[rng.integers(0, len(up_keys), 3 * len(up_keys))]
        vals = rng.integers(1, 1000, len(ups)).astype(np.uint64)
        if how == "mixed":
            ops = np.concatenate([np.full(len(er), OP_ERASE), np.full(len(ups), OP_UPSERT | (2 << 4)),
                                  np.full(len(q_keys), OP_QUERY)]).astype(np.uint8)
            keys = np.concatenate([er, ups, q_keys])
            vv = np.concatenate([np.zeros(len(er), np.uint64), vals, np.zeros(len(q_keys), np.uint64)])
            p = rng.permutation(len(ops))
            st, vo = t.mixed_batch(_cuda(ops[p]), _cuda(keys[p]), _cuda(vv[p]))
            inv = np.empty_like(p)
            inv[p] = np.arange(len(p))
            st, vo = _np(st)[inv], _np(vo)[inv]
            s_er, s_up, s_q = st[: len(er)], st[len(er): len(er) + len(ups)], st[len(er) + len(ups):]
            v_q = vo[len(er) + len(ups):]
        else:
            s_er = _np(t.erase_batch(_cuda(er))).astype(np.uint8) if len(er) else np.zeros(0, np.uint8)
            s_up = _np(t.upsert_batch(_cuda(ups), _cuda(vals), merge="add", combine=how == "split_combine"))
            f, v = t.query_batch(_cuda(q_keys))
            s_q, v_q = _np(f).astype(np.uint8), _np(v)
        # erases: every erased key was live
        assert s_er.astype(bool).all(), (it, design)
        # queries: disjoint from this batch's writers -> pre-batch state
        want_f = np.array([k in live_set for k in q_keys.tolist()])
        np.testing.assert_array_equal(s_q.astype(bool), want_f)
        want_v = np.array([model.get(k, 0) for k in q_keys.tolist()], dtype=np.uint64)
        np.testing.assert_array_equal(v_q[want_f], want_v[want_f])
        # upserts: one INSERTED per key new to the table, no FULL
        assert not (s_up == 2).any(), (it, design, np.bincount(s_up))
        new_keys = set(k for k in ups.tolist() if k not in live_set)
        assert int((s_up == 0).sum()) == len(new_keys), (it, design)
        for k in er.tolist():
            del model[k]
        for k, v in zip(ups.tolist(), vals.tolist()):
            model[k] = model.get(k, 0) + v
    assert dict(t.items()) == model
    assert t.duplicate_scan() == {}

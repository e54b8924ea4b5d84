"""Device workload runners for the BASELINE.json configs (the GPU counterparts
of reference bench/runners.py).  Every runner verifies results, times the
device batches with CUDA events, and returns a report dict plus reference-
schema CSV rows (instrument.Row).

* ``run_config1``  double hashing 2^20: insert to 0.85, 2^19 interleaved
  50/50 queries (reference runners.py:130-144, 172-181)
* ``run_load_sweep``  insert / query / probes per load point, then an erase
  drain (reference runners.py:172-256); config 4 = cuckoo / chaining sweeps
* ``run_aging``  prefill 0.85, then mixed batches: Zipf upsert-ADD on live
  keys + fresh inserts, erase of the oldest slice, queries on untouched live
  keys and on absent keys (reference runners.py:259-353; config 3)
* ``run_aging_uniform``  the reference's own aging workload with its
  instrumented probe phase (SPEC acceptance 8, Table 1 aging probes)
* ``run_scaling``  probe means / throughput per table size (reference
  runners.py:356-405; SPEC acceptance 13)
* ``run_kmer``  canonical 31-mer counting with upsert-ADD (config 5 on one
  table / shard)
"""

from __future__ import annotations

import contextlib
import json
import os
import time

import numpy as np

from .core import TableConfig
from .instrument import Row, write_csv
from .workload import derive_seed, gen_uniform_keys, kmer_keys, mix64_np, zipf_ranks

U64 = np.uint64
LOAD_POINTS = tuple(round(0.05 * i, 2) for i in range(1, 19))


def _torch():
    import torch
    return torch


def _dev(a, device):
    torch = _torch()
    a = np.ascontiguousarray(a)
    if a.dtype == np.uint8:
        return torch.from_numpy(a).to(device)
    return torch.from_numpy(a.astype(U64, copy=False).view(np.int64)).to(device).view(torch.uint64)


def _np(t):
    torch = _torch()
    t = t.cpu()
    if t.dtype == torch.uint64:
        return t.view(torch.int64).numpy().view(U64)
    return t.numpy()


class _Timer:
    def __init__(self):
        torch = _torch()
        self.a = torch.cuda.Event(enable_timing=True)
        self.b = torch.cuda.Event(enable_timing=True)

    def __enter__(self):
        self.a.record()
        return self

    def __exit__(self, *exc):
        self.b.record()
        self.b.synchronize()
        self.ms = self.a.elapsed_time(self.b)


def _mops(n, ms):
    return n / ms / 1e3 if ms > 0 else 0.0


# ------------------------------------------------------------ CSV + manifest

def manifest_lines(benchmark: str, table, seed: int, extra=()) -> list:
    """The reference's '#'-prefixed CSV manifest (bench/runners.py:66-86),
    field for field; `threads` is 0 (one device launch per batch, no host
    thread pool) and `slot_engine` / `wide_atomic` come from the table's
    capability report."""
    from . import __version__
    cfg = table.config
    cap = table.capability_report()
    lines = [
        f"benchmark={benchmark}",
        f"design={cfg.design}",
        f"capacity_slots={table.capacity_slots}",
        f"bucket_size={table.bucket_size}",
        f"line_bytes={cfg.line_bytes}",
        f"probe_cap={cfg.probe_cap}",
        f"mode={cfg.mode}",
        f"seed={seed}",
        "threads=0",
        f"slot_engine={cap['slot_engine']}",
        f"wide_atomic={cap['wide_atomic']}",
        f"num_buckets={table.num_buckets}",
        f"version={__version__}",
        f"timestamp={time.strftime('%Y-%m-%dT%H:%M:%S')}",
    ]
    lines.extend(extra)
    return lines


def write_report_csv(out_dir, benchmark: str, table, rows, seed: int, extra=()) -> str:
    """`{out_dir}/{benchmark}_{design}.csv` in the reference schema
    (instrument.CSV_HEADER) with the manifest above; returns the path."""
    path = os.path.join(out_dir, f"{benchmark}_{table.config.design}.csv")
    write_csv(path, manifest_lines(benchmark, table, seed, extra), rows)
    return path


# ------------------------------------------------------- ncu range markers
# WS_NCU_RANGES=<file>: every timed batch of the runners becomes one
# cudaProfilerStart/Stop range opened by a one-element torch fill (the range
# marker), and the range's (design, op, load) label is appended to <file>.
# Under `ncu --profile-from-start off` the launch list is then the marker,
# the batch's kernels, the next marker, ... -- scripts/ncu_ranges.py joins
# it with the labels into DRAM sectors per op for every load point.
_NCU_MARK = None


@contextlib.contextmanager
def _ncu_range(label: dict, ops: int):
    path = os.environ.get("WS_NCU_RANGES")
    if not path:
        yield
        return
    global _NCU_MARK
    torch = _torch()
    if _NCU_MARK is None:
        _NCU_MARK = torch.zeros(1, dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    _NCU_MARK.fill_(1)
    try:
        yield
    finally:
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
        with open(path, "a", encoding="utf-8") as fh:
            fh.write(json.dumps({**label, "ops": int(ops)}) + "\n")


def run_config1(seed: int = 42, capacity: int = 1 << 20, design: str = "double") -> dict:
    from .tables import make_table
    t = make_table(TableConfig(design=design, capacity_slots=capacity, seed=seed))
    dev = t.device
    n = int(capacity * 0.85)
    keys = gen_uniform_keys(seed, n)
    nq = min(1 << 19, 2 * (n // 2))
    miss = gen_uniform_keys(derive_seed(seed, 0xFEED), nq // 2)
    hits = keys[: nq // 2]
    q = np.empty(nq, dtype=U64)
    q[0::2], q[1::2] = hits, miss
    dk, dv, dq = _dev(keys, dev), _dev(keys & U64(0xFFFF), dev), _dev(q, dev)
    t.upsert_batch(dk, dv)  # warm the kernels (lazy module loading) outside the timed region
    t.query_batch(dq)
    t.clear()
    with _Timer() as ti:
        st = t.upsert_batch(dk, dv, check=False)
    with _Timer() as tq:
        found, vals = t.query_batch(dq, check=False)
    f, v = _np(found).astype(bool), _np(vals)
    ok = (_np(st) == 0).all() and f[0::2].all() and not f[1::2].any() and \
        (v[0::2] == (hits & U64(0xFFFF))).all()
    rows = [Row(design, "concurrent", capacity, 128, "throughput", "insert", 0.85, 0, n, ti.ms / 1e3,
                _mops(n, ti.ms)),
            Row(design, "concurrent", capacity, 128, "throughput", "query_5050", 0.85, 0, nq, tq.ms / 1e3,
                _mops(nq, tq.ms))]
    return {"ok": bool(ok), "insert_mops": _mops(n, ti.ms), "query_mops": _mops(nq, tq.ms), "rows": rows}


def run_load_sweep(design: str, capacity: int, seed: int = 42, load_points=LOAD_POINTS,
                   query_sample: int = 1 << 20, probe_sample: int = 4096, mode: str = "concurrent",
                   drain: bool = True, out_dir: str | None = None) -> dict:
    """Insert to each load point (timed batch), 50/50 queries (timed), probe
    means from instrumented batches (reference ProbeRecorder semantics), then
    an erase drain in 18 slices."""
    from .tables import OP_QUERY, OP_UPSERT, make_table
    cfg = TableConfig(design=design, capacity_slots=capacity, seed=seed, mode=mode)
    t = make_table(cfg)
    dev = t.device
    cap = t.capacity_slots
    n_max = int(cap * load_points[-1])
    keys = gen_uniform_keys(seed, n_max)
    neg = gen_uniform_keys(derive_seed(seed, 0xFEED), query_sample)
    rows, points, fulls = [], [], 0
    placed = 0
    inserted_mask = np.ones(n_max, dtype=bool)
    t.query_batch(_dev(neg[:4096], dev), check=False)  # first-launch costs outside the timed region
    # first-batch allocation costs (status tensors, pool growth) outside the
    # timed region: run the first load point's batch once on a scratch table
    scratch = make_table(cfg)
    w0 = _dev(keys[: int(cap * load_points[0])], dev)
    scratch.upsert_batch(w0, w0, check=False)
    del scratch, w0
    for point in load_points:
        target = int(cap * point)
        batch = keys[placed:target]
        # the batch's last probe_sample inserts run instrumented
        np_ins = min(probe_sample, len(batch) // 4)
        timed = batch[: len(batch) - np_ins]
        d_timed = _dev(timed, dev)  # H2D outside the timed region
        with _ncu_range({"design": design, "op": "insert", "load": point}, len(timed)), _Timer() as ti:
            st = t.upsert_batch(d_timed, d_timed, check=False)
        st_np = _np(st)
        fulls += int((st_np == 2).sum())
        if (st_np == 2).any():  # FULLed keys are legitimately absent: keep them out of the hit set
            inserted_mask[placed:placed + len(timed)] &= st_np != 2
        ins_probe = 0.0
        if np_ins:
            pst, _v, pr, _l = t.probe_batch(np.full(np_ins, OP_UPSERT, np.uint8), batch[-np_ins:],
                                            batch[-np_ins:], serial=False)
            fulls += int((pst == 2).sum())
            inserted_mask[target - np_ins:target] &= pst != 2
            ins_probe = float(pr.mean())
        placed = target
        qn = min(query_sample, placed)
        live_keys = keys[:placed][inserted_mask[:placed]]
        pos = live_keys[np.linspace(0, len(live_keys) - 1, qn // 2).astype(np.int64)]
        q = np.concatenate([pos, neg[: qn - len(pos)]])
        d_q = _dev(q, dev)
        with _ncu_range({"design": design, "op": "query_5050", "load": point}, qn), _Timer() as tq:
            found, _vals = t.query_batch(d_q, check=False)
        f = _np(found).astype(bool)
        ok = bool(f[: len(pos)].all() and not f[len(pos):].any())
        ps = min(probe_sample, len(pos))
        _s, _v, prp, _l = t.probe_batch(np.full(ps, OP_QUERY, np.uint8), pos[:ps], serial=False)
        _s, _v, prn, _l = t.probe_batch(np.full(ps, OP_QUERY, np.uint8), neg[:ps], serial=False)
        rows += [
            Row(design, mode, cap, 128, "throughput", "insert", point, 0, len(timed), ti.ms / 1e3,
                _mops(len(timed), ti.ms)),
            Row(design, mode, cap, 128, "probe", "insert", point, 0, np_ins, 0, 0, ins_probe),
            Row(design, mode, cap, 128, "throughput", "query_5050", point, 0, qn, tq.ms / 1e3, _mops(qn, tq.ms)),
            Row(design, mode, cap, 128, "probe", "query_pos", point, 0, ps, 0, 0, float(prp.mean())),
            Row(design, mode, cap, 128, "probe", "query_neg", point, 0, ps, 0, 0, float(prn.mean())),
        ]
        points.append({"load": point, "insert_mops": _mops(len(timed), ti.ms), "query_mops": _mops(qn, tq.ms),
                       "probes_insert": ins_probe, "probes_query_pos": float(prp.mean()),
                       "probes_query_neg": float(prn.mean()), "queries_ok": ok, "fulls_so_far": fulls})
    if drain:
        live = keys[:placed][inserted_mask[:placed]]
        chunk = -(-len(live) // 18)
        for off in range(0, len(live), chunk):
            sl = live[off:off + chunk]
            d_sl = _dev(sl, dev)
            with _ncu_range({"design": design, "op": "erase", "load": round((len(live) - off) / cap, 4)},
                            len(sl)), _Timer() as te:
                gone = t.erase_batch(d_sl, check=False)
            rows.append(Row(design, mode, cap, 128, "throughput", "erase", round((len(live) - off) / cap, 4), 0,
                            len(sl), te.ms / 1e3, _mops(len(sl), te.ms)))
            if not bool(_np(gone).all()):
                points.append({"drain_error": off})
        points.append({"after_drain_occupied": t.occupied_count()})
    csv = write_report_csv(out_dir, "load", t, rows, seed, [f"fulls={fulls}"]) if out_dir else None
    return {"design": design, "capacity": cap, "fulls": fulls, "points": points, "rows": rows, "csv": csv}


def run_aging(design: str = "iceberg_md", capacity: int = 1 << 26, iterations: int = 20,
              slice_fraction: float = 0.01, seed: int = 42, theta: float = 0.99,
              zipf_ops_per_slice: float = 1.0, combine: bool = True) -> dict:
    """Aging with Zipf upsert-ADD (config 3).  Per iteration one mixed launch:
    fresh keys inserted (ADD), a Zipf(theta) sample of live keys upsert-ADDed,
    the oldest slice erased, the next slice queried (present) and absent keys
    queried -- key roles disjoint, so results are order-independent.  Every
    status / found flag / value is checked against a numpy model; the final
    table checksum is compared to the model's."""
    from .tables import OP_ERASE, OP_QUERY, OP_UPSERT, make_table
    torch = _torch()
    t = make_table(TableConfig(design=design, capacity_slots=capacity, seed=seed))
    dev = t.device
    cap = t.capacity_slots
    fill = int(cap * 0.85)
    sl = max(8, int(fill * slice_fraction))
    stream = gen_uniform_keys(seed, fill + sl * iterations)
    absent = gen_uniform_keys(derive_seed(seed, 0xADAE), sl * iterations)
    values = np.zeros(len(stream), dtype=U64)  # model: value of stream[i] while live
    values[:fill] = stream[:fill] & U64(0xFFFF)
    st = t.upsert_batch(_dev(stream[:fill], dev), _dev(values[:fill], dev))
    if int((_np(st) != 0).sum()):
        raise RuntimeError("aging prefill did not insert every key")
    head, tail = 0, fill
    ADD = OP_UPSERT | (2 << 4)
    rows, its = [], []
    total_ok = True
    for it in range(iterations):
        new = np.arange(tail, tail + sl)
        old = np.arange(head, head + sl)
        pos = np.arange(head + sl, head + 2 * sl)
        live_lo = head + 2 * sl  # Zipf universe: live keys outside the erase / query slices
        uni = tail - live_lo
        nz = int(sl * zipf_ops_per_slice)
        zr = zipf_ranks(uni, nz, theta, seed=derive_seed(seed, it)) - 1
        zidx = live_lo + zr
        zval = (mix64_np(np.arange(nz, dtype=U64) + U64(it)) & U64(0xFF))
        ops = np.concatenate([np.full(sl, ADD), np.full(nz, ADD), np.full(sl, OP_ERASE),
                              np.full(sl, OP_QUERY), np.full(sl, OP_QUERY)]).astype(np.uint8)
        keys = np.concatenate([stream[new], stream[zidx], stream[old], stream[pos],
                               absent[it * sl:(it + 1) * sl]])
        newv = stream[new] & U64(0xFFFF)
        vals = np.concatenate([newv, zval, np.zeros(3 * sl, U64)])
        perm = np.argsort((keys * U64(0x9E3779B97F4A7C15)) & U64(0xFFFFFFFF), kind="stable")
        d_ops, d_keys, d_vals = _dev(ops[perm], dev), _dev(keys[perm], dev), _dev(vals[perm], dev)
        with _Timer() as tm:
            s, v = t.mixed_batch(d_ops, d_keys, d_vals, check=False, combine=combine)
        s, v = _np(s), _np(v)
        inv = np.empty_like(perm)
        inv[perm] = np.arange(len(perm))
        s, v = s[inv], v[inv]
        # model: statuses and values
        o = 0
        ok = (s[o:o + sl] == 0).all()  # fresh inserts
        o += sl
        ok &= (s[o:o + nz] == 1).all()  # Zipf adds hit live keys
        o += nz
        ok &= (s[o:o + sl] == 1).all()  # erases found
        o += sl
        ok &= (s[o:o + sl] == 1).all() and (v[o:o + sl] == values[pos]).all()  # present, pre-add values
        o += sl
        ok &= not s[o:o + sl].any()  # absent
        with np.errstate(over="ignore"):
            np.add.at(values, zidx, zval)
        values[new] = newv
        values[old] = 0
        head += sl
        tail += sl
        total_ok &= bool(ok)
        n_ops = len(ops)
        its.append({"iteration": it, "ops": n_ops, "ms": tm.ms, "mops": _mops(n_ops, tm.ms), "ok": bool(ok)})
        rows.append(Row(design, "concurrent", cap, 128, "throughput", "mixed", round(fill / cap, 4), 0, n_ops,
                        tm.ms / 1e3, _mops(n_ops, tm.ms)))
    live = np.arange(head, tail)
    with np.errstate(over="ignore"):
        lk, lv = stream[live], values[live]
        want = (len(live), int(lk.sum(dtype=U64)), int(lv.sum(dtype=U64)),
                int(np.bitwise_xor.reduce(mix64_np(lk ^ mix64_np(lv)))))
    got = t.checksum()
    del torch
    return {"design": design, "capacity": cap, "slice": sl, "iterations": its, "ok": total_ok,
            "checksum_ok": got == want, "duplicates": t.duplicate_count(),
            "mean_mops": float(np.mean([i["mops"] for i in its])), "rows": rows}


def _probe_means(t, ops, keys, vals, kinds, serial=False):
    """Instrumented pass; returns {kind: mean distinct lines} for the
    contiguous op groups in `kinds`.  The ops of one pass touch distinct keys,
    so each op's probe count is that of its own path whether the pass runs
    serially (the reference's single recorder) or one thread per op."""
    st, vo, pr, _locks = t.probe_batch(ops, keys, vals, serial=serial)
    out, o = {}, 0
    for kind, n in kinds:
        if n:
            out[kind] = float(pr[o:o + n].mean())
        o += n
    return st, vo, out


def run_aging_uniform(design: str, capacity: int, iterations: int = 200, slice_fraction: float = 0.01,
                      seed: int = 42, probe_sample: int = 200, line_bytes: int = 128,
                      out_dir: str | None = None, interleaved: bool = False, concurrent: bool = False) -> dict:
    """The reference's aging workload restated (bench/runners.py:259-353):
    fill to 85%, then per iteration one concurrent mixed launch that inserts
    a 1% slice of new keys (value k & 0xFFFF), erases the oldest 1%, queries
    1% known-present and 1% known-absent keys -- interleaved by the
    reference's (k * 0x9E3779B97F4A7C15) & 0xFFFFFFFF sort -- followed by the
    instrumented probe phase on the first `probe_sample` keys of each slice
    (upsert value 1, erase, present query, absent query; serial, as the
    reference's single-threaded recorder).  Every result is checked.
    interleaved=True runs each mixed batch as ONE launch with the kinds
    interleaved (WS_F_INTERLEAVED), so erases race inserts and queries inside
    the kernel as the reference's threads do; concurrent=True runs the
    per-kind segments concurrently on three streams with the tuned kernels;
    the default runs them one after another (one serial order of the batch)."""
    from .tables import OP_ERASE, OP_QUERY, OP_UPSERT, make_table
    t = make_table(TableConfig(design=design, capacity_slots=capacity, seed=seed, line_bytes=line_bytes))
    dev = t.device
    cap = t.capacity_slots
    fill_n = int(cap * 0.85)
    slice_n = max(4, int(fill_n * slice_fraction))
    stream = gen_uniform_keys(seed, fill_n + slice_n * iterations + 16)
    neg_stream = gen_uniform_keys(derive_seed(seed, 0xADAE), slice_n * iterations + 16)
    st = t.upsert_batch(_dev(stream[:fill_n], dev), _dev(stream[:fill_n] & U64(0xFFFF), dev))
    if int((_np(st) == 2).sum()):
        raise RuntimeError("aging prefill hit full")
    probe_n = min(probe_sample, slice_n)
    head, nxt = 0, fill_n
    its, rows, ok_all = [], [], True
    for it in range(iterations):
        new_k = stream[nxt:nxt + slice_n]
        old_k = stream[head:head + slice_n]          # FIFO = insertion order of the stream
        pos_k = stream[head + slice_n:head + 2 * slice_n]
        neg_k = neg_stream[it * slice_n:(it + 1) * slice_n]
        kinds = np.concatenate([np.full(slice_n - probe_n, c, np.uint8) for c in (0, 1, 2, 3)])
        keys = np.concatenate([new_k[probe_n:], old_k[probe_n:], pos_k[probe_n:], neg_k[probe_n:]])
        order = np.argsort((keys * U64(0x9E3779B97F4A7C15)) & U64(0xFFFFFFFF), kind="stable")
        kinds, keys = kinds[order], keys[order]
        ops = np.where(kinds == 0, OP_UPSERT, np.where(kinds == 1, OP_ERASE, OP_QUERY)).astype(np.uint8)
        vals = np.where(kinds == 0, keys & U64(0xFFFF), U64(0))
        d_ops, d_keys, d_vals = _dev(ops, dev), _dev(keys, dev), _dev(vals, dev)
        with _ncu_range({"design": design, "op": "mixed", "load": round(fill_n / cap, 4), "iteration": it},
                        len(ops)), _Timer() as tm:
            s, _v = t.mixed_batch(d_ops, d_keys, d_vals, check=False, interleaved=interleaved,
                                  concurrent=concurrent)
        s = _np(s)
        ok = bool((s[kinds == 0] == 0).all() and (s[kinds == 1] == 1).all() and
                  (s[kinds == 2] == 1).all() and not s[kinds == 3].any())
        p_ops = np.concatenate([np.full(probe_n, OP_UPSERT), np.full(probe_n, OP_ERASE),
                                np.full(2 * probe_n, OP_QUERY)]).astype(np.uint8)
        p_keys = np.concatenate([new_k[:probe_n], old_k[:probe_n], pos_k[:probe_n], neg_k[:probe_n]])
        p_vals = np.concatenate([np.ones(probe_n, U64), np.zeros(3 * probe_n, U64)])
        ps, _pv, means = _probe_means(t, p_ops, p_keys, p_vals,
                                      [("insert", probe_n), ("erase", probe_n), ("query_pos", probe_n),
                                       ("query_neg", probe_n)])
        ok &= bool((ps[:probe_n] == 0).all() and (ps[probe_n:3 * probe_n] == 1).all() and
                   not ps[3 * probe_n:].any())
        ok_all &= ok
        head += slice_n
        nxt += slice_n
        lf = round(fill_n / cap, 4)
        rows.append(Row(design, "concurrent", cap, line_bytes, "throughput", "mixed", lf, 0, len(ops),
                        tm.ms / 1e3, _mops(len(ops), tm.ms)))
        for kind, m in means.items():
            rows.append(Row(design, "concurrent", cap, line_bytes, "probe", kind, lf, 1, probe_n, 0.0, 0.0, m))
        its.append({"iteration": it, "probe_means": means, "mops": _mops(len(ops), tm.ms), "ok": ok})
    csv = write_report_csv(out_dir, "aging", t, rows, seed) if out_dir else None
    return {"design": design, "capacity": cap, "slice": slice_n, "iterations": its, "ok": ok_all,
            "occupied": t.occupied_count(), "fill_n": fill_n, "rows": rows, "csv": csv}


def run_scaling(design: str, sizes=(1 << 17, 1 << 20, 1 << 23), seed: int = 42, probe_sample: int = 4096,
                query_sample: int = 1 << 20, line_bytes: int = 128, probe_window: float = 0.0,
                out_dir: str | None = None) -> dict:
    """Insert to 90% and positive-query throughput plus probe means per table
    size (reference bench/runners.py:356-405): the last stretch of the fill
    is inserted instrumented, then instrumented positive / negative queries.
    probe_window > 0 sizes that stretch as a load fraction (the same load
    window at every size) instead of the reference's min(probe_sample,
    fill / 5) keys."""
    from .tables import OP_QUERY, OP_UPSERT, make_table
    per_size, rows = [], []
    for size in sizes:
        t = make_table(TableConfig(design=design, capacity_slots=size, seed=seed, line_bytes=line_bytes))
        dev = t.device
        cap = t.capacity_slots
        fill_n = int(cap * 0.9)
        probe_ins_n = (max(1, int(cap * probe_window)) if probe_window > 0
                       else min(probe_sample, max(1, fill_n // 5)))
        n = fill_n - probe_ins_n
        keys = gen_uniform_keys(derive_seed(seed, size), fill_n)
        dk, dv = _dev(keys[:n], dev), _dev(keys[:n] & U64(0xFFFF), dev)  # H2D outside the timed region
        with _ncu_range({"design": design, "op": "insert", "load": 0.9, "size": cap}, n), _Timer() as ti:
            st = t.upsert_batch(dk, dv, check=False)
        fulls = int((_np(st) == 2).sum())
        stride = max(1, n // min(query_sample, n))
        pos = keys[:n][::stride][:min(query_sample, n)]
        d_pos = _dev(pos, dev)
        with _ncu_range({"design": design, "op": "query_pos", "load": 0.9, "size": cap}, len(pos)), \
                _Timer() as tq:
            f, _v = t.query_batch(d_pos, check=False)
        miss = int((~_np(f).astype(bool)).sum())
        ins_ops = np.full(probe_ins_n, OP_UPSERT, np.uint8)
        pst, _pv, m_ins = _probe_means(t, ins_ops, keys[n:], np.ones(probe_ins_n, U64),
                                       [("insert", probe_ins_n)])
        fulls += int((pst == 2).sum())
        ps = min(probe_sample, n)
        pstride = max(1, fill_n // ps)
        psample = keys[::pstride][:ps]
        negs = gen_uniform_keys(derive_seed(seed, size, 3), probe_sample)
        q_ops = np.full(len(psample) + len(negs), OP_QUERY, np.uint8)
        _s, _v2, m_q = _probe_means(t, q_ops, np.concatenate([psample, negs]), None,
                                    [("query_pos", len(psample)), ("query_neg", len(negs))])
        means = {**m_ins, **m_q}
        rows.append(Row(design, "concurrent", cap, line_bytes, "throughput", "insert", 0.9, 0, n, ti.ms / 1e3,
                        _mops(n, ti.ms)))
        rows.append(Row(design, "concurrent", cap, line_bytes, "throughput", "query_pos", 0.9, 0, len(pos),
                        tq.ms / 1e3, _mops(len(pos), tq.ms)))
        for kind, m in means.items():
            rows.append(Row(design, "concurrent", cap, line_bytes, "probe", kind, 0.9, 1, 0, 0.0, 0.0, m))
        per_size.append({"size": cap, "probe_means": means, "fulls": fulls, "missing": miss,
                         "insert_mops": _mops(n, ti.ms), "query_mops": _mops(len(pos), tq.ms)})
        last = t
    csv = write_report_csv(out_dir, "scaling", last, rows, seed) if out_dir and sizes else None
    return {"design": design, "per_size": per_size, "rows": rows, "csv": csv}


def run_kmer(genome_len: int = 1 << 24, k: int = 31, capacity: int = 1 << 25, design: str = "p2_md",
             seed: int = 7, batches: int = 4, repeats: int = 4, combine: bool = False) -> dict:
    """Count canonical k-mers of a synthetic genome with upsert-ADD; every
    count is checked against numpy's.  The genome is `repeats` copies of a
    random base sequence, so k-mer multiplicities are known (~repeats)."""
    from .tables import make_table
    t = make_table(TableConfig(design=design, capacity_slots=capacity, seed=seed))
    dev = t.device
    km = kmer_keys(genome_len, k, seed, repeats=repeats)
    rng = np.random.default_rng(seed)
    km = km[rng.permutation(len(km))]  # reads arrive in arbitrary order
    ones = np.ones(len(km), dtype=U64)
    parts = np.array_split(np.arange(len(km)), batches)
    # warm-up on a scratch table: the first launch of a new batch size grows
    # the stream-ordered memory pool (combining scratch), outside the timing
    scratch = make_table(TableConfig(design=design, capacity_slots=capacity, seed=seed))
    scratch.upsert_batch(_dev(km[parts[0]], dev), _dev(ones[parts[0]], dev), merge="add", check=False,
                         combine=combine)
    del scratch
    ms = 0.0
    for part in parts:
        d_k, d_o = _dev(km[part], dev), _dev(ones[part], dev)
        with _Timer() as tm:
            st = t.upsert_batch(d_k, d_o, merge="add", check=False, combine=combine)
        ms += tm.ms
        if int((_np(st) == 2).sum()):
            raise RuntimeError("k-mer table hit FULL: raise capacity")
    u, c = np.unique(km, return_counts=True)
    found, vals = t.query_batch(_dev(u, dev))
    ok = bool(_np(found).all() and (_np(vals) == c.astype(U64)).all())
    return {"kmers": len(km), "distinct": len(u), "load": len(u) / t.capacity_slots, "ok": ok,
            "ms": ms, "mops": _mops(len(km), ms), "occupied": t.occupied_count()}


def _kmers_device(genome, lo: int, m: int, k: int = 31):
    """Canonical k-mers (2 bits/base, +1) starting at genome[lo:lo+m] of a
    device uint8 base tensor -- the device twin of workload.kmer_keys (test
    workload generation for config 5 at full size, not a table path)."""
    torch = _torch()
    fwd = torch.zeros(m, dtype=torch.int64, device=genome.device)
    rev = torch.zeros(m, dtype=torch.int64, device=genome.device)
    for j in range(k):
        b = genome[lo + j:lo + j + m].to(torch.int64)
        fwd = (fwd << 2) | b
        rev = rev | ((3 - b) << (2 * j))
    return (torch.minimum(fwd, rev) + 1).view(torch.uint64)


def run_kmer_full(log2_slots: int = 32, load: float = 0.9, repeats: int = 2, k: int = 31, seed: int = 7,
                  chunk: int = 1 << 27, design: str = "p2_md") -> dict:
    """BASELINE config 5 at its stated size on one B200 (2^32 P2-MD slots =
    64 GiB of cells + 8 GiB of tags, SURVEY 8(a) sizing): a seeded random
    genome of load * 2^32 bases is generated on the device, and its canonical
    31-mers are upsert-ADDed `repeats` times in chunks of `chunk` k-mers, so
    the distinct-key load is ~`load` and every k-mer's count is `repeats`
    times its multiplicity in the genome.  Checked: no FULL, no duplicates,
    the table's value sum equals repeats x the number of k-mers, every k-mer
    of the genome is found with a positive multiple of `repeats`."""
    from .tables import make_table
    torch = _torch()
    cap = 1 << log2_slots
    t = make_table(TableConfig(design=design, capacity_slots=cap, seed=seed))
    dev = t.device
    n_kmers = int(cap * load)
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    genome = torch.randint(0, 4, (n_kmers + k - 1,), dtype=torch.uint8, device=dev, generator=g)
    ones = torch.ones(chunk, dtype=torch.int64, device=dev).view(torch.uint64)
    ms, fulls = 0.0, 0
    for _rep in range(repeats):
        for lo in range(0, n_kmers, chunk):
            m = min(chunk, n_kmers - lo)
            km = _kmers_device(genome, lo, m, k)
            with _Timer() as tm:
                st = t.upsert_batch(km, ones[:m], merge="add", check=False)
            ms += tm.ms
            fulls += int((st == 2).sum())
    occupied, _sk, sv, _x = t.checksum()
    found_all, mult_ok = True, True
    for lo in range(0, n_kmers, chunk):
        m = min(chunk, n_kmers - lo)
        f, v = t.query_batch(_kmers_device(genome, lo, m, k), check=False)
        found_all &= bool(f.bool().all())
        vv = v.view(torch.int64)
        mult_ok &= bool(((vv > 0) & (vv % repeats == 0)).all())
    dups = t.duplicate_count()
    ok = fulls == 0 and dups == 0 and sv == repeats * n_kmers and found_all and mult_ok
    return {"ok": ok, "slots": cap, "kmers": n_kmers, "repeats": repeats, "upserts": repeats * n_kmers,
            "distinct": occupied, "load": occupied / cap, "fulls": fulls, "duplicates": dups,
            "value_sum_exact": sv == repeats * n_kmers, "ms": ms, "mops": _mops(repeats * n_kmers, ms)}


YCSB_MIX = {"A": 0.50, "B": 0.05, "C": 0.0}  # update fraction (reference apps/ycsb.py:21)


def run_ycsb(workload: str, universe: int = 1 << 24, ops: int = 1 << 26, capacity: int = 0,
             design: str = "p2_md", theta: float = 0.99, seed: int = 42, batch: int = 1 << 24,
             combine: bool = True) -> dict:
    """YCSB A/B/C on the device table (reference apps/ycsb.py:37-93): the
    universe is preloaded (values k & 0xFFFF), keys are Zipf(theta) ranks,
    one update every 1/ratio ops (REPLACE with value i & 0xFFFFFFFF), the rest
    queries.  Each chunk of `batch` ops is one mixed launch.  Every query must
    hit; with combining (stable sort keeps index order) the final values are
    exactly those of the reference's sequential run (last update wins)."""
    from .tables import OP_QUERY, OP_UPSERT, make_table
    frac = YCSB_MIX[workload]
    cap = capacity or int(universe / 0.85) // 32 * 32
    t = make_table(TableConfig(design=design, capacity_slots=cap, seed=seed))
    dev = t.device
    keys = gen_uniform_keys(seed, universe)
    st = t.upsert_batch(_dev(keys, dev), _dev(keys & U64(0xFFFF), dev))
    if int((_np(st) != 0).sum()):
        raise RuntimeError("YCSB preload did not insert every key")
    period = round(1 / frac) if frac else 0
    ranks = zipf_ranks(universe, ops, theta, seed=derive_seed(seed, 1)) - 1
    idx = np.arange(ops, dtype=np.int64)
    is_up = (idx % period == 0) if period else np.zeros(ops, dtype=bool)
    op_b = np.where(is_up, OP_UPSERT, OP_QUERY).astype(np.uint8)  # merge 0 = REPLACE
    ks = keys[ranks]
    vs = (idx.astype(np.uint64) & U64(0xFFFFFFFF))
    ms, missing = 0.0, 0
    # warm-up at full batch size with the workload's op mix, updates as
    # upsert-KEEP of present keys (table unchanged): the first launch of a new
    # size grows the stream-ordered memory pool (~0.1 s) on the same path the
    # timed batches take
    wq = min(batch, ops)
    w_ops = np.where(is_up[:wq], OP_UPSERT | (1 << 4), OP_QUERY).astype(np.uint8)
    t.mixed_batch(_dev(w_ops, dev), _dev(ks[:wq], dev), _dev(vs[:wq], dev), combine=combine)
    for lo in range(0, ops, batch):
        hi = min(ops, lo + batch)
        d_o, d_k, d_v = _dev(op_b[lo:hi], dev), _dev(ks[lo:hi], dev), _dev(vs[lo:hi], dev)
        with _Timer() as tm:
            s, _v = t.mixed_batch(d_o, d_k, d_v, check=False, combine=combine)
        ms += tm.ms
        s = _np(s)
        missing += int((~is_up[lo:hi] & (s == 0)).sum())
    # model of the final values: preload, then the last update of each key in index order
    final = keys & U64(0xFFFF)
    if period:
        up_i = np.nonzero(is_up)[0]
        final[ranks[up_i]] = vs[up_i]  # fancy assignment keeps the last write per index
    found, vals = t.query_batch(_dev(keys, dev))
    values_ok = bool(_np(found).all() and (_np(vals) == final).all()) if combine else bool(_np(found).all())
    return {"workload": workload, "universe": universe, "ops": ops, "updates": int(is_up.sum()),
            "ms": ms, "mops": _mops(ops, ms), "missing_queries": missing, "final_values_exact": values_ok,
            "combine": combine}


def run_phased_overhead(designs=("double", "double_md", "iceberg", "iceberg_md", "p2", "p2_md", "cuckoo",
                                 "chaining"), capacity: int = 1 << 24, seed: int = 42, reps: int = 3) -> dict:
    """Concurrent vs phased (BSP) query throughput per design (paper Table 1,
    PAPER.md:1390-1415; reference runners.py:408-476): the same fill, then the
    same 50/50 hit/miss query batch against a `mode="concurrent"` and a
    `mode="phased"` table; overhead = 1 - concurrent / phased."""
    from .tables import make_table
    torch = _torch()
    out = {}
    for design in designs:
        load = 0.85 if design.startswith("double") else (1.0 if design == "chaining" else 0.9)
        res = {}
        for mode in ("concurrent", "phased"):
            cfg = TableConfig(design=design, capacity_slots=capacity if design != "chaining" else 7 * (capacity // 8),
                              seed=seed, mode=mode)
            t = make_table(cfg)
            dev = t.device
            n = int(t.capacity_slots * load)
            keys = gen_uniform_keys(seed, n)
            dk = _dev(keys, dev)
            t.upsert_batch(dk, dk, check=False)
            miss = gen_uniform_keys(derive_seed(seed, 0xFEED), n // 2)
            q = np.concatenate([keys[: n // 2], miss])
            np.random.default_rng(seed).shuffle(q)
            dq = _dev(q, dev)
            t.query_batch(dq, check=False)  # warm-up
            best = 1e30
            for _ in range(reps):
                with _Timer() as tm:
                    f, _v = t.query_batch(dq, check=False)
                best = min(best, tm.ms)
            hits = int(_np(f).astype(bool).sum())
            res[mode] = {"query_mops": _mops(len(q), best), "hits": hits}
            del t, dk, dq
            torch.cuda.empty_cache()
        c, p = res["concurrent"]["query_mops"], res["phased"]["query_mops"]
        out[design] = {"concurrent_mops": c, "phased_mops": p, "overhead_pct": 100.0 * (1 - c / p) if p else 0.0,
                       "same_hits": res["concurrent"]["hits"] == res["phased"]["hits"]}
    return out

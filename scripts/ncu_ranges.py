"""DRAM sectors per op for every timed batch of a runner script.

  python scripts/ncu_ranges.py OUT.json -- python scripts/run_table1.py --skip aging,scaling ...

runs the command under `ncu --profile-from-start off` with WS_NCU_RANGES set:
the runners open one cudaProfilerStart/Stop range per timed batch, started by
a one-element torch fill (the marker kernel), and log the batch's label
(design, op, load, ops).  The launch list is split at the markers, the
batch's kernels summed, and per label the script writes DRAM sectors read /
written per op, L2 write sectors per op, bytes per op and the (serialised,
cold-cache) kernel time.  DRAM writes are only those written back while the
kernel ran: a batch whose dirty lines fit in the 126 MB L2 shows ~0, and its
L2 write sectors are the better per-op write figure.
"""
import csv
import json
import os
import subprocess
import sys
import tempfile


def main():
    out_path = sys.argv[1]
    cmd = sys.argv[sys.argv.index("--") + 1:]
    labels = tempfile.NamedTemporaryFile(suffix=".jsonl", delete=False).name
    log = tempfile.NamedTemporaryFile(suffix=".csv", delete=False).name
    ncu = os.environ.get("NCU", "ncu")
    full = [ncu, "--profile-from-start", "off", "--clock-control", "none",
            "--metrics", "dram__sectors_read.sum,dram__sectors_write.sum,lts__t_sectors_op_write.sum,"
            "gpu__time_duration.sum",
            "--csv", "--log-file", log, *cmd]
    r = subprocess.run(full, env={**os.environ, "WS_NCU_RANGES": labels})
    lab = [json.loads(x) for x in open(labels) if x.strip()]
    rows = [x for x in csv.reader(open(log)) if len(x) > 10]
    hdr = rows[0]
    ii, ki, mi, vi, ui = (hdr.index(h) for h in ("ID", "Kernel Name", "Metric Name", "Metric Value",
                                                  "Metric Unit"))
    kern = {}
    order = []
    for x in rows[1:]:
        k = kern.get(x[ii])
        if k is None:
            k = kern[x[ii]] = {"name": x[ki], "rd": 0.0, "wr": 0.0, "l2w": 0.0, "ms": 0.0}
            order.append(x[ii])
        v = float(x[vi].replace(",", ""))
        if x[mi] == "dram__sectors_read.sum":
            k["rd"] = v
        elif x[mi] == "dram__sectors_write.sum":
            k["wr"] = v
        elif x[mi] == "lts__t_sectors_op_write.sum":
            k["l2w"] = v
        elif x[mi] == "gpu__time_duration.sum":
            k["ms"] = v / 1e6 if x[ui] == "ns" else v / 1e3 if x[ui] in ("us", "usecond") else v
    groups = []
    for i in order:
        k = kern[i]
        if "FillFunctor" in k["name"] or "fill" in k["name"].lower() and "ws::" not in k["name"]:
            groups.append([])
        elif groups:
            groups[-1].append(k)
    res = []
    for lb, g in zip(lab, groups):
        rd, wr, ms = sum(k["rd"] for k in g), sum(k["wr"] for k in g), sum(k["ms"] for k in g)
        l2w = sum(k["l2w"] for k in g)
        n = max(1, lb["ops"])
        res.append({**lb, "kernels": len(g), "sectors_read_per_op": round(rd / n, 3),
                    "sectors_write_per_op": round(wr / n, 3), "dram_bytes_per_op": round(32 * (rd + wr) / n, 1),
                    # sectors stored into L2 (each written back to DRAM once unless
                    # re-dirtied while resident); dram__sectors_write misses the dirty
                    # lines ncu's cache flush writes back after the kernel
                    "l2_write_sectors_per_op": round(l2w / n, 3),
                    "ncu_ms": round(ms, 4), "top_kernel": max(g, key=lambda k: k["ms"])["name"][:120] if g else None})
    json.dump({"command": cmd, "rc": r.returncode, "ranges": len(lab), "marker_groups": len(groups),
               "points": res}, open(out_path, "w"), indent=1)
    print(f"{len(res)} ranges -> {out_path} (labels {len(lab)}, groups {len(groups)}, rc {r.returncode})")


if __name__ == "__main__":
    main()

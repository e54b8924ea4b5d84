"""Independent pin of the random-access ceiling with PyTorch's own kernels
(not this repo's code): random 8-byte gathers x[idx] and random 64-byte row
gathers x.index_select(0, idx) from tables far larger than the 126 MB L2,
plus random 8-byte scatters x[idx] = v.  Reports G random accesses/s to set
beside scripts/gather_bench.cu (profiles/random_access_ceiling.json).

    python scripts/torch_gather_ceiling.py
"""
import json

import torch


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


def main():
    torch.manual_seed(0)
    dev = "cuda"
    res = {}
    # 8-byte elements from a 16 GiB table
    x = torch.zeros(1 << 31, dtype=torch.int64, device=dev)
    n = 1 << 28
    idx = torch.randint(0, x.numel(), (n,), device=dev)
    out = torch.empty(n, dtype=torch.int64, device=dev)
    ms = timed(lambda: torch.index_select(x, 0, idx, out=out))
    res["gather_8B_16GiB"] = {"ms": ms, "G_access_per_s": n / ms / 1e6}
    v = torch.ones(n, dtype=torch.int64, device=dev)
    ms = timed(lambda: x.index_put_((idx,), v))
    res["scatter_8B_16GiB"] = {"ms": ms, "G_access_per_s": n / ms / 1e6}
    del x, out, v
    # 64-byte rows (one tag block's size) from a 16 GiB table
    rows = torch.zeros((1 << 28, 8), dtype=torch.int64, device=dev)
    m = 1 << 26
    ridx = torch.randint(0, rows.shape[0], (m,), device=dev)
    rout = torch.empty((m, 8), dtype=torch.int64, device=dev)
    ms = timed(lambda: torch.index_select(rows, 0, ridx, out=rout))
    res["gather_64B_rows_16GiB"] = {"ms": ms, "G_access_per_s": m / ms / 1e6,
                                    "note": "includes the 4 GiB streaming write of the gathered rows"}
    for k, r in res.items():
        print(f"{k}: {r['ms']:.3f} ms  {r['G_access_per_s']:.1f} G accesses/s", flush=True)
    print(json.dumps(res))


if __name__ == "__main__":
    main()

"""Host<->device copy rates from pinned memory on this box: one stream vs
two / four concurrent streams, chunk sizes 4-64 MiB, H2D alone, D2H alone and
both directions at once -- the ceiling of bench.py's e2e (PCIe-bound)."""
import torch

GB = 1 << 30
n = 4 * GB
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")


def run(nstreams, chunk, h2d=True, d2h=False):
    ss = [torch.cuda.Stream() for _ in range(nstreams)]
    ss2 = [torch.cuda.Stream() for _ in range(nstreams)]
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for s in ss + ss2:
        s.wait_event(a)
    for k, off in enumerate(range(0, n, chunk)):
        if h2d:
            with torch.cuda.stream(ss[k % nstreams]):
                d[off:off + chunk].copy_(h[off:off + chunk], non_blocking=True)
        if d2h:
            with torch.cuda.stream(ss2[k % nstreams]):
                h2[off:off + chunk].copy_(d2[off:off + chunk], non_blocking=True)
    for s in ss + ss2:
        b.wait_stream(s) if hasattr(b, "wait_stream") else None
        torch.cuda.current_stream().wait_stream(s)
    b.record()
    b.synchronize()
    ms = a.elapsed_time(b)
    return n * (int(h2d) + int(d2h)) / ms / 1e6


for mode in ((True, False), (False, True), (True, True)):
    for ns in (1, 2, 4):
        for ch in (4 << 20, 16 << 20, 64 << 20):
            r = max(run(ns, ch, *mode) for _ in range(3))
            print(f"h2d={mode[0]} d2h={mode[1]} streams={ns} chunk={ch >> 20:3d} MiB: {r:6.1f} GB/s total", flush=True)

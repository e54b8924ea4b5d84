"""Host-side cost of one batched API call, split into its parts (device
batches, so no staging): Python argument handling, the ctypes call into
libwarpspeed (pointer classification, scratch allocation, launches) and the
GPU work, for a small uniform batch and an aging-sized mixed batch.

  python scripts/host_overhead.py
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_16407_b200 import TableConfig, _native, make_table  # noqa: E402
from paper_2509_16407_b200.tables import _as_u8, _as_u64  # noqa: E402
from paper_2509_16407_b200.workload import gen_uniform_keys  # noqa: E402


def tm(f, reps=200):
    f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e6


t = make_table(TableConfig(design="iceberg_md", capacity_slots=1 << 24, seed=1))
for n in (1024, 1 << 21):
    keys = torch.from_numpy(gen_uniform_keys(3, n).view(np.int64)).cuda().view(torch.uint64)
    ops = torch.full((n,), 2, dtype=torch.uint8, device="cuda")
    ops[: n // 3] = 0x20
    ops[n // 3: n // 2] = 1
    vals = torch.ones(n, dtype=torch.uint64, device="cuda")
    st = torch.empty(n, dtype=torch.uint8, device="cuda")
    vo = torch.empty(n, dtype=torch.uint64, device="cuda")
    lib = t._lib
    h = t._h
    s = torch.cuda.current_stream().cuda_stream
    res = {
        "python_args_only": tm(lambda: (_as_u8(ops, torch), _as_u64(keys, torch), _as_u64(vals, torch),
                                        torch.empty(n, dtype=torch.uint8, device="cuda"),
                                        torch.empty(n, dtype=torch.uint64, device="cuda"), t._stream())),
        "ctypes_mixed_query_only": tm(lambda: lib.ws_query(h, keys.data_ptr(), n, vo.data_ptr(), st.data_ptr(),
                                                           s, _native.WS_F_NO_CHECK)),
        "ctypes_mixed": tm(lambda: lib.ws_mixed(h, ops.data_ptr(), keys.data_ptr(), vals.data_ptr(), n,
                                                st.data_ptr(), vo.data_ptr(), s, _native.WS_F_NO_CHECK)),
        "ctypes_mixed_combine": tm(lambda: lib.ws_mixed(h, ops.data_ptr(), keys.data_ptr(), vals.data_ptr(), n,
                                                        st.data_ptr(), vo.data_ptr(), s,
                                                        _native.WS_F_NO_CHECK | _native.WS_F_COMBINE)),
        "mixed_batch_api": tm(lambda: t.mixed_batch(ops, keys, vals, check=False, combine=True)),
        "query_batch_api": tm(lambda: t.query_batch(keys, check=False)),
    }
    print(n, {k: round(v, 1) for k, v in res.items()}, "us per call (incl. GPU time)", flush=True)

# cost of the pointer classification run_batch does for each of its (up to 5)
# pointers, and of one stream-ordered scratch allocation
from cuda.bindings import runtime as rt  # noqa: E402

p = keys.data_ptr()
print("cudaPointerGetAttributes us:", round(tm(lambda: rt.cudaPointerGetAttributes(p), 2000), 2), flush=True)


def _ma():
    e, q = rt.cudaMallocAsync(4096, s)
    rt.cudaFreeAsync(q, s)


print("cudaMallocAsync+cudaFreeAsync us:", round(tm(_ma, 2000), 2), flush=True)
print("empty torch kernel launch us:", round(tm(lambda: st.fill_(0), 2000), 2), flush=True)

"""Trace of the double-buffered p2p exchange (csrc/ws_shard.cu, WS_XCHG_TRACE):
two ranks share one GPU over CUDA IPC (the harness of tests/test_gpu_sharded.py),
each upserts then queries its batch through ShardedTable(exchange="p2p") in
several rounds.  Every round's route / apply+reply / recv+copy intervals are
CUDA-event timestamps on their own streams; the summary reports, per rank,
how much of each round's routing overlaps the previous round's apply.

    python scripts/xchg_trace.py [out.csv]
"""
import os
import socket
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def worker(rank, world, port, path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WS_XCHG_TRACE=path)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2509_16407_b200 import TableConfig
    from paper_2509_16407_b200.sharded import ShardedTable
    from paper_2509_16407_b200.workload import gen_uniform_keys
    st = ShardedTable(TableConfig(design="p2_md", capacity_slots=1 << 27, seed=42), exchange="p2p",
                      chunk_ops=1 << 22)
    n = 1 << 24
    k = torch.from_numpy(gen_uniform_keys(300 + rank, n).view(np.int64)).cuda().view(torch.uint64)
    s = st.upsert_batch(k, k, check=False)
    f, v = st.query_batch(k, check=False)
    assert int((s != 0).sum()) == 0 and bool(f.all())
    dist.barrier()
    dist.destroy_process_group()


def summarize(path):
    rows = [ln.strip().split(",") for ln in open(path) if ln.strip()]
    by = {}
    for rank, r, ph, a, e in rows:
        by.setdefault(int(rank), []).append((int(r), ph, float(a), float(e)))
    for rank, ev in sorted(by.items()):
        # calls append in order; split into calls at round 0 of "route"
        calls, cur = [], []
        for x in ev:
            if x[0] == 0 and x[1] == "route" and cur:
                calls.append(cur)
                cur = []
            cur.append(x)
        calls.append(cur)
        for ci, c in enumerate(calls):
            d = {(r, ph): (a, e) for r, ph, a, e in c}
            rounds = max(r for r, _, _, _ in c) + 1
            ov, tot = 0.0, 0.0
            for r in range(1, rounds):
                ra, re_ = d[(r, "route")]
                aa, ae = d[(r - 1, "apply+reply")]
                ov += max(0.0, min(re_, ae) - max(ra, aa))
                tot += re_ - ra
            span = max(e for _, _, _, e in c) - min(a for _, _, a, _ in c)
            print(f"rank {rank} call {ci}: {rounds} rounds, {span:.2f} ms; routing of rounds 1.. overlapping "
                  f"the previous round's apply: {ov:.3f} of {tot:.3f} ms ({100 * ov / tot if tot else 0:.0f}%)")


if __name__ == "__main__":
    path = os.path.abspath(sys.argv[1] if len(sys.argv) > 1 else "xchg_trace.csv")
    if os.path.exists(path):
        os.remove(path)
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    mp.spawn(worker, args=(2, port, path), nprocs=2)
    summarize(path)

// ws_batch.cu -- mixed batches and same-key combining (host orchestration
// and their kernels); the ABI entry points live in ws_capi.cu.
//
//   * run_device_split / run_device_by_kind: a large mixed batch runs as one
//     uniform segment per op kind through the design's tuned kernels;
//   * combine_uniform: WS_F_COMBINE's same-key folding by hash aggregation.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <vector>

#include <cub/cub.cuh>

#include "ws_host.cuh"

using namespace ws;

namespace ws_host {

__global__ void k_comb_iota(u64 n, u32* idx);

__global__ void k_kind_gather(const u32* __restrict__ perm, const u64* __restrict__ keys,
                              const u64* __restrict__ vals, u64 n, u64* kp, u64* vp) {
  for (u64 j = blockIdx.x * (u64)blockDim.x + threadIdx.x; j < n; j += (u64)gridDim.x * blockDim.x) {
    const u32 i = perm[j];
    kp[j] = keys[i];
    if (vals) vp[j] = vals[i];
  }
}
__global__ void k_kind_scatter(const u32* __restrict__ perm, const u8* __restrict__ sp, const u64* __restrict__ vop,
                               u64 n, u8* status, u64* vout) {
  for (u64 j = blockIdx.x * (u64)blockDim.x + threadIdx.x; j < n; j += (u64)gridDim.x * blockDim.x) {
    const u32 i = perm[j];
    if (status) status[i] = sp[j];
    if (vout) vout[i] = vop[j];
  }
}


// first index of every op-byte value in the sorted op array (~0 when absent)
__global__ void k_seg_starts(const u8* __restrict__ op_sorted, u64 n, u64* start) {
  for (u64 j = blockIdx.x * (u64)blockDim.x + threadIdx.x; j < n; j += (u64)gridDim.x * blockDim.x)
    if (j == 0 || op_sorted[j] != op_sorted[j - 1]) start[op_sorted[j]] = j;
}

// Mixed batches: the generic op kernel carries every op kind's code path
// (~100 KB of SASS for a 32-slot md design); with kinds interleaved at random
// every warp walks all of them and the SMs stall on instruction fetch (ncu:
// 65% "no instruction" stalls in the iceberg aging batch).  Large mixed
// batches are therefore stably partitioned by op byte (kind | merge << 4) and
// each segment runs as its own uniform launch -- upserts of one merge through
// the design's upsert kernel (the tuned lock-round kernel for P2-MD), erases,
// queries through the lock-free query kernel -- one after another on the
// stream, then the results are scattered back.  Running the segments in
// sequence is one serial order of the concurrent batch.

// ---- split by kind without a sort or a blocking read-back
// A counting partition by op byte (one histogram pass, a scan of the
// bin-major [256 x blocks] counts, one scatter pass; order within a bin is
// arbitrary, so every op carries its batch index) writes the erases and the
// queries into regions of their own, whose bases the host knows, and every
// other op byte into a third region ordered by op byte.  The erase and query
// segments are launched at once with their device-resident counts; the host
// waits only for the 257 bin starts (an event behind the partition) while
// the GPU runs them, then launches the upsert segments at known offsets.
constexpr int kKindTile = 256;

// per-block chunk, a multiple of 32 so every warp's lanes share one loop bound
__device__ __forceinline__ u32 kind_chunk(u64 n, u32 nblk) { return (u32)(((n + nblk - 1) / nblk + 31) & ~31ull); }

__global__ void __launch_bounds__(kKindTile) k_kind_hist(const u8* __restrict__ ops, u64 n, u32* H) {
  __shared__ u32 h[256];
  for (int b = threadIdx.x; b < 256; b += blockDim.x) h[b] = 0;
  __syncthreads();
  const u32 ch = kind_chunk(n, gridDim.x);
  const u64 lo = (u64)blockIdx.x * ch, hi = lo + ch < n ? lo + ch : n;
  for (u64 i = lo + threadIdx.x; i < ((hi + 31) & ~31ull) && lo < hi; i += blockDim.x) {
    const bool act = i < hi;
    const u32 b = act ? ops[i] : 256u;
    const unsigned peers = __match_any_sync(0xFFFFFFFFu, b);
    if (act && (threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&h[b], (u32)__popc(peers));
  }
  __syncthreads();
  for (int b = threadIdx.x; b < 256; b += blockDim.x) H[(u64)b * gridDim.x + blockIdx.x] = h[b];
}

struct KindOut {
  u64 *ke, *kq, *kr, *vr;
  u32 *ie, *iq, *ir;
  u8* opr;
};

// S: exclusive scan of H (bin-major).  Bin 1 (erase) and bin 2 (query) go to
// their own regions; every other bin to the rest region, shifted down by the
// erase and query counts when it sorts above them.
__global__ void __launch_bounds__(kKindTile) k_kind_split(const u8* __restrict__ ops, const u64* __restrict__ keys,
                                                          const u64* __restrict__ vals, u64 n, const u32* S,
                                                          KindOut o) {
  __shared__ u32 cur[256];
  const u32 nb = gridDim.x;
  for (int b = threadIdx.x; b < 256; b += blockDim.x) cur[b] = S[(u64)b * nb + blockIdx.x];
  const u32 s1 = S[1ull * nb], s2 = S[2ull * nb], s3 = S[3ull * nb];
  __syncthreads();
  const u32 ch = kind_chunk(n, nb);
  const u64 lo = (u64)blockIdx.x * ch, hi = lo + ch < n ? lo + ch : n;
  for (u64 i = lo + threadIdx.x; i < ((hi + 31) & ~31ull) && lo < hi; i += blockDim.x) {
    const bool act = i < hi;
    const u32 b = act ? ops[i] : 256u;
    const unsigned peers = __match_any_sync(0xFFFFFFFFu, b);
    const int lane = threadIdx.x & 31, first = __ffs(peers) - 1;
    u32 base = 0;
    if (act && lane == first) base = atomicAdd(&cur[b], (u32)__popc(peers));
    base = __shfl_sync(0xFFFFFFFFu, base, first);
    if (!act) continue;
    const u32 p = base + __popc(peers & ((1u << lane) - 1));
    const u64 k = keys[i];
    if (b == 1) {
      o.ke[p - s1] = k;
      o.ie[p - s1] = (u32)i;
    } else if (b == 2) {
      o.kq[p - s2] = k;
      o.iq[p - s2] = (u32)i;
    } else {
      const u32 r = b > 2 ? p - (s3 - s1) : p;
      o.kr[r] = k;
      o.vr[r] = vals[i];
      o.ir[r] = (u32)i;
      o.opr[r] = (u8)b;
    }
  }
}

// bin starts S[b][0] (b = 0..255) and n, plus the erase / query / rest counts
__global__ void k_kind_starts(const u32* S, u32 nb, u64 n, u64* starts, u64* cnt) {
  const int b = threadIdx.x;
  starts[b] = S[(u64)b * nb];
  if (b == 0) {
    starts[256] = n;
    const u64 s1 = S[1ull * nb], s2 = S[2ull * nb], s3 = S[3ull * nb];
    cnt[0] = s2 - s1;
    cnt[1] = s3 - s2;
    cnt[2] = n - (s3 - s1);
  }
}

// results back to batch order; region 0 erases, 1 queries, 2 the rest
__global__ void k_kind_unsplit(const u64* cnt, const u32* ie, const u8* ste, const u32* iq, const u8* stq,
                               const u64* voq, const u32* ir, const u8* str, const u64* vor, const u8* opr,
                               u8* status, u64* vout) {
  const int g = blockIdx.y;
  const u64 m = cnt[g];
  for (u64 j = blockIdx.x * (u64)blockDim.x + threadIdx.x; j < m; j += (u64)gridDim.x * blockDim.x) {
    if (g == 0) {
      const u32 i = ie[j];
      if (status) status[i] = ste[j];
      if (vout) vout[i] = 0;
    } else if (g == 1) {
      const u32 i = iq[j];
      if (status) status[i] = stq[j];
      if (vout) vout[i] = voq[j];
    } else {
      const u32 i = ir[j];
      if (status) status[i] = str[j];
      if (vout) vout[i] = (opr[j] & 15) == OP_QUERY ? vor[j] : 0;
    }
  }
}

int run_device_split(ws_table* t, const u8* ops, const u64* keys, const u64* vals, u64 n, u8* status, u64* vout,
                     cudaStream_t s, u32 flags, bool has_erase, bool has_upsert, const CallCtx& cx) {
  const u32 nblk = (u32)std::max<u64>(1, std::min<u64>((u64)kSMs * 8, (n + 2047) / 2048));
  const u64 nh = 256ull * nblk;
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, (u32*)nullptr, (u32*)nullptr, (int64_t)nh, s);
  // one scratch allocation, carved
  const u64 need = n * (8 + 4 + 1) + n * (8 + 4 + 1 + 8) + n * (8 + 8 + 4 + 1 + 1 + 8) + 8 * nh + 257 * 8 + 3 * 8 +
                   tb + 24 * 128;
  char* buf = nullptr;
  WS_CK(cudaMallocAsync((void**)&buf, need, s));
  char* p = buf;
  auto carve = [&](u64 bytes) { char* r = p; p += (bytes + 127) & ~127ull; return (void*)r; };
  KindOut o;
  o.ke = (u64*)carve(8 * n); o.ie = (u32*)carve(4 * n); u8* ste = (u8*)carve(n);
  o.kq = (u64*)carve(8 * n); o.iq = (u32*)carve(4 * n); u8* stq = (u8*)carve(n); u64* voq = (u64*)carve(8 * n);
  o.kr = (u64*)carve(8 * n); o.vr = (u64*)carve(8 * n); o.ir = (u32*)carve(4 * n); o.opr = (u8*)carve(n);
  u8* str = (u8*)carve(n); u64* vor = (u64*)carve(8 * n);
  u32* H = (u32*)carve(4 * nh); u32* S = (u32*)carve(4 * nh);
  u64* starts = (u64*)carve(257 * 8); u64* cnt = (u64*)carve(3 * 8);
  void* tmp = carve(tb + 16);
  // WS_F_CONCURRENT_KINDS: erases on se, queries on sq, upserts on s, all
  // concurrent; every segment launch then assumes concurrent erases (the
  // tombstone flag re-read behind a fence, as for multi_stream tables)
  const bool par = (flags & WS_F_CONCURRENT_KINDS) != 0;
  const u32 inner = (flags & ~(WS_F_SYNC_CHECK | WS_F_COMBINE | WS_F_CONCURRENT_KINDS)) | kF_NO_KIND_SORT |
                    ((flags & WS_F_NO_CHECK) ? 0u : (kF_VALIDATED | WS_F_NO_CHECK)) | (par ? kF_CONC_ERASE : 0u);
  const bool comb = (flags & WS_F_COMBINE) != 0;
  Staging* sg = par ? staging(t->device) : nullptr;
  if (par && !sg) { cudaFreeAsync(buf, s); return WS_ERR_ALLOC; }
  cudaStream_t se = par ? sg->s_in : s, sq = par ? sg->s_aux : s;
  cudaEvent_t ev_fork = nullptr, ev_e = nullptr, ev_q = nullptr;
  k_kind_hist<<<nblk, kKindTile, 0, s>>>(ops, n, H);
  cub::DeviceScan::ExclusiveSum(tmp, tb, H, S, (int64_t)nh, s);
  k_kind_split<<<nblk, kKindTile, 0, s>>>(ops, keys, vals, n, S, o);
  k_kind_starts<<<1, 256, 0, s>>>(S, nblk, n, starts, cnt);
  int rc = cuda_err(cudaGetLastError());
  u64* hst = pin_call();
  if (!hst) rc = WS_ERR_ALLOC;
  cudaEvent_t ev = nullptr;
  if (!rc) rc = cuda_err(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  if (!rc) rc = cuda_err(cudaMemcpyAsync(hst, starts, 257 * 8, cudaMemcpyDeviceToHost, s));
  if (!rc) rc = cuda_err(cudaEventRecord(ev, s));
  if (par && !rc) {
    for (cudaEvent_t* e : {&ev_fork, &ev_e, &ev_q})
      if (!rc) rc = cuda_err(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    if (!rc) rc = cuda_err(cudaEventRecord(ev_fork, s));
    if (!rc) rc = cuda_err(cudaStreamWaitEvent(se, ev_fork, 0));
    if (!rc) rc = cuda_err(cudaStreamWaitEvent(sq, ev_fork, 0));
  }
  // erases and queries at once, their counts read on the device
  if (!rc) {
    CallCtx ce = cx;
    ce.dn = cnt;
    rc = run_device_plain(t, nullptr, OP_ERASE, o.ke, nullptr, n, ste, nullptr, se, inner, true, false, false, ce);
  }
  if (!rc) {
    CallCtx cq = cx;
    cq.dn = cnt + 1;
    rc = run_device_plain(t, nullptr, OP_QUERY, o.kq, nullptr, n, stq, voq, sq, inner, par, false, true, cq);
  }
  if (par && !rc) rc = cuda_err(cudaEventRecord(ev_e, se));
  if (par && !rc) rc = cuda_err(cudaEventRecord(ev_q, sq));
  if (!rc) rc = cuda_err(cudaEventSynchronize(ev));
  std::vector<u64> st_h(257, 0);
  if (!rc) std::copy(hst, hst + 257, st_h.begin());
  const u64* hs = st_h.data();
  // the rest region, one segment per op byte present, in op-byte order
  const u64 c1 = hs[2] - hs[1], c2 = hs[3] - hs[2];
  for (int v = 0; v < 256 && !rc; v++) {
    if (v == 1 || v == 2) continue;
    const u64 lo = hs[v] - (v > 2 ? c1 + c2 : 0), m = hs[v + 1] - hs[v];
    if (!m) continue;
    const int kind = v & 15, merge = v >> 4;
    if (kind == OP_UPSERT && merge <= M_MIN) {
      rc = comb && m >= 2 ? combine_uniform(t, (u8)v, o.kr + lo, o.vr + lo, m, str + lo, s, inner, cx, o.ir + lo,
                                            nullptr, n)
                          : run_device_plain(t, nullptr, (u8)v, o.kr + lo, o.vr + lo, m, str + lo, nullptr, s, inner,
                                             par, true, false, cx);
    } else {  // erase / query bytes with stray merge bits, invalid bytes (gated): the generic kernel
      rc = run_device_plain(t, o.opr + lo, 0, o.kr + lo, o.vr + lo, m, str + lo, vor + lo, s, inner,
                            has_erase || par, has_upsert, false, cx);
    }
  }
  if (par) {  // join the side streams before the results are gathered (and before any error return)
    if (ev_e) cudaStreamWaitEvent(s, ev_e, 0);
    if (ev_q) cudaStreamWaitEvent(s, ev_q, 0);
  }
  if (!rc) {
    dim3 g(grid_for(n, kThreads, kTableGridPerSM), 3);
    k_kind_unsplit<<<g, kThreads, 0, s>>>(cnt, o.ie, ste, o.iq, stq, voq, o.ir, str, vor, o.opr, status, vout);
    rc = cuda_err(cudaGetLastError());
  }
  for (cudaEvent_t e : {ev, ev_fork, ev_e, ev_q})
    if (e) cudaEventDestroy(e);
  cudaFreeAsync(buf, s);
  return rc;
}

int run_device_by_kind(ws_table* t, const u8* ops, u8 uop, const u64* keys, const u64* vals, u64 n, u8* status,
                       u64* vout, cudaStream_t s, u32 flags, bool has_erase, bool has_upsert, const CallCtx& cx) {
  int rc = validate(keys, ops, n, s, (flags & WS_F_SYNC_CHECK) != 0, flags, cx);
  if (rc) return rc;
  if (vals && n < (1ull << 31)) return run_device_split(t, ops, keys, vals, n, status, vout, s, flags, has_erase,
                                                          has_upsert, cx);
  u8 *op_p = nullptr, *st_p = nullptr;
  u32 *idx = nullptr, *perm = nullptr;
  u64 *k_p = nullptr, *v_p = nullptr, *vo_p = nullptr, *starts = nullptr;
  void* tmp = nullptr;
  size_t tb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tb, ops, op_p, idx, perm, (int64_t)n, 0, 8, s);
  WS_CK(cudaMallocAsync((void**)&op_p, n, s));
  WS_CK(cudaMallocAsync((void**)&st_p, n, s));
  WS_CK(cudaMallocAsync((void**)&idx, 4 * n, s));
  WS_CK(cudaMallocAsync((void**)&perm, 4 * n, s));
  WS_CK(cudaMallocAsync((void**)&k_p, 8 * n, s));
  WS_CK(cudaMallocAsync((void**)&starts, 8 * 256, s));
  if (vals) WS_CK(cudaMallocAsync((void**)&v_p, 8 * n, s));
  if (vout) WS_CK(cudaMallocAsync((void**)&vo_p, 8 * n, s));
  WS_CK(cudaMallocAsync(&tmp, tb + 16, s));
  k_comb_iota<<<grid_for(n), kThreads, 0, s>>>(n, idx);
  cub::DeviceRadixSort::SortPairs(tmp, tb, ops, op_p, idx, perm, (int64_t)n, 0, 8, s);
  k_kind_gather<<<grid_for(n), kThreads, 0, s>>>(perm, keys, vals, n, k_p, v_p);
  WS_CK(cudaMemsetAsync(starts, 0xFF, 8 * 256, s));
  k_seg_starts<<<grid_for(n), kThreads, 0, s>>>(op_p, n, starts);
  rc = cuda_err(cudaGetLastError());
  std::vector<u64> st_h(256);
  if (!rc) rc = cuda_err(cudaMemcpyAsync(st_h.data(), starts, 8 * 256, cudaMemcpyDeviceToHost, s));
  if (!rc) rc = cuda_err(cudaStreamSynchronize(s));
  const bool comb = (flags & WS_F_COMBINE) != 0;
  const u32 inner = (flags & ~(WS_F_SYNC_CHECK | WS_F_COMBINE)) | kF_NO_KIND_SORT |
                    ((flags & WS_F_NO_CHECK) ? 0u : (kF_VALIDATED | WS_F_NO_CHECK));
  // segments in op-byte order
  std::vector<std::pair<u64, int>> seg;
  for (int v = 0; v < 256; v++)
    if (st_h[v] != ~0ull) seg.push_back({st_h[v], v});
  std::sort(seg.begin(), seg.end());
  for (size_t q = 0; q < seg.size() && !rc; q++) {
    const u64 lo = seg[q].first, hi = q + 1 < seg.size() ? seg[q + 1].first : n;
    const u8 v = (u8)seg[q].second;
    const int kind = v & 15, merge = v >> 4;
    const u64 m = hi - lo;
    if (kind == OP_UPSERT && merge <= M_MIN && v_p) {
      rc = comb && m >= 2 ? combine_uniform(t, v, k_p + lo, v_p + lo, m, st_p + lo, s, inner, cx, nullptr, nullptr, 0)
                          : run_device_plain(t, nullptr, v, k_p + lo, v_p + lo, m, st_p + lo, nullptr, s, inner,
                                             false, true, false, cx);
      if (vo_p && !rc) rc = cuda_err(cudaMemsetAsync(vo_p + lo, 0, 8 * m, s));
    } else if (kind == OP_ERASE && merge == 0) {
      rc = run_device_plain(t, nullptr, v, k_p + lo, nullptr, m, st_p + lo, nullptr, s, inner, true, false, false,
                            cx);
      if (vo_p && !rc) rc = cuda_err(cudaMemsetAsync(vo_p + lo, 0, 8 * m, s));
    } else if (kind == OP_QUERY && merge == 0) {
      rc = run_device_plain(t, nullptr, v, k_p + lo, nullptr, m, st_p + lo, vo_p ? vo_p + lo : nullptr, s, inner,
                            false, false, true, cx);
    } else {  // value-less upserts or invalid op bytes (gated): the generic kernel handles them
      rc = run_device_plain(t, op_p + lo, 0, k_p + lo, v_p ? v_p + lo : nullptr, m, st_p + lo,
                            vo_p ? vo_p + lo : nullptr, s, inner, has_erase, has_upsert, false, cx);
    }
  }
  if (!rc) {
    k_kind_scatter<<<grid_for(n), kThreads, 0, s>>>(perm, st_p, vo_p, n, status, vout);
    rc = cuda_err(cudaGetLastError());
  }
  for (void* p : {(void*)op_p, (void*)st_p, (void*)idx, (void*)perm, (void*)k_p, (void*)v_p, (void*)vo_p,
                  (void*)starts, tmp})
    if (p) cudaFreeAsync(p, s);
  return rc;
}

// ------------------------------------------------------------------ combining
// WS_F_COMBINE: same-key upserts of one batch are reduced before they touch
// the table; one op per (key, merge) group is applied and the statuses are
// expanded: the group leader gets the real status, the other members
// UPDATED (FULL if the leader was).  Equivalent to a serial order of the
// batch in which each group's upserts run back to back, in batch-index order;
// the point is Zipf hot keys, whose ops would otherwise serialise on one
// bucket lock.
//   * mixed batches are first split by op byte (run_device_by_kind); every
//     upsert segment (one merge) is then combined on its own;
//   * every merge uses hash aggregation into an L2-resident open-addressing
//     table (claim by CAS): ADD / MAX / MIN fold the values with one atomic
//     per warp group; REPLACE keeps the value of the group's HIGHEST batch
//     index (atomicMax on index+1: the last write of the serial order), KEEP
//     the value of its LOWEST (the first write; later KEEPs keep it).  The
//     leader -- the op reporting INSERTED for a new key -- is the lowest batch
//     index.  Compaction of the leaders, then the apply, with the group count
//     read on the device: no sort and no host synchronisation.
//   * `oidx` (optional) maps a segment position to its batch index when the
//     segment was gathered out of order (run_device_by_kind); `dn` (optional)
//     is the segment's device-resident length (n = its upper bound).
__global__ void k_comb_iota(u64 n, u32* idx) {
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) idx[i] = (u32)i;
}

__device__ __forceinline__ u64 merge_of(int merge, u64 a, u64 b) {
  return merge == M_ADD ? a + b : merge == M_MAX ? (a > b ? a : b) : (a < b ? a : b);
}
__device__ __forceinline__ u64 dev_n(u64 n, const u64* dn) { return dn && *dn < n ? *dn : n; }

// one slot of the scratch aggregation table: key, folded value (REPLACE: the
// group's highest batch index + 1), leader (lowest batch index) and group
// number share one 32-byte sector, so an op touches one DRAM line
struct __align__(32) AggSlot {
  u64 key;
  u64 val;
  u32 leader;
  u32 slot2g;
  u64 pad;
};
__global__ void k_agg_init(AggSlot* tab, u64 cap, u64 ident) {
  for (u64 h = blockIdx.x * (u64)blockDim.x + threadIdx.x; h < cap; h += (u64)gridDim.x * blockDim.x)
    tab[h] = AggSlot{0ull, ident, 0xFFFFFFFFu, 0u, 0ull};
}

// Lanes of a warp holding the same key fold first (__match_any_sync), so a
// Zipf hot key costs one table atomic per warp instead of one per op.
__global__ void __launch_bounds__(256) k_agg_insert(const u64* __restrict__ keys, const u64* __restrict__ vals,
                                                    const u32* __restrict__ oidx, u64 n, const u64* dn, int merge,
                                                    AggSlot* tab, u64 mask, u32* grp) {
  n = dev_n(n, dn);
  const int lane = threadIdx.x & 31;
  const bool fold = merge == M_ADD || merge == M_MAX || merge == M_MIN;
  for (u64 base = (blockIdx.x * (u64)blockDim.x + threadIdx.x) & ~31ull; base < n;
       base += (u64)gridDim.x * blockDim.x) {
    const u64 i = base + lane;
    const bool act = i < n;
    const u64 key = act ? __ldg(keys + i) : 0ull;
    const u64 v0 = act && fold ? __ldg(vals + i) : 0ull;
    u64 v = v0;
    const u32 bi = act ? (oidx ? __ldg(oidx + i) : (u32)i) : 0xFFFFFFFFu;  // batch index
    const unsigned act_m = __ballot_sync(0xFFFFFFFFu, act);
    const unsigned same = __match_any_sync(0xFFFFFFFFu, key) & act_m;
    // the group's lowest and highest batch index, and (fold) its folded value,
    // gathered into every member lane (all lanes take part in every shuffle)
    u32 lo = bi, hi = act ? bi : 0u;
    for (int j = 0; j < 32; j++) {
      const u64 vj = __shfl_sync(0xFFFFFFFFu, v0, j);  // members' own values, not partial folds
      const u32 bj = __shfl_sync(0xFFFFFFFFu, bi, j);
      if (act && j != lane && ((same >> j) & 1u)) {
        if (fold && j < lane) v = merge_of(merge, v, vj);
        lo = bj < lo ? bj : lo;
        hi = bj > hi ? bj : hi;
      }
    }
    // one lane per warp group talks to the table: the group's last lane,
    // which (fold) now holds the fold of every member
    const int last = same ? 31 - __clz(same) : -1;
    u64 h = 0;
    if (act && lane == last) {
      h = mix64(key ^ 0x9E3779B97F4A7C15ull) & mask;
      while (true) {
        const u64 cur = *(volatile const u64*)&tab[h].key;
        if (cur == key) break;
        if (cur == 0) {
          const u64 prev = atomicCAS((unsigned long long*)&tab[h].key, 0ull, (unsigned long long)key);
          if (prev == 0 || prev == key) break;
        }
        h = (h + 1) & mask;
      }
      // key, value and leader share the slot's 32-byte sector: one DRAM line
      // per op.  The leader and the MAX / MIN / REPLACE values only ever move
      // one way, so an atomic is issued only when the current value (a plain
      // read; a stale one only costs an extra atomic) would change: a hot
      // key's group then takes ~ln(m) of them instead of one per warp
      AggSlot& e = tab[h];
      if (*(volatile const u32*)&e.leader > lo) atomicMin(&e.leader, lo);
      unsigned long long* tv = (unsigned long long*)&e.val;
      const u64 cur = merge == M_ADD ? 0ull : *(volatile const u64*)&e.val;
      if (merge == M_ADD) atomicAdd(tv, (unsigned long long)v);
      else if (merge == M_MAX) { if (cur < v) atomicMax(tv, (unsigned long long)v); }
      else if (merge == M_MIN) { if (cur > v) atomicMin(tv, (unsigned long long)v); }
      else if (merge == M_REPLACE) { if (cur < (u64)hi + 1) atomicMax(tv, (unsigned long long)hi + 1); }
    }
    h = __shfl_sync(0xFFFFFFFFu, h, last < 0 ? 0 : last);
    if (act) grp[i] = (u32)h;
  }
}

// one group per leader op (ops, not table slots, are scanned).  REPLACE /
// KEEP: the winning op's value is read back through a batch-index -> segment
// position map (pos), the identity when the segment is in batch order.
__global__ void __launch_bounds__(256) k_agg_compact(const u64* __restrict__ keys, const u64* __restrict__ vals,
                                                     const u32* __restrict__ oidx, const u32* __restrict__ grp,
                                                     AggSlot* tab, const u32* pos, u64 n,
                                                     const u64* dn, int merge, u64* gkey, u64* gval,
                                                     u64* ng) {
  n = dev_n(n, dn);
  const int lane = threadIdx.x & 31;
  for (u64 base = (blockIdx.x * (u64)blockDim.x + threadIdx.x) & ~31ull; base < n;
       base += (u64)gridDim.x * blockDim.x) {
    const u64 i = base + lane;
    const u32 h = i < n ? grp[i] : 0u;
    const u32 bi = i < n ? (oidx ? oidx[i] : (u32)i) : 0u;
    const bool lead = i < n && tab[h].leader == bi;
    const u32 m = __ballot_sync(0xFFFFFFFFu, lead);
    if (!m) continue;
    u64 at = 0;
    if (lane == 0) at = atomicAdd((unsigned long long*)ng, (unsigned long long)__popc(m));
    at = __shfl_sync(0xFFFFFFFFu, at, 0);
    if (lead) {
      const u64 g = at + __popc(m & ((1u << lane) - 1));
      gkey[g] = __ldg(keys + i);
      u64 v;
      if (merge == M_KEEP) v = __ldg(vals + i);  // the leader is the first write
      else if (merge == M_REPLACE) {
        const u32 w = (u32)(tab[h].val - 1);  // highest batch index of the group
        v = __ldg(vals + (pos ? pos[w] : w));
      } else v = tab[h].val;
      gval[g] = v;
      tab[h].slot2g = (u32)g;
    }
  }
}

__global__ void k_pos_of(const u32* __restrict__ oidx, u64 n, const u64* dn, u32* pos) {
  n = dev_n(n, dn);
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x)
    pos[oidx[i]] = (u32)i;
}

__global__ void k_agg_expand(const u32* grp, const AggSlot* tab, const u32* __restrict__ oidx,
                             u64 n, const u64* dn, const u8* gst, u8* status) {
  n = dev_n(n, dn);
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
    const u32 h = grp[i];
    const u8 gs = gst[tab[h].slot2g];
    const u32 bi = oidx ? oidx[i] : (u32)i;
    status[i] = tab[h].leader == bi ? gs : (gs == S_FULL ? (u8)S_FULL : (u8)S_UPDATED);
  }
}

// Large plain batches (round 2, "combining"): the
// scratch table above is L2-resident only up to ~2M ops; past that every
// aggregation atomic is a random DRAM access and combining a uniform batch
// cost 3x the uncombined apply.  So a plain batch of more than kCombineChunk
// ops is (1) validated once, (2) sampled: kCombineSample keys at a fixed
// stride go into a small hash set.  If fewer than 1/64 of them repeat (no hot
// keys: same-key ops rarely meet on a lock) and the merge is commutative, so
// the result does not depend on combining, the batch is applied uncombined
// (same final map; the one INSERTED status of a new key may then go to any
// of its ops, as in any concurrent batch).  If at least 1/4 repeat (heavy
// skew, few distinct keys) it is folded whole.  Otherwise (3) it is combined
// chunk by chunk, each chunk with an L2-resident scratch table.  Chunks apply
// in batch order, so REPLACE / KEEP keep their serial last- / first-write
// result and each key's first op in the batch is still the one reporting
// INSERTED.
constexpr u64 kCombineChunk = 1ull << 21;
constexpr u32 kCombineSample = 1u << 16;
constexpr u32 kSampleSetMask = (1u << 18) - 1;

__global__ void k_sample_dups(const u64* __restrict__ keys, u64 stride, u64* set, u32* dups) {
  const u32 i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= kCombineSample) return;
  const u64 key = __ldg(keys + (u64)i * stride);
  u32 h = (u32)mix64(key) & kSampleSetMask;
  for (;;) {  // 2^16 keys in 2^18 slots: short probes; key 0 (a sentinel) counts as placed
    const u64 prev = atomicCAS((unsigned long long*)(set + h), 0ull, (unsigned long long)key);
    if (prev == 0ull) return;
    if (prev == key) { atomicAdd(dups, 1u); return; }
    h = (h + 1) & kSampleSetMask;
  }
}

int combine_chunk(ws_table* t, u8 uop, const u64* keys, const u64* vals, u64 n, u8* status, cudaStream_t s,
                  u32 flags, const CallCtx& cx, const u32* oidx, const u64* dn, u64 nbatch);

// one uniform upsert batch (merge = uop >> 4), combined; see above.  oidx /
// dn / nbatch: a gathered segment (positions -> batch indices < nbatch, the
// device-resident length dn); all null / 0 for a plain batch.
int combine_uniform(ws_table* t, u8 uop, const u64* keys, const u64* vals, u64 n, u8* status, cudaStream_t s,
                    u32 flags, const CallCtx& cx, const u32* oidx, const u64* dn, u64 nbatch) {
  if (oidx || dn || n <= kCombineChunk)
    return combine_chunk(t, uop, keys, vals, n, status, s, flags, cx, oidx, dn, nbatch);
  int rc = validate(keys, nullptr, n, s, (flags & WS_F_SYNC_CHECK) != 0, flags, cx);
  if (rc) return rc;
  // the chunks run unchecked but stay gated on this call's verdict
  const u32 sub = (flags & ~WS_F_SYNC_CHECK) | WS_F_NO_CHECK |
                  ((flags & WS_F_NO_CHECK) && !(flags & kF_VALIDATED) ? 0u : kF_VALIDATED);
  const int m = uop >> 4;
  const bool commutative = m == M_ADD || m == M_MAX || m == M_MIN;
  {
    u64* set = nullptr;
    if (cudaMallocAsync((void**)&set, 8ull * (kSampleSetMask + 1) + 64, s) != cudaSuccess) return WS_ERR_ALLOC;
    u32* dups = (u32*)(set + kSampleSetMask + 1);
    rc = cuda_err(cudaMemsetAsync(set, 0, 8ull * (kSampleSetMask + 1) + 64, s));
    if (!rc) {
      k_sample_dups<<<kCombineSample / 256, 256, 0, s>>>(keys, n / kCombineSample, set, dups);
      rc = cuda_err(cudaGetLastError());
    }
    u64* hp = pin();
    if (!rc && !hp) rc = WS_ERR_ALLOC;
    if (!rc) rc = cuda_err(cudaMemcpyAsync(hp, dups, 4, cudaMemcpyDeviceToHost, s));
    if (!rc) rc = cuda_err(cudaStreamSynchronize(s));
    const u32 nd = rc ? 0u : *(const u32*)hp;
    cudaFreeAsync(set, s);
    if (rc) return rc;
    if (commutative && (u64)nd * 64 < kCombineSample)
      return run_device_plain(t, nullptr, uop, keys, vals, n, status, nullptr, s, sub & ~WS_F_COMBINE, false, true,
                              false, cx);
    // heavily skewed (>= 1/4 of the sample repeats): few distinct keys, so
    // one whole-batch fold touches few scratch slots and applies each hot key
    // once, where chunks would re-apply it per chunk
    if ((u64)nd * 4 >= kCombineSample) return combine_chunk(t, uop, keys, vals, n, status, s, sub, cx, nullptr, nullptr, 0);
  }
  for (u64 lo = 0; lo < n && !rc; lo += kCombineChunk)
    rc = combine_chunk(t, uop, keys + lo, vals + lo, std::min(kCombineChunk, n - lo), status ? status + lo : nullptr,
                       s, sub, cx, nullptr, nullptr, 0);
  return rc;
}

int combine_chunk(ws_table* t, u8 uop, const u64* keys, const u64* vals, u64 n, u8* status, cudaStream_t s,
                  u32 flags, const CallCtx& cx, const u32* oidx, const u64* dn, u64 nbatch) {
  int rc = dn ? WS_OK : validate(keys, nullptr, n, s, (flags & WS_F_SYNC_CHECK) != 0, flags, cx);
  if (rc) return rc;
  // the folded batch keeps the kernels gated on this call's validation verdict
  // (an asynchronous check is not read back here, but a batch holding a
  // sentinel key still mutates nothing)
  const u32 inner = (flags & ~(WS_F_COMBINE | WS_F_SYNC_CHECK)) | WS_F_NO_CHECK |
                    ((flags & WS_F_NO_CHECK) && !(flags & kF_VALIDATED) ? 0u : kF_VALIDATED);
  const int m = uop >> 4;
  std::vector<void*> mem;
  auto alloc = [&](size_t bytes) -> void* {
    void* p = nullptr;
    if (cudaMallocAsync(&p, bytes ? bytes : 16, s) != cudaSuccess) return nullptr;
    mem.push_back(p);
    return p;
  };
  auto release = [&]() { for (void* p : mem) cudaFreeAsync(p, s); };
  const u64 cap = next_pow2(n + n / 2);  // load <= 2/3; 32 B/slot, L2-resident up to ~2M ops
  u8* gst = (u8*)alloc(n);
  u64* gkey = (u64*)alloc(8 * n);
  u64* gval = (u64*)alloc(8 * n);
  u64* ng = (u64*)alloc(8);
  AggSlot* tab = (AggSlot*)alloc(sizeof(AggSlot) * cap);
  u32* grp = (u32*)alloc(4 * n);
  u32* pos = (oidx && m == M_REPLACE) ? (u32*)alloc(4 * std::max<u64>(nbatch, 1)) : nullptr;
  if (!gst || !gkey || !gval || !ng || !tab || !grp || (oidx && m == M_REPLACE && !pos)) {
    release();
    return WS_ERR_ALLOC;
  }
  k_agg_init<<<grid_for(cap), kThreads, 0, s>>>(tab, cap, m == M_MIN ? ~0ull : 0ull);  // merge identity
  WS_CK(cudaMemsetAsync(ng, 0, 8, s));
  if (pos) k_pos_of<<<grid_for(n), kThreads, 0, s>>>(oidx, n, dn, pos);
  // random table accesses: the table kernels' launch shape (ws_kernels.cuh kTableGridPerSM)
  k_agg_insert<<<grid_for(n, 256, kTableGridPerSM), 256, 0, s>>>(keys, vals, oidx, n, dn, m, tab, cap - 1, grp);
  k_agg_compact<<<grid_for(n, 256, kTableGridPerSM), 256, 0, s>>>(keys, vals, oidx, grp, tab, pos, n, dn, m, gkey,
                                                                   gval, ng);
  rc = cuda_err(cudaGetLastError());
  CallCtx gcx = cx;
  gcx.dn = ng;  // the group count stays on the device
  if (!rc) rc = run_device_plain(t, nullptr, uop, gkey, gval, n, gst, nullptr, s, inner, false, true, false, gcx);
  if (!rc && status) {
    k_agg_expand<<<grid_for(n, kThreads, kTableGridPerSM), kThreads, 0, s>>>(grp, tab, oidx, n, dn, gst, status);
    rc = cuda_err(cudaGetLastError());
  }
  release();
  return rc;
}


}  // namespace ws_host

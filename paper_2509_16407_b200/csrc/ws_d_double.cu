// Kernel instantiations for the double design (see ws_kernels.cuh), plus
// lock-round upsert and line-at-a-time query kernels for the default 8-slot
// (128-byte) buckets.
#include "ws_kernels.cuh"

#include <algorithm>

namespace ws {

// one 8-cell bucket (a 128-byte line) as four 32-byte loads issued together
template <bool RO>
__device__ __forceinline__ void ld_bucket8(const u64* p, u64 (&w)[16]) {
#pragma unroll
  for (int q = 0; q < 4; q++) {
    if (RO)
      asm volatile("ld.global.nc.L1::no_allocate.v4.u64 {%0,%1,%2,%3}, [%4];"
                   : "=l"(w[4 * q]), "=l"(w[4 * q + 1]), "=l"(w[4 * q + 2]), "=l"(w[4 * q + 3])
                   : "l"(p + 4 * q));
    else
      asm volatile("ld.relaxed.gpu.global.v4.u64 {%0,%1,%2,%3}, [%4];"
                   : "=l"(w[4 * q]), "=l"(w[4 * q + 1]), "=l"(w[4 * q + 2]), "=l"(w[4 * q + 3])
                   : "l"(p + 4 * q) : "memory");
  }
}

// Scan of one bucket with the semantics of sync.py:184-207 (probe_range):
// stop at the key or at the first EMPTY; `hint` = first reusable cell.
__device__ __forceinline__ void scan8(const u64 (&w)[16], u64 lo, u64 key, i64& idx, u64& val, i64& hint,
                                      bool& saw_empty) {
#pragma unroll
  for (int j = 0; j < 8; j++) {
    if (idx >= 0 || saw_empty) break;
    const u64 k = w[2 * j];
    if (k == key) { idx = (i64)(lo + j); val = w[2 * j + 1]; }
    else if (k == EMPTY) { if (hint < 0) hint = (i64)(lo + j); saw_empty = true; }
    else if (k == TOMB) { if (hint < 0) hint = (i64)(lo + j); }
  }
}

// Double-hashing query (reference openaddr.py:266-280): walk b0, b0+step, ...
// for at most min(probe_cap, nb) buckets, stop at the key or at a bucket that
// holds an EMPTY cell.  Lock-free, one line fetch per bucket.
template <bool RO>
__global__ void __launch_bounds__(256) k_query_double_lines(Dev d, const u64* __restrict__ keys, u64 n, u64* vout,
                                                            u8* found, int gated) {
  WS_PROLOGUE(d, gated, n);
  const u64 len = (u64)d.probe_cap < d.nb ? (u64)d.probe_cap : d.nb;
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
    const u64 key = __ldg(keys + i);
    u64 b = d.nbm(mix64(key ^ d.seeds[0]) >> 16);
    const u64 sm = (mix64(key ^ d.seeds[1]) | 1ull) % d.nb;
    i64 idx = -1, hint = -1;
    u64 val = 0;
    for (u64 s = 0; s < len; s++) {
      u64 w[16];
      ld_bucket8<RO>(d.cells + 16 * b, w);
      bool saw_empty = false;
      scan8(w, b * 8, key, idx, val, hint, saw_empty);
      if (idx >= 0 || saw_empty) break;
      b = b + sm >= d.nb ? b + sm - d.nb : b + sm;
    }
    if (found) found[i] = idx >= 0;
    if (vout) vout[i] = idx >= 0 ? val : 0;
  }
}

// Double-hashing upsert (reference openaddr.py:232-264, Ctx::dbl_upsert) in
// warp-synchronous lock rounds: the primary-bucket lock is try-locked and kept
// across rounds; the holder walks the probe sequence a line at a time, merges
// into a match, else publishes into the first reusable cell it passed by CAS
// (writers into a foreign bucket do not hold its lock, sync.py's reserve
// protocol); a lost CAS re-walks next round.  One fence per warp-round.
__global__ void __launch_bounds__(256, 4) k_upsert_double_rounds(Dev d, const u64* __restrict__ keys,
                                                              const u64* __restrict__ vals, u64 n, int merge,
                                                              u8* status, int gated) {
  WS_PROLOGUE(d, gated, n);
  const int lane = threadIdx.x & 31;
  const u64 nwarps = ((u64)gridDim.x * blockDim.x) >> 5;
  const u64 len = (u64)d.probe_cap < d.nb ? (u64)d.probe_cap : d.nb;
  for (u64 c = (blockIdx.x * (u64)blockDim.x + threadIdx.x) >> 5; c * 32 < n; c += nwarps) {
    const u64 i = c * 32 + lane;
    bool pending = i < n;
    const u64 key = pending ? __ldg(keys + i) : 0;
    const u64 val = pending ? __ldg(vals + i) : 0;
    const u64 b0 = d.nbm(mix64(key ^ d.seeds[0]) >> 16);
    const u64 sm = (mix64(key ^ d.seeds[1]) | 1ull) % d.nb;
    bool held = false;
    u8 st = S_INSERTED;
    unsigned backoff = 64;
    while (__any_sync(0xFFFFFFFFu, pending)) {
      if (pending && !held) held = try_lock_bucket(d.locks, b0);
      if (pending && held) {
        u64 b = b0, hv = 0;
        i64 idx = -1, fh = -1;
        for (u64 s = 0; s < len; s++) {
          u64 w[16];
          ld_bucket8<false>(d.cells + 16 * b, w);
          i64 hint = -1;
          bool saw_empty = false;
          scan8(w, b * 8, key, idx, hv, hint, saw_empty);
          if (idx >= 0) break;
          if (fh < 0 && hint >= 0) fh = hint;
          if (saw_empty) break;
          b = b + sm >= d.nb ? b + sm - d.nb : b + sm;
        }
        if (idx >= 0) {
          st_cell(d.cells + 2 * (u64)idx, key, apply_merge(merge, hv, val));
          st = S_UPDATED;
          pending = false;
        } else if (fh < 0) {
          st = S_FULL;
          pending = false;
        } else if (publish_cell(d.cells + 2 * (u64)fh, key, val)) {
          st = S_INSERTED;
          pending = false;
        }  // else a foreign writer took the cell: walk again next round
      }
      __syncwarp();
      fence_acq_rel();
      if (!pending && held) {
        asm volatile("red.relaxed.gpu.global.and.b32 [%0], %1;" ::"l"(d.locks + (b0 >> 5)), "r"(~(1u << (b0 & 31)))
                     : "memory");
        held = false;
      }
      if (pending) {
        __nanosleep(backoff + 8 * lane);
        if (backoff < 4096) backoff <<= 1;
      }
    }
    if (i < n && status) status[i] = st;
  }
}

// the fused mixed / erase kernel shared with double_md (ws_d_double_md.cu)
void launch_mixed_dbl(const OpsArgs& a, bool md);
bool mixed_dbl_ok(const OpsArgs& a);

static void double_ops(const OpsArgs& a, bool def) {
  if (def && mixed_dbl_ok(a)) {
    launch_mixed_dbl(a, false);
    return;
  }
  const bool upsert_only = !a.ops && (a.uop & 15) == OP_UPSERT;
  if (def && upsert_only && !a.instr && !a.d.delay_ns && !a.serial && !a.redo && !a.d.phased &&
      a.d.tune_upsert == 4) {
    u64 g = (a.n + 255) / 256;
    g = std::max<u64>(std::min<u64>(g, (u64)kSMs * table_grid_per_sm(a.d)), 1);
    k_upsert_double_rounds<<<(unsigned)g, 256, 0, a.s>>>(a.d, a.keys, a.vals, a.n, a.uop >> 4, a.status, a.gated);
    return;
  }
  if (def) launch_ops_t<D_DOUBLE, 8>(a); else launch_ops_t<D_DOUBLE, 0>(a);
}
static void double_query(const QueryArgs& a, bool def) {
  if (def && !a.conc_erase && a.d.tune_qilp > 0) {
    // whole-line scans (86-90 registers, 2 CTAs/SM) measured 3-10% faster
    // with the default 8 CTAs/SM grid than with kTableGridPerSM
    const unsigned g = grid_for(a.n);
    if (a.ro) k_query_double_lines<true><<<g, kThreads, 0, a.s>>>(a.d, a.keys, a.n, a.vout, a.found, a.gated);
    else k_query_double_lines<false><<<g, kThreads, 0, a.s>>>(a.d, a.keys, a.n, a.vout, a.found, a.gated);
    return;
  }
  if (def) launch_query_t<D_DOUBLE, 8>(a); else launch_query_t<D_DOUBLE, 0>(a);
}
static void double_locate(const LocateArgs& a, bool def) {
  if (def) launch_locate_t<D_DOUBLE, 8>(a); else launch_locate_t<D_DOUBLE, 0>(a);
}
static void double_preload(bool def) {
  if (!def) { preload_t<D_DOUBLE, 0>(); return; }
  preload_t<D_DOUBLE, 8>();
  preload_fn(k_query_double_lines<false>);
  preload_fn(k_query_double_lines<true>);
  preload_fn(k_upsert_double_rounds);
}
Launchers launchers_double() { return Launchers{double_ops, double_query, double_locate, double_preload}; }

}  // namespace ws

// Kernel instantiations for the p2 design (see ws_kernels.cuh), plus a
// line-at-a-time lock-free query for the default 32-slot buckets.
#include "ws_kernels.cuh"
#include "ws_scan32.cuh"

#include <algorithm>

namespace ws {

// P2 query (reference openaddr.py:433-447, Ctx::p2_find with the early exit):
// scan b0; stop if found, or if b0 holds an EMPTY cell, the table never
// tombstoned and b0 is below the shortcut threshold; else scan b1.
template <bool RO>
__global__ void __launch_bounds__(256) k_query_p2_lines(Dev d, const u64* __restrict__ keys, u64 n, u64* vout,
                                                        u8* found, int conc_erase, int gated) {
  WS_PROLOGUE(d, gated, n);
  const u32 te0 = ld_u32_relaxed(d.state);
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
    const u64 key = __ldg(keys + i);
    const u64 b0 = d.nbm(mix64(key ^ d.seeds[0]) >> 16);
    i64 idx, hint;
    u64 val = 0;
    int used;
    bool saw_empty;
    scan32_all<RO>(d.cells, b0 * 32, key, idx, val, used, hint, saw_empty);
    if (idx < 0) {
      bool te = te0 != 0;
      if (conc_erase) { fence_acq_rel(); te = ld_u32_relaxed(d.state) != 0; }
      if (!(saw_empty && !te && used < d.shortcut)) {
        const u64 b1 = d.nbm(mix64(key ^ d.seeds[1]) >> 16);
        if (b1 != b0) scan32_all<RO>(d.cells, b1 * 32, key, idx, val, used, hint, saw_empty);
      }
    }
    if (found) found[i] = idx >= 0;
    if (vout) vout[i] = idx >= 0 ? val : 0;
  }
}

// P2 upsert (reference openaddr.py:370-418 with the serialisable routing of
// Ctx::p2_upsert) in the warp-synchronous lock rounds of k_upsert_p2md_rounds
// (ws_fast.cuh), with the bucket scans of a design without metadata: lock
// b0, scan it a half-bucket at a time (scan32_all); found -> merge; the
// shortcut (never tombstoned, fewer than `shortcut` claimed cells before the
// first EMPTY) claims b0's first free cell; otherwise lock and scan b1 and
// claim in the less-used bucket (ties to b0), else FULL.  Exclusive plain
// publication under the bucket lock, one fence per warp-round, and the same
// ascending-order retry rule (keep b0 while retrying b1 > b0; release b0 and
// take b1 first when b1 < b0).
__global__ void __launch_bounds__(256, 3) k_upsert_p2_rounds(Dev d, const u64* __restrict__ keys,
                                                          const u64* __restrict__ vals, u64 n, int merge,
                                                          u8* status, int conc_erase, int gated) {
  WS_PROLOGUE(d, gated, n);
  const u32 te0 = ld_u32_relaxed(d.state);
  const int lane = threadIdx.x & 31;
  const u64 nwarps = ((u64)gridDim.x * blockDim.x) >> 5;
  for (u64 c = (blockIdx.x * (u64)blockDim.x + threadIdx.x) >> 5; c * 32 < n; c += nwarps) {
    const u64 i = c * 32 + lane;
    bool pending = i < n;
    const u64 key = pending ? __ldg(keys + i) : 0;
    const u64 val = pending ? __ldg(vals + i) : 0;
    const u64 b0 = d.nbm(mix64(key ^ d.seeds[0]) >> 16);
    const u64 b1 = d.nbm(mix64(key ^ d.seeds[1]) >> 16);
    u8 st = 0;
    unsigned backoff = 64;
    bool held0 = false, held1 = false, lofirst = false;
    while (__any_sync(0xFFFFFFFFu, pending)) {
      if (pending) {
        if (lofirst) {
          if (!held1) held1 = try_lock_bucket(d.locks, b1);
          if (held1 && !held0) held0 = try_lock_bucket(d.locks, b0);
        } else if (!held0) {
          held0 = try_lock_bucket(d.locks, b0);
        }
      }
      bool drop0 = false;
      if (pending && held0) {
        // one scan call site (b0, then b1 when needed) keeps one 256-byte
        // half-bucket of registers live instead of two
        i64 slot = -1, hint0 = -1;
        int used0 = 0;
        bool decided = false, te = te0 != 0;
#pragma unroll 1
        for (int q = 0; q < 2; q++) {
          const u64 b = q ? b1 : b0;
          i64 idx, hint;
          u64 old = 0;
          int used;
          bool se;
          scan32_all<false>(d.cells, b * 32, key, idx, old, used, hint, se);
          if (idx >= 0) {
            st_cell(d.cells + 2 * (u64)idx, key, apply_merge(merge, old, val));
            st = S_UPDATED;
            pending = false;
            break;
          }
          if (q == 1) {
            const bool prim = used0 <= used;  // ties go to the primary
            slot = prim ? hint0 : hint;
            if (slot < 0) slot = prim ? hint : hint0;
            decided = true;
            break;
          }
          used0 = used;
          hint0 = hint;
          if (conc_erase) { fence_acq_rel(); te = ld_u32_relaxed(d.state) != 0; }
          if (!(te || used0 >= d.shortcut) || b1 == b0) {
            slot = hint0;  // shortcut (or b1 == b0): the primary it is
            decided = true;
            break;
          }
          if (!held1) {
            held1 = try_lock_bucket(d.locks, b1);
            if (!held1) {
              if (b1 < b0) {
                lofirst = true;
                drop0 = true;
              }
              break;  // retry next round
            }
          }
        }
        if (decided) {
          if (slot < 0) {
            st = S_FULL;
          } else {
            if (conc_erase) fence_acq_rel();
            // never tombstoned: every cell after the first EMPTY is EMPTY, so
            // an even slot's partner is ours too -- write the whole sector
            if (!te && !(slot & 1)) st_cell(d.cells + 2 * ((u64)slot + 1), 0, 0);
            st_cell(d.cells + 2 * (u64)slot, key, val);
            st = S_INSERTED;
          }
          pending = false;
        }
      }
      __syncwarp();
      fence_acq_rel();
      if (held1 && !pending) {
        asm volatile("red.relaxed.gpu.global.and.b32 [%0], %1;" ::"l"(d.locks + (b1 >> 5)), "r"(~(1u << (b1 & 31)))
                     : "memory");
        held1 = false;
      }
      if (held0 && (!pending || drop0)) {
        asm volatile("red.relaxed.gpu.global.and.b32 [%0], %1;" ::"l"(d.locks + (b0 >> 5)), "r"(~(1u << (b0 & 31)))
                     : "memory");
        held0 = false;
      }
      if (pending) {
        __nanosleep(backoff + 8 * lane);
        if (backoff < 4096) backoff <<= 1;
      }
    }
    if (i < n && status) status[i] = st;
  }
}

static void p2_ops(const OpsArgs& a, bool def) {
  const bool upsert_only = !a.ops && (a.uop & 15) == OP_UPSERT;
  if (def && upsert_only && !a.instr && !a.d.delay_ns && !a.serial && !a.redo && !a.d.phased && !a.d.lock_elided &&
      a.d.tune_upsert == 4) {
    u64 g = (a.n + 255) / 256;
    const u64 lim = std::max<u64>((a.d.nb + 255) / 256, 4);  // <= ~1 op in flight per bucket
    g = std::max<u64>(std::min<u64>(std::min<u64>(g, (u64)kSMs * table_grid_per_sm(a.d)), lim), 1);
    k_upsert_p2_rounds<<<(unsigned)g, 256, 0, a.s>>>(a.d, a.keys, a.vals, a.n, a.uop >> 4, a.status, a.conc_erase,
                                                     a.gated);
    return;
  }
  if (def) launch_ops_t<D_P2, 32>(a); else launch_ops_t<D_P2, 0>(a);
}
static void p2_query(const QueryArgs& a, bool def) {
  if (def && a.d.tune_qilp > 0) {
    // whole-line scans (86-90 registers, 2 CTAs/SM) measured 3-10% faster
    // with the default 8 CTAs/SM grid than with kTableGridPerSM
    const unsigned g = grid_for(a.n);
    if (a.ro) k_query_p2_lines<true><<<g, kThreads, 0, a.s>>>(a.d, a.keys, a.n, a.vout, a.found, a.conc_erase, a.gated);
    else k_query_p2_lines<false><<<g, kThreads, 0, a.s>>>(a.d, a.keys, a.n, a.vout, a.found, a.conc_erase, a.gated);
    return;
  }
  if (def) launch_query_t<D_P2, 32>(a); else launch_query_t<D_P2, 0>(a);
}
static void p2_locate(const LocateArgs& a, bool def) {
  if (def) launch_locate_t<D_P2, 32>(a); else launch_locate_t<D_P2, 0>(a);
}
static void p2_preload(bool def) {
  if (!def) { preload_t<D_P2, 0>(); return; }
  preload_t<D_P2, 32>();
  preload_fn(k_query_p2_lines<false>);
  preload_fn(k_query_p2_lines<true>);
  preload_fn(k_upsert_p2_rounds);
}
Launchers launchers_p2() { return Launchers{p2_ops, p2_query, p2_locate, p2_preload}; }

}  // namespace ws

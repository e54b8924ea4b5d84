// Kernel instantiations for the iceberg design (see ws_kernels.cuh), plus a
// line-at-a-time lock-free query for the default 32-slot buckets.
#include "ws_kernels.cuh"
#include "ws_scan32.cuh"

#include <algorithm>

namespace ws {

// Iceberg query (reference openaddr.py:589-609, Ctx::ice_find with the early
// exit): scan the front bucket; stop if found or if it holds an EMPTY cell;
// else scan the backyard pair.
template <bool RO>
__global__ void __launch_bounds__(256) k_query_ice_lines(Dev d, const u64* __restrict__ keys, u64 n, u64* vout,
                                                         u8* found, int gated) {
  WS_PROLOGUE(d, gated, n);
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
    const u64 key = __ldg(keys + i);
    const u64 b0 = d.frontm(mix64(key ^ d.seeds[0]) >> 16);
    i64 idx, hint;
    u64 val = 0;
    int used;
    bool saw_empty;
    scan32_lines<RO>(d.cells, b0 * 32, key, idx, val, used, hint, saw_empty);
    if (idx < 0 && !saw_empty) {
      const u64 b1 = d.front + d.backm(mix64(key ^ d.seeds[1]) >> 16);
      const u64 b2 = d.front + d.backm(mix64(key ^ d.seeds[2]) >> 16);
      scan32_lines<RO>(d.cells, b1 * 32, key, idx, val, used, hint, saw_empty);
      if (idx < 0 && b2 != b1) scan32_lines<RO>(d.cells, b2 * 32, key, idx, val, used, hint, saw_empty);
    }
    if (found) found[i] = idx >= 0;
    if (vout) vout[i] = idx >= 0 ? val : 0;
  }
}

// Iceberg upsert (reference openaddr.py:540-578 with the serialisable
// routing of Ctx::ice_upsert) in warp-synchronous lock rounds
// (k_upsert_icemd_rounds without metadata): try-lock the front bucket and
// keep it; scan it; found -> merge; an EMPTY in the front -> claim its first
// free cell (the backyard cannot hold the key); otherwise try-lock both
// backyard buckets (indices above every front bucket: ascending order),
// search them, then claim in the front if it has a TOMB, else in the
// backyard bucket with a free cell and the fewest claimed cells (ties to the
// lower index, sorted((used, bucket))), else FULL.  One scan call site for
// the three buckets; one fence per warp-round.
__global__ void __launch_bounds__(256) k_upsert_ice_rounds(Dev d, const u64* __restrict__ keys,
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
    const u64 b0 = d.frontm(mix64(key ^ d.seeds[0]) >> 16);
    u64 bl = d.front + d.backm(mix64(key ^ d.seeds[1]) >> 16);
    u64 bh = d.front + d.backm(mix64(key ^ d.seeds[2]) >> 16);
    if (bh < bl) { const u64 x = bl; bl = bh; bh = x; }  // ascending; bh == bl -> one bucket
    u8 st = 0;
    unsigned backoff = 64;
    bool held0 = false, heldb = false;
    while (__any_sync(0xFFFFFFFFu, pending)) {
      if (pending && !held0) held0 = try_lock_bucket(d.locks, b0);
      if (pending && held0) {
        i64 slot = -1, hint0 = -1, hint1 = -1;
        int used1 = 0;
        bool decided = false;
        const int nq = bh == bl ? 2 : 3;
#pragma unroll 1
        for (int q = 0; q < nq; q++) {
          const u64 b = q == 0 ? b0 : (q == 1 ? bl : bh);
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
          if (q == 0) {
            hint0 = hint;
            if (se) {  // the front never filled: the key can only be here
              slot = hint0;
              decided = true;
              break;
            }
            if (!heldb) {
              const bool l1 = try_lock_bucket(d.locks, bl);
              const bool l2 = !l1 || bh == bl || try_lock_bucket(d.locks, bh);
              if (l1 && l2) {
                heldb = true;
              } else {
                if (l1)
                  asm volatile("red.relaxed.gpu.global.and.b32 [%0], %1;" ::"l"(d.locks + (bl >> 5)),
                               "r"(~(1u << (bl & 31))) : "memory");
                break;  // keep the front lock, retry the backyard next round
              }
            }
          } else {
            if (q == 1 && nq == 3) {
              used1 = used;
              hint1 = hint;
              continue;
            }
            if (hint0 >= 0) {
              slot = hint0;  // a reusable front cell
            } else if (nq == 2) {
              slot = hint;
            } else {
              const bool lo = hint1 >= 0 && (hint < 0 || used1 <= used);
              slot = lo ? hint1 : hint;
            }
            decided = true;
          }
        }
        if (decided) {
          if (slot < 0) {
            st = S_FULL;
          } else {
            bool te = te0 != 0;
            if (conc_erase) { fence_acq_rel(); te = ld_u32_relaxed(d.state) != 0; }
            // never tombstoned: cells after a bucket's first EMPTY are EMPTY,
            // so an even slot's partner is ours too -- write the whole sector
            if (!te && !(slot & 1)) st_cell(d.cells + 2 * ((u64)slot + 1), 0, 0);
            st_cell(d.cells + 2 * (u64)slot, key, val);
            st = S_INSERTED;
          }
          pending = false;
        }
      }
      __syncwarp();
      fence_acq_rel();
      if (!pending) {
        if (heldb) {
          if (bh != bl)
            asm volatile("red.relaxed.gpu.global.and.b32 [%0], %1;" ::"l"(d.locks + (bh >> 5)),
                         "r"(~(1u << (bh & 31))) : "memory");
          asm volatile("red.relaxed.gpu.global.and.b32 [%0], %1;" ::"l"(d.locks + (bl >> 5)),
                       "r"(~(1u << (bl & 31))) : "memory");
          heldb = false;
        }
        if (held0) {
          asm volatile("red.relaxed.gpu.global.and.b32 [%0], %1;" ::"l"(d.locks + (b0 >> 5)),
                       "r"(~(1u << (b0 & 31))) : "memory");
          held0 = false;
        }
      }
      if (pending) {
        __nanosleep(backoff + 8 * lane);
        if (backoff < 4096) backoff <<= 1;
      }
    }
    if (i < n && status) status[i] = st;
  }
}

static void iceberg_ops(const OpsArgs& a, bool def) {
  const bool upsert_only = !a.ops && (a.uop & 15) == OP_UPSERT;
  if (def && upsert_only && !a.instr && !a.d.delay_ns && !a.serial && !a.redo && !a.d.phased && !a.d.lock_elided &&
      a.d.tune_upsert == 4) {
    u64 g = (a.n + 255) / 256;
    const u64 lim = std::max<u64>((a.d.nb + 255) / 256, 4);  // <= ~1 op in flight per bucket
    g = std::max<u64>(std::min<u64>(std::min<u64>(g, (u64)kSMs * table_grid_per_sm(a.d)), lim), 1);
    k_upsert_ice_rounds<<<(unsigned)g, 256, 0, a.s>>>(a.d, a.keys, a.vals, a.n, a.uop >> 4, a.status, a.conc_erase,
                                                      a.gated);
    return;
  }
  if (def) launch_ops_t<D_ICEBERG, 32>(a); else launch_ops_t<D_ICEBERG, 0>(a);
}
static void iceberg_query(const QueryArgs& a, bool def) {
  if (def && a.d.tune_qilp > 0) {
    // whole-line scans (86-90 registers, 2 CTAs/SM) measured 3-10% faster
    // with the default 8 CTAs/SM grid than with kTableGridPerSM
    const unsigned g = grid_for(a.n);
    if (a.ro) k_query_ice_lines<true><<<g, kThreads, 0, a.s>>>(a.d, a.keys, a.n, a.vout, a.found, a.gated);
    else k_query_ice_lines<false><<<g, kThreads, 0, a.s>>>(a.d, a.keys, a.n, a.vout, a.found, a.gated);
    return;
  }
  if (def) launch_query_t<D_ICEBERG, 32>(a); else launch_query_t<D_ICEBERG, 0>(a);
}
static void iceberg_locate(const LocateArgs& a, bool def) {
  if (def) launch_locate_t<D_ICEBERG, 32>(a); else launch_locate_t<D_ICEBERG, 0>(a);
}
static void iceberg_preload(bool def) {
  if (!def) { preload_t<D_ICEBERG, 0>(); return; }
  preload_t<D_ICEBERG, 32>();
  preload_fn(k_query_ice_lines<false>);
  preload_fn(k_query_ice_lines<true>);
  preload_fn(k_upsert_ice_rounds);
}
Launchers launchers_iceberg() { return Launchers{iceberg_ops, iceberg_query, iceberg_locate, iceberg_preload}; }

}  // namespace ws

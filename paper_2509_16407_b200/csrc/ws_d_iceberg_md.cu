// Kernel instantiations for the iceberg_md design (see ws_kernels.cuh), plus
// the tuned lock-round upsert for uniform upsert launches.
#include "ws_fast.cuh"
#include "ws_kernels.cuh"

#include <algorithm>

namespace ws {

// Iceberg-MD upsert (reference openaddr.py:540-578 with the serialisable
// routing of Ctx::ice_upsert), one thread per op in warp-synchronous lock
// rounds like k_upsert_p2md_rounds (ws_fast.cuh): try-locks that never block,
// pair-cooperative 64-byte tag fetches, exclusive plain-store publication,
// one fence per warp-round.
//   * front bucket b0 = (h0 >> 16) % front, locked first;
//   * found in b0 -> merge; b0 has a never-used slot (a zero tag while the
//     table never tombstoned) -> claim its first zero tag (the backyard is
//     not read: a key of a front that never filled can only be in that front);
//   * otherwise lock both backyard buckets (indices above every front bucket,
//     so ascending order holds), search them, then claim in the front if it
//     has any zero tag, else in the least-loaded backyard bucket with a free
//     slot (ties to the lower index, as sorted((used, bucket))), else FULL.
// Lock retries follow the ascending-order rule of the P2-MD kernel: a lane
// keeps its front lock while it retries the (higher) backyard locks.
template <bool FILL>
__global__ void __launch_bounds__(256) k_upsert_icemd_rounds(Dev d, const u64* __restrict__ keys,
                                                             const u64* __restrict__ vals, u64 n, int merge,
                                                             u8* status, int conc_erase, int gated) {
  WS_PROLOGUE(d, gated, n);
  const u32 te0 = ld_u32_relaxed(d.state);
  const int lane = threadIdx.x & 31;
  const u64 nwarps = ((u64)gridDim.x * blockDim.x) >> 5;
  for (u64 c = (blockIdx.x * (u64)blockDim.x + threadIdx.x) >> 5; c * 32 < n; c += nwarps) {
    const u64 i = c * 32 + lane;
    bool pending = i < n;
    u64 key = 0, val = 0, b0 = 0, b1 = 0, b2 = 0;
    u16 tag = 1;
    if (pending) {
      key = __ldg(keys + i);
      val = __ldg(vals + i);
      const u64 h0 = mix64(key ^ d.seeds[0]);
      b0 = d.frontm(h0 >> 16);
      const u16 t = (u16)(h0 & 0xFFFF);
      tag = t ? t : (u16)1;
      b1 = d.front + d.backm(mix64(key ^ d.seeds[1]) >> 16);
      b2 = d.front + d.backm(mix64(key ^ d.seeds[2]) >> 16);
      if (b2 < b1) { const u64 x = b1; b1 = b2; b2 = x; }  // ascending; b2 == b1 -> one bucket
    }
    u8 st = 0;
    unsigned backoff = 64;
    bool held0 = false, heldb = false;
    while (__any_sync(0xFFFFFFFFu, pending)) {
      if (pending && !held0) held0 = try_lock_bucket(d.locks, b0);
      const bool hold0 = pending && held0;
      u32 M0, Z0;
      coop_masks<false, true>(d, hold0, b0, tag, M0, Z0);
      bool needb = false, decided = false, te_last = true;
      u64 target = 0;
      u32 Zt = 0;
      u64 old;
      if (hold0) {
        const int j = M0 ? pair_confirm<false, true>(d, b0, M0, key, old) : -1;
        if (j >= 0) {
          st_cell(d.cells + 2 * (b0 * 32 + j), key, apply_merge(merge, old, val));
          st = S_UPDATED;
          pending = false;
        } else {
          bool te = te0 != 0;
          if (conc_erase) { fence_acq_rel(); te = ld_u32_relaxed(d.state) != 0; }
          te_last = te;
          if (Z0 && !te) {  // saw_empty: the front never filled
            target = b0;
            Zt = Z0;
            decided = true;
          } else {
            if (!heldb) {
              const bool l1 = try_lock_bucket(d.locks, b1);
              const bool l2 = !l1 || b2 == b1 || try_lock_bucket(d.locks, b2);
              if (l1 && l2) {
                heldb = true;
              } else if (l1) {
                red_and_relaxed(d.locks + (b1 >> 5), ~(1u << (b1 & 31)));  // keep b0, retry next round
              }
            }
            needb = heldb;
          }
        }
      }
      // backyard tag blocks of the lanes that hold them
      u32 M1 = 0, Z1 = 0, M2 = 0, Z2 = 0;
      const bool need2 = needb && b2 != b1;
      if (__any_sync(0xFFFFFFFFu, needb)) coop_masks<false, true>(d, needb, b1, tag, M1, Z1);
      if (__any_sync(0xFFFFFFFFu, need2)) coop_masks<false, true>(d, need2, b2, tag, M2, Z2);
      if (needb) {
        int j = M1 ? pair_confirm<false, true>(d, b1, M1, key, old) : -1;
        u64 bj = b1;
        if (j < 0 && need2 && M2) {
          j = pair_confirm<false, true>(d, b2, M2, key, old);
          bj = b2;
        }
        if (j >= 0) {
          st_cell(d.cells + 2 * (bj * 32 + j), key, apply_merge(merge, old, val));
          st = S_UPDATED;
          pending = false;
        } else if (Z0) {  // front has a reusable slot (tombstoned table)
          target = b0;
          Zt = Z0;
          decided = true;
        } else {
          const int zc1 = __popc(Z1), zc2 = need2 ? __popc(Z2) : 0;
          const int u1 = 32 - (zc1 < d.zcc ? zc1 : d.zcc), u2 = 32 - (zc2 < d.zcc ? zc2 : d.zcc);
          // sorted((used, bucket)) over the backyard buckets with a free slot; b1 < b2
          if (Z1 && (!need2 || !Z2 || u1 <= u2)) { target = b1; Zt = Z1; }
          else if (need2 && Z2) { target = b2; Zt = Z2; }
          decided = true;  // Zt == 0 -> FULL
        }
      }
      if (decided) {
        if (!Zt) {
          st = S_FULL;
          pending = false;
        } else {
          const u64 slot = target * 32 + (__ffs(Zt) - 1);
          if (conc_erase) fence_acq_rel();
          if (FILL && !te_last && ((Zt >> ((slot & 31) ^ 1)) & 1u)) st_cell(d.cells + 2 * (slot ^ 1), 0, 0);
          st_cell(d.cells + 2 * slot, key, val);
          st_tag(d.tags + slot, tag);
          st = S_INSERTED;
          pending = false;
        }
      }
      // one MEMBAR for the warp, then relaxed releases of finished lanes
      __syncwarp();
      fence_acq_rel();
      if (!pending) {
        if (heldb) {
          if (b2 != b1) red_and_relaxed(d.locks + (b2 >> 5), ~(1u << (b2 & 31)));
          red_and_relaxed(d.locks + (b1 >> 5), ~(1u << (b1 & 31)));
          heldb = false;
        }
        if (held0) {
          red_and_relaxed(d.locks + (b0 >> 5), ~(1u << (b0 & 31)));
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

static void iceberg_md_ops(const OpsArgs& a, bool def) {
  const bool upsert_only = !a.ops && (a.uop & 15) == OP_UPSERT;
  if (def && upsert_only && !a.instr && !a.d.delay_ns && !a.serial && !a.redo && !a.d.phased && !a.d.lock_elided &&
      a.d.tune_upsert == 4) {
    u64 g = (a.n + 255) / 256;
    const u64 lim = std::max<u64>((a.d.nb + 255) / 256, 4);  // <= ~1 op in flight per bucket
    g = std::max<u64>(std::min<u64>(std::min<u64>(g, (u64)kSMs * 8), lim), 1);
    k_upsert_icemd_rounds<true><<<(unsigned)g, 256, 0, a.s>>>(a.d, a.keys, a.vals, a.n, a.uop >> 4, a.status,
                                                               a.conc_erase, a.gated);
    return;
  }
  if (def) launch_ops_t<D_ICEBERG_MD, 32>(a); else launch_ops_t<D_ICEBERG_MD, 0>(a);
}
static void iceberg_md_query(const QueryArgs& a, bool def) {
  if (def) launch_query_t<D_ICEBERG_MD, 32>(a); else launch_query_t<D_ICEBERG_MD, 0>(a);
}
static void iceberg_md_locate(const LocateArgs& a, bool def) {
  if (def) launch_locate_t<D_ICEBERG_MD, 32>(a); else launch_locate_t<D_ICEBERG_MD, 0>(a);
}
static void iceberg_md_preload(bool def) {
  if (!def) { preload_t<D_ICEBERG_MD, 0>(); return; }
  preload_t<D_ICEBERG_MD, 32>();
  preload_fn(k_upsert_icemd_rounds<true>);
}
Launchers launchers_iceberg_md() {
  return Launchers{iceberg_md_ops, iceberg_md_query, iceberg_md_locate, iceberg_md_preload};
}

}  // namespace ws

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
__global__ void __launch_bounds__(256, 4) k_upsert_icemd_rounds(Dev d, const u64* __restrict__ keys,
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

// Iceberg-MD query (reference openaddr.py:593-610, Ctx::ice_find with the
// early exit), one thread per op with the pair-cooperative 64-byte tag
// fetches of k_query_p2md_coop: front bucket tags -> confirm; a front with a
// zero tag while the table never tombstoned proves the key never reached the
// backyard (early exit); else both backyard buckets, b2 only when b2 != b1.
template <bool RO, bool F64>
__global__ void __launch_bounds__(256) k_query_icemd_coop(Dev d, const u64* __restrict__ keys, u64 n, u64* vout,
                                                          u8* found, int conc_erase, int gated) {
  WS_PROLOGUE(d, gated, n);
  const u32 te0 = ld_u32_relaxed(d.state);
  const u64 stride = (u64)gridDim.x * blockDim.x;
  const u64 first = (blockIdx.x * (u64)blockDim.x + threadIdx.x) & ~31ull;  // warp-uniform loop bound
  for (u64 base = first; base < n; base += stride) {
    const u64 i = base + (threadIdx.x & 31);
    const bool act = i < n;
    const u64 key = act ? __ldg(keys + i) : 0;
    const u64 h0 = mix64(key ^ d.seeds[0]);
    const u64 b0 = d.frontm(h0 >> 16);
    const u16 t = (u16)(h0 & 0xFFFF);
    const u16 tag = t ? t : (u16)1;
    u32 M, Z;
    coop_masks<RO, F64>(d, act, b0, tag, M, Z);
    u64 val = 0;
    bool hit = act && M && pair_confirm<RO, F64>(d, b0, M, key, val) >= 0;
    bool te = te0 != 0;
    if (conc_erase) { fence_acq_rel(); te = ld_u32_relaxed(d.state) != 0; }
    const u64 b1 = d.front + d.backm(mix64(key ^ d.seeds[1]) >> 16);
    const u64 b2 = d.front + d.backm(mix64(key ^ d.seeds[2]) >> 16);
    const bool need1 = act && !hit && !(Z && !te);
    if (__any_sync(0xFFFFFFFFu, need1)) {
      coop_masks<RO, F64>(d, need1, b1, tag, M, Z);
      if (need1 && M) hit = pair_confirm<RO, F64>(d, b1, M, key, val) >= 0;
      const bool need2 = need1 && !hit && b2 != b1;
      if (__any_sync(0xFFFFFFFFu, need2)) {
        coop_masks<RO, F64>(d, need2, b2, tag, M, Z);
        if (need2 && M) hit = pair_confirm<RO, F64>(d, b2, M, key, val) >= 0;
      }
    }
    if (act) {
      if (found) found[i] = hit;
      if (vout) vout[i] = hit ? val : 0;
    }
  }
}

// Iceberg-MD erase (reference openaddr.py:612-631, Ctx::ice_erase): the
// front lock only, as the reference; warp-synchronous lock rounds with
// non-blocking try-locks, the ice_find search above with coherent loads, and
// the tombstone protocol of Ctx::tombstone (tombstones_ever set, fence, cell
// := TOMB, fence, tag := 0) with one fence per step for the whole warp.
template <bool F64>
__global__ void __launch_bounds__(256) k_erase_icemd_rounds(Dev d, const u64* __restrict__ keys, u64 n,
                                                            u8* found, int conc_erase, int gated) {
  WS_PROLOGUE(d, gated, n);
  const int lane = threadIdx.x & 31;
  const u64 nwarps = ((u64)gridDim.x * blockDim.x) >> 5;
  for (u64 c = (blockIdx.x * (u64)blockDim.x + threadIdx.x) >> 5; c * 32 < n; c += nwarps) {
    const u64 i = c * 32 + lane;
    bool pending = i < n;
    const u64 key = pending ? __ldg(keys + i) : 0;
    const u64 h0 = mix64(key ^ d.seeds[0]);
    const u64 b0 = d.frontm(h0 >> 16);
    const u16 t = (u16)(h0 & 0xFFFF);
    const u16 tag = t ? t : (u16)1;
    const u64 b1 = d.front + d.backm(mix64(key ^ d.seeds[1]) >> 16);
    const u64 b2 = d.front + d.backm(mix64(key ^ d.seeds[2]) >> 16);
    bool gone = false, held = false;
    unsigned backoff = 64;
    while (__any_sync(0xFFFFFFFFu, pending)) {
      if (pending && !held) held = try_lock_bucket(d.locks, b0);
      const bool hold = pending && held;
      u32 M, Z;
      coop_masks<false, F64>(d, hold, b0, tag, M, Z);
      i64 slot = -1;
      u64 v;
      if (hold && M) {
        const int j = pair_confirm<false, F64>(d, b0, M, key, v);
        if (j >= 0) slot = (i64)(b0 * 32 + j);
      }
      bool te = true;
      if (__any_sync(0xFFFFFFFFu, hold && slot < 0)) {
        fence_acq_rel();  // as Ctx::tomb_ever under concurrent erases
        te = ld_u32_relaxed(d.state) != 0;
      }
      const bool need1 = hold && slot < 0 && !(Z && !te);
      if (__any_sync(0xFFFFFFFFu, need1)) {
        coop_masks<false, F64>(d, need1, b1, tag, M, Z);
        if (need1 && M) {
          const int j = pair_confirm<false, F64>(d, b1, M, key, v);
          if (j >= 0) slot = (i64)(b1 * 32 + j);
        }
        const bool need2 = need1 && slot < 0 && b2 != b1;
        if (__any_sync(0xFFFFFFFFu, need2)) {
          coop_masks<false, F64>(d, need2, b2, tag, M, Z);
          if (need2 && M) {
            const int j = pair_confirm<false, F64>(d, b2, M, key, v);
            if (j >= 0) slot = (i64)(b2 * 32 + j);
          }
        }
      }
      // tombstone protocol, one fence per step for the warp
      const bool del = slot >= 0;
      if (__any_sync(0xFFFFFFFFu, del)) {
        if (del && ld_u32_relaxed(d.state) == 0) st_u32_relaxed(d.state, 1u);
        fence_acq_rel();
        if (del) st_cell(d.cells + 2 * (u64)slot, TOMB, 0);
        fence_acq_rel();  // the tombstone is visible before the zero tag that advertises it
        if (del) st_tag(d.tags + (u64)slot, 0);
      }
      if (hold) {
        gone = del;
        pending = false;
      }
      __syncwarp();
      fence_acq_rel();
      if (held && !pending) {
        red_and_relaxed(d.locks + (b0 >> 5), ~(1u << (b0 & 31)));
        held = false;
      }
      if (pending) {
        __nanosleep(backoff + 8 * lane);
        if (backoff < 4096) backoff <<= 1;
      }
    }
    if (i < n && found) found[i] = gone;
  }
}

// Iceberg-MD mixed batches in ONE launch (interleaved / small mixed batches,
// the split's remainder): k_upsert_icemd_rounds extended with erase lanes
// (front lock only, as openaddr.py:612-631; front, then -- unless the front
// provably never filled -- both backyard buckets; tombstone protocol of
// Ctx::tombstone with one fence per step for the warp) and lock-free query
// lanes (openaddr.py:593-610) that finish in the first round.  Op bytes of
// another kind run as queries, merges above MIN as REPLACE (Ctx::run).
__global__ void __launch_bounds__(256, 4) k_mixed_icemd_rounds(Dev d, const u8* __restrict__ ops, u8 uop,
                                                            const u64* __restrict__ keys,
                                                            const u64* __restrict__ vals, u64 n, u8* status,
                                                            u64* vout, int conc_erase, int gated) {
  WS_PROLOGUE(d, gated, n);
  const u32 te0 = ld_u32_relaxed(d.state);
  const bool conc = conc_erase == 2 ? ld_u32_relaxed(d.cs + 3) != 0 : conc_erase != 0;
  const int lane = threadIdx.x & 31;
  const u64 nwarps = ((u64)gridDim.x * blockDim.x) >> 5;
  for (u64 c = (blockIdx.x * (u64)blockDim.x + threadIdx.x) >> 5; c * 32 < n; c += nwarps) {
    const u64 i = c * 32 + lane;
    bool pending = i < n;
    int kind = OP_QUERY, merge = 0;
    u64 key = 0, val = 0, b0 = 0, b1 = 0, b2 = 0;
    u16 tag = 1;
    if (pending) {
      const u8 op = ops ? __ldg(ops + i) : uop;
      kind = op & 15;
      if (kind > OP_QUERY) kind = OP_QUERY;
      merge = op >> 4;
      key = __ldg(keys + i);
      val = vals ? __ldg(vals + i) : 0ull;
      const u64 h0 = mix64(key ^ d.seeds[0]);
      b0 = d.frontm(h0 >> 16);
      const u16 t = (u16)(h0 & 0xFFFF);
      tag = t ? t : (u16)1;
      b1 = d.front + d.backm(mix64(key ^ d.seeds[1]) >> 16);
      b2 = d.front + d.backm(mix64(key ^ d.seeds[2]) >> 16);
      if (b2 < b1) { const u64 x = b1; b1 = b2; b2 = x; }  // ascending; b2 == b1 -> one bucket
    }
    const bool locker = kind != OP_QUERY;
    u8 st = 0;
    u64 qv = 0;
    unsigned backoff = 64;
    bool held0 = false, heldb = false;
    while (__any_sync(0xFFFFFFFFu, pending)) {
      if (pending && locker && !held0) held0 = try_lock_bucket(d.locks, b0);
      const bool hold0 = pending && (!locker || held0);
      u32 M0, Z0;
      coop_masks<false, true>(d, hold0, b0, tag, M0, Z0);
      bool needb = false, decided = false, te_last = true;
      i64 del = -1;
      u64 target = 0;
      u32 Zt = 0;
      u64 old;
      if (hold0) {
        const int j = M0 ? pair_confirm<false, true>(d, b0, M0, key, old) : -1;
        if (j >= 0) {
          if (kind == OP_UPSERT) {
            st_cell(d.cells + 2 * (b0 * 32 + j), key, apply_merge(merge, old, val));
            st = S_UPDATED;
            pending = false;
          } else if (kind == OP_ERASE) {
            del = (i64)(b0 * 32 + j);
          } else {
            st = 1;
            qv = old;
            pending = false;
          }
        } else {
          bool te = te0 != 0;
          if (conc) { fence_acq_rel(); te = ld_u32_relaxed(d.state) != 0; }
          te_last = te;
          if (Z0 && !te) {  // saw_empty: the front never filled
            if (kind == OP_UPSERT) {
              target = b0;
              Zt = Z0;
              decided = true;
            } else {
              st = 0;  // provably absent
              pending = false;
            }
          } else if (kind == OP_UPSERT) {
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
          } else {
            needb = true;  // erase / query: search the backyard (no locks)
          }
        }
      }
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
        if (kind == OP_UPSERT) {
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
            if (Z1 && (!need2 || !Z2 || u1 <= u2)) { target = b1; Zt = Z1; }
            else if (need2 && Z2) { target = b2; Zt = Z2; }
            decided = true;  // Zt == 0 -> FULL
          }
        } else if (kind == OP_ERASE) {
          if (j >= 0) del = (i64)(bj * 32 + j);
          else { st = 0; pending = false; }
        } else {
          if (j >= 0) { st = 1; qv = old; }
          pending = false;
        }
      }
      if (decided) {
        if (!Zt) {
          st = S_FULL;
          pending = false;
        } else {
          const u64 slot = target * 32 + (__ffs(Zt) - 1);
          if (conc) fence_acq_rel();
          if (!te_last && ((Zt >> ((slot & 31) ^ 1)) & 1u)) st_cell(d.cells + 2 * (slot ^ 1), 0, 0);
          st_cell(d.cells + 2 * slot, key, val);
          st_tag(d.tags + slot, tag);
          st = S_INSERTED;
          pending = false;
        }
      }
      if (__any_sync(0xFFFFFFFFu, del >= 0)) {  // tombstones, one fence per step for the warp
        if (del >= 0 && ld_u32_relaxed(d.state) == 0) st_u32_relaxed(d.state, 1u);
        fence_acq_rel();
        if (del >= 0) st_cell(d.cells + 2 * (u64)del, TOMB, 0);
        fence_acq_rel();  // the tombstone is visible before the zero tag that advertises it
        if (del >= 0) {
          st_tag(d.tags + (u64)del, 0);
          st = 1;
          pending = false;
        }
      }
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
    if (i < n) {
      if (status) status[i] = st;
      if (vout) vout[i] = kind == OP_QUERY && st ? qv : 0;
    }
  }
}

static void iceberg_md_ops(const OpsArgs& a, bool def) {
  if (def && a.ops && !a.instr && !a.d.delay_ns && !a.serial && !a.redo && !a.rlist && !a.d.phased &&
      a.d.tune_upsert == 4) {
    u64 g = (a.n + 255) / 256;
    const u64 lim = std::max<u64>((a.d.front + 255) / 256, 4);  // <= ~1 op in flight per front bucket
    g = std::max<u64>(std::min<u64>(std::min<u64>(g, (u64)kSMs * table_grid_per_sm(a.d)), lim), 1);
    k_mixed_icemd_rounds<<<(unsigned)g, 256, 0, a.s>>>(a.d, a.ops, a.uop, a.keys, a.vals, a.n, a.status, a.vout,
                                                        a.conc_erase, a.gated);
    return;
  }
  const bool erase_only = !a.ops && (a.uop & 15) == OP_ERASE;
  if (def && erase_only && !a.instr && !a.d.delay_ns && !a.serial && !a.redo && !a.d.phased &&
      a.d.tune_upsert == 4) {
    u64 g = (a.n + 255) / 256;
    const u64 lim = std::max<u64>((a.d.front + 255) / 256, 4);  // <= ~1 op in flight per front bucket
    g = std::max<u64>(std::min<u64>(std::min<u64>(g, (u64)kSMs * table_grid_per_sm(a.d)), lim), 1);
    if (a.d.tune_l2pol == 2)
      k_erase_icemd_rounds<true><<<(unsigned)g, 256, 0, a.s>>>(a.d, a.keys, a.n, a.status, a.conc_erase, a.gated);
    else
      k_erase_icemd_rounds<false><<<(unsigned)g, 256, 0, a.s>>>(a.d, a.keys, a.n, a.status, a.conc_erase, a.gated);
    return;
  }
  const bool upsert_only = !a.ops && (a.uop & 15) == OP_UPSERT;
  if (def && upsert_only && !a.instr && !a.d.delay_ns && !a.serial && !a.redo && !a.d.phased && !a.d.lock_elided &&
      a.d.tune_upsert == 4) {
    u64 g = (a.n + 255) / 256;
    const u64 lim = std::max<u64>((a.d.nb + 255) / 256, 4);  // <= ~1 op in flight per bucket
    g = std::max<u64>(std::min<u64>(std::min<u64>(g, (u64)kSMs * table_grid_per_sm(a.d)), lim), 1);
    k_upsert_icemd_rounds<true><<<(unsigned)g, 256, 0, a.s>>>(a.d, a.keys, a.vals, a.n, a.uop >> 4, a.status,
                                                               a.conc_erase, a.gated);
    return;
  }
  if (def) launch_ops_t<D_ICEBERG_MD, 32>(a); else launch_ops_t<D_ICEBERG_MD, 0>(a);
}
static void iceberg_md_query(const QueryArgs& a, bool def) {
  // opt-in (query_ilp = 6): the pair-cooperative query measured slower than
  // the generic one at 2^26, where the tag array is largely L2-resident
  if (def && a.d.tune_qilp == 6) {
    u64 g = (a.n + 255) / 256;
    g = std::min<u64>(std::max<u64>(g, 1), (u64)kSMs * table_grid_per_sm(a.d));
#define WS_QI(RO, F) k_query_icemd_coop<RO, F><<<(unsigned)g, 256, 0, a.s>>>(a.d, a.keys, a.n, a.vout, a.found, \
                                                                            a.conc_erase, a.gated)
    const bool f64 = a.d.tune_l2pol == 2;
    if (a.ro) { if (f64) WS_QI(true, true); else WS_QI(true, false); }
    else { if (f64) WS_QI(false, true); else WS_QI(false, false); }
#undef WS_QI
    return;
  }
  if (def) launch_query_t<D_ICEBERG_MD, 32>(a); else launch_query_t<D_ICEBERG_MD, 0>(a);
}
static void iceberg_md_locate(const LocateArgs& a, bool def) {
  if (def) launch_locate_t<D_ICEBERG_MD, 32>(a); else launch_locate_t<D_ICEBERG_MD, 0>(a);
}
static void iceberg_md_preload(bool def) {
  if (!def) { preload_t<D_ICEBERG_MD, 0>(); return; }
  preload_t<D_ICEBERG_MD, 32>();
  preload_fn(k_upsert_icemd_rounds<true>);
  preload_fn(k_query_icemd_coop<false, true>);
  preload_fn(k_query_icemd_coop<true, true>);
  preload_fn(k_erase_icemd_rounds<true>);
  preload_fn(k_mixed_icemd_rounds);
}
Launchers launchers_iceberg_md() {
  return Launchers{iceberg_md_ops, iceberg_md_query, iceberg_md_locate, iceberg_md_preload};
}

}  // namespace ws

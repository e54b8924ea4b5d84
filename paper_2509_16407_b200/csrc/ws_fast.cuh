// ws_fast.cuh -- tuned kernels for the headline path (P2 + fingerprint
// metadata, 32-slot buckets): the pair-cooperative lock-free query, the
// warp-synchronous lock-round upsert and the fused mixed-batch kernel.
//
// Why: beyond the 126 MB L2 a B200 sustains ~45 G random line REQUESTS/s
// (scripts/gather_bench.cu), whatever their width up to 128 B, so each kernel
// minimises requests per op (one request per 64-byte tag block, 64-byte L2
// fills) and keeps every lane's op in flight.  Variants measured slower and
// removed in round 2: Q independent lookups per thread,
// 2-lane tiles per op, L2 evict-first/last policies, L2 prefetch of the next
// op's tag block, deferring lock releases behind the next round's loads.
//
// Semantics are exactly Ctx::p2_find / p2_upsert / p2_erase (reference
// openaddr.py:370-473).
#pragma once
#include "ws_ops.cuh"

namespace ws {

// 64-byte L2 fetch: the default promotes every random miss to a 128-byte
// line fill (4 sectors, measured); a 64-byte tag block or a 16-byte cell only
// needs 2 (scripts/gather_bench.cu: 3.92 -> 1.98 DRAM sectors per access).
__device__ __forceinline__ void ld_tags32_64(const u16* p, u32 (&w)[8]) {
  asm volatile("ld.relaxed.gpu.global.L2::64B.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7])
               : "l"(p) : "memory");
}
__device__ __forceinline__ void ld_tags32_ro64(const u16* p, u32 (&w)[8]) {
  asm volatile("ld.global.nc.L1::no_allocate.L2::64B.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7])
               : "l"(p));
}
template <bool RO, bool F64>
__device__ __forceinline__ void ld_cell_f(const u64* p, u64& k, u64& v) {
  if (!F64) { load_cell<RO>(p, k, v); return; }
  if (RO)
    asm volatile("ld.global.nc.L1::no_allocate.L2::64B.v2.u64 {%0, %1}, [%2];" : "=l"(k), "=l"(v) : "l"(p));
  else
    asm volatile("{.reg .b128 t; ld.relaxed.gpu.global.L2::64B.b128 t, [%2]; mov.b128 {%0, %1}, t;}"
                 : "=l"(k), "=l"(v) : "l"(p) : "memory");
}

// first slot (0..31) of bucket b holding key among the tag matches M, or -1
template <bool RO, bool F64 = false>
__device__ __forceinline__ int pair_confirm(const Dev& d, u64 b, u32 M, u64 key, u64& val) {
  while (M) {
    const int j = __ffs(M) - 1;
    M &= M - 1;
    u64 k, v;
    ld_cell_f<RO, F64>(d.cells + 2 * (b * 32 + j), k, v);
    if (k == key) { val = v; return j; }
  }
  return -1;
}

__device__ __forceinline__ void red_and_relaxed(u32* p, u32 m) {
  asm volatile("red.relaxed.gpu.global.and.b32 [%0], %1;" :: "l"(p), "r"(m) : "memory");
}

// ------------------------------------------------ pair-cooperative loads
//
// One thread per op, but the 64-byte tag blocks of lanes 2k and 2k+1 are
// fetched cooperatively: in the first instruction both lanes load the two
// halves of op 2k's block, in the second the two halves of op 2k+1's block --
// one line request per block and still 32 ops per warp.  Each lane then swaps
// the 16-slot mask half it holds for its partner's op.  Must be called by all
// 32 lanes (converged); `active` gates the lane's own op.
__device__ __forceinline__ void half_masks(const u32 (&w)[8], u16 tag, u32& m, u32& z) {
  const u32 pat = (u32)tag * 0x10001u;
  m = 0;
  z = 0;
#pragma unroll
  for (int i = 0; i < 8; i++) {
    const u32 mm = __vcmpeq2(w[i], pat), zz = __vcmpeq2(w[i], 0u);
    m |= ((mm & 1u) | ((mm >> 15) & 2u)) << (2 * i);
    z |= ((zz & 1u) | ((zz >> 15) & 2u)) << (2 * i);
  }
}

template <bool RO, bool F64>
__device__ __forceinline__ void coop_masks(const Dev& d, bool active, u64 b, u16 tag, u32& M, u32& Z) {
  const int half = threadIdx.x & 1;
  const u64 pb = __shfl_xor_sync(0xFFFFFFFFu, b, 1);
  const u32 pt = __shfl_xor_sync(0xFFFFFFFFu, (u32)tag, 1);
  const u32 pa = __shfl_xor_sync(0xFFFFFFFFu, (u32)active, 1);
  // op A = even lane's op, op B = odd lane's op
  const u64 bA = half ? pb : b, bB = half ? b : pb;
  const u16 tA = (u16)(half ? pt : tag), tB = (u16)(half ? tag : pt);
  const bool aA = half ? pa != 0 : active, aB = half ? active : pa != 0;
  u32 wA[8], wB[8];
#pragma unroll
  for (int i = 0; i < 8; i++) { wA[i] = 0xFFFFFFFFu; wB[i] = 0xFFFFFFFFu; }
  const u16* pA = d.tags + bA * 32 + half * 16;
  const u16* pB = d.tags + bB * 32 + half * 16;
  if (aA) {
    if (F64) { if (RO) ld_tags32_ro64(pA, wA); else ld_tags32_64(pA, wA); }
    else { if (RO) ld_tags32_ro(pA, wA); else ld_tags32(pA, wA); }
  }
  if (aB) {
    if (F64) { if (RO) ld_tags32_ro64(pB, wB); else ld_tags32_64(pB, wB); }
    else { if (RO) ld_tags32_ro(pB, wB); else ld_tags32(pB, wB); }
  }
  u32 mA, zA, mB, zB;
  half_masks(wA, tA, mA, zA);
  half_masks(wB, tB, mB, zB);
  // even lane holds A-lo (needs A-hi from odd); odd holds B-hi (needs B-lo)
  const u32 rm = __shfl_xor_sync(0xFFFFFFFFu, half ? mA : mB, 1);
  const u32 rz = __shfl_xor_sync(0xFFFFFFFFu, half ? zA : zB, 1);
  if (!half) { M = mA | (rm << 16); Z = zA | (rz << 16); }
  else { M = rm | (mB << 16); Z = rz | (zB << 16); }
}

// One thread per query, pair-cooperative tag fetches (see coop_masks).
template <bool RO, bool F64, int MINB>
__global__ void __launch_bounds__(256, MINB) k_query_p2md_coop(Dev d, const u64* __restrict__ keys, u64 n, u64* vout,
                                                         u8* found, int conc_erase, int gated, int check_keys = 0) {
  WS_PROLOGUE(d, gated, n);
  const u32 te0 = ld_u32_relaxed(d.state);
  const u64 stride = (u64)gridDim.x * blockDim.x;
  // the loop runs warp-uniformly: the bound is the warp's first index
  const u64 first = (blockIdx.x * (u64)blockDim.x + threadIdx.x) & ~31ull;
  for (u64 base = first; base < n; base += stride) {
    const u64 i = base + (threadIdx.x & 31);
    const bool act = i < n;
    const u64 key = act ? __ldg(keys + i) : 0;
    if (check_keys && __any_sync(0xFFFFFFFFu, act && is_sentinel(key)) && (threadIdx.x & 31) == 0)
      atomicAdd(d.cs, 1u);  // a sentinel (0, 2^64-2, 2^64-1) among this warp's keys (k_validate's rule)
    const u64 h0 = mix64(key ^ d.seeds[0]);
    const u64 b0 = d.nbm(h0 >> 16);
    const u16 t = (u16)(h0 & 0xFFFF);
    const u16 tag = t ? t : (u16)1;
    u32 M, Z;
    coop_masks<RO, F64>(d, act, b0, tag, M, Z);
    u64 val = 0;
    bool hit = act && M && pair_confirm<RO, F64>(d, b0, M, key, val) >= 0;
    bool te = te0 != 0;
    if (conc_erase) { fence_acq_rel(); te = ld_u32_relaxed(d.state) != 0; }
    const int zc = __popc(Z);
    const int used0 = 32 - (zc < d.zcc ? zc : d.zcc);
    const u64 b1 = d.nbm(mix64(key ^ d.seeds[1]) >> 16);
    const bool need1 = act && !hit && !(Z && !te && used0 < d.shortcut) && b1 != b0;
    if (__any_sync(0xFFFFFFFFu, need1)) {
      coop_masks<RO, F64>(d, need1, b1, tag, M, Z);
      if (need1 && M) hit = pair_confirm<RO, F64>(d, b1, M, key, val) >= 0;
    }
    if (act) {
      if (found) found[i] = hit;
      if (vout) vout[i] = hit ? val : 0;
    }
  }
}

// PHASED: the reference's bulk-synchronous mode (mode="phased",
// sync.py:70-102): bucket locks are no-ops, so there is no try-lock, fence
// or release, and publication falls back to a 128-bit CAS (foreign writers
// race for free slots); a lost CAS retries the op next round.
// FILL: when the target cell's sector partner (slot ^ 1) is a zero tag and
// the table never tombstoned, the partner is EMPTY (0,0) and exclusively ours
// under the bucket lock; storing (0,0) there too makes the 32-byte sector
// fully valid in L2, so its eviction needs no ECC read-modify-write of the
// untouched half (measured ~1 DRAM sector per insert without it).
template <bool F64, int MINB, bool PHASED, bool FILL = false>
__global__ void __launch_bounds__(256, MINB) k_upsert_p2md_rounds(Dev d, const u64* __restrict__ keys,
                                                            const u64* __restrict__ vals, u64 n, int merge,
                                                            u8* status, int conc_erase, int gated) {
  WS_PROLOGUE(d, gated, n);
  const u32 te0 = ld_u32_relaxed(d.state);
  const int lane = threadIdx.x & 31;
  const u64 nwarps = ((u64)gridDim.x * blockDim.x) >> 5;
  const u64 c0 = (blockIdx.x * (u64)blockDim.x + threadIdx.x) >> 5;
  for (u64 c = c0; c * 32 < n; c += nwarps) {
    const u64 i = c * 32 + lane;
    bool pending = i < n;
    u64 key = 0, val = 0, b0 = 0, b1 = 0;
    u16 tag = 1;
    if (pending) {
      key = __ldg(keys + i);
      val = __ldg(vals + i);
      const u64 h0 = mix64(key ^ d.seeds[0]);
      b0 = d.nbm(h0 >> 16);
      const u16 t = (u16)(h0 & 0xFFFF);
      tag = t ? t : (u16)1;
      b1 = d.nbm(mix64(key ^ d.seeds[1]) >> 16);
    }
    u8 st = 0;
    unsigned backoff = 64;
    // Locks a lane holds across rounds.  Retries must not be symmetric: two
    // lanes of one warp that each hold their primary and want the other's
    // (b1(A) = b0(B), b1(B) = b0(A)) would fail, release and collide again in
    // every lockstep round -- a livelock, hit in tombstoned small tables where
    // every insert needs its alternate.  The first attempt try-locks b1 in any
    // order (non-blocking, so no deadlock); after a failure a lane only ever
    // waits for a HIGHER bucket while holding a lower one: holding b0 it
    // retries b1 > b0 next round without releasing b0; needing b1 < b0 it
    // releases b0 and next round takes b1 first, then b0 (`lofirst`).
    bool held0 = false, held1 = false, lofirst = false;
    while (__any_sync(0xFFFFFFFFu, pending)) {
      // phase 1: try-locks in ascending order (never block)
      if (!PHASED && pending) {
        if (lofirst) {
          if (!held1) held1 = try_lock_bucket(d.locks, b1);
          if (held1 && !held0) held0 = try_lock_bucket(d.locks, b0);
        } else if (!held0) {
          held0 = try_lock_bucket(d.locks, b0);
        }
      }
      const bool hold0 = pending && (PHASED || held0);
      bool drop0 = false;
      // phase 2: primary tag blocks, one request per op
      u32 M0, Z0;
      coop_masks<false, F64>(d, hold0, b0, tag, M0, Z0);
      bool hold1 = false, need1 = false, decided = false, te_last = true;
      u64 old;
      int used0 = 0;
      if (hold0) {
        const int j = M0 ? pair_confirm<false, F64>(d, b0, M0, key, old) : -1;
        if (j >= 0) {
          st_cell(d.cells + 2 * (b0 * 32 + j), key, apply_merge(merge, old, val));
          st = S_UPDATED;
          pending = false;
        } else {
          bool te = te0 != 0;
          if (conc_erase) { fence_acq_rel(); te = ld_u32_relaxed(d.state) != 0; }
          te_last = te;
          const int zc0 = __popc(Z0);
          used0 = 32 - (zc0 < d.zcc ? zc0 : d.zcc);
          if ((te || used0 >= d.shortcut) && b1 != b0) {
            if (PHASED || held1) {
              hold1 = true;
            } else {
              held1 = try_lock_bucket(d.locks, b1);
              hold1 = held1;
              // on failure: b1 above b0 -> keep b0 and retry b1 next round;
              // b1 below b0 -> release b0, next round take b1 first, then b0
              if (!held1 && b1 < b0) {
                lofirst = true;
                drop0 = true;
              }
            }
            need1 = hold1;
          } else {
            decided = true;  // shortcut (or b1 == b0): the primary it is
          }
        }
      }
      // phase 3: alternate tag blocks of the lanes that need them
      u32 M1 = 0, Z1 = 0;
      if (__any_sync(0xFFFFFFFFu, need1)) coop_masks<false, F64>(d, need1, b1, tag, M1, Z1);
      u64 target = b0;
      u32 Zt = Z0;
      if (need1) {
        const int j = M1 ? pair_confirm<false, F64>(d, b1, M1, key, old) : -1;
        if (j >= 0) {
          st_cell(d.cells + 2 * (b1 * 32 + j), key, apply_merge(merge, old, val));
          st = S_UPDATED;
          pending = false;
        } else {
          const int zc1 = __popc(Z1);
          const int used1 = 32 - (zc1 < d.zcc ? zc1 : d.zcc);
          const bool prim = used0 <= used1;  // ties go to the primary
          target = prim ? b0 : b1;
          Zt = prim ? Z0 : Z1;
          if (!Zt) { target = prim ? b1 : b0; Zt = prim ? Z1 : Z0; }
          decided = true;
        }
      }
      if (decided) {
        if (!Zt) {
          st = S_FULL;
          pending = false;
        } else {
          const u64 slot = target * 32 + (__ffs(Zt) - 1);
          if (conc_erase) fence_acq_rel();
          if (PHASED) {
            if (publish_cell(d.cells + 2 * slot, key, val)) {
              st_tag(d.tags + slot, tag);
              st = S_INSERTED;
              pending = false;
            }
          } else {
            if (FILL && !te_last && ((Zt >> ((slot & 31) ^ 1)) & 1u)) st_cell(d.cells + 2 * (slot ^ 1), 0, 0);
            st_cell(d.cells + 2 * slot, key, val);
            st_tag(d.tags + slot, tag);
            st = S_INSERTED;
            pending = false;
          }
        }
      }
      // phase 4: one MEMBAR for the warp, then relaxed releases of the
      // finished lanes' locks (pending lanes keep what they hold, see above)
      if (!PHASED) {
        __syncwarp();
        fence_acq_rel();
        if (held1 && !pending) {
          red_and_relaxed(d.locks + (b1 >> 5), ~(1u << (b1 & 31)));
          held1 = false;
        }
        if (held0 && (!pending || drop0)) {
          red_and_relaxed(d.locks + (b0 >> 5), ~(1u << (b0 & 31)));
          held0 = false;
        }
      }
      if (pending) {
        __nanosleep(backoff + 8 * (threadIdx.x & 31));
        if (backoff < 4096) backoff <<= 1;
      }
    }
    if (status && i < n) status[i] = st;
  }
}

// Mixed batches in ONE launch (the paper's single-kernel aging; interleaved
// batches, small mixed batches): k_upsert_p2md_rounds extended with erase and
// query lanes.  Every lane runs its own op kind in the same warp-synchronous
// rounds, so the pair-cooperative tag fetches stay warp-collective:
//   * upsert lanes: exactly the upsert kernel's lock rounds (b0, then b1 when
//     the shortcut does not apply), per-op merge from the op byte;
//   * erase lanes (reference openaddr.py:449-473): lock b0 only, find in b0,
//     else (no early exit) in b1, then the tombstone protocol of
//     Ctx::tombstone (tombstones_ever, fence, cell := TOMB, fence, tag := 0),
//     one fence per step for the warp;
//   * query lanes: lock-free (openaddr.py:433-447), done in the first round.
// Op bytes whose kind is not upsert / erase run as queries and merges above
// MIN as REPLACE, as Ctx::run / apply_merge do.  conc_erase 2: the launch's
// erase count (k_count_erases) decides whether the tombstone flag must be
// re-read behind a fence.
template <int MINB>
__global__ void __launch_bounds__(256, MINB) k_mixed_p2md_rounds(Dev d, const u8* __restrict__ ops, u8 uop,
                                                           const u64* __restrict__ keys,
                                                           const u64* __restrict__ vals, u64 n, u8* status,
                                                           u64* vout, int conc_erase, int gated) {
  WS_PROLOGUE(d, gated, n);
  const u32 te0 = ld_u32_relaxed(d.state);
  const bool conc = conc_erase == 2 ? ld_u32_relaxed(d.cs + 3) != 0 : conc_erase != 0;
  const int lane = threadIdx.x & 31;
  const u64 nwarps = ((u64)gridDim.x * blockDim.x) >> 5;
  const u64 c0 = (blockIdx.x * (u64)blockDim.x + threadIdx.x) >> 5;
  for (u64 c = c0; c * 32 < n; c += nwarps) {
    const u64 i = c * 32 + lane;
    bool pending = i < n;
    int kind = OP_QUERY, merge = 0;
    u64 key = 0, val = 0, b0 = 0, b1 = 0;
    u16 tag = 1;
    if (pending) {
      const u8 op = ops ? __ldg(ops + i) : uop;
      kind = op & 15;
      if (kind > OP_QUERY) kind = OP_QUERY;
      merge = op >> 4;
      key = __ldg(keys + i);
      val = vals ? __ldg(vals + i) : 0ull;
      const u64 h0 = mix64(key ^ d.seeds[0]);
      b0 = d.nbm(h0 >> 16);
      const u16 t = (u16)(h0 & 0xFFFF);
      tag = t ? t : (u16)1;
      b1 = d.nbm(mix64(key ^ d.seeds[1]) >> 16);
    }
    const bool locker = kind != OP_QUERY;
    u8 st = 0;
    u64 qv = 0;
    unsigned backoff = 64;
    // lock discipline of k_upsert_p2md_rounds (ascending waits only); erase
    // lanes only ever hold b0
    bool held0 = false, held1 = false, lofirst = false;
    while (__any_sync(0xFFFFFFFFu, pending)) {
      if (pending && locker) {
        if (lofirst) {
          if (!held1) held1 = try_lock_bucket(d.locks, b1);
          if (held1 && !held0) held0 = try_lock_bucket(d.locks, b0);
        } else if (!held0) {
          held0 = try_lock_bucket(d.locks, b0);
        }
      }
      const bool hold0 = pending && (!locker || held0);
      bool drop0 = false;
      u32 M0, Z0;
      coop_masks<false, true>(d, hold0, b0, tag, M0, Z0);
      bool hold1 = false, need1 = false, decided = false, te_last = true;
      i64 del = -1;
      u64 old;
      int used0 = 0;
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
          const int zc0 = __popc(Z0);
          used0 = 32 - (zc0 < d.zcc ? zc0 : d.zcc);
          if (kind == OP_UPSERT) {
            if ((te || used0 >= d.shortcut) && b1 != b0) {
              if (held1) {
                hold1 = true;
              } else {
                held1 = try_lock_bucket(d.locks, b1);
                hold1 = held1;
                if (!held1 && b1 < b0) {
                  lofirst = true;
                  drop0 = true;
                }
              }
              need1 = hold1;
            } else {
              decided = true;
            }
          } else if (!(Z0 && !te && used0 < d.shortcut) && b1 != b0) {
            need1 = true;  // erase / query: the key may live in the alternate
          } else {
            st = 0;  // early exit: provably absent
            pending = false;
          }
        }
      }
      u32 M1 = 0, Z1 = 0;
      if (__any_sync(0xFFFFFFFFu, need1)) coop_masks<false, true>(d, need1, b1, tag, M1, Z1);
      u64 target = b0;
      u32 Zt = Z0;
      if (need1) {
        const int j = M1 ? pair_confirm<false, true>(d, b1, M1, key, old) : -1;
        if (kind == OP_UPSERT) {
          if (j >= 0) {
            st_cell(d.cells + 2 * (b1 * 32 + j), key, apply_merge(merge, old, val));
            st = S_UPDATED;
            pending = false;
          } else {
            const int zc1 = __popc(Z1);
            const int used1 = 32 - (zc1 < d.zcc ? zc1 : d.zcc);
            const bool prim = used0 <= used1;  // ties go to the primary
            target = prim ? b0 : b1;
            Zt = prim ? Z0 : Z1;
            if (!Zt) { target = prim ? b1 : b0; Zt = prim ? Z1 : Z0; }
            decided = true;
          }
        } else if (kind == OP_ERASE) {
          if (j >= 0) del = (i64)(b1 * 32 + j);
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
      // tombstones (one fence per step for the warp)
      if (__any_sync(0xFFFFFFFFu, del >= 0)) {
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
      if (held1 && !pending) {
        red_and_relaxed(d.locks + (b1 >> 5), ~(1u << (b1 & 31)));
        held1 = false;
      }
      if (held0 && (!pending || drop0)) {
        red_and_relaxed(d.locks + (b0 >> 5), ~(1u << (b0 & 31)));
        held0 = false;
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

}  // namespace ws

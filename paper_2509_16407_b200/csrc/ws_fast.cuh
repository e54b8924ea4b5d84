// ws_fast.cuh -- tuned kernels for the headline path (P2 + fingerprint
// metadata, 32-slot buckets): lock-free batched queries with Q lookups per
// thread advanced phase by phase.
//
// Why: beyond the 126 MB L2 a B200 sustains ~45 G random line accesses/s
// (scripts/gather_bench.cu: 43-46 G/s for 16-128 B accesses from 512 MiB to
// 64 GiB buffers, i.e. a DRAM row-activation ceiling, not a byte ceiling), and
// reaching it needs ~10^4 accesses in flight per SM.  The one-op-per-thread
// kernel has exactly one dependent access in flight per thread (tags -> slot
// -> alternate tags -> slot).  Here every thread keeps Q independent lookups
// in flight: all Q primary tag blocks are requested before any is examined,
// then all Q slot confirmations, then all Q alternate tag blocks, ...
//
// Semantics are exactly Ctx::p2_find(early_exit=true) (reference
// openaddr.py:433-447): tag scan of b0, full-key confirmation of every tag
// match, early exit when b0 provably never overflowed, else b1.
#pragma once
#include "ws_ops.cuh"

namespace ws {

// POL: 0 = no L2 hint, 1 = tags evict_last + cells evict_first
template <bool RO, int POL>
__device__ __forceinline__ void fast_tags32(const u16* p, u32 (&w)[8], u64 pol) {
  if (POL == 0) {
    if (RO) ld_tags32_ro(p, w); else ld_tags32(p, w);
  } else if (RO) {
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
                 : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7])
                 : "l"(p), "l"(pol));
  } else {
    asm volatile("ld.relaxed.gpu.global.L2::cache_hint.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
                 : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7])
                 : "l"(p), "l"(pol) : "memory");
  }
}

template <bool RO, int POL>
__device__ __forceinline__ void fast_cell(const u64* p, u64& k, u64& v, u64 pol) {
  if (POL == 0) {
    load_cell<RO>(p, k, v);
  } else if (RO) {
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u64 {%0, %1}, [%2], %3;"
                 : "=l"(k), "=l"(v) : "l"(p), "l"(pol));
  } else {
    asm volatile("{.reg .b128 t; ld.relaxed.gpu.global.L2::cache_hint.b128 t, [%2], %3; mov.b128 {%0, %1}, t;}"
                 : "=l"(k), "=l"(v) : "l"(p), "l"(pol) : "memory");
  }
}

__device__ __forceinline__ void masks_from(const u32 (&a)[8], const u32 (&b)[8], u16 tag, u32& match, u32& zero) {
  const u32 pat = (u32)tag * 0x10001u;
  match = 0;
  zero = 0;
#pragma unroll
  for (int i = 0; i < 8; i++) {
    u32 m = __vcmpeq2(a[i], pat), z = __vcmpeq2(a[i], 0u);
    match |= ((m & 1u) | ((m >> 15) & 2u)) << (2 * i);
    zero |= ((z & 1u) | ((z >> 15) & 2u)) << (2 * i);
    m = __vcmpeq2(b[i], pat);
    z = __vcmpeq2(b[i], 0u);
    match |= ((m & 1u) | ((m >> 15) & 2u)) << (2 * i + 16);
    zero |= ((z & 1u) | ((z >> 15) & 2u)) << (2 * i + 16);
  }
}

template <bool RO, int POL>
__device__ __forceinline__ void block_masks(const Dev& d, u64 b, u16 tag, u32& M, u32& Z, u64 pol) {
  u32 a[8], c[8];
  fast_tags32<RO, POL>(d.tags + b * 32, a, pol);
  fast_tags32<RO, POL>(d.tags + b * 32 + 16, c, pol);
  masks_from(a, c, tag, M, Z);
}

// Confirm the tag matches M of bucket b against key; -> found / value.
template <bool RO, int POL>
__device__ __forceinline__ bool confirm(const Dev& d, u64 b, u32 M, u64 key, u64& val, u64 pol) {
  while (M) {
    const int j = __ffs(M) - 1;
    M &= M - 1;
    u64 k, v;
    fast_cell<RO, POL>(d.cells + 2 * (b * 32 + j), k, v, pol);
    if (k == key) { val = v; return true; }
  }
  return false;
}

template <int Q, bool RO, int POL>
__global__ void __launch_bounds__(256) k_query_p2md(Dev d, const u64* __restrict__ keys, u64 n, u64* vout,
                                                    u8* found, int conc_erase, int gated) {
  WS_PROLOGUE(d, gated, n);
  u64 pol_tag = 0, pol_cell = 0;
  if (POL) {
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_tag));
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_cell));
  }
  const u32 te0 = ld_u32_relaxed(d.state);
  const u64 chunk = (u64)blockDim.x * Q;
  for (u64 base = blockIdx.x * chunk; base < n; base += (u64)gridDim.x * chunk) {
    u64 key[Q], b0[Q], b1[Q], val[Q];
    u16 tag[Q];
    u32 M[Q], Z[Q];
    bool done[Q], hit[Q];
#pragma unroll
    for (int q = 0; q < Q; q++) {
      const u64 i = base + threadIdx.x + (u64)q * blockDim.x;
      done[q] = i >= n;
      key[q] = done[q] ? 0 : __ldg(keys + i);
      const u64 h0 = mix64(key[q] ^ d.seeds[0]);
      b0[q] = d.nbm(h0 >> 16);
      const u16 t = (u16)(h0 & 0xFFFF);
      tag[q] = t ? t : (u16)1;
      hit[q] = false;
      val[q] = 0;
    }
    // phase 1: every primary tag block in flight
#pragma unroll
    for (int q = 0; q < Q; q++)
      if (!done[q]) block_masks<RO, POL>(d, b0[q], tag[q], M[q], Z[q], pol_tag);
    // phase 2: confirm primary matches
#pragma unroll
    for (int q = 0; q < Q; q++)
      if (!done[q] && M[q]) hit[q] = confirm<RO, POL>(d, b0[q], M[q], key[q], val[q], pol_cell);
    // early exit (openaddr.py:440-442): b0 has a never-used slot, the table
    // never tombstoned and b0 is below the shortcut threshold
    bool te = te0 != 0;
    if (conc_erase) {
      fence_acq_rel();
      te = ld_u32_relaxed(d.state) != 0;
    }
#pragma unroll
    for (int q = 0; q < Q; q++) {
      if (done[q] || hit[q]) { done[q] = true; continue; }
      const int zc = __popc(Z[q]);
      const int used0 = 32 - (zc < d.zcc ? zc : d.zcc);
      if (Z[q] && !te && used0 < d.shortcut) { done[q] = true; continue; }
      b1[q] = d.nbm(mix64(key[q] ^ d.seeds[1]) >> 16);
      if (b1[q] == b0[q]) done[q] = true;
    }
    // phase 3: alternate tag blocks
#pragma unroll
    for (int q = 0; q < Q; q++)
      if (!done[q]) block_masks<RO, POL>(d, b1[q], tag[q], M[q], Z[q], pol_tag);
    // phase 4: confirm alternate matches
#pragma unroll
    for (int q = 0; q < Q; q++)
      if (!done[q] && M[q]) hit[q] = confirm<RO, POL>(d, b1[q], M[q], key[q], val[q], pol_cell);
#pragma unroll
    for (int q = 0; q < Q; q++) {
      const u64 i = base + threadIdx.x + (u64)q * blockDim.x;
      if (i < n) {
        if (found) found[i] = hit[q];
        if (vout) vout[i] = hit[q] ? val[q] : 0;
      }
    }
  }
}

// ===================================================== lane-pair kernels
//
// A 2-lane cooperative tile owns one operation.  Each lane loads one 32-byte
// half of the 64-byte tag block, so the warp instruction carries ONE line
// request per operation instead of two (beyond L2 the B200 sustains ~45 G
// L2-missing requests/s, scripts/gather_bench.cu; a single thread reading 64 B
// issues 2).  The lanes exchange their 16-slot masks with one shuffle and then
// run identical control flow on identical data; loads of the same address by
// both lanes in one instruction merge into one request.  Side effects (lock
// atomics, publication stores) are issued by the even lane only.

struct Pair {
  u32 mask;
  int half;
  __device__ __forceinline__ Pair() {
    const int lane = threadIdx.x & 31;
    half = lane & 1;
    mask = 3u << (lane & 30);
  }
  __device__ __forceinline__ u32 xchg(u32 v) const { return __shfl_xor_sync(mask, v, 1); }
  __device__ __forceinline__ u32 from_lead(u32 v) const { return __shfl_sync(mask, v, (threadIdx.x & 31) & 30); }
};

// Software pipelining across grid-stride iterations: a lane hashes the key it
// will handle `dist` iterations later and prefetches that op's primary tag
// block (64 B, exactly the block: cp.async.bulk.prefetch) into L2, so when the
// op comes up its tag load is an L2 hit instead of a DRAM round trip.  Pure
// cache hint -- the op still reads the block itself (under its lock for
// mutations), so correctness never depends on the prefetched copy.
// (a bulk prefetch per lane goes through the TMA unit and measured 28-38%
// slower: the LSU prefetch below is what a per-lane random block wants)
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" :: "l"(p) : "memory");
}
__device__ __forceinline__ void prefetch_tag_block(const Dev& d, const u64* __restrict__ keys, u64 i, u64 n) {
  if (i >= n) return;
  const u16* blk = d.tags + d.nbm(mix64(__ldg(keys + i) ^ d.seeds[0]) >> 16) * 32;
  prefetch_l2(blk);
}

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

template <bool RO, bool F64 = false>
__device__ __forceinline__ void pair_masks(const Dev& d, const Pair& p, u64 b, u16 tag, u32& M, u32& Z) {
  u32 w[8];
  const u16* blk = d.tags + b * 32 + p.half * 16;
  if (F64) { if (RO) ld_tags32_ro64(blk, w); else ld_tags32_64(blk, w); }
  else { if (RO) ld_tags32_ro(blk, w); else ld_tags32(blk, w); }
  const u32 pat = (u32)tag * 0x10001u;
  u32 m = 0, z = 0;
#pragma unroll
  for (int i = 0; i < 8; i++) {
    const u32 mm = __vcmpeq2(w[i], pat), zz = __vcmpeq2(w[i], 0u);
    m |= ((mm & 1u) | ((mm >> 15) & 2u)) << (2 * i);
    z |= ((zz & 1u) | ((zz >> 15) & 2u)) << (2 * i);
  }
  const u32 om = p.xchg(m), oz = p.xchg(z);
  M = p.half ? (om | (m << 16)) : (m | (om << 16));
  Z = p.half ? (oz | (z << 16)) : (z | (oz << 16));
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

template <bool RO, bool F64>
__global__ void __launch_bounds__(256) k_query_p2md_pair(Dev d, const u64* __restrict__ keys, u64 n, u64* vout,
                                                         u8* found, int conc_erase, int gated) {
  WS_PROLOGUE(d, gated, n);
  const Pair p;
  const u32 te0 = ld_u32_relaxed(d.state);
  const u64 stride = ((u64)gridDim.x * blockDim.x) >> 1;
  for (u64 i = (blockIdx.x * (u64)blockDim.x + threadIdx.x) >> 1; i < n; i += stride) {
    const u64 key = __ldg(keys + i);
    const u64 h0 = mix64(key ^ d.seeds[0]);
    const u64 b0 = d.nbm(h0 >> 16);
    const u16 t = (u16)(h0 & 0xFFFF);
    const u16 tag = t ? t : (u16)1;
    u32 M, Z;
    pair_masks<RO, F64>(d, p, b0, tag, M, Z);
    u64 val = 0;
    bool hit = M && pair_confirm<RO, F64>(d, b0, M, key, val) >= 0;
    if (!hit) {
      bool te = te0 != 0;
      if (conc_erase) { fence_acq_rel(); te = ld_u32_relaxed(d.state) != 0; }
      const int zc = __popc(Z);
      const int used0 = 32 - (zc < d.zcc ? zc : d.zcc);
      if (!(Z && !te && used0 < d.shortcut)) {  // no early exit (openaddr.py:440-442)
        const u64 b1 = d.nbm(mix64(key ^ d.seeds[1]) >> 16);
        if (b1 != b0) {
          pair_masks<RO, F64>(d, p, b1, tag, M, Z);
          hit = M && pair_confirm<RO, F64>(d, b1, M, key, val) >= 0;
        }
      }
    }
    if (p.half == 0) {
      if (found) found[i] = hit;
      if (vout) vout[i] = hit ? val : 0;
    }
  }
}

// P2-MD upsert (reference openaddr.py:370-418 plus the serialisable routing
// of Ctx::p2_upsert) for exclusive-mode tables (locks on, not lock-elided).
__device__ __forceinline__ void pair_lock(const Dev& d, const Pair& p, u64 b) {
  if (p.half == 0) lock_bucket(d.locks, b);
  __syncwarp(p.mask);
}
__device__ __forceinline__ void pair_unlock(const Dev& d, const Pair& p, u64 b) {
  __syncwarp(p.mask);
  if (p.half == 0) unlock_bucket(d.locks, b);
}
// extra bucket lock in ascending order; false when `held` had to be dropped
__device__ __forceinline__ bool pair_lock_extra(const Dev& d, const Pair& p, u64 b, u64 held) {
  u32 ok = 1;
  if (p.half == 0) {
    if (b > held) {
      lock_bucket(d.locks, b);
    } else if (!try_lock_bucket(d.locks, b)) {
      unlock_bucket(d.locks, held);
      lock_bucket(d.locks, b);
      lock_bucket(d.locks, held);
      ok = 0;
    }
  }
  return p.from_lead(ok) != 0;
}

static __global__ void __launch_bounds__(256) k_upsert_p2md_pair(Dev d, const u64* __restrict__ keys,
                                                          const u64* __restrict__ vals, u64 n, int merge,
                                                          u8* status, int conc_erase, int gated) {
  WS_PROLOGUE(d, gated, n);
  const Pair p;
  const bool lead = p.half == 0;
  const u32 te0 = ld_u32_relaxed(d.state);
  const u64 stride = ((u64)gridDim.x * blockDim.x) >> 1;
  for (u64 i = (blockIdx.x * (u64)blockDim.x + threadIdx.x) >> 1; i < n; i += stride) {
    const u64 key = __ldg(keys + i);
    const u64 val = __ldg(vals + i);
    const u64 h0 = mix64(key ^ d.seeds[0]);
    const u64 b0 = d.nbm(h0 >> 16);
    const u16 t = (u16)(h0 & 0xFFFF);
    const u16 tag = t ? t : (u16)1;
    bool have_b1 = false;
    u64 b1l = 0;
    u8 st;
    pair_lock(d, p, b0);
    for (;;) {
      u32 M0, Z0;
      pair_masks<false>(d, p, b0, tag, M0, Z0);
      u64 old;
      int j = M0 ? pair_confirm<false>(d, b0, M0, key, old) : -1;
      if (j >= 0) {
        if (lead) st_cell(d.cells + 2 * (b0 * 32 + j), key, apply_merge(merge, old, val));
        st = S_UPDATED;
        break;
      }
      bool te = te0 != 0;
      if (conc_erase) { fence_acq_rel(); te = ld_u32_relaxed(d.state) != 0; }
      const int zc0 = __popc(Z0);
      const int used0 = 32 - (zc0 < d.zcc ? zc0 : d.zcc);
      u64 target = b0;
      u32 Zt = Z0;
      if (te || used0 >= d.shortcut) {  // no shortcut: consult the alternate
        const u64 b1 = d.nbm(mix64(key ^ d.seeds[1]) >> 16);
        if (b1 != b0) {
          if (!have_b1) {
            have_b1 = true;
            b1l = b1;
            if (!pair_lock_extra(d, p, b1, b0)) continue;  // b0 was dropped: re-read it
          }
          u32 M1, Z1;
          pair_masks<false>(d, p, b1, tag, M1, Z1);
          j = M1 ? pair_confirm<false>(d, b1, M1, key, old) : -1;
          if (j >= 0) {
            if (lead) st_cell(d.cells + 2 * (b1 * 32 + j), key, apply_merge(merge, old, val));
            st = S_UPDATED;
            break;
          }
          const int zc1 = __popc(Z1);
          const int used1 = 32 - (zc1 < d.zcc ? zc1 : d.zcc);
          const bool prim = used0 <= used1;  // ties go to the primary
          target = prim ? b0 : b1;
          Zt = prim ? Z0 : Z1;
          if (!Zt) { target = prim ? b1 : b0; Zt = prim ? Z1 : Z0; }
        }
      }
      if (!Zt) { st = S_FULL; break; }
      const u64 slot = target * 32 + (__ffs(Zt) - 1);
      if (lead) {
        if (conc_erase) fence_acq_rel();
        st_cell(d.cells + 2 * slot, key, val);
        st_tag(d.tags + slot, tag);
      }
      st = S_INSERTED;
      break;
    }
    if (have_b1) pair_unlock(d, p, b1l);
    pair_unlock(d, p, b0);
    if (lead && status) status[i] = st;
  }
}

// =============================================== warp-synchronous rounds
//
// P2-MD upsert, one thread per op, in warp-synchronous lock rounds.  A
// release fence (MEMBAR.GPU) waits for every memory operation the warp has in
// flight; issued per lane at unlock time -- while warp-mates still have DRAM
// loads outstanding -- it was 35% of the one-thread kernel's stall samples.
// Here each round is:
//   1. every pending lane TRY-locks its primary (atom.acquire; never blocks),
//   2. lanes holding their lock read tags, decide, try-lock the alternate if
//      routing needs it (serialisable routing, see Ctx::lock_extra) and
//      publish (plain 128-bit store + tag store, exclusive bucket),
//   3. the warp reconverges and issues ONE fence.acq_rel, then every lane
//      releases its locks with relaxed reds (fence-based release),
//   4. lanes whose try-lock failed keep their op for the next round (after a
//      lane-staggered backoff, holding no lock -- no deadlock, and warp-mates
//      never wait on each other's locks).
template <bool F64>
__device__ __forceinline__ void tag_masks_t(const Dev& d, u64 b, u16 tag, u32& M, u32& Z) {
  u32 a[8], c[8];
  const u16* blk = d.tags + b * 32;
  if (F64) { ld_tags32_64(blk, a); ld_tags32_64(blk + 16, c); }
  else { ld_tags32(blk, a); ld_tags32(blk + 16, c); }
  masks_from(a, c, tag, M, Z);
}

__device__ __forceinline__ u32 atom_or_relaxed(u32* p, u32 m) {
  u32 old;
  asm volatile("atom.relaxed.gpu.global.or.b32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(m) : "memory");
  return old;
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

// fence_after_issue (warp-uniform): one fence.acq_rel between issuing the
// tag loads and consuming them -- the insert kernel's deferred lock release
// (k_upsert_p2md_rounds, DEFER) overlaps the previous round's store
// acknowledgements with this round's tag-load latency.
template <bool RO, bool F64>
__device__ __forceinline__ void coop_masks(const Dev& d, bool active, u64 b, u16 tag, u32& M, u32& Z,
                                           bool fence_after_issue = false) {
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
  if (fence_after_issue) fence_acq_rel();
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
                                                         u8* found, int conc_erase, int gated) {
  WS_PROLOGUE(d, gated, n);
  const u32 te0 = ld_u32_relaxed(d.state);
  const u64 stride = (u64)gridDim.x * blockDim.x;
  // the loop runs warp-uniformly: the bound is the warp's first index
  const u64 first = (blockIdx.x * (u64)blockDim.x + threadIdx.x) & ~31ull;
  const int pf = d.tune_pf;
  for (int k = 1; k < pf; k++) prefetch_tag_block(d, keys, first + k * stride + (threadIdx.x & 31), n);
  for (u64 base = first; base < n; base += stride) {
    const u64 i = base + (threadIdx.x & 31);
    if (pf) prefetch_tag_block(d, keys, i + pf * stride, n);
    const bool act = i < n;
    const u64 key = act ? __ldg(keys + i) : 0;
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
template <bool F64, int MINB, bool PHASED, bool FILL = false, bool DEFER = false>
__global__ void __launch_bounds__(256, MINB) k_upsert_p2md_rounds(Dev d, const u64* __restrict__ keys,
                                                            const u64* __restrict__ vals, u64 n, int merge,
                                                            u8* status, int conc_erase, int gated) {
  WS_PROLOGUE(d, gated, n);
  const u32 te0 = ld_u32_relaxed(d.state);
  const int lane = threadIdx.x & 31;
  const u64 nwarps = ((u64)gridDim.x * blockDim.x) >> 5;
  const u64 c0 = (blockIdx.x * (u64)blockDim.x + threadIdx.x) >> 5;
  const int pf = d.tune_pf;
  // DEFER: locks of ops finished in a warp's last round of a chunk are
  // released after the NEXT chunk's first tag loads are issued, behind the
  // one fence that also orders those loads -- the fence's wait for this
  // round's store acknowledgements overlaps the next op's DRAM latency
  // instead of stalling the warp on its own (ncu: membar was 31% of stalls)
  u64 rel0 = ~0ull, rel1 = ~0ull;
  for (int k = 1; k < pf; k++) prefetch_tag_block(d, keys, (c0 + k * nwarps) * 32 + lane, n);
  for (u64 c = c0; c * 32 < n; c += nwarps) {
    const u64 i = c * 32 + lane;
    if (pf) prefetch_tag_block(d, keys, (c + pf * nwarps) * 32 + lane, n);
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
      const bool dfence = DEFER && __any_sync(0xFFFFFFFFu, rel0 != ~0ull || rel1 != ~0ull);
      coop_masks<false, F64>(d, hold0, b0, tag, M0, Z0, dfence);
      if (DEFER && dfence) {  // the fence inside coop_masks ordered the deferred ops' stores
        if (rel1 != ~0ull) red_and_relaxed(d.locks + (rel1 >> 5), ~(1u << (rel1 & 31)));
        if (rel0 != ~0ull) red_and_relaxed(d.locks + (rel0 >> 5), ~(1u << (rel0 & 31)));
        rel0 = rel1 = ~0ull;
      }
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
        // DEFER: when the chunk is done (no lane retries -- a retrying lane's
        // backoff would stretch the hold), hand the releases to the next
        // chunk's fence instead of fencing here
        if (DEFER && !__any_sync(0xFFFFFFFFu, pending)) {
          if (held1) { rel1 = b1; held1 = false; }
          if (held0) { rel0 = b0; held0 = false; }
        } else {
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
      }
      if (pending) {
        __nanosleep(backoff + 8 * (threadIdx.x & 31));
        if (backoff < 4096) backoff <<= 1;
      }
    }
    if (status && i < n) status[i] = st;
  }
  if (DEFER && !PHASED && __any_sync(0xFFFFFFFFu, rel0 != ~0ull || rel1 != ~0ull)) {
    fence_acq_rel();
    if (rel1 != ~0ull) red_and_relaxed(d.locks + (rel1 >> 5), ~(1u << (rel1 & 31)));
    if (rel0 != ~0ull) red_and_relaxed(d.locks + (rel0 >> 5), ~(1u << (rel0 & 31)));
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

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
  if (gated && (ld_u32_relaxed(d.state + 2) | ld_u32_relaxed(d.state + 3))) return;
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

template <bool RO>
__device__ __forceinline__ void pair_masks(const Dev& d, const Pair& p, u64 b, u16 tag, u32& M, u32& Z) {
  u32 w[8];
  const u16* blk = d.tags + b * 32 + p.half * 16;
  if (RO) ld_tags32_ro(blk, w); else ld_tags32(blk, w);
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
template <bool RO>
__device__ __forceinline__ int pair_confirm(const Dev& d, u64 b, u32 M, u64 key, u64& val) {
  while (M) {
    const int j = __ffs(M) - 1;
    M &= M - 1;
    u64 k, v;
    load_cell<RO>(d.cells + 2 * (b * 32 + j), k, v);
    if (k == key) { val = v; return j; }
  }
  return -1;
}

template <bool RO>
__global__ void __launch_bounds__(256) k_query_p2md_pair(Dev d, const u64* __restrict__ keys, u64 n, u64* vout,
                                                         u8* found, int conc_erase, int gated) {
  if (gated && (ld_u32_relaxed(d.state + 2) | ld_u32_relaxed(d.state + 3))) return;
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
    pair_masks<RO>(d, p, b0, tag, M, Z);
    u64 val = 0;
    bool hit = M && pair_confirm<RO>(d, b0, M, key, val) >= 0;
    if (!hit) {
      bool te = te0 != 0;
      if (conc_erase) { fence_acq_rel(); te = ld_u32_relaxed(d.state) != 0; }
      const int zc = __popc(Z);
      const int used0 = 32 - (zc < d.zcc ? zc : d.zcc);
      if (!(Z && !te && used0 < d.shortcut)) {  // no early exit (openaddr.py:440-442)
        const u64 b1 = d.nbm(mix64(key ^ d.seeds[1]) >> 16);
        if (b1 != b0) {
          pair_masks<RO>(d, p, b1, tag, M, Z);
          hit = M && pair_confirm<RO>(d, b1, M, key, val) >= 0;
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

__global__ void __launch_bounds__(256) k_upsert_p2md_pair(Dev d, const u64* __restrict__ keys,
                                                          const u64* __restrict__ vals, u64 n, int merge,
                                                          u8* status, int conc_erase, int gated) {
  if (gated && (ld_u32_relaxed(d.state + 2) | ld_u32_relaxed(d.state + 3))) return;
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

}  // namespace ws

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

}  // namespace ws

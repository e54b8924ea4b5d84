// ws_scan32.cuh -- line-at-a-time scan of a 32-cell (512-byte) bucket for the
// designs without fingerprint metadata (p2, iceberg): the bucket is fetched
// as two halves of eight 32-byte loads issued together (2 round trips instead
// of the generic four 8-cell chunks), then scanned with the semantics of
// reference sync.py:184-207 (probe_range): stop at the key or at the first
// EMPTY; `used` counts claimed cells passed, `hint` the first reusable cell.
#pragma once
#include "ws_ops.cuh"

namespace ws {

template <bool RO>
__device__ __forceinline__ void scan32_lines(const u64* cells, u64 lo, u64 key, i64& idx, u64& val, int& used,
                                             i64& hint, bool& saw_empty) {
  idx = -1;
  used = 0;
  hint = -1;
  saw_empty = false;
#pragma unroll
  for (int half = 0; half < 2; half++) {
    u64 w[32];
    const u64* p = cells + 2 * (lo + 16 * half);
#pragma unroll
    for (int q = 0; q < 8; q++) {
      if (RO)
        asm volatile("ld.global.nc.L1::no_allocate.v4.u64 {%0,%1,%2,%3}, [%4];"
                     : "=l"(w[4 * q]), "=l"(w[4 * q + 1]), "=l"(w[4 * q + 2]), "=l"(w[4 * q + 3])
                     : "l"(p + 4 * q));
      else
        asm volatile("ld.relaxed.gpu.global.v4.u64 {%0,%1,%2,%3}, [%4];"
                     : "=l"(w[4 * q]), "=l"(w[4 * q + 1]), "=l"(w[4 * q + 2]), "=l"(w[4 * q + 3])
                     : "l"(p + 4 * q) : "memory");
    }
    bool stop = false;
#pragma unroll
    for (int j = 0; j < 16; j++) {
      const u64 k = w[2 * j];
      const i64 slot = (i64)(lo + 16 * half + j);
      if (!stop) {
        if (k == key) { idx = slot; val = w[2 * j + 1]; stop = true; }
        else if (k == EMPTY) { if (hint < 0) hint = slot; saw_empty = true; stop = true; }
        else if (k == TOMB) { if (hint < 0) hint = slot; }
        else used++;
      }
    }
    if (stop) return;
  }
}

// Variant for mutations (reference _find_in_bucket plus _used_and_free,
// openaddr.py:59-130), the same results as scan32_lines: claims always take a
// bucket's first EMPTY/TOMB cell and erasures leave TOMB, so nothing is ever
// claimed past the first EMPTY and the claimed count of the whole bucket is
// the count before it.  The chunks are NOT unrolled: one chunk of registers
// stays live (122 instead of 171 registers in the iceberg upsert, 2 CTAs per
// SM instead of 1), at no extra round trip.
template <bool RO, int CH = 16>
__device__ __forceinline__ void scan32_all(const u64* cells, u64 lo, u64 key, i64& idx, u64& val, int& used,
                                           i64& hint, bool& saw_empty) {
  idx = -1;
  used = 0;
  hint = -1;
  saw_empty = false;
#pragma unroll 1
  for (int part = 0; part < 32 / CH; part++) {
    u64 w[2 * CH];
    const u64* p = cells + 2 * (lo + CH * part);
#pragma unroll
    for (int q = 0; q < CH / 2; q++) {
      if (RO)
        asm volatile("ld.global.nc.L1::no_allocate.v4.u64 {%0,%1,%2,%3}, [%4];"
                     : "=l"(w[4 * q]), "=l"(w[4 * q + 1]), "=l"(w[4 * q + 2]), "=l"(w[4 * q + 3])
                     : "l"(p + 4 * q));
      else
        asm volatile("ld.relaxed.gpu.global.v4.u64 {%0,%1,%2,%3}, [%4];"
                     : "=l"(w[4 * q]), "=l"(w[4 * q + 1]), "=l"(w[4 * q + 2]), "=l"(w[4 * q + 3])
                     : "l"(p + 4 * q) : "memory");
    }
#pragma unroll
    for (int j = 0; j < CH; j++) {
      const u64 k = w[2 * j];
      const i64 slot = (i64)(lo + CH * part + j);
      if (k == key) { idx = slot; val = w[2 * j + 1]; }
      if (k == EMPTY || k == TOMB) { if (hint < 0) hint = slot; }
      else used++;
      saw_empty |= k == EMPTY;
    }
    if (idx >= 0 || saw_empty) return;  // nothing is ever claimed past an EMPTY
  }
}

}  // namespace ws

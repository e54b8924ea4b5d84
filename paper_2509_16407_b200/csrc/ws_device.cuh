// ws_device.cuh -- sm_100a device primitives for the WarpSpeed table kernels.
//
// Memory-model choices (the device form of reference sync.py:1-26):
//  * A slot is one 16-byte cell (key u64, value u64).  Every read of a cell
//    is a single 128-bit access (LDG.E.128.STRONG.GPU, `ld.relaxed.gpu.b128`)
//    and every publication a single 128-bit CAS or store, so a reader can
//    never see a torn pair; the reference's RESERVED intermediate state
//    (sync.py:144-169) collapses into one `atom.cas.b128` EMPTY/TOMB -> (k,v).
//  * Tags (u16 per slot) and cells of tables that are being mutated are read
//    with `.relaxed.gpu` loads, which are served by L2 (the coherence point),
//    never by a stale L1 line.  Query-only launches read through the
//    non-coherent path with L1::no_allocate (the table is immutable for the
//    kernel's lifetime; L1 is invalidated at every launch boundary).
//  * Bucket locks are 1 bit per bucket in a u32 array (reference
//    sync.py:54-119): acquire = `atom.acquire.gpu.or`, release =
//    `red.release.gpu.and`.  At 2^25 buckets the array is 4 MiB and stays
//    resident in the 126 MB L2.
#pragma once
#include <cstdint>

namespace ws {

typedef unsigned long long u64;
typedef long long i64;
typedef uint32_t u32;
typedef uint16_t u16;
typedef uint8_t u8;

constexpr u64 EMPTY = 0ull;
constexpr u64 TOMB = ~0ull;
constexpr u64 RESV = ~0ull - 1ull;
constexpr u64 TAG_BASE = 1ull << 44;   // reference tables/base.py:38
constexpr u64 LOCK_BASE = 1ull << 45;  // reference tables/base.py:39

__device__ __forceinline__ bool is_sentinel(u64 k) { return k == EMPTY || k >= RESV; }
__device__ __forceinline__ bool free_key(u64 k) { return k == EMPTY || k == TOMB; }

// splitmix64 finaliser, reference core.py:120-129
__host__ __device__ __forceinline__ u64 mix64(u64 x) {
  x ^= x >> 30;
  x *= 0xBF58476D1CE4E5B9ull;
  x ^= x >> 27;
  x *= 0x94D049BB133111EBull;
  x ^= x >> 31;
  return x;
}

// x % d with a mask fast path for power-of-two d.
struct Mod {
  u64 d, mask;  // mask = d-1 when d is a power of two, else 0
  __device__ __forceinline__ u64 operator()(u64 x) const { return mask ? (x & mask) : (x % d); }
};

// ----------------------------------------------------------------- cells

__device__ __forceinline__ void ld_cell(const u64* p, u64& k, u64& v) {
  asm volatile("{.reg .b128 t; ld.relaxed.gpu.global.b128 t, [%2]; mov.b128 {%0, %1}, t;}"
               : "=l"(k), "=l"(v) : "l"(p) : "memory");
}
__device__ __forceinline__ void ld_cell_ro(const u64* p, u64& k, u64& v) {
  asm volatile("ld.global.nc.L1::no_allocate.v2.u64 {%0, %1}, [%2];"
               : "=l"(k), "=l"(v) : "l"(p));
}
template <bool RO>
__device__ __forceinline__ void load_cell(const u64* p, u64& k, u64& v) {
  if (RO) ld_cell_ro(p, k, v); else ld_cell(p, k, v);
}
__device__ __forceinline__ void st_cell(u64* p, u64 k, u64 v) {
  asm volatile("{.reg .b128 t; mov.b128 t, {%1, %2}; st.relaxed.gpu.global.b128 [%0], t;}"
               :: "l"(p), "l"(k), "l"(v) : "memory");
}
__device__ __forceinline__ void st_cell_release(u64* p, u64 k, u64 v) {
  asm volatile("{.reg .b128 t; mov.b128 t, {%1, %2}; st.release.gpu.global.b128 [%0], t;}"
               :: "l"(p), "l"(k), "l"(v) : "memory");
}
// 128-bit compare-and-swap; returns the previous cell in (ok, ov).
__device__ __forceinline__ bool cas_cell(u64* p, u64 ek, u64 ev, u64 nk, u64 nv, u64& ok, u64& ov) {
  asm volatile(
      "{.reg .b128 e, n, o; mov.b128 e, {%2, %3}; mov.b128 n, {%4, %5};"
      " atom.relaxed.gpu.global.cas.b128 o, [%6], e, n; mov.b128 {%0, %1}, o;}"
      : "=l"(ok), "=l"(ov) : "l"(ek), "l"(ev), "l"(nk), "l"(nv), "l"(p) : "memory");
  return ok == ek && ov == ev;
}
// Publish (k, v) into a reusable cell (EMPTY or TOMBSTONE); false if taken.
__device__ __forceinline__ bool publish_cell(u64* p, u64 k, u64 v) {
  u64 ok, ov;
  if (cas_cell(p, EMPTY, 0, k, v, ok, ov)) return true;
  if (ok == TOMB && ov == 0) return cas_cell(p, TOMB, 0, k, v, ok, ov);
  return false;
}

__device__ __forceinline__ u64 ld_u64_acquire(const u64* p) {
  u64 r;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(r) : "l"(p) : "memory");
  return r;
}
__device__ __forceinline__ void st_u64_release(u64* p, u64 v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ u32 ld_u32_relaxed(const u32* p) {
  u32 r;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(r) : "l"(p) : "memory");
  return r;
}
__device__ __forceinline__ void st_u32_relaxed(u32* p, u32 v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_acq_rel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

// ------------------------------------------------------------------ tags

__device__ __forceinline__ u16 ld_tag(const u16* p) {
  u16 r;
  asm volatile("ld.relaxed.gpu.global.u16 %0, [%1];" : "=h"(r) : "l"(p) : "memory");
  return r;
}
__device__ __forceinline__ u16 ld_tag_ro(const u16* p) {
  u16 r;
  asm volatile("ld.global.nc.L1::no_allocate.u16 %0, [%1];" : "=h"(r) : "l"(p));
  return r;
}
__device__ __forceinline__ void st_tag(u16* p, u16 t) {
  asm volatile("st.relaxed.gpu.global.u16 [%0], %1;" :: "l"(p), "h"(t) : "memory");
}

// 32 bytes (16 tags) in one LDG.E.ENL2.256.
__device__ __forceinline__ void ld_tags32(const u16* p, u32 (&w)[8]) {
  asm volatile("ld.relaxed.gpu.global.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]),
                 "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7])
               : "l"(p) : "memory");
}
__device__ __forceinline__ void ld_tags32_ro(const u16* p, u32 (&w)[8]) {
  asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]),
                 "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7])
               : "l"(p));
}

// Per-slot bit masks of a 32-slot tag block: which tags equal `tag`, which are 0.
template <bool RO>
__device__ __forceinline__ void tag_masks32(const u16* blk, u16 tag, u32& match, u32& zero) {
  u32 a[8], b[8];
  if (RO) { ld_tags32_ro(blk, a); ld_tags32_ro(blk + 16, b); }
  else { ld_tags32(blk, a); ld_tags32(blk + 16, b); }
  const u32 pat = (u32)tag * 0x10001u;
  match = 0; zero = 0;
#pragma unroll
  for (int i = 0; i < 8; i++) {
    u32 m = __vcmpeq2(a[i], pat), z = __vcmpeq2(a[i], 0u);
    match |= ((m & 1u) | ((m >> 15) & 2u)) << (2 * i);
    zero |= ((z & 1u) | ((z >> 15) & 2u)) << (2 * i);
    m = __vcmpeq2(b[i], pat); z = __vcmpeq2(b[i], 0u);
    match |= ((m & 1u) | ((m >> 15) & 2u)) << (2 * i + 16);
    zero |= ((z & 1u) | ((z >> 15) & 2u)) << (2 * i + 16);
  }
}

// ----------------------------------------------------------------- locks

__device__ __forceinline__ u32 atom_or_acquire(u32* p, u32 m) {
  u32 old;
  asm volatile("atom.acquire.gpu.global.or.b32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(m) : "memory");
  return old;
}
__device__ __forceinline__ void red_and_release(u32* p, u32 m) {
  asm volatile("red.release.gpu.global.and.b32 [%0], %1;" :: "l"(p), "r"(m) : "memory");
}
__device__ __forceinline__ void lock_bucket(u32* locks, u64 b) {
  u32* w = locks + (b >> 5);
  const u32 bit = 1u << (b & 31);
  unsigned ns = 16;
  while (atom_or_acquire(w, bit) & bit) {
    __nanosleep(ns);
    if (ns < 256) ns <<= 1;  // short cap: hot keys hand the lock over quickly
  }
}
__device__ __forceinline__ void unlock_bucket(u32* locks, u64 b) {
  red_and_release(locks + (b >> 5), ~(1u << (b & 31)));
}
__device__ __forceinline__ bool try_lock_bucket(u32* locks, u64 b) {
  const u32 bit = 1u << (b & 31);
  return !(atom_or_acquire(locks + (b >> 5), bit) & bit);
}

// ------------------------------------------------------ probe accounting
// Distinct line-sized regions touched by one op, in the reference's idealised
// address image (instrument.py:26-85, tables/base.py:38-39).

constexpr int PROBE_CAP = 192;

struct Probe {
  u64 line[PROBE_CAP];
  u32 n, extra, locks;
  u32 lb;
  __device__ void reset(u32 line_bytes) { n = 0; extra = 0; locks = 0; lb = line_bytes; }
  __device__ void add_line(u64 l) {
    for (u32 i = 0; i < n; i++)
      if (line[i] == l) return;
    if (n < PROBE_CAP) line[n++] = l; else extra++;
  }
  __device__ void touch(u64 off) { add_line(off / lb); }
  __device__ void touch_range(u64 off, u64 nbytes) {
    for (u64 l = off / lb; l <= (off + nbytes - 1) / lb; l++) add_line(l);
  }
  __device__ u32 count() const { return n + extra; }
};

}  // namespace ws

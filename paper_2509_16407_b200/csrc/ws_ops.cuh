// ws_ops.cuh -- per-design upsert / query / erase on the device.
//
// One thread owns one operation (a "tile" of 1 lane).  Each function cites the
// reference routine it restates (paths under /root/reference/pkg/src/warpbench).
// Sequential behaviour (a batch of one op) is identical to the reference: the
// same bucket routing, shortcut / least-loaded decisions, first-reusable-slot
// claims and probe accounting, so a replay of a reference op stream through
// the device reproduces the reference's slot layout exactly.
//
// Concurrency (a batch of many ops in one launch): inserts and erases hold the
// key's primary-bucket lock, writes into foreign buckets (P2 alternate,
// iceberg backyard, double-hash path) only CAS reusable cells, queries are
// lock-free (cuckoo: ordered locks on all of the key's buckets, as the
// reference).  See ws_device.cuh for the memory-model details.
#pragma once
#include "ws_device.cuh"

namespace ws {

enum Design { D_DOUBLE = 0, D_DOUBLE_MD, D_P2, D_P2_MD, D_ICEBERG, D_ICEBERG_MD, D_CUCKOO,
              D_CHAINING, D_UNSAFE };
enum Merge { M_REPLACE = 0, M_KEEP, M_ADD, M_MAX, M_MIN };
enum Status { S_INSERTED = 0, S_UPDATED = 1, S_FULL = 2, S_RETRY = 3 };
enum OpKind { OP_UPSERT = 0, OP_ERASE = 1, OP_QUERY = 2 };

constexpr int CUCKOO_RETRIES = 16;  // reference cuckoo.py:26
constexpr int BFS_BUDGET = 4096;    // reference cuckoo.py:29

struct Dev {
  u64* cells;        // 2 words per slot, or the chaining node arena
  u16* tags;         // md designs
  u32* locks;        // 1 bit per bucket
  u32* state;        // [0] tombstones_ever (table-wide, persistent)
  // per-call state (each API call gets its own 4 words, so concurrent calls on
  // one table never see each other's verdicts): [0] invalid keys  [1] invalid
  // op bytes  [2] chain pool exhausted  [3] erase count of a mixed batch
  u32* cs;
  // per-call device-resident batch size (multi-GPU exchange: the owner's
  // inbox count is known only on the device); nullptr = the launch's n
  const u64* dn;
  u64* chain_next;   // chaining bump allocator
  u64 chain_cap;     // physical node capacity of the arena
  u64* bfs_mem;      // cuckoo BFS workspaces
  u32* bfs_busy;
  u64 bfs_entries, bfs_seen_cap, bfs_stride;  // per-workspace sizes (entries / words)
  u32 n_bfs;
  u64 cap, nb, front, back;
  Mod nbm, frontm, backm;
  u64 seeds[8];
  int design, bs, md, shortcut, zcc, probe_cap, ways, depth, phased, lock_elided, line_bytes, wpn;
  int tune_qilp;   // > 0: the per-design tuned query kernels, 0: the generic kernel
  int tune_l2pol;  // 2: 64-byte L2 fills for tag blocks and cells (default)
  int tune_upsert; // 4: the per-design tuned upsert kernels (default), 0: generic; P2-MD 2/3 = rounds
                   // without 64-byte fills / whole-sector writes; cuckoo 6 = serial eviction launch
  // cuckoo: this launch continues ops whose first attempt (the locked scan
  // that found every bucket full) already ran in k_upsert_cuckoo_rounds, so
  // ck_upsert starts at the eviction search (launch-local, never stored)
  int ck_resume;
  // delay injection at the reference's scheduling-hook stages
  // (tables/base.py:66-69, bench/adversarial.py:40-93): with probability
  // delay_p16/65536 a stage sleeps up to delay_ns; 0 = off (generic kernels)
  u32 delay_ns, delay_p16;
  u64 delay_seed;
};

// Kernel prologue of every batch kernel: a batch whose validation failed
// (this call's cs words) does nothing; a device-resident batch size clamps n.
#define WS_PROLOGUE(d, gated, n)                                                    \
  do {                                                                              \
    if ((gated) && (ld_u32_relaxed((d).cs) | ld_u32_relaxed((d).cs + 1))) return;   \
    if ((d).dn) { const u64 dn_ = *(const volatile u64*)(d).dn; if (dn_ < (n)) (n) = dn_; } \
  } while (0)

__device__ __forceinline__ u64 apply_merge(int m, u64 old, u64 nv) {
  switch (m) {
    case M_KEEP: return old;
    case M_ADD: return old + nv;  // mod 2^64, reference openaddr.py:200
    case M_MAX: return old > nv ? old : nv;
    case M_MIN: return old < nv ? old : nv;
    default: return nv;
  }
}

struct Find {
  i64 idx;
  u64 val;
  int used;
  i64 hint;
  bool saw_empty;
};

struct OpOut {
  u8 status;
  u64 val;
};

// DES: design (compile time).  BS_T: compile-time bucket size (0 = runtime
// d.bs).  RO: launch contains no mutation.  INSTR: record probe lines.
template <int DES, int BS_T, bool RO, bool INSTR>
struct Ctx {
  static constexpr bool MD = DES == D_DOUBLE_MD || DES == D_P2_MD || DES == D_ICEBERG_MD;
  const Dev& d;
  Probe* pr;
  bool conc_erase;  // erases may run concurrently in this launch
  u32 te0;          // tombstones_ever as seen at launch (valid when !conc_erase)

  __device__ __forceinline__ int B() const { return BS_T ? BS_T : d.bs; }
  __device__ __forceinline__ u64* cell(u64 i) const { return d.cells + 2 * i; }
  __device__ __forceinline__ void touch(u64 off) { if (INSTR) pr->touch(off); }
  __device__ __forceinline__ void touch_range(u64 off, u64 n) { if (INSTR) pr->touch_range(off, n); }
  __device__ __forceinline__ void touch_lock(u64 b) {
    if (INSTR && !d.phased) { pr->locks++; pr->touch(LOCK_BASE + (b >> 3)); }
  }
  __device__ __forceinline__ bool tomb_ever() {
    if (!conc_erase) return te0 != 0;
    fence_acq_rel();  // pairs with the fence in tombstone(): tag/cell reads above happen-before
    return ld_u32_relaxed(d.state) != 0;
  }
  __device__ __forceinline__ void lock(u64 b) {
    touch_lock(b);
    if (!d.phased) lock_bucket(d.locks, b);
  }
  __device__ __forceinline__ void unlock(u64 b) {
    if (!d.phased) unlock_bucket(d.locks, b);
  }
  // Lock a bucket an insert routes INTO besides its primary.  Not part of the
  // reference's discipline (openaddr.py:8-10 lets foreign writers rely on the
  // slot CAS alone): with ~10^5 inserts in flight, unsynchronised
  // least-loaded decisions read stale occupancy and overfill buckets, so a
  // concurrent fill could report FULL where every sequential order succeeds.
  // Holding the lock of every bucket whose occupancy drives a routing decision
  // makes inserts serialisable.  Not counted as a probe (the reference's
  // idealised accounting has no such lock).  Returns false when it had to
  // drop `held` to respect ascending lock order -- the caller must re-read.
  __device__ __forceinline__ bool lock_extra(u64 b, u64 held) {
    if (d.phased) return true;
    if (b > held) { lock_bucket(d.locks, b); return true; }
    if (try_lock_bucket(d.locks, b)) return true;
    unlock_bucket(d.locks, held);
    lock_bucket(d.locks, b);
    lock_bucket(d.locks, held);
    return false;
  }
  __device__ __forceinline__ void ldc(u64 i, u64& k, u64& v) { load_cell<RO>(cell(i), k, v); }
  enum Stage { PRE_RESERVE = 1, PRE_PUBLISH = 2, PRE_TOMBSTONE = 3, PRE_SCAN = 4 };
  __device__ __forceinline__ void hook(int stage, u64 key) {
    if (RO || INSTR || !d.delay_ns) return;
    const u64 r = mix64(d.delay_seed ^ (key * 0x9E3779B97F4A7C15ull) ^ ((u64)stage << 56) ^
                        ((u64)(blockIdx.x * blockDim.x + threadIdx.x) << 20) ^ clock64());
    if ((u32)(r & 0xFFFF) < d.delay_p16) __nanosleep((u32)((r >> 32) % d.delay_ns));
  }
  __device__ __forceinline__ u16 ldt(u64 i) { return RO ? ld_tag_ro(d.tags + i) : ld_tag(d.tags + i); }
  __device__ __forceinline__ u64 hb(int i, u64 key, const Mod& m) const {
    return m(mix64(key ^ d.seeds[i]) >> 16);
  }
  __device__ __forceinline__ u16 md_tag(u64 h0) const {
    if constexpr (!MD) return 0;
    u16 t = (u16)(h0 & 0xFFFF);
    return t ? t : (u16)1;
  }

  // ---------------------------------------------------------------- scans

  // reference sync.py:184-207 (probe_range): cells [lo, lo+n), stopping at
  // the first EMPTY.  Cells are fetched a line (8 cells) at a time.
  __device__ Find scan_cells(u64 lo, int n, u64 key) {
    Find r{-1, 0, 0, -1, false};
    for (int base = 0; base < n; base += 8) {
      const int cnt = n - base < 8 ? n - base : 8;
      u64 k[8], v[8];
#pragma unroll
      for (int j = 0; j < 8; j++)
        if (j < cnt) ldc(lo + base + j, k[j], v[j]);
#pragma unroll
      for (int j = 0; j < 8; j++) {
        if (j >= cnt) break;
        const u64 i = lo + base + j;
        touch(16 * i);
        if (k[j] == key) { r.idx = (i64)i; r.val = v[j]; r.used = -1; return r; }
        if (k[j] == EMPTY) {
          if (r.hint < 0) r.hint = (i64)i;
          r.saw_empty = true;
          return r;
        }
        if (k[j] == TOMB) { if (r.hint < 0) r.hint = (i64)i; } else { r.used++; }
      }
    }
    return r;
  }

  // first EMPTY/TOMB cell of [lo, lo+n) or -1 (reference sync.py:230-239)
  __device__ i64 find_free(u64 lo, int n) {
    for (int base = 0; base < n; base += 8) {
      const int cnt = n - base < 8 ? n - base : 8;
      u64 k[8], v[8];
#pragma unroll
      for (int j = 0; j < 8; j++)
        if (j < cnt) ldc(lo + base + j, k[j], v[j]);
#pragma unroll
      for (int j = 0; j < 8; j++)
        if (j < cnt && free_key(k[j])) return (i64)(lo + base + j);
    }
    return -1;
  }

  __device__ int used_cells(u64 lo, int n) {
    int u = 0;
    for (int base = 0; base < n; base += 8) {
      const int cnt = n - base < 8 ? n - base : 8;
      u64 k[8], v[8];
#pragma unroll
      for (int j = 0; j < 8; j++)
        if (j < cnt) ldc(lo + base + j, k[j], v[j]);
#pragma unroll
      for (int j = 0; j < 8; j++)
        if (j < cnt && !free_key(k[j])) u++;
    }
    return u;
  }

  // md helpers over live tags (generic bucket size)
  __device__ i64 md_next_zero(u64 from, u64 hi) {
    for (u64 j = from; j < hi; j++)
      if (ldt(j) == 0) return (i64)j;
    return -1;
  }
  __device__ int md_count_zeros(u64 lo, u64 hi, int cap) {
    int z = 0;
    for (u64 j = lo; j < hi; j++)
      if (ldt(j) == 0 && ++z >= cap) return z;
    return z;
  }

  // reference openaddr.py:59-116 (_find_in_bucket)
  __device__ Find find(u64 b, u64 key, u16 tag, bool classify) {
    const int n = B();
    const u64 lo = b * (u64)n;
    if constexpr (!MD) return scan_cells(lo, n, key);
    Find r{-1, 0, 0, -1, false};
    touch_range(TAG_BASE + 2 * lo, 2 * (u64)n);
    if constexpr (BS_T == 32) {
      u32 M, Z;
      tag_masks32<RO>(d.tags + lo, tag, M, Z);
      while (M) {
        const int j = __ffs(M) - 1;
        M &= M - 1;
        u64 k, v;
        ldc(lo + j, k, v);
        touch(16 * (lo + j));
        if (k == key) { r.idx = (i64)(lo + j); r.val = v; r.used = -1; return r; }
      }
      if (!Z) { r.used = 32; return r; }
      const int zc = __popc(Z);
      r.used = 32 - (zc < d.zcc ? zc : d.zcc);
      r.hint = (i64)(lo + __ffs(Z) - 1);
      if (!tomb_ever()) { r.saw_empty = true; return r; }
      if (classify) {
        while (Z) {
          const int j = __ffs(Z) - 1;
          Z &= Z - 1;
          u64 k, v;
          ldc(lo + j, k, v);
          touch(16 * (lo + j));
          if (k == EMPTY) { r.saw_empty = true; return r; }
        }
      }
      return r;
    }
    const u64 hi = lo + n;
    for (u64 j = lo; j < hi; j++) {
      if (ldt(j) != tag) continue;
      u64 k, v;
      ldc(j, k, v);
      touch(16 * j);
      if (k == key) { r.idx = (i64)j; r.val = v; r.used = -1; return r; }
    }
    const i64 fz = md_next_zero(lo, hi);
    if (fz < 0) { r.used = n; return r; }
    r.used = n - md_count_zeros(lo, hi, d.zcc);
    r.hint = fz;
    if (!tomb_ever()) { r.saw_empty = true; return r; }
    if (classify) {
      for (i64 z = fz; z >= 0; z = md_next_zero((u64)z + 1, hi)) {
        u64 k, v;
        ldc((u64)z, k, v);
        touch(16 * (u64)z);
        if (k == EMPTY) { r.saw_empty = true; return r; }
      }
    }
    return r;
  }

  // reference openaddr.py:118-130 (_used_and_free)
  __device__ void used_and_free(u64 b, int& used, bool& has_free) {
    const int n = B();
    const u64 lo = b * (u64)n;
    if constexpr (MD) {
      touch_range(TAG_BASE + 2 * lo, 2 * (u64)n);
      int z;
      if constexpr (BS_T == 32) {
        u32 M, Z;
        tag_masks32<RO>(d.tags + lo, 0xFFFF, M, Z);
        z = __popc(Z);
        if (z > d.zcc) z = d.zcc;
      } else {
        z = md_count_zeros(lo, lo + n, d.zcc);
      }
      used = n - z;
      has_free = z > 0;
      return;
    }
    touch_range(16 * lo, 16 * (u64)n);
    used = used_cells(lo, n);
    has_free = used < n;
  }

  // reference openaddr.py:132-185: claim the first reusable slot of bucket b
  // (hint first) and publish (key, val); the md tag is written right after
  // the 128-bit publication.  Returns the slot or -1 when the bucket is full.
  //
  // Exclusive buckets: in P2 / iceberg / cuckoo every writer into a bucket's
  // free slots holds that bucket's lock (see lock_extra), so a free slot seen
  // under the lock cannot be taken concurrently and the 128-bit publication
  // is a plain store -- no CAS, hence no DRAM read of the slot's sector.
  static constexpr bool EXCL_DES = DES == D_P2 || DES == D_P2_MD || DES == D_ICEBERG ||
                                   DES == D_ICEBERG_MD || DES == D_CUCKOO;
  __device__ __forceinline__ bool exclusive() const { return EXCL_DES && !d.phased && !d.lock_elided; }

  __device__ i64 claim_publish(u64 b, i64 hint, u64 key, u64 val, u16 tag) {
    const int n = B();
    const u64 lo = b * (u64)n, hi = lo + n;
    if (exclusive()) {
      if constexpr (!MD) {
        if (hint < 0) hint = find_free(lo, n);
        if (hint < 0) return -1;
        hook(PRE_PUBLISH, key);
        st_cell(cell((u64)hint), key, val);
        touch(16 * (u64)hint);
        return hint;
      } else {
        const i64 z = hint >= 0 ? hint : md_first_zero(lo, hi, lo);
        if (z < 0) return -1;
        touch(16 * (u64)z);
        // a zero tag may be a slot an eraser just tombstoned: order its
        // tombstone store (released by the eraser's fence) before ours
        hook(PRE_PUBLISH, key);
        if (conc_erase) fence_acq_rel();
        st_cell(cell((u64)z), key, val);
        st_tag(d.tags + z, tag);
        touch(TAG_BASE + 2 * (u64)z);
        return z;
      }
    }
    if constexpr (!MD) {
      for (;;) {
        if (hint < 0) hint = find_free(lo, n);
        if (hint < 0) return -1;
        touch(16 * (u64)hint);
        hook(PRE_RESERVE, key);
        if (publish_cell(cell((u64)hint), key, val)) break;
        hint = -1;
      }
      touch(16 * (u64)hint);
      return hint;
    }
    i64 z = hint >= 0 ? hint : md_first_zero(lo, hi, lo);
    for (;;) {
      if (z < 0) {
        z = md_first_zero(lo, hi, lo);
        if (z < 0) return -1;
      }
      touch(16 * (u64)z);
      hook(PRE_RESERVE, key);
      if (publish_cell(cell((u64)z), key, val)) break;
      z = md_first_zero(lo, hi, (u64)z + 1);
    }
    st_tag(d.tags + z, tag);
    touch(TAG_BASE + 2 * (u64)z);
    return z;
  }
  __device__ i64 md_first_zero(u64 lo, u64 hi, u64 from) {
    if constexpr (BS_T == 32) {
      u32 M, Z;
      tag_masks32<false>(d.tags + lo, 0xFFFF, M, Z);
      const u32 off = (u32)(from - lo);
      if (off >= 32) return -1;
      Z &= ~0u << off;
      return Z ? (i64)(lo + __ffs(Z) - 1) : -1;
    }
    return md_next_zero(from, hi);
  }

  // reference openaddr.py:187-197: flag, tombstone, then clear the tag
  __device__ void tombstone(u64 idx) {
    hook(PRE_TOMBSTONE, idx);
    if (ld_u32_relaxed(d.state) == 0) st_u32_relaxed(d.state, 1u);
    fence_acq_rel();
    st_cell(cell(idx), TOMB, 0);
    touch(16 * idx);
    if constexpr (MD) {
      fence_acq_rel();  // the tombstone is visible before the zero tag that advertises it
      st_tag(d.tags + idx, 0);
      touch(TAG_BASE + 2 * idx);
    }
  }

  // reference openaddr.py:199-204 (caller holds the key's primary lock)
  __device__ u8 update(i64 idx, u64 key, u64 old, u64 val, int merge) {
    st_cell(cell((u64)idx), key, apply_merge(merge, old, val));
    touch(16 * (u64)idx);
    return S_UPDATED;
  }

  // ======================================================= double hashing
  // reference openaddr.py:207-318

  __device__ u64 dbl_len() const { return (u64)d.probe_cap < d.nb ? (u64)d.probe_cap : d.nb; }
  __device__ u64 dbl_next(u64 b, u64 sm) const { const u64 x = b + sm; return x >= d.nb ? x - d.nb : x; }

  __device__ u8 dbl_upsert(u64 key, u64 val, int merge) {
    const u64 b0 = hb(0, key, d.nbm);
    lock(b0);
    const u8 st = dbl_upsert_held(key, val, merge);
    unlock(b0);
    return st;
  }
  // the body of dbl_upsert with the primary-bucket lock already held (also
  // run by the lock-round kernel of ws_d_double_md.cu)
  __device__ u8 dbl_upsert_held(u64 key, u64 val, int merge) {
    const u64 h0 = mix64(key ^ d.seeds[0]);
    const u64 b0 = d.nbm(h0 >> 16);
    const u16 tag = md_tag(h0);
    const u64 sm = (mix64(key ^ d.seeds[1]) | 1ull) % d.nb;  // (b+step)%nb without 2^64 wrap
    const u64 len = dbl_len();
    u8 st;
    for (;;) {
      i64 fb = -1, fh = -1;
      u64 b = b0;
      bool done = false;
      for (u64 i = 0; i < len; i++) {
        Find r = find(b, key, tag, true);
        if (r.idx >= 0) { st = update(r.idx, key, r.val, val, merge); done = true; break; }
        if (fb < 0 && r.hint >= 0) { fb = (i64)b; fh = r.hint; }
        if (r.saw_empty) break;
        b = dbl_next(b, sm);
      }
      if (done) break;
      if (fb < 0) { st = S_FULL; break; }
      if (claim_publish((u64)fb, fh, key, val, tag) >= 0) { st = S_INSERTED; break; }
    }
    return st;
  }

  __device__ i64 dbl_find(u64 key, u64& val) {
    const u64 h0 = mix64(key ^ d.seeds[0]);
    u64 b = d.nbm(h0 >> 16);
    const u16 tag = md_tag(h0);
    const u64 sm = (mix64(key ^ d.seeds[1]) | 1ull) % d.nb;
    const u64 len = dbl_len();
    for (u64 i = 0; i < len; i++) {
      Find r = find(b, key, tag, true);
      if (r.idx >= 0) { val = r.val; return r.idx; }
      if (r.saw_empty) return -1;
      b = dbl_next(b, sm);
    }
    return -1;
  }

  __device__ bool dbl_erase(u64 key) {
    const u64 b0 = hb(0, key, d.nbm);
    lock(b0);
    u64 v;
    const i64 idx = dbl_find(key, v);
    if (idx >= 0) tombstone((u64)idx);
    unlock(b0);
    return idx >= 0;
  }

  // ================================================= power of two choice
  // reference openaddr.py:326-483 (lock_elided = UnsafeP2Table)

  __device__ u8 p2_upsert(u64 key, u64 val, int merge) {
    const u64 h0 = mix64(key ^ d.seeds[0]);
    const u64 b0 = d.nbm(h0 >> 16);
    const u16 tag = md_tag(h0);
    const bool locked = !d.lock_elided;
    u8 st;
    bool have_b1 = false;
    u64 b1_locked = 0;
    if (locked) lock(b0);
    for (;;) {
      Find r0 = find(b0, key, tag, false);
      if (r0.idx >= 0) { st = update(r0.idx, key, r0.val, val, merge); break; }
      const bool shortcut = !tomb_ever() && r0.used < d.shortcut;
      i64 b1 = -1, h1 = -1;
      int used1 = 0;
      if (!shortcut) {
        b1 = (i64)hb(1, key, d.nbm);
        if ((u64)b1 != b0) {
          if (locked && !have_b1) {
            have_b1 = true;
            b1_locked = (u64)b1;
            if (!lock_extra((u64)b1, b0)) continue;  // b0 was released: re-read it
          }
          Find r1 = find((u64)b1, key, tag, false);
          if (r1.idx >= 0) { st = update(r1.idx, key, r1.val, val, merge); break; }
          used1 = r1.used;
          h1 = r1.hint;
        } else {
          b1 = -1;
        }
      }
      i64 idx;
      if (shortcut || b1 < 0) {
        idx = claim_publish(b0, r0.hint, key, val, tag);
        if (idx < 0) {
          if (shortcut) continue;  // primary crossed the threshold meanwhile
          st = S_FULL;
          break;
        }
      } else {
        const bool prim = r0.used <= used1;  // ties go to the primary
        idx = claim_publish(prim ? b0 : (u64)b1, prim ? r0.hint : h1, key, val, tag);
        if (idx < 0) idx = claim_publish(prim ? (u64)b1 : b0, prim ? h1 : r0.hint, key, val, tag);
        if (idx < 0) { st = S_FULL; break; }
      }
      st = S_INSERTED;
      break;
    }
    if (have_b1) unlock(b1_locked);
    if (locked) unlock(b0);
    return st;
  }

  __device__ i64 p2_find(u64 key, u64& val, bool early_exit) {
    const u64 h0 = mix64(key ^ d.seeds[0]);
    const u64 b0 = d.nbm(h0 >> 16);
    const u16 tag = md_tag(h0);
    Find r0 = find(b0, key, tag, false);
    if (r0.idx >= 0) { val = r0.val; return r0.idx; }
    if (early_exit && r0.saw_empty && r0.used < d.shortcut && !tomb_ever()) return -1;
    const u64 b1 = hb(1, key, d.nbm);
    if (b1 == b0) return -1;
    Find r1 = find(b1, key, tag, false);
    if (r1.idx >= 0) { val = r1.val; return r1.idx; }
    return -1;
  }

  __device__ bool p2_erase(u64 key) {
    const u64 b0 = hb(0, key, d.nbm);
    const bool locked = !d.lock_elided;
    if (locked) lock(b0);
    hook(PRE_SCAN, key);
    u64 v;
    const i64 idx = p2_find(key, v, true);
    if (idx >= 0) tombstone((u64)idx);
    if (locked) unlock(b0);
    return idx >= 0;
  }

  // ============================================================== iceberg
  // reference openaddr.py:486-631

  __device__ void ice_backs(u64 key, u64& b1, u64& b2) const {
    b1 = d.front + hb(1, key, d.backm);
    b2 = d.front + hb(2, key, d.backm);
  }

  __device__ u8 ice_upsert(u64 key, u64 val, int merge) {
    const u64 h0 = mix64(key ^ d.seeds[0]);
    const u64 b0 = d.frontm(h0 >> 16);
    const u16 tag = md_tag(h0);
    u8 st;
    bool backs_locked = false;
    u64 bl[2] = {0, 0};
    int nbl = 0;
    lock(b0);
    for (;;) {
      Find r0 = find(b0, key, tag, false);
      if (r0.idx >= 0) { st = update(r0.idx, key, r0.val, val, merge); break; }
      u64 bk[2];
      int nbk = 0;
      bool found = false;
      if (!r0.saw_empty) {
        ice_backs(key, bk[0], bk[1]);
        nbk = bk[1] == bk[0] ? 1 : 2;
        if (!backs_locked) {  // backyard indices exceed every front index: ascending order holds
          backs_locked = true;
          bl[0] = bk[0] < bk[1] ? bk[0] : bk[1];
          bl[1] = bk[0] < bk[1] ? bk[1] : bk[0];
          nbl = nbk;
          for (int i = 0; i < nbl; i++) lock_extra(bl[i], b0);
        }
        for (int i = 0; i < nbk; i++) {
          Find r = find(bk[i], key, tag, false);
          if (r.idx >= 0) { st = update(r.idx, key, r.val, val, merge); found = true; break; }
        }
      }
      if (found) break;
      i64 idx = claim_publish(b0, r0.hint, key, val, tag);
      if (idx < 0) {
        if (!nbk) continue;  // front filled since the scan: rescan everything
        int u[2];
        bool f[2];
        for (int i = 0; i < nbk; i++) used_and_free(bk[i], u[i], f[i]);
        // sorted((used, bucket)) over the buckets with a free slot
        int order[2] = {0, 1};
        if (nbk == 2 && (u[1] < u[0] || (u[1] == u[0] && bk[1] < bk[0]))) { order[0] = 1; order[1] = 0; }
        for (int oi = 0; oi < nbk && idx < 0; oi++) {
          const int i = order[oi];
          if (f[i]) idx = claim_publish(bk[i], -1, key, val, tag);
        }
        if (idx < 0) { st = S_FULL; break; }
      }
      st = S_INSERTED;
      break;
    }
    for (int i = nbl - 1; i >= 0; i--) unlock(bl[i]);
    unlock(b0);
    return st;
  }

  __device__ i64 ice_find(u64 key, u64& val, bool early_exit) {
    const u64 h0 = mix64(key ^ d.seeds[0]);
    const u64 b0 = d.frontm(h0 >> 16);
    const u16 tag = md_tag(h0);
    Find r0 = find(b0, key, tag, false);
    if (r0.idx >= 0) { val = r0.val; return r0.idx; }
    if (early_exit && r0.saw_empty) return -1;
    u64 b1, b2;
    ice_backs(key, b1, b2);
    Find r = find(b1, key, tag, false);
    if (r.idx >= 0) { val = r.val; return r.idx; }
    if (b2 != b1 || !early_exit) {
      r = find(b2, key, tag, false);
      if (r.idx >= 0) { val = r.val; return r.idx; }
    }
    return -1;
  }

  __device__ bool ice_erase(u64 key) {
    const u64 b0 = hb(0, key, d.frontm);
    lock(b0);
    u64 v;
    const i64 idx = ice_find(key, v, true);
    if (idx >= 0) tombstone((u64)idx);
    unlock(b0);
    return idx >= 0;
  }

  // =============================================================== cuckoo
  // reference cuckoo.py:32-222

  __device__ int ck_buckets(u64 key, u64* uq) const {  // dict.fromkeys order
    int nu = 0;
    for (int i = 0; i < d.ways; i++) {
      const u64 b = hb(i, key, d.nbm);
      bool dup = false;
      for (int j = 0; j < nu; j++) dup |= uq[j] == b;
      if (!dup) uq[nu++] = b;
    }
    return nu;
  }
  // Phased mode (locks are no-ops in the reference, sync.py:70-102) keeps the
  // locks of cuckoo MUTATIONS: displacement chains move other keys, and two
  // unlocked movers of one key would both copy it (a duplicate).  Phased
  // queries stay lock-free (`mut` false).
  __device__ void ck_lock_all(const u64* uq, int nu, bool mut = true) {  // ascending order: deadlock free
    for (int i = 0; i < nu; i++) touch_lock(uq[i]);
    if (d.phased && !mut) return;
    u64 s[8];
    for (int i = 0; i < nu; i++) s[i] = uq[i];
    for (int i = 1; i < nu; i++)
      for (int j = i; j > 0 && s[j - 1] > s[j]; j--) { const u64 t = s[j]; s[j] = s[j - 1]; s[j - 1] = t; }
    for (int i = 0; i < nu; i++) lock_bucket(d.locks, s[i]);
  }
  __device__ void ck_unlock_all(const u64* uq, int nu, bool mut = true) {
    if (d.phased && !mut) return;
    for (int i = 0; i < nu; i++) unlock_bucket(d.locks, uq[i]);
  }

  // BFS workspace: [entries x 4 words: bucket | parent<<32 | depth, slot, key, -]
  //                [seen_cap words keys][seen_cap/2 words epochs]
  __device__ u64* ws_acquire(u32& id) {
    u32 i = (u32)((blockIdx.x * blockDim.x + threadIdx.x) % d.n_bfs);
    unsigned ns = 64;
    for (;;) {
      for (u32 t = 0; t < d.n_bfs; t++) {
        const u32 w = (i + t) % d.n_bfs;
        if (atomicCAS(d.bfs_busy + w, 0u, 1u) == 0u) {
          __threadfence();
          id = w;
          return d.bfs_mem + (u64)w * d.bfs_stride;
        }
      }
      __nanosleep(ns);
      if (ns < 4096) ns <<= 1;
    }
  }
  __device__ void ws_release(u32 id) {
    __threadfence();
    atomicExch(d.bfs_busy + id, 0u);
  }

  // reference cuckoo.py:107-156; returns #moves (written at ws[0..]) or -1
  __device__ int ck_find_path(u64* ws, const u64* uq, int nu) {
    const u64 E = d.bfs_entries, SC = d.bfs_seen_cap;
    u64* ent = ws;                 // 4 words per visited entry
    u64* skey = ws + 4 * E;        // seen set keys
    u32* sep = (u32*)(skey + SC);  // seen set epochs
    u32* hdr = sep + SC;           // [0] epoch
    u32 epoch = hdr[0] + 1;
    if (epoch == 0) {
      for (u64 i = 0; i < SC; i++) sep[i] = 0;
      epoch = 1;
    }
    hdr[0] = epoch;
    const u64 smask = SC - 1;
    auto seen_has = [&](u64 b) {
      for (u64 h = mix64(b) & smask;; h = (h + 1) & smask) {
        if (sep[h] != epoch) return false;
        if (skey[h] == b) return true;
      }
    };
    auto seen_add = [&](u64 b) {
      for (u64 h = mix64(b) & smask;; h = (h + 1) & smask) {
        if (sep[h] != epoch) { sep[h] = epoch; skey[h] = b; return; }
        if (skey[h] == b) return;
      }
    };
    u64 vn = 0;
    for (int i = 0; i < nu; i++) {
      ent[4 * vn] = uq[i] | (0xFFFFFFull << 40);  // parent = none
      ent[4 * vn + 1] = 0;
      ent[4 * vn + 2] = 0;
      ent[4 * vn + 3] = 0;
      vn++;
      seen_add(uq[i]);
    }
    const int n = B();
    const u64 NOPAR = 0xFFFFFFull;
    u64 head = 0;
    int expanded = 0;
    while (head < vn && expanded < BFS_BUDGET) {
      const u64 vi = head++;
      const u64 bucket = ent[4 * vi] & ((1ull << 40) - 1);
      const int depth = (int)ent[4 * vi + 3];
      if (depth >= d.depth) continue;
      expanded++;
      for (int j = 0; j < n; j++) {
        const u64 slot = bucket * (u64)n + j;
        u64 k, v;
        ldc(slot, k, v);
        if (k == EMPTY || k >= RESV) continue;
        for (int s = 0; s < d.ways; s++) {
          const u64 alt = hb(s, k, d.nbm);
          if (alt == bucket || seen_has(alt)) continue;
          if (find_free(alt * (u64)n, n) >= 0) {
            // unwind parent edges into moves, root-most first, stored in the
            // top `len` entries of the workspace (host sizing keeps them free)
            int len = 1;
            for (u64 c = vi; ((ent[4 * c] >> 40) & NOPAR) != NOPAR; c = (ent[4 * c] >> 40) & NOPAR) len++;
            u64* mv = ent + 4 * (E - (u64)len);  // moves live in the top entries
            int pos = len - 1;
            mv[4 * pos] = bucket; mv[4 * pos + 1] = slot; mv[4 * pos + 2] = k; mv[4 * pos + 3] = alt;
            pos--;
            for (u64 c = vi; ((ent[4 * c] >> 40) & NOPAR) != NOPAR; c = (ent[4 * c] >> 40) & NOPAR) {
              const u64 p = (ent[4 * c] >> 40) & NOPAR;
              mv[4 * pos] = ent[4 * p] & ((1ull << 40) - 1);
              mv[4 * pos + 1] = ent[4 * c + 1];
              mv[4 * pos + 2] = ent[4 * c + 2];
              mv[4 * pos + 3] = ent[4 * c] & ((1ull << 40) - 1);
              pos--;
            }
            return len;
          }
          if (vn + 64 >= E) continue;  // workspace exhausted (cannot happen with host sizing)
          ent[4 * vn] = alt | (vi << 40);
          ent[4 * vn + 1] = slot;
          ent[4 * vn + 2] = k;
          ent[4 * vn + 3] = (u64)(depth + 1);
          vn++;
          seen_add(alt);
        }
      }
    }
    return -1;
  }

  // Depth-1 prefix of the reference BFS (cuckoo.py:107-156) without a
  // workspace: start buckets in order, their resident slots in order, seeds
  // in order, skipping alternates already seen; the first alternate with a
  // free slot is exactly the path the full BFS returns when one of length 1
  // exists.  1: found (move in mv[0..3]), 0: no length-1 path (run the full
  // BFS), -1: seen set overflowed the local budget (run the full BFS).
  __device__ int ck_find_path1(const u64* uq, int nu, u64* mv) {
    constexpr int kSeen = 96;
    u64 seen[kSeen];
    int ns = 0;
    for (int i = 0; i < nu; i++) seen[ns++] = uq[i];
    const int n = B();
    for (int i = 0; i < nu; i++) {
      const u64 bucket = uq[i];
      for (int j = 0; j < n; j++) {
        const u64 slot = bucket * (u64)n + j;
        u64 k, v;
        ldc(slot, k, v);
        if (k == EMPTY || k >= RESV) continue;
        for (int sd = 0; sd < d.ways; sd++) {
          const u64 alt = hb(sd, k, d.nbm);
          if (alt == bucket) continue;
          bool dup = false;
          for (int q = 0; q < ns && !dup; q++) dup = seen[q] == alt;
          if (dup) continue;
          if (find_free(alt * (u64)n, n) >= 0) {
            mv[0] = bucket; mv[1] = slot; mv[2] = k; mv[3] = alt;
            return 1;
          }
          if (ns == kSeen) return -1;
          seen[ns++] = alt;
        }
      }
    }
    return 0;
  }

  // reference cuckoo.py:158-183, deepest move first, each under {src, dst}
  __device__ bool ck_execute(const u64* mv, int len) {
    const int n = B();
    for (int i = len - 1; i >= 0; i--) {
      const u64 src_b = mv[4 * i], src = mv[4 * i + 1], key = mv[4 * i + 2], dst_b = mv[4 * i + 3];
      u64 pair[2] = {src_b, dst_b};
      const int np = dst_b == src_b ? 1 : 2;
      ck_lock_all(pair, np);
      u64 k, v;
      ldc(src, k, v);
      bool ok = k == key;
      if (ok) {
        const i64 f = find_free(dst_b * (u64)n, n);
        ok = f >= 0 && publish_cell(cell((u64)f), key, v);
        if (ok) {
          if (ld_u32_relaxed(d.state) == 0) st_u32_relaxed(d.state, 1u);
          st_cell(cell(src), TOMB, 0);
          touch(16 * src);
          touch(16 * (u64)f);
        }
      }
      ck_unlock_all(pair, np);
      if (!ok) return false;
    }
    return true;
  }

  __device__ u8 ck_upsert(u64 key, u64 val, int merge) {
    const int n = B();
    u64 uq[8];
    const int nu = ck_buckets(key, uq);
    bool final_scan = false;  // a resumed op that found no path rescans its own buckets once
    for (int attempt = 0; attempt < CUCKOO_RETRIES; attempt++) {
      if (attempt > 0 || !d.ck_resume) {
        ck_lock_all(uq, nu);
        i64 free_at = -1;
        u8 st = 0xFF;
        for (int i = 0; i < nu && st == 0xFF; i++) {
          Find r = scan_cells(uq[i] * (u64)n, n, key);
          if (r.idx >= 0) st = update(r.idx, key, r.val, val, merge);
          else if (free_at < 0 && r.hint >= 0) free_at = r.hint;
        }
        if (st == 0xFF && free_at >= 0) {
          if (publish_cell(cell((u64)free_at), key, val)) {
            touch(16 * (u64)free_at);
            st = S_INSERTED;
          }
        }
        ck_unlock_all(uq, nu);
        if (st != 0xFF) return st;
        if (free_at >= 0) continue;  // lost a race for the free cell: retry
        if (final_scan) return S_FULL;
      }
      if (d.depth >= 1) {
        u64 mv1[4];
        const int r1 = ck_find_path1(uq, nu, mv1);
        if (r1 == 1) {
          ck_execute(mv1, 1);  // a failed move means the world changed: retry
          continue;
        }
      }
      u32 wid;
      u64* ws = ws_acquire(wid);
      const int len = ck_find_path(ws, uq, nu);
      bool ok = false;
      if (len > 0) ok = ck_execute(ws + 4 * (d.bfs_entries - (u64)len), len);
      ws_release(wid);
      if (len < 0) {
        // a resumed op skipped the locked scan of attempt 0; its buckets may
        // have gained the key or a free cell during the eviction launch
        if (attempt == 0 && d.ck_resume) { final_scan = true; continue; }
        return S_FULL;
      }
      (void)ok;  // a failed move means the world changed: retry the insert
    }
    return S_FULL;
  }

  __device__ i64 ck_find(u64 key, u64& val, bool take_locks) {
    const int n = B();
    u64 uq[8];
    const int nu = ck_buckets(key, uq);
    if (take_locks) ck_lock_all(uq, nu, false);
    i64 idx = -1;
    for (int i = 0; i < nu && idx < 0; i++) {
      Find r = scan_cells(uq[i] * (u64)n, n, key);
      if (r.idx >= 0) { idx = r.idx; val = r.val; }
    }
    if (take_locks) ck_unlock_all(uq, nu, false);
    return idx;
  }

  __device__ bool ck_erase(u64 key) {
    const int n = B();
    u64 uq[8];
    const int nu = ck_buckets(key, uq);
    ck_lock_all(uq, nu);
    i64 idx = -1;
    for (int i = 0; i < nu && idx < 0; i++) {
      Find r = scan_cells(uq[i] * (u64)n, n, key);
      if (r.idx >= 0) idx = r.idx;
    }
    if (idx >= 0) {
      if (ld_u32_relaxed(d.state) == 0) st_u32_relaxed(d.state, 1u);
      st_cell(cell((u64)idx), TOMB, 0);
      touch(16 * (u64)idx);
    }
    ck_unlock_all(uq, nu);
    return idx >= 0;
  }

  // ============================================================= chaining
  // reference chaining.py:32-226.  Node m = d.wpn words at cells + m*wpn;
  // pair j at words (2j, 2j+1), link at word 2*bs.  Node 0 is the null link,
  // the head of bucket b is node b+1, overflow nodes come from a bump
  // allocator over a preallocated pool (the host grows it between launches).

  struct Walk { i64 m, j; u64 val, tail; i64 fm, fj; };

  __device__ u64* node(u64 m) const { return d.cells + (u64)d.wpn * m; }

  __device__ Walk ch_walk(u64 key) {
    Walk w{-1, -1, 0, 0, -1, -1};
    const int pairs = B();
    u64 m = hb(0, key, d.nbm) + 1;
    for (;;) {
      touch((u64)d.line_bytes * m);
      u64* nd = node(m);
      for (int base = 0; base < pairs; base += 8) {
        const int cnt = pairs - base < 8 ? pairs - base : 8;
        u64 k[8], v[8];
#pragma unroll
        for (int j = 0; j < 8; j++)
          if (j < cnt) load_cell<RO>(nd + 2 * (base + j), k[j], v[j]);
#pragma unroll
        for (int jj = 0; jj < 8; jj++) {
          if (jj >= cnt) break;
          const int j = base + jj;
          if (k[jj] == key) { w.m = (i64)m; w.j = j; w.val = v[jj]; w.tail = m; return w; }
          if (k[jj] == EMPTY) {
            if (w.fm < 0) { w.fm = (i64)m; w.fj = j; }
            w.tail = m;
            return w;
          }
          if (k[jj] == TOMB && w.fm < 0) { w.fm = (i64)m; w.fj = j; }
        }
      }
      const u64 nxt = ld_u64_acquire(nd + 2 * pairs);
      if (!nxt) { w.tail = m; return w; }
      m = nxt;
    }
  }

  __device__ u8 ch_upsert(u64 key, u64 val, int merge) {
    const u64 b = hb(0, key, d.nbm);
    u8 st;
    lock(b);
    // Phased mode (sync.py:70-102) makes the chain lock a no-op while inserts
    // of distinct keys into one chain still run concurrently: a free pair is
    // then claimed by CAS and a new node is linked by CAS on the tail's link
    // before its first pair is claimed (a loser walks the chain again; an
    // unlinked node stays EMPTY).  Under the lock plain stores suffice.
    for (;;) {
      Walk w = ch_walk(key);
      if (w.m >= 0) {
        st_cell(node((u64)w.m) + 2 * w.j, key, apply_merge(merge, w.val, val));
        st = S_UPDATED;
        break;
      }
      if (w.fm >= 0) {
        if (!d.phased) {
          st_cell(node((u64)w.fm) + 2 * w.fj, key, val);
          st = S_INSERTED;
          break;
        }
        if (publish_cell(node((u64)w.fm) + 2 * w.fj, key, val)) { st = S_INSERTED; break; }
        continue;
      }
      const u64 m = atomicAdd(d.chain_next, 1ull);
      if (m >= d.chain_cap) {
        st_u32_relaxed(d.cs + 2, 1u);  // host grows the pool and re-runs this op
        st = S_RETRY;
        break;
      }
      touch((u64)d.line_bytes * m);
      if (!d.phased) {
        st_cell(node(m), key, val);
        st_u64_release(node(w.tail) + 2 * B(), m);
        st = S_INSERTED;
        break;
      }
      if (atomicCAS((unsigned long long*)(node(w.tail) + 2 * B()), 0ull, (unsigned long long)m) != 0ull) continue;
      if (publish_cell(node(m), key, val)) { st = S_INSERTED; break; }
    }
    unlock(b);
    return st;
  }

  __device__ bool ch_erase(u64 key) {
    const u64 b = hb(0, key, d.nbm);
    lock(b);
    Walk w = ch_walk(key);
    if (w.m >= 0) {
      if (ld_u32_relaxed(d.state) == 0) st_u32_relaxed(d.state, 1u);
      fence_acq_rel();
      st_cell(node((u64)w.m) + 2 * w.j, TOMB, 0);
    }
    unlock(b);
    return w.m >= 0;
  }

  // ============================================================ dispatch

  template <int DESIGN>
  __device__ u8 upsert(u64 key, u64 val, int merge) {
    if constexpr (DESIGN == D_DOUBLE || DESIGN == D_DOUBLE_MD) return dbl_upsert(key, val, merge);
    else if constexpr (DESIGN == D_P2 || DESIGN == D_P2_MD || DESIGN == D_UNSAFE) return p2_upsert(key, val, merge);
    else if constexpr (DESIGN == D_ICEBERG || DESIGN == D_ICEBERG_MD) return ice_upsert(key, val, merge);
    else if constexpr (DESIGN == D_CUCKOO) return ck_upsert(key, val, merge);
    else return ch_upsert(key, val, merge);
  }

  template <int DESIGN>
  __device__ bool erase(u64 key) {
    if constexpr (DESIGN == D_DOUBLE || DESIGN == D_DOUBLE_MD) return dbl_erase(key);
    else if constexpr (DESIGN == D_P2 || DESIGN == D_P2_MD || DESIGN == D_UNSAFE) return p2_erase(key);
    else if constexpr (DESIGN == D_ICEBERG || DESIGN == D_ICEBERG_MD) return ice_erase(key);
    else if constexpr (DESIGN == D_CUCKOO) return ck_erase(key);
    else return ch_erase(key);
  }

  // lock-free lookup (cuckoo takes its ordered locks unless phased)
  template <int DESIGN>
  __device__ bool query(u64 key, u64& v) {
    i64 idx;
    if constexpr (DESIGN == D_DOUBLE || DESIGN == D_DOUBLE_MD) idx = dbl_find(key, v);
    else if constexpr (DESIGN == D_P2 || DESIGN == D_P2_MD || DESIGN == D_UNSAFE) idx = p2_find(key, v, true);
    else if constexpr (DESIGN == D_ICEBERG || DESIGN == D_ICEBERG_MD) idx = ice_find(key, v, true);
    else if constexpr (DESIGN == D_CUCKOO) idx = ck_find(key, v, true);
    else { Walk w = ch_walk(key); idx = w.m; v = w.val; }
    if (idx < 0) v = 0;
    return idx >= 0;
  }

  template <int DESIGN>
  __device__ OpOut run(int kind, int merge, u64 key, u64 val) {
    OpOut o{0, 0};
    if (kind == OP_UPSERT) o.status = upsert<DESIGN>(key, val, merge);
    else if (kind == OP_ERASE) o.status = erase<DESIGN>(key);
    else o.status = query<DESIGN>(key, o.val);
    return o;
  }

  // slot_of (reference tables/base.py:136-143 -> each design's _locate)
  template <int DESIGN>
  __device__ i64 locate(u64 key) {
    u64 v;
    if constexpr (DESIGN == D_DOUBLE || DESIGN == D_DOUBLE_MD) return dbl_find(key, v);
    else if constexpr (DESIGN == D_P2 || DESIGN == D_P2_MD || DESIGN == D_UNSAFE) return p2_find(key, v, false);
    else if constexpr (DESIGN == D_ICEBERG || DESIGN == D_ICEBERG_MD) return ice_find(key, v, false);
    else if constexpr (DESIGN == D_CUCKOO) return ck_find(key, v, false);
    else { Walk w = ch_walk(key); return w.m >= 0 ? w.m * B() + w.j : -1; }
  }
};

}  // namespace ws

// Kernel instantiations for the cuckoo design (see ws_kernels.cuh), plus the
// tuned lock-round query and upsert fast path for the default 8-slot buckets.
#include "ws_kernels.cuh"

#include <algorithm>

namespace ws {

__device__ __forceinline__ void ld32b(const u64* p, u64* w) {
  asm volatile("ld.relaxed.gpu.global.v4.u64 {%0,%1,%2,%3}, [%4];"
               : "=l"(w[0]), "=l"(w[1]), "=l"(w[2]), "=l"(w[3]) : "l"(p) : "memory");
}
// Scan of one 8-cell bucket (a 128-byte line) in hash-slot order, stopping
// at the key or the first EMPTY, in stages of 32-byte sectors: the first
// sector alone (one request; at low load it usually holds an EMPTY), then
// (STAGED) the second alone, then the remaining sectors together -- fewer
// round trips than sector by sector, at most one extra request.  The query
// (loads around 0.9, most buckets need every sector) takes the rest in one
// stage; the upsert, whose fills start from an empty table, takes two.
// `fr` = first reusable cell (TOMB / EMPTY).
template <bool STAGED>
__device__ __forceinline__ void scan_line8(const u64* p, u64 lo, u64 key, i64& hit, u64& val, i64& fr) {
  u64 w[16];
  bool stop = false;
  auto scan = [&](int j0, int j1) {
#pragma unroll
    for (int j = j0; j < j1; j++) {
      if (!stop) {
        if (w[2 * j] == key) { hit = (i64)(lo + j); val = w[2 * j + 1]; stop = true; }
        else if (w[2 * j] == EMPTY) { if (fr < 0) fr = (i64)(lo + j); stop = true; }
        else if (w[2 * j] == TOMB) { if (fr < 0) fr = (i64)(lo + j); }
      }
    }
  };
  ld32b(p, w);
  scan(0, 2);
  if (stop) return;
  if (STAGED) {
    ld32b(p + 4, w + 4);
    scan(2, 4);
    if (stop) return;
  } else {
    ld32b(p + 4, w + 4);
  }
  ld32b(p + 8, w + 8);
  ld32b(p + 12, w + 12);
  if (!STAGED) scan(2, 4);
  scan(4, 8);
}

// Per-op bucket set of the lock-round query with compile-time capacity W
// (3 for the default table, 8 otherwise): hash-order distinct buckets in uq
// (dict.fromkeys), ascending copy in srt (unused entries sort last as ~0).
// Every loop runs to W with predicates, so the arrays stay in registers
// (the upsert keeps its runtime-bounded arrays: measured no faster there).
template <int W>
__device__ __forceinline__ int ck_setup(const Dev& d, bool pending, u64 key, u64 (&uq)[W], u64 (&srt)[W]) {
  const int ways = W == 3 ? 3 : d.ways;
  int nu = 0;
#pragma unroll
  for (int w = 0; w < W; w++) {
    uq[w] = ~0ull;
    if (pending && w < ways) {
      const u64 b = d.nbm(mix64(key ^ d.seeds[w]) >> 16);
      bool dup = false;
#pragma unroll
      for (int j = 0; j < W; j++) dup |= j < nu && uq[j] == b;
      if (!dup) {
#pragma unroll
        for (int j = 0; j < W; j++)
          if (j == nu) uq[j] = b;
        nu++;
      }
    }
  }
#pragma unroll
  for (int j = 0; j < W; j++) srt[j] = j < nu ? uq[j] : ~0ull;
#pragma unroll
  for (int a = 0; a < W; a++)
#pragma unroll
    for (int b = 0; b + 1 < W - a; b++)
      if (srt[b] > srt[b + 1]) { const u64 t = srt[b]; srt[b] = srt[b + 1]; srt[b + 1] = t; }
  return nu;
}
// uq[q] without dynamic indexing (a select chain keeps the array in registers)
template <int W>
__device__ __forceinline__ u64 ck_pick(const u64 (&a)[W], int q) {
  u64 r = a[0];
#pragma unroll
  for (int j = 1; j < W; j++)
    if (q == j) r = a[j];
  return r;
}
// try-lock the sorted buckets from `held` on, stopping at the first failure
template <int W>
__device__ __forceinline__ int ck_trylock_prefix(const Dev& d, const u64 (&srt)[W], int nu, int held) {
#pragma unroll
  for (int j = 0; j < W; j++)
    if (j == held && j < nu && try_lock_bucket(d.locks, srt[j])) held++;
  return held;
}
template <int W>
__device__ __forceinline__ void ck_release(const Dev& d, const u64 (&srt)[W], int nu) {
#pragma unroll
  for (int q = 0; q < W; q++)
    if (q < nu)
      asm volatile("red.relaxed.gpu.global.and.b32 [%0], %1;" ::"l"(d.locks + (srt[q] >> 5)),
                   "r"(~(1u << (srt[q] & 31))) : "memory");
}

// Cuckoo query (reference cuckoo.py:185-198): take the locks of the key's
// distinct buckets in ascending order, scan them in hash order (stopping at
// the first EMPTY, sync.py:184-207), release.  One thread per op in
// warp-synchronous rounds: each pending lane try-locks its sorted buckets
// one after another and stops at the first failure, KEEPING the prefix it
// holds (it only ever waits for a higher lock, so there is no cycle, and two
// lanes of a warp racing for the same lowest lock get exactly one winner);
// lanes holding all their locks scan with 32-byte loads, then the warp issues
// one fence and the finished lanes release with relaxed reductions.
template <int W>
__global__ void __launch_bounds__(256, 5) k_query_cuckoo_rounds(Dev d, const u64* __restrict__ keys, u64 n,
                                                             u64* vout, u8* found, int gated) {
  WS_PROLOGUE(d, gated, n);
  const int lane = threadIdx.x & 31;
  const u64 nwarps = ((u64)gridDim.x * blockDim.x) >> 5;
  const bool locked = !d.phased;
  for (u64 c = (blockIdx.x * (u64)blockDim.x + threadIdx.x) >> 5; c * 32 < n; c += nwarps) {
    const u64 i = c * 32 + lane;
    bool pending = i < n;
    const u64 key = pending ? __ldg(keys + i) : 0;
    u64 uq[W], srt[W];
    const int nu = ck_setup<W>(d, pending, key, uq, srt);
    int held = 0;
    bool hit = false;
    u64 val = 0;
    unsigned backoff = 64;
    while (__any_sync(0xFFFFFFFFu, pending)) {
      if (pending && locked) held = ck_trylock_prefix<W>(d, srt, nu, held);
      const bool ready = pending && (!locked || held == nu);
      if (ready) {
#pragma unroll 1
        for (int q = 0; q < nu && !hit; q++) {
          const u64 b = ck_pick<W>(uq, q);
          i64 h = -1, fr = -1;
          scan_line8<false>(d.cells + 2 * (b * 8), b * 8, key, h, val, fr);
          hit = h >= 0;
        }
        pending = false;
      }
      if (locked) {
        __syncwarp();
        fence_acq_rel();
        if (ready) ck_release<W>(d, srt, nu);
      }
      if (pending) {
        __nanosleep(backoff + 8 * lane);
        if (backoff < 4096) backoff <<= 1;
      }
    }
    if (i < n) {
      if (found) found[i] = hit;
      if (vout) vout[i] = hit ? val : 0;
    }
  }
}

// Cuckoo upsert fast path (reference cuckoo.py:68-97, the part before the
// eviction search): same lock rounds as the query; with all of the key's
// bucket locks held, scan the buckets in hash order -- a match is merged, else
// the first bucket with a reusable cell (first TOMB / EMPTY before the
// bucket's first EMPTY) receives the key.  Ops whose buckets are all full
// are marked S_RETRY and left to the generic kernel (BFS eviction chains),
// launched right after on the same stream: one serial order of the batch.
__global__ void __launch_bounds__(256, 6) k_upsert_cuckoo_rounds(Dev d, const u64* __restrict__ keys,
                                                              const u64* __restrict__ vals, u64 n, int merge,
                                                              u8* st_out, int gated) {
  WS_PROLOGUE(d, gated, n);
  const int lane = threadIdx.x & 31;
  const u64 nwarps = ((u64)gridDim.x * blockDim.x) >> 5;
  const bool locked = true;  // mutations lock even in phased mode (Ctx::ck_lock_all)
  for (u64 c = (blockIdx.x * (u64)blockDim.x + threadIdx.x) >> 5; c * 32 < n; c += nwarps) {
    const u64 i = c * 32 + lane;
    bool pending = i < n;
    const u64 key = pending ? __ldg(keys + i) : 0;
    const u64 val = pending ? __ldg(vals + i) : 0;
    u64 uq[8], srt[8];
    int nu = 0;
    if (pending) {
      for (int w = 0; w < d.ways; w++) {
        const u64 b = d.nbm(mix64(key ^ d.seeds[w]) >> 16);
        bool dup = false;
        for (int j = 0; j < nu; j++) dup |= uq[j] == b;
        if (!dup) uq[nu++] = b;
      }
      for (int j = 0; j < nu; j++) srt[j] = uq[j];
      for (int a = 1; a < nu; a++)
        for (int b = a; b > 0 && srt[b - 1] > srt[b]; b--) { const u64 t = srt[b]; srt[b] = srt[b - 1]; srt[b - 1] = t; }
    }
    int held = 0;
    u8 st = S_RETRY;
    unsigned backoff = 64;
    while (__any_sync(0xFFFFFFFFu, pending)) {
      if (pending && locked)
        while (held < nu && try_lock_bucket(d.locks, srt[held])) held++;
      const bool ready = pending && (!locked || held == nu);
      if (ready) {
        i64 hit = -1, free_at = -1;
        u64 old = 0;
        for (int q = 0; q < nu && hit < 0; q++) {
          const u64 lo = uq[q] * 8;
          i64 fr = -1;
          scan_line8<true>(d.cells + 2 * lo, lo, key, hit, old, fr);
          if (free_at < 0 && fr >= 0) free_at = fr;
        }
        if (hit >= 0) {
          st_cell(d.cells + 2 * (u64)hit, key, apply_merge(merge, old, val));
          st = S_UPDATED;
        } else if (free_at >= 0 && publish_cell(d.cells + 2 * (u64)free_at, key, val)) {
          st = S_INSERTED;
        }  // else S_RETRY: every bucket full (eviction chain) -> generic kernel
        pending = false;
      }
      if (locked) {
        __syncwarp();
        fence_acq_rel();
        if (ready) {
          for (int q = 0; q < nu; q++)
            asm volatile("red.relaxed.gpu.global.and.b32 [%0], %1;" ::"l"(d.locks + (srt[q] >> 5)),
                         "r"(~(1u << (srt[q] & 31))) : "memory");
        }
      }
      if (pending) {
        __nanosleep(backoff + 8 * lane);
        if (backoff < 4096) backoff <<= 1;
      }
    }
    if (i < n) st_out[i] = st;
  }
}

// Warp-aggregated compaction of the S_RETRY ops into an index list (order
// within a warp kept, across warps arbitrary: the ops are concurrent anyway).
__global__ void __launch_bounds__(256) k_compact_retry(const u8* __restrict__ st, u64 n, u32* list, u32* count,
                                                       const u64* dn) {
  if (dn && *dn < n) n = *dn;  // device-resident batch size (multi-GPU exchange)
  const int lane = threadIdx.x & 31;
  for (u64 base = (blockIdx.x * (u64)blockDim.x + threadIdx.x) & ~31ull; base < n;
       base += (u64)gridDim.x * blockDim.x) {
    const u64 i = base + lane;
    const bool r = i < n && st[i] == S_RETRY;
    const u32 m = __ballot_sync(0xFFFFFFFFu, r);
    if (!m) continue;
    u32 at = 0;
    if (lane == 0) at = atomicAdd(count, (u32)__popc(m));
    at = __shfl_sync(0xFFFFFFFFu, at, 0);
    if (r) list[at + __popc(m & ((1u << lane) - 1))] = (u32)i;
  }
}

// Eviction launch (the S_RETRY ops of k_upsert_cuckoo_rounds, compacted),
// one op per 8-lane group, 4 ops per warp.  Exactly Ctx::ck_upsert with
// ck_resume (reference cuckoo.py:58-105) except that its depth-1 path search
// (Ctx::ck_find_path1: start buckets in order, their resident slots in order,
// seeds in order, the first alternate with a free cell wins) runs across the
// group: lane j loads slot j of every start bucket, then the candidates
// (bucket, slot, seed) are checked in the serial order in waves of 8, one
// alternate per lane (whole-line key loads), and the first wave holding a
// free alternate yields its lowest-order one -- the path the serial search
// returns: duplicates of an earlier alternate are free exactly when it is, so
// skipping them (the serial seen-set) cannot change the first free one.  Locked scans, moves and the full BFS fallback
// run on the group's leader lane with the generic code.
__device__ __forceinline__ bool line8_has_free(const u64* line) {
  bool f = false;
#pragma unroll
  for (int q = 0; q < 4; q++) {
    u64 a, b, c, e;
    asm volatile("ld.relaxed.gpu.global.v4.u64 {%0,%1,%2,%3}, [%4];"
                 : "=l"(a), "=l"(b), "=l"(c), "=l"(e) : "l"(line + 4 * q) : "memory");
    f |= free_key(a) | free_key(c);
  }
  return f;
}

__global__ void __launch_bounds__(256, 5) k_ck_evict_coop(Dev d, const u64* __restrict__ keys,
                                                       const u64* __restrict__ vals, int merge, u8* status,
                                                       const u32* __restrict__ rlist, const u32* rcount,
                                                       int conc_erase) {
  Ctx<D_CUCKOO, 8, false, false> c{d, nullptr, conc_erase != 0, ld_u32_relaxed(d.state)};
  const int lane = threadIdx.x & 31, lj = lane & 7, lead = lane & ~7;
  const unsigned gm = 0xFFu << lead;
  const bool leader = lj == 0;
  const u64 ngroups = ((u64)gridDim.x * blockDim.x) >> 3;
  const u32 cnt = *rcount;
  for (u64 t = (blockIdx.x * (u64)blockDim.x + threadIdx.x) >> 3; t < cnt; t += ngroups) {
    const u32 i = rlist[t];
    const u64 key = keys[i], val = vals[i];
    u64 uq[8];
    const int nu = c.ck_buckets(key, uq);
    u8 st = 0xFF;
    bool final_scan = false;
    for (int attempt = 0; attempt < CUCKOO_RETRIES; attempt++) {
      if (attempt > 0 || !d.ck_resume) {  // locked scan of the op's own buckets (leader)
        int code = 0;                     // 1: decided (st), 2: lost a race for a free cell
        if (leader) {
          c.ck_lock_all(uq, nu);
          i64 free_at = -1;
          for (int b = 0; b < nu && st == 0xFF; b++) {
            Find r = c.scan_cells(uq[b] * 8, 8, key);
            if (r.idx >= 0) st = c.update(r.idx, key, r.val, val, merge);
            else if (free_at < 0 && r.hint >= 0) free_at = r.hint;
          }
          if (st == 0xFF && free_at >= 0 && publish_cell(c.cell((u64)free_at), key, val)) st = S_INSERTED;
          c.ck_unlock_all(uq, nu);
          code = st != 0xFF ? 1 : free_at >= 0 ? 2 : 0;
        }
        code = __shfl_sync(gm, code, lead);
        if (code == 1) break;
        if (code == 2) continue;
        if (final_scan) { st = S_FULL; break; }
      }
      if (d.depth >= 1 && nu <= 3 && d.ways == 3) {
        // resident keys: lane j holds slot j of every start bucket
        u64 k[3];
#pragma unroll
        for (int b = 0; b < 3; b++) {
          k[b] = 0;
          if (b < nu) { u64 v; c.ldc(uq[b] * 8 + lj, k[b], v); }
        }
        // candidates in the serial search's order c = (bucket * 8 + slot) * 3 + seed,
        // checked in waves of 8 (one per lane) until a wave holds a free alternate
        int found = -1;
        u64 falt = 0, fkey = 0;
        for (int w = 0; w < nu * 3 && found < 0; w++) {
          const int cidx = 8 * w + lj, b = cidx / 24, slot = (cidx % 24) / 3, sd = cidx % 3;
          const u64 k0 = __shfl_sync(gm, k[0], lead + slot), k1 = __shfl_sync(gm, k[1], lead + slot),
                    k2 = __shfl_sync(gm, k[2], lead + slot);
          const u64 kk = b == 0 ? k0 : b == 1 ? k1 : k2;
          bool fr = false;
          u64 alt = 0;
          if (b < nu && !free_key(kk) && kk < RESV) {
            alt = c.hb(sd, kk, d.nbm);
            bool dup = false;
            for (int q = 0; q < nu; q++) dup |= alt == uq[q];
            fr = !dup && line8_has_free(d.cells + 16 * alt);
          }
          const unsigned m = __ballot_sync(gm, fr) & gm;
          if (m) {
            const int src = __ffs(m) - 1;
            found = __shfl_sync(gm, b * 8 + slot, src);
            falt = __shfl_sync(gm, alt, src);
            fkey = __shfl_sync(gm, kk, src);
          }
        }
        if (found >= 0) {
          if (leader) {
            const int b = found / 8, slot = found % 8;
            const u64 mv[4] = {uq[b], uq[b] * 8 + (u64)slot, fkey, falt};
            c.ck_execute(mv, 1);  // a failed move means the world changed: retry
          }
          __syncwarp(gm);
          continue;
        }
      } else if (d.depth >= 1) {  // more than three distinct buckets: the serial depth-1 search
        int r1 = 0;
        if (leader) {
          u64 mv1[4];
          r1 = c.ck_find_path1(uq, nu, mv1);
          if (r1 == 1) c.ck_execute(mv1, 1);
        }
        r1 = __shfl_sync(gm, r1, lead);
        if (r1 == 1) continue;
      }
      int len = 0;
      if (leader) {
        u32 wid;
        u64* ws = c.ws_acquire(wid);
        len = c.ck_find_path(ws, uq, nu);
        if (len > 0) c.ck_execute(ws + 4 * (d.bfs_entries - (u64)len), len);
        c.ws_release(wid);
      }
      len = __shfl_sync(gm, len, lead);
      if (len < 0) {
        if (attempt == 0 && d.ck_resume) { final_scan = true; continue; }
        st = S_FULL;
        break;
      }
    }
    if (st == 0xFF) st = S_FULL;
    if (leader && status) status[i] = st;
  }
}

static void cuckoo_ops(const OpsArgs& a, bool def) {
  const bool upsert_only = !a.ops && (a.uop & 15) == OP_UPSERT;
  // tune_upsert 6: the same fast path with the round-1 one-thread-per-op eviction launch (A/B)
  if (def && upsert_only && !a.instr && !a.d.delay_ns && !a.serial && !a.redo && a.d.ways <= 8 &&
      (a.d.tune_upsert == 4 || a.d.tune_upsert == 6)) {
    u8* st = a.status;
    if (!st && cudaMallocAsync((void**)&st, a.n, a.s) != cudaSuccess) st = nullptr;
    if (st) {
      u64 g = (a.n + 255) / 256;
      const u64 lim = std::max<u64>((a.d.nb + 255) / 256, 4);  // <= ~1 op in flight per bucket
      g = std::max<u64>(std::min<u64>(std::min<u64>(g, (u64)kSMs * table_grid_per_sm(a.d)), lim), 1);
      k_upsert_cuckoo_rounds<<<(unsigned)g, 256, 0, a.s>>>(a.d, a.keys, a.vals, a.n, a.uop >> 4, st, a.gated);
      OpsArgs lo = a;
      lo.status = st;
      lo.redo = st;  // the generic kernel runs only the S_RETRY ops (eviction chains)
      lo.d.ck_resume = 1;  // ...starting at their eviction search
      // compacted, so the eviction searches fill whole warps instead of the
      // ~1/3 of lanes whose buckets were full
      u32* rl = nullptr;
      if (a.n < 0xFFFFFFFFull && cudaMallocAsync((void**)&rl, 4 * (a.n + 1), a.s) == cudaSuccess) {
        cudaMemsetAsync(rl + a.n, 0, 4, a.s);
        k_compact_retry<<<(unsigned)std::max<u64>(std::min<u64>((a.n + 255) / 256, (u64)kSMs * table_grid_per_sm(a.d)), 1), 256, 0,
                          a.s>>>(st, a.n, rl, rl + a.n, a.d.dn);
        lo.rlist = rl;
        lo.rcount = rl + a.n;
      }
      if (rl && a.vals && a.d.tune_upsert == 4) {
        // 8 lanes per op; the grid covers the worst case (every op retries)
        const u64 g = std::max<u64>(std::min<u64>((8 * a.n + 255) / 256, (u64)kSMs * table_grid_per_sm(a.d)), 1);
        k_ck_evict_coop<<<(unsigned)g, 256, 0, a.s>>>(lo.d, a.keys, a.vals, a.uop >> 4, st, rl, rl + a.n,
                                                      a.conc_erase);
      } else {
        launch_ops_t<D_CUCKOO, 8>(lo);
      }
      if (rl) cudaFreeAsync(rl, a.s);
      if (st != a.status) cudaFreeAsync(st, a.s);
      return;
    }
  }
  if (def) launch_ops_t<D_CUCKOO, 8>(a); else launch_ops_t<D_CUCKOO, 0>(a);
}
static void cuckoo_query(const QueryArgs& a, bool def) {
  if (def && a.d.ways <= 8 && a.d.tune_qilp > 0) {
    u64 g = (a.n + 255) / 256;
    g = std::max<u64>(std::min<u64>(g, (u64)kSMs * table_grid_per_sm(a.d)), 1);
    if (a.d.ways == 3)
      k_query_cuckoo_rounds<3><<<(unsigned)g, 256, 0, a.s>>>(a.d, a.keys, a.n, a.vout, a.found, a.gated);
    else
      k_query_cuckoo_rounds<8><<<(unsigned)g, 256, 0, a.s>>>(a.d, a.keys, a.n, a.vout, a.found, a.gated);
    return;
  }
  if (def) launch_query_t<D_CUCKOO, 8>(a); else launch_query_t<D_CUCKOO, 0>(a);
}
static void cuckoo_locate(const LocateArgs& a, bool def) {
  if (def) launch_locate_t<D_CUCKOO, 8>(a); else launch_locate_t<D_CUCKOO, 0>(a);
}
static void cuckoo_preload(bool def) {
  if (!def) { preload_t<D_CUCKOO, 0>(); return; }
  preload_t<D_CUCKOO, 8>();
  preload_fn(k_query_cuckoo_rounds<3>);
  preload_fn(k_query_cuckoo_rounds<8>);
  preload_fn(k_upsert_cuckoo_rounds);
  preload_fn(k_compact_retry);
  preload_fn(k_ck_evict_coop);
}
Launchers launchers_cuckoo() { return Launchers{cuckoo_ops, cuckoo_query, cuckoo_locate, cuckoo_preload}; }

}  // namespace ws

// ws_bulk.cu -- bucket-partitioned bulk upsert for P2-MD (the headline design).
//
// Why: the one-op-per-thread upsert (k_upsert_p2md_rounds) costs ~3.2 random
// DRAM line accesses per insert -- primary tag block read, the tag line's
// write-back and the cell line's write-back -- and runs at ~90% of the
// measured random-access ceiling.  A large batch carries
// ~29 inserts per bucket (2^28 slots at 0.9 load), so most of that work can be
// done with STREAMING traffic: partition the batch by primary bucket, let one
// CTA own a group of consecutive buckets, read their tag blocks once, apply
// their shortcut inserts and write tags and new cells back as whole sectors.
//
// Semantics (reference tables/openaddr.py:370-418).  While the table has
// never tombstoned, an insert whose primary bucket b0 holds fewer than
// `shortcut` (24) claimed slots goes to b0 without reading the alternate, and
// such a key can only live in b0 (occupancy is monotone, so every earlier
// insert of it also shortcut).  The batch is executed as the serial order
//   phase A: every op whose key is found in b0 or that takes the shortcut
//            (capped, below), bucket by bucket, in batch order per bucket;
//   phase B: every remaining op (b0 already at the threshold),
// which is a valid linearisation of the concurrent batch:
//   * a phase-A op sees exactly the b0 state the serial order gives it (only
//     phase-A ops of the same b0 precede it there; foreign writers into b0 --
//     P2 alternates -- run in phase B);
//   * a deferred op was not found in b0 and b0 was at the threshold; b0 stays
//     at or above it, and later same-key ops of the bucket are deferred too,
//     so the key cannot appear in b0 before phase B runs it.
// Phase A claims slots only while b0 holds fewer than cap = shortcut - 4 (20)
// slots; ops past that are deferred even if they could still shortcut.  Any
// cap <= shortcut keeps the argument above.  Why not the full 24: the serial
// order "every bucket to the threshold, then all overflow" squeezes the
// overflow into the last 8 slots of every bucket and a 0.9 fill then reports
// FULL for a few keys whose two buckets are both full (measured 11 per 2^28
// fill; load simulation 2.25 per 2^26) where batch (random) order reports
// none.  With the cap at 20 the remaining 31% of ops run in random order from
// a balanced half-full table and the simulation shows 0 FULL (6 fills at
// 2^28, 8 at 2^26), as for random order.
// Phase B is the ordinary locked kernel (k_upsert_p2md_rounds) over the
// deferred ops (a bit per batch index), so alternate-bucket routing, FULL
// handling and statuses are exactly those of the per-op path.  It visits them
// in BATCH order, like a plain per-op launch: processed in partition (bucket)
// order, the least-loaded choices of early buckets starve late ones and a
// 0.9 fill reports FULLs that no random order produces (oracle-checked:
// bucket order 5 FULL at 2^16 slots, 33 at 2^20; random 0), and any
// structured order (group order, a Weyl stride) measurably does the same.
//
// Ownership instead of locks: phase A takes no bucket locks because each
// bucket is touched by exactly one CTA (the owner of its group); the path is
// only taken for tables that are not declared multi_stream (ws_capi.cu).
//
// Kernels:
//   k_part_hist / k_part_scatter  stable LSD partition of (key, value, batch
//       index) by group id = b0 >> log2(GB), R <= 10 bits per pass.  Each CTA
//       owns a contiguous input range; sub-tiles of 2048 are double-buffered
//       into shared memory with cp.async, ranked (__match_any_sync), sorted
//       by digit in place and written out as per-digit runs;
//   k_bulk_apply  persistent, one group at a time per CTA, the next chunk's
//       ops and tag blocks prefetched with cp.async.  Ops are stable-sorted by
//       bucket; a bucket whose ops have no key collision (no tag hit on a
//       claimed slot, no repeated key in the chunk -- shared-memory hash) is
//       applied one thread per op (slot = used + rank, coalesced cell
//       stores); the rest run a warp-per-bucket path with key confirmation
//       and same-key folding in batch order.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>

#include <cub/cub.cuh>

#include "ws_bulk.cuh"
#include "ws_kernels.cuh"

namespace ws {
namespace {

__device__ __forceinline__ u64 umin64(u64 a, u64 b) { return a < b ? a : b; }

__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc, int src_bytes) {
  const u32 s = (u32)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gsrc), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
// m elements of `esz` bytes at g (16-byte aligned) -> s, zero-filling the tail
template <int NT>
__device__ __forceinline__ void cp_async_elems(void* s, const void* g, u32 m, u32 esz) {
  const u32 bytes = m * esz, chunks = (bytes + 15) / 16;
  for (u32 c = threadIdx.x; c < chunks; c += NT) {
    const u32 left = bytes - 16 * c;
    cp_async16((char*)s + 16 * c, (const char*)g + 16 * c, left < 16 ? (int)left : 16);
  }
}
template <int NB, int NT>
__device__ __forceinline__ void block_exclusive_scan(const u32* total, u32* start) {
  typedef cub::BlockScan<u32, NT> BS;
  __shared__ typename BS::TempStorage ts;
  constexpr int PER = NB >= NT ? NB / NT : 1;
  u32 loc[PER];
  u32 sum = 0;
#pragma unroll
  for (int j = 0; j < PER; j++) {
    const int i = threadIdx.x * PER + j;
    loc[j] = i < NB ? total[i] : 0;
    sum += loc[j];
  }
  u32 ex;
  BS(ts).ExclusiveSum(sum, ex);
#pragma unroll
  for (int j = 0; j < PER; j++) {
    const int i = threadIdx.x * PER + j;
    if (i < NB) start[i] = ex;
    ex += loc[j];
  }
}

// ------------------------------------------------------------ partition

constexpr int PT = 256;             // partition CTA threads
constexpr int PW = PT / 32;         // warps per partition CTA
constexpr int PTILE = 2048;         // elements per shared-memory sub-tile
constexpr int PSTEP = PTILE / PT;   // elements per lane per sub-tile
constexpr int PWE = PTILE / PW;     // contiguous elements per warp per sub-tile

struct GroupFn {
  Mod nbm;
  u64 s0;
  int gshift;
  __device__ __forceinline__ u32 operator()(u64 key) const {
    return (u32)(nbm(mix64(key ^ s0) >> 16) >> gshift);
  }
};

template <int R>
__global__ void __launch_bounds__(PT) k_part_hist(const u64* __restrict__ keys, u64 n, u64 per, GroupFn gf,
                                                  int dshift, u32* __restrict__ counts) {
  constexpr int NB = 1 << R;
  __shared__ u32 h[NB];
  for (int i = threadIdx.x; i < NB; i += PT) h[i] = 0;
  __syncthreads();
  const u64 lo = blockIdx.x * per, hi = umin64(n, lo + per);
  for (u64 b = lo; b < hi; b += (u64)PT * 8) {
    u64 k[8];
#pragma unroll
    for (int j = 0; j < 8; j++) {
      const u64 i = b + (u64)j * PT + threadIdx.x;
      k[j] = i < hi ? __ldcs(keys + i) : 0;
    }
#pragma unroll
    for (int j = 0; j < 8; j++) {
      const u64 i = b + (u64)j * PT + threadIdx.x;
      if (i < hi) atomicAdd(&h[(gf(k[j]) >> dshift) & (NB - 1)], 1u);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < NB; i += PT) counts[(u64)i * gridDim.x + blockIdx.x] = h[i];
}

struct PBuf {
  u64 k[PTILE];
  u64 v[PTILE];
  u32 i[PTILE];
  u32 g[PTILE];
};

template <int R>
constexpr size_t part_smem() {
  return 2 * sizeof(PBuf) + 3 * sizeof(u32) * (1 << R) + sizeof(u16) * PW * (1 << R);
}

template <bool FIRST>
__device__ __forceinline__ void part_load(PBuf& B, const u64* ik, const u64* iv, const u32* ii, u64 base, u32 m,
                                          u64 pol) {
  (void)pol;
  cp_async_elems<PT>(B.k, ik + base, m, 8);
  cp_async_elems<PT>(B.v, iv + base, m, 8);
  if (!FIRST) cp_async_elems<PT>(B.i, ii + base, m, 4);
}

// Stable scatter of one LSD pass.  CTA c owns input range [c*per, (c+1)*per)
// and digit d's output run starts at offs[d*C + c] (exclusive scan of the
// digit-major histogram).  LAST: also counts elements per group (one atomic
// per run of equal group in the sorted sub-tile).
template <int R, bool FIRST, bool LAST>
__global__ void __launch_bounds__(PT, 2) k_part_scatter(const u64* __restrict__ ik, const u64* __restrict__ iv,
                                                        const u32* __restrict__ ii, u64 n, u64 per, GroupFn gf,
                                                        int dshift, const u32* __restrict__ offs,
                                                        u64* __restrict__ ok, u64* __restrict__ ov,
                                                        u32* __restrict__ oi, u32* __restrict__ gcount) {
  constexpr int NB = 1 << R;
  extern __shared__ __align__(16) unsigned char smem[];
  PBuf* buf = reinterpret_cast<PBuf*>(smem);
  u32* cursor = reinterpret_cast<u32*>(buf + 2);
  u32* total = cursor + NB;
  u32* dstart = total + NB;
  u16* whist = reinterpret_cast<u16*>(dstart + NB);  // [PW][NB]
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  for (int d = tid; d < NB; d += PT) cursor[d] = offs[(u64)d * gridDim.x + blockIdx.x];
  const u64 lo = blockIdx.x * per, hi = umin64(n, lo + per);
  const u32 ntiles = hi > lo ? (u32)((hi - lo + PTILE - 1) / PTILE) : 0;
  const u64 pol = 0;
  if (ntiles) part_load<FIRST>(buf[0], ik, iv, ii, lo, (u32)umin64(PTILE, hi - lo), pol);
  cp_async_commit();
  for (u32 t = 0; t < ntiles; t++) {
    PBuf& B = buf[t & 1];
    const u64 base = lo + (u64)t * PTILE;
    const u32 m = (u32)umin64(PTILE, hi - base);
    if (t + 1 < ntiles) {
      const u64 nb2 = base + PTILE;
      part_load<FIRST>(buf[(t + 1) & 1], ik, iv, ii, nb2, (u32)umin64(PTILE, hi - nb2), pol);
    }
    cp_async_commit();
    for (int d = lane; d < NB; d += 32) whist[w * NB + d] = 0;
    cp_async_wait<1>();
    __syncthreads();
    u64 k[PSTEP], v[PSTEP];
    u32 ix[PSTEP], g[PSTEP], r[PSTEP];
#pragma unroll
    for (int s = 0; s < PSTEP; s++) {
      const u32 p = w * PWE + s * 32 + lane;
      const bool in = p < m;
      k[s] = B.k[p];
      v[s] = B.v[p];
      ix[s] = FIRST ? (u32)(base + p) : B.i[p];
      g[s] = in ? gf(k[s]) : 0;
      const u32 dg = in ? ((g[s] >> dshift) & (NB - 1)) : (u32)NB;
      const u32 peers = __match_any_sync(0xFFFFFFFFu, dg);
      const u32 rank = __popc(peers & ((1u << lane) - 1));
      const u32 cnt = in ? whist[w * NB + dg] : 0;
      r[s] = cnt + rank;
      __syncwarp();
      if (in && rank == 0) whist[w * NB + dg] = (u16)(cnt + __popc(peers));
      __syncwarp();
    }
    __syncthreads();
    for (int d = tid; d < NB; d += PT) {
      u32 run = 0;
#pragma unroll
      for (int x = 0; x < PW; x++) {
        const u32 c = whist[x * NB + d];
        whist[x * NB + d] = (u16)run;
        run += c;
      }
      total[d] = run;
    }
    __syncthreads();
    block_exclusive_scan<NB, PT>(total, dstart);
    __syncthreads();
#pragma unroll
    for (int s = 0; s < PSTEP; s++) {
      const u32 p = w * PWE + s * 32 + lane;
      if (p < m) {
        const u32 dg = (g[s] >> dshift) & (NB - 1);
        const u32 pos = dstart[dg] + whist[w * NB + dg] + r[s];
        B.k[pos] = k[s];
        B.v[pos] = v[s];
        B.i[pos] = ix[s];
        B.g[pos] = g[s];
      }
    }
    __syncthreads();
    for (u32 p = tid; p < m; p += PT) {
      const u32 gg = B.g[p];
      const u32 dg = (gg >> dshift) & (NB - 1);
      const u64 o = (u64)cursor[dg] + (p - dstart[dg]);
      __stcg(ok + o, B.k[p]);
      __stcg(ov + o, B.v[p]);
      __stcg(oi + o, B.i[p]);
      if (LAST && (p == 0 || B.g[p - 1] != gg)) {
        u32 e = p + 1;
        while (e < m && B.g[e] == gg) e++;
        atomicAdd(gcount + gg, e - p);
      }
    }
    __syncthreads();
    for (int d = tid; d < NB; d += PT) cursor[d] += total[d];
  }
  cp_async_wait<0>();
}

// ---------------------------------------------------------------- apply

constexpr int AT = 512;       // apply CTA threads
constexpr int AW = AT / 32;   // warps
constexpr int ACAP = 2048;    // ops staged per chunk
constexpr int AWE = ACAP / AW;
constexpr int GBMAX = 128;    // buckets per group (max)
constexpr int HCAP = 4096;    // shared-memory key hash (same-key detection), power of two

struct ABuf {  // chunk ops start at element ok (keys / values) and oi (indices): 16-byte aligned copies
  u64 k[ACAP + 2];
  u64 v[ACAP + 2];
  u32 idx[ACAP + 4];
  u16 tags[GBMAX * 32];
};

struct ApplySmem {
  ABuf buf[2];
  u32 hkey[HCAP];       // 32-bit key fingerprints: in-chunk repeated-key filter
  u32 lbt[ACAP];        // local bucket << 16 | tag
  u16 rank[ACAP];
  u16 order[ACAP];      // bucket-sorted op positions
  u16 whist[AW][GBMAX];
  u32 btot[GBMAX];
  u32 bstart[GBMAX];
  u32 bflag[GBMAX];     // 1: bucket needs the warp path (key collision)
  u32 used0[GBMAX];     // claimed slots before the chunk
  u32 wback[GBMAX];     // 1: the bucket's tag block must be written back
  u32 slow[GBMAX];      // list of warp-path buckets
  u64 wk[AW][32];       // warp path: slot keys / values of the bucket
  u64 wv[AW][32];
  u64 fv[AW][32];       // warp path: op values (same-key folding)
  u32 nslow;
};

// The chunk list: group g's ops [goff[g], goff[g+1]) split into ACAP pieces.
struct ChunkIt {
  u64 g, c_lo, o_hi;
};

__device__ __forceinline__ void apply_prefetch(ABuf& B, const Dev& d, const u64* K, const u64* V, const u32* I,
                                               const ChunkIt& c, int gb_log2, bool tags) {
  const u32 m = (u32)umin64(ACAP, c.o_hi - c.c_lo);
  const u32 ok = (u32)(c.c_lo & 1), oi = (u32)(c.c_lo & 3);
  cp_async_elems<AT>(B.k, K + c.c_lo - ok, m + ok, 8);
  cp_async_elems<AT>(B.v, V + c.c_lo - ok, m + ok, 8);
  cp_async_elems<AT>(B.idx, I + c.c_lo - oi, m + oi, 4);
  if (tags) {
    const u64 b_lo = c.g << gb_log2;
    const u32 nbk = (u32)umin64(1u << gb_log2, d.nb - b_lo);
    cp_async_elems<AT>(B.tags, d.tags + b_lo * 32, nbk * 32, 2);
  }
}

// warp path for one bucket: ops order[bs0 .. bs0+cnt), exact serial semantics
__device__ void apply_bucket_warp(ApplySmem& S, ABuf& B, const u64* bk, const u64* bv, const u32* bi,
                                  const Dev& d, u64 b, u32 lb, u32 bs0, u32 cnt, bool te, int cap, int merge,
                                  u8* status, u32* dmask) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const u32 lane_lt = (1u << lane) - 1;
  u16* bt = B.tags + lb * 32;
  const u32 zmask = __ballot_sync(0xFFFFFFFFu, bt[lane] == 0);
  const int used_old = zmask ? __ffs(zmask) - 1 : 32;
  int used = used_old;
  u32 loaded = 0, newm = 0, dirty = 0;
  for (u32 c0 = 0; c0 < cnt; c0 += 32) {
    const u32 i = c0 + lane;
    const bool act = i < cnt;
    const u32 p = act ? S.order[bs0 + i] : 0;
    const u64 key = act ? bk[p] : ~0ull;  // ~0 is a sentinel, never a batch key
    const u64 val = act ? bv[p] : 0;
    const u16 tag = act ? (u16)(S.lbt[p] & 0xFFFF) : 0;
    u32 M = 0;
    if (act) {
      const u32* bw = reinterpret_cast<const u32*>(bt);
      const u32 pat = (u32)tag * 0x10001u;
#pragma unroll
      for (int q = 0; q < 16; q++) {
        const u32 mm = __vcmpeq2(bw[q], pat);
        M |= ((mm & 1u) | ((mm >> 15) & 2u)) << (2 * q);
      }
    }
    // pre-existing slots behind a tag match: load their cells (coalesced)
    const u32 need = __reduce_or_sync(0xFFFFFFFFu, M) & ~newm & ~loaded;
    if (need) {
      if ((need >> lane) & 1u) {
        u64 k2, v2;
        ld_cell(d.cells + 2 * (b * 32 + lane), k2, v2);
        S.wk[w][lane] = k2;
        S.wv[w][lane] = v2;
      }
      loaded |= need;
      __syncwarp();
    }
    int j = -1;
    for (u32 MM = M; MM; MM &= MM - 1) {
      const int c = __ffs(MM) - 1;
      if (S.wk[w][c] == key) { j = c; break; }
    }
    const u32 actm = __ballot_sync(0xFFFFFFFFu, act);
    const u32 peers = __match_any_sync(0xFFFFFFFFu, key) & actm;
    const int leader = peers ? __ffs(peers) - 1 : lane;
    const bool isl = act && lane == leader;
    const bool found = j >= 0;
    const bool newl = isl && !found;
    const u32 nlm = __ballot_sync(0xFFFFFFFFu, newl);
    const int room = te ? 0 : max(0, cap - used);
    const int r = __popc(nlm & lane_lt);
    const int slot = (newl && r < room) ? used + r : -1;
    const int lslot = __shfl_sync(0xFFFFFFFFu, slot, leader);
    S.fv[w][lane] = val;
    __syncwarp();
    int tgt = -1;
    if (isl && (found || slot >= 0)) {
      tgt = found ? j : slot;
      u64 acc = found ? apply_merge(merge, S.wv[w][j], val) : val;
      for (u32 rest = peers & ~(1u << lane); rest; rest &= rest - 1)
        acc = apply_merge(merge, acc, S.fv[w][__ffs(rest) - 1]);
      S.wk[w][tgt] = key;
      S.wv[w][tgt] = acc;
      if (!found) bt[tgt] = tag;
    }
    dirty |= __reduce_or_sync(0xFFFFFFFFu, tgt >= 0 ? (1u << tgt) : 0u);
    const int ins = min(__popc(nlm), room);
    if (ins) newm |= ((ins == 32 ? 0xFFFFFFFFu : ((1u << ins) - 1)) << used);
    used += ins;
    if (act && status && (found || (lslot >= 0 && !isl))) status[bi[p]] = S_UPDATED;
    if (act && !found && lslot < 0) atomicOr(dmask + (bi[p] >> 5), 1u << (bi[p] & 31));
    __syncwarp();
  }
  if (dirty) {
    if ((dirty >> lane) & 1u) st_cell(d.cells + 2 * (b * 32 + lane), S.wk[w][lane], S.wv[w][lane]);
    if (used > used_old && (used & 1) && lane == used && used < 32) st_cell(d.cells + 2 * (b * 32 + lane), 0, 0);
  }
  if (used > used_old && lane == 0) S.wback[lb] = 1;
}

__global__ void __launch_bounds__(AT, 1) k_bulk_apply(Dev d, const u64* __restrict__ K, const u64* __restrict__ V,
                                                      const u32* __restrict__ I, const u32* __restrict__ goff, u64 G,
                                                      int gb_log2, int cap, int merge, u8* status, u32* dmask,
                                                      int gated) {
  if (gated && (ld_u32_relaxed(d.cs) | ld_u32_relaxed(d.cs + 1))) return;
  if (blockIdx.x >= G) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  ApplySmem& S = *reinterpret_cast<ApplySmem*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const u32 lane_lt = (1u << lane) - 1;
  const u32 GB = 1u << gb_log2;
  const bool te = ld_u32_relaxed(d.state) != 0;  // tombstoned table: everything goes to phase B
  ChunkIt cur{blockIdx.x, goff[blockIdx.x], goff[blockIdx.x + 1]};
  apply_prefetch(S.buf[0], d, K, V, I, cur, gb_log2, true);
  cp_async_commit();
  for (u32 it = 0;; it++) {
    ABuf& B = S.buf[it & 1];
    ABuf& Bn = S.buf[(it + 1) & 1];
    // next chunk: rest of this group, else this CTA's next group
    ChunkIt nxt = cur;
    bool same = false, have_next = true;
    if (cur.c_lo + ACAP < cur.o_hi) {
      nxt.c_lo += ACAP;
      same = true;
    } else if (cur.g + gridDim.x < G) {
      const u64 g2 = cur.g + gridDim.x;
      nxt = ChunkIt{g2, goff[g2], goff[g2 + 1]};
    } else {
      have_next = false;
    }
    if (have_next) apply_prefetch(Bn, d, K, V, I, nxt, gb_log2, !same);
    cp_async_commit();
    const u64 b_lo = cur.g << gb_log2;
    const u32 nbk = (u32)umin64(GB, d.nb - b_lo);
    const u32 m = (u32)umin64(ACAP, cur.o_hi - cur.c_lo);
    const u64* bk = B.k + (cur.c_lo & 1);
    const u64* bv = B.v + (cur.c_lo & 1);
    const u32* bi = B.idx + (cur.c_lo & 3);
    // --- clear per-chunk state; per-op bucket and tag
    for (u32 x = lane; x < GBMAX; x += 32) S.whist[w][x] = 0;
    for (u32 q = tid; q < HCAP / 4; q += AT) reinterpret_cast<uint4*>(S.hkey)[q] = make_uint4(0, 0, 0, 0);
    for (u32 x = tid; x < GBMAX; x += AT) { S.bflag[x] = 0; S.wback[x] = 0; }
    if (tid == 0) S.nslow = 0;
    cp_async_wait<1>();
    __syncthreads();
    for (u32 p = tid; p < m; p += AT) {
      const u64 h0 = mix64(bk[p] ^ d.seeds[0]);
      const u32 lb = (u32)(d.nbm(h0 >> 16) - b_lo);
      const u16 t = (u16)(h0 & 0xFFFF);
      S.lbt[p] = (lb << 16) | (t ? t : 1u);
    }
    __syncthreads();
    // --- stable counting sort of the chunk by local bucket; same-key detection
    for (int s = 0; s < AWE / 32; s++) {
      const u32 p = w * AWE + s * 32 + lane;
      const bool in = p < m;
      const u32 lb = in ? (S.lbt[p] >> 16) : 0xFFFFu;
      const u32 peers = __match_any_sync(0xFFFFFFFFu, lb);
      const u32 rk = __popc(peers & lane_lt);
      const u32 cnt = in ? S.whist[w][lb] : 0;
      if (in) S.rank[p] = (u16)(cnt + rk);
      __syncwarp();
      if (in && rk == 0) S.whist[w][lb] = (u16)(cnt + __popc(peers));
      __syncwarp();
      if (in) {
        // a repeated fingerprint sends the bucket to the warp path, which is
        // exact; fingerprint collisions of distinct keys only cost speed
        const u64 hk = mix64(bk[p] ^ 0x9E3779B97F4A7C15ull);
        const u32 fp = (u32)(hk >> 32) | 1u;  // never 0 (free slot)
        u32 h = (u32)hk & (HCAP - 1);
        for (;;) {
          const u32 old = atomicCAS(&S.hkey[h], 0u, fp);
          if (old == 0) break;
          if (old == fp) { S.bflag[lb] = 1; break; }
          h = (h + 1) & (HCAP - 1);
        }
      }
    }
    __syncthreads();
    for (u32 x = tid; x < GBMAX; x += AT) {
      u32 run = 0;
      if (x < GB) {
#pragma unroll
        for (int y = 0; y < AW; y++) {
          const u32 c = S.whist[y][x];
          S.whist[y][x] = (u16)run;
          run += c;
        }
      }
      S.btot[x] = run;
      u32 u = 32;
      if (x < nbk) {
        const u32* bw = reinterpret_cast<const u32*>(B.tags + x * 32);
        for (int q = 0; q < 16; q++) {
          const u32 wd = bw[q];
          if (!(wd & 0xFFFFu)) { u = 2 * q; break; }
          if (!(wd >> 16)) { u = 2 * q + 1; break; }
        }
      }
      S.used0[x] = u;
    }
    __syncthreads();
    block_exclusive_scan<GBMAX, AT>(S.btot, S.bstart);
    __syncthreads();
    // --- bucket order; a tag hit on a claimed slot sends the bucket to the warp path
    for (u32 p = tid; p < m; p += AT) {
      const u32 lbt = S.lbt[p];
      const u32 lb = lbt >> 16;
      S.order[S.bstart[lb] + S.whist[p / AWE][lb] + S.rank[p]] = (u16)p;
      const u32 u0 = S.used0[lb];
      if (u0) {  // claimed slots are a prefix of the bucket (no tombstones)
        const uint4* bw = reinterpret_cast<const uint4*>(B.tags + lb * 32);
        const u32 pat = (lbt & 0xFFFFu) * 0x10001u;
        u32 hit = 0;
        for (u32 q = 0; q < (u0 + 7) / 8; q++) {
          const uint4 t4 = bw[q];
          hit |= __vcmpeq2(t4.x, pat) | __vcmpeq2(t4.y, pat) | __vcmpeq2(t4.z, pat) | __vcmpeq2(t4.w, pat);
        }
        if (hit) S.bflag[lb] = 1;
      }
    }
    __syncthreads();
    // --- fast path: one thread per op of a collision-free bucket
    for (u32 q = tid; q < m; q += AT) {
      const u32 p = S.order[q];
      const u32 lbt = S.lbt[p];
      const u32 lb = lbt >> 16;
      if (S.bflag[lb]) continue;
      const u32 u0 = S.used0[lb];
      const u32 slot = u0 + (q - S.bstart[lb]);
      if (!te && (int)slot < cap) {
        const u64 b = b_lo + lb;
        st_cell(d.cells + 2 * (b * 32 + slot), bk[p], bv[p]);
        B.tags[lb * 32 + slot] = (u16)(lbt & 0xFFFF);
        // last insert of the bucket at an even slot: complete its sector
        const u32 last = min(u0 + S.btot[lb], (u32)cap) - 1;
        if (slot == last && !(slot & 1)) st_cell(d.cells + 2 * (b * 32 + slot + 1), 0, 0);
      } else {
        atomicOr(dmask + (bi[p] >> 5), 1u << (bi[p] & 31));  // phase B runs it
      }
    }
    for (u32 x = tid; x < nbk; x += AT) {
      if (S.bflag[x]) {
        if (S.btot[x]) S.slow[atomicAdd(&S.nslow, 1u)] = x;
      } else if (S.btot[x] && !te && (int)S.used0[x] < cap) {
        S.wback[x] = 1;
      }
    }
    __syncthreads();
    // --- warp path for buckets with key collisions
    for (u32 e = w; e < S.nslow; e += AW) {
      const u32 lb = S.slow[e];
      apply_bucket_warp(S, B, bk, bv, bi, d, b_lo + lb, lb, S.bstart[lb], S.btot[lb], te, cap, merge, status,
                        dmask);
    }
    __syncthreads();
    // --- tag blocks of buckets that claimed slots; deferred ops
    for (u32 q = tid; q < nbk * 16; q += AT) {
      if (S.wback[q >> 4])
        st_u32_relaxed(reinterpret_cast<u32*>(d.tags + b_lo * 32) + q, reinterpret_cast<const u32*>(B.tags)[q]);
    }
    if (!have_next) break;
    // the rest of a group continues from this chunk's (updated) tag blocks
    if (same) {
      for (u32 q = tid; q < nbk * 16; q += AT)
        reinterpret_cast<u32*>(Bn.tags)[q] = reinterpret_cast<const u32*>(B.tags)[q];
    }
    __syncthreads();
    cur = nxt;
  }
  cp_async_wait<0>();
}

// ------------------------------------------------------------ host side

template <int R>
struct Part {
  static constexpr size_t sm = part_smem<R>();
  template <bool F, bool L>
  static void set_attr() {
    static bool done = false;
    if (!done) {
      cudaFuncSetAttribute(k_part_scatter<R, F, L>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      done = true;
    }
  }
  static int occupancy() {
    set_attr<true, false>();
    set_attr<false, true>();
    set_attr<true, true>();
    set_attr<false, false>();
    int a = 1, b = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, k_part_scatter<R, true, false>, PT, sm);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_part_scatter<R, false, true>, PT, sm);
    return std::max(1, std::min(a, b));
  }
  static void hist(const u64* keys, u64 n, u64 per, unsigned C, GroupFn gf, int dshift, u32* counts,
                   cudaStream_t s) {
    k_part_hist<R><<<C, PT, 0, s>>>(keys, n, per, gf, dshift, counts);
  }
  static void pass(bool first, bool last, const u64* ik, const u64* iv, const u32* ii, u64 n, u64 per, unsigned C,
                   GroupFn gf, int dshift, const u32* offs, u64* ok, u64* ov, u32* oi, u32* gcount,
                   cudaStream_t s) {
    if (first && last)
      k_part_scatter<R, true, true><<<C, PT, sm, s>>>(ik, iv, ii, n, per, gf, dshift, offs, ok, ov, oi, gcount);
    else if (first)
      k_part_scatter<R, true, false><<<C, PT, sm, s>>>(ik, iv, ii, n, per, gf, dshift, offs, ok, ov, oi, gcount);
    else if (last)
      k_part_scatter<R, false, true><<<C, PT, sm, s>>>(ik, iv, ii, n, per, gf, dshift, offs, ok, ov, oi, gcount);
    else
      k_part_scatter<R, false, false><<<C, PT, sm, s>>>(ik, iv, ii, n, per, gf, dshift, offs, ok, ov, oi, gcount);
  }
};

typedef void (*PassFn)(bool, bool, const u64*, const u64*, const u32*, u64, u64, unsigned, GroupFn, int,
                       const u32*, u64*, u64*, u32*, u32*, cudaStream_t);
typedef void (*HistFn)(const u64*, u64, u64, unsigned, GroupFn, int, u32*, cudaStream_t);
typedef int (*OccFn)();

#define WS_BULK_CK(x) do { const cudaError_t e_ = (x); if (e_ != cudaSuccess) return e_; } while (0)

void apply_attr() {
  static bool done = false;
  if (!done) {
    cudaFuncSetAttribute(k_bulk_apply, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(ApplySmem));
    done = true;
  }
}

}  // namespace

BulkPlan bulk_plan(u64 n, u64 nb, int gb_log2) {
  BulkPlan p{};
  const double rho = nb ? (double)n / (double)nb : 0.0;
  // groups sized so a group's ops fit two staging chunks (4 sigma headroom):
  // larger groups mean fewer partition digits and longer output runs
  const double budget = 2.0 * ACAP - 4.0 * std::sqrt(2.0 * ACAP);
  int gl = 0;
  while ((2 << gl) <= GBMAX && (double)(2u << gl) * rho <= budget) gl++;
  if (gb_log2 >= 0) gl = std::min(gb_log2, 7);
  p.gb_log2 = gl;
  p.groups = (nb + (1ull << gl) - 1) >> gl;
  int gbits = 0;
  while ((1ull << gbits) < p.groups) gbits++;
  p.passes = gbits <= 10 ? 1 : gbits <= 20 ? 2 : 3;
  p.radix = std::max(6, (gbits + p.passes - 1) / p.passes);
  return p;
}

bool bulk_aligned(const void* keys, const void* vals) {
  return (((uintptr_t)keys | (uintptr_t)vals) & 15) == 0;
}

cudaError_t bulk_upsert_p2md(const Dev& d, const u64* keys, const u64* vals, u64 n, int merge, u8* status,
                             int gated, cudaStream_t s, const BulkPlan& plan) {
  if (!n) return cudaSuccess;
  const int R = plan.radix;
  const int NB = 1 << R;
  PassFn pass = R <= 6 ? Part<6>::pass : R == 7 ? Part<7>::pass : R == 8 ? Part<8>::pass
              : R == 9 ? Part<9>::pass : Part<10>::pass;
  HistFn hist = R <= 6 ? Part<6>::hist : R == 7 ? Part<7>::hist : R == 8 ? Part<8>::hist
              : R == 9 ? Part<9>::hist : Part<10>::hist;
  OccFn occf = R <= 6 ? Part<6>::occupancy : R == 7 ? Part<7>::occupancy : R == 8 ? Part<8>::occupancy
              : R == 9 ? Part<9>::occupancy : Part<10>::occupancy;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  u64 C = (u64)sms * occf();
  const u64 tiles = (n + PTILE - 1) / PTILE;
  if (C > tiles) C = tiles;
  const u64 per = ((tiles + C - 1) / C) * PTILE;
  C = (n + per - 1) / per;
  const GroupFn gf{d.nbm, d.seeds[0], plan.gb_log2};

  // scratch: two (key, value, index) buffers, digit histograms, group
  // offsets, the deferral bitmap (one bit per batch op)
  u64 *K0 = nullptr, *V0 = nullptr, *K1 = nullptr, *V1 = nullptr;
  u32 *I0 = nullptr, *I1 = nullptr, *counts = nullptr, *offs = nullptr, *gcnt = nullptr, *goff = nullptr;
  u32* dmask = nullptr;
  void* tmp = nullptr;
  const u64 G = plan.groups;
  const u64 mwords = (n + 31) / 32;
  size_t tb1 = 0, tb2 = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb1, counts, offs, (int64_t)(NB * C), s);
  cub::DeviceScan::ExclusiveSum(nullptr, tb2, gcnt, goff, (int64_t)(G + 1), s);
  WS_BULK_CK(cudaMallocAsync((void**)&K0, 8 * n, s));
  WS_BULK_CK(cudaMallocAsync((void**)&V0, 8 * n, s));
  WS_BULK_CK(cudaMallocAsync((void**)&I0, 4 * n, s));
  WS_BULK_CK(cudaMallocAsync((void**)&K1, 8 * n, s));
  WS_BULK_CK(cudaMallocAsync((void**)&V1, 8 * n, s));
  WS_BULK_CK(cudaMallocAsync((void**)&I1, 4 * n, s));
  WS_BULK_CK(cudaMallocAsync((void**)&dmask, 4 * mwords, s));
  WS_BULK_CK(cudaMallocAsync((void**)&counts, 4 * NB * C, s));
  WS_BULK_CK(cudaMallocAsync((void**)&offs, 4 * NB * C, s));
  WS_BULK_CK(cudaMallocAsync((void**)&gcnt, 4 * (G + 1), s));
  WS_BULK_CK(cudaMallocAsync((void**)&goff, 4 * (G + 1), s));
  WS_BULK_CK(cudaMallocAsync(&tmp, std::max(tb1, tb2) + 16, s));
  WS_BULK_CK(cudaMemsetAsync(gcnt, 0, 4 * (G + 1), s));
  WS_BULK_CK(cudaMemsetAsync(dmask, 0, 4 * mwords, s));
  if (status) WS_BULK_CK(cudaMemsetAsync(status, S_INSERTED, n, s));

  const u64* ik = keys;
  const u64* iv = vals;
  const u32* ii = nullptr;
  u64* bk[2] = {K0, K1};
  u64* bv[2] = {V0, V1};
  u32* bi[2] = {I0, I1};
  int out = 0;
  for (int ps = 0; ps < plan.passes; ps++) {
    const int dshift = ps * R;
    const bool first = ps == 0, last = ps == plan.passes - 1;
    hist(ik, n, per, (unsigned)C, gf, dshift, counts, s);
    cub::DeviceScan::ExclusiveSum(tmp, tb1, counts, offs, (int64_t)(NB * C), s);
    pass(first, last, ik, iv, ii, n, per, (unsigned)C, gf, dshift, offs, bk[out], bv[out], bi[out], gcnt, s);
    ik = bk[out];
    iv = bv[out];
    ii = bi[out];
    out ^= 1;
  }
  WS_BULK_CK(cudaGetLastError());
  cub::DeviceScan::ExclusiveSum(tmp, tb2, gcnt, goff, (int64_t)(G + 1), s);
  apply_attr();
  const u64 gA = std::min<u64>(G, (u64)sms);
  k_bulk_apply<<<(unsigned)gA, AT, sizeof(ApplySmem), s>>>(d, ik, iv, ii, goff, G, plan.gb_log2,
                                                            std::min(plan.cap, d.shortcut), merge, status, dmask,
                                                            gated);
  WS_BULK_CK(cudaGetLastError());
  if (!plan.skip_b) {
    // phase B: the locked per-op kernel over the deferred ops, in batch order
    u64 gB = (n + 255) / 256;
    gB = std::min<u64>(gB, (u64)sms * 8);
    gB = std::min<u64>(gB, std::max<u64>((d.nb + 255) / 256, 4));
    bulk_phase_b(d, keys, vals, n, merge, status, gated, dmask, (unsigned)std::max<u64>(gB, 1), s);
    WS_BULK_CK(cudaGetLastError());
  }
  for (void* p : {(void*)K0, (void*)V0, (void*)I0, (void*)K1, (void*)V1, (void*)I1, (void*)counts, (void*)offs,
                  (void*)gcnt, (void*)goff, tmp, (void*)dmask})
    cudaFreeAsync(p, s);
  return cudaSuccess;
}

void bulk_preload() {
  Part<8>::occupancy();
  Part<9>::occupancy();
  apply_attr();
  preload_fn(k_bulk_apply);
  preload_fn(k_part_hist<8>);
  preload_fn(k_part_hist<9>);
}

}  // namespace ws

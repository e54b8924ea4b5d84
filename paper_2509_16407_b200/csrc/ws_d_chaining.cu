// Kernel instantiations for the chaining design (see ws_kernels.cuh), plus a
// line-at-a-time lock-free query for the default 7-pair (128-byte) nodes.
#include "ws_kernels.cuh"

#include <algorithm>

namespace ws {

// Chaining query (reference chaining.py:137-171, 205-207): walk the chain
// from head node b+1, stop at the key, at the first EMPTY, or at a null link.
// The generic walk loads a node's seven 16-byte pairs, scans them and only
// then loads the link -- two dependent DRAM round trips per node.  Here a
// node (7 pairs + link + pad = 128 bytes, one line) is fetched as four
// 32-byte loads issued together, so the link comes with the pairs.  Used for
// launches with no concurrent mutation (the next node is then fully
// published before this launch started; concurrent launches keep the
// acquire-ordered generic walk).
template <bool RO>
__global__ void __launch_bounds__(256) k_query_chain_lines(Dev d, const u64* __restrict__ keys, u64 n, u64* vout,
                                                           u8* found, int gated) {
  WS_PROLOGUE(d, gated, n);
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
    const u64 key = __ldg(keys + i);
    u64 m = d.nbm(mix64(key ^ d.seeds[0]) >> 16) + 1;
    bool hit = false;
    u64 val = 0;
    for (;;) {
      const u64* nd = d.cells + 16 * m;
      u64 w[16];
#pragma unroll
      for (int q = 0; q < 4; q++) {
        if (RO)
          asm volatile("ld.global.nc.L1::no_allocate.v4.u64 {%0,%1,%2,%3}, [%4];"
                       : "=l"(w[4 * q]), "=l"(w[4 * q + 1]), "=l"(w[4 * q + 2]), "=l"(w[4 * q + 3])
                       : "l"(nd + 4 * q));
        else
          asm volatile("ld.relaxed.gpu.global.v4.u64 {%0,%1,%2,%3}, [%4];"
                       : "=l"(w[4 * q]), "=l"(w[4 * q + 1]), "=l"(w[4 * q + 2]), "=l"(w[4 * q + 3])
                       : "l"(nd + 4 * q) : "memory");
      }
      bool stop = false;
#pragma unroll
      for (int j = 0; j < 7; j++) {
        if (stop) break;
        if (w[2 * j] == key) { hit = true; val = w[2 * j + 1]; stop = true; }
        else if (w[2 * j] == EMPTY) stop = true;
      }
      if (stop || !w[14]) break;
      m = w[14];
    }
    if (found) found[i] = hit;
    if (vout) vout[i] = hit ? val : 0;
  }
}

// Chaining upsert (reference chaining.py:173-199, Ctx::ch_upsert): one thread
// per op in warp-synchronous lock rounds (try-lock the key's bucket; one
// fence per warp-round before the relaxed releases).  The holder walks the
// chain a line at a time (four 32-byte loads per 128-byte node), then merges
// into the match, fills the first reusable pair, or appends a node from the
// bump allocator -- node contents stored first, then the link with release
// semantics, so lock-free readers only ever see a whole node.  An exhausted
// pool marks the op S_RETRY and raises the flag the host's grow-and-redo
// loop (ws_capi.cu) reacts to, exactly as the generic kernel does.
__global__ void __launch_bounds__(256) k_upsert_chain_rounds(Dev d, const u64* __restrict__ keys,
                                                             const u64* __restrict__ vals, u64 n, int merge,
                                                             u8* status, int gated) {
  WS_PROLOGUE(d, gated, n);
  const int lane = threadIdx.x & 31;
  const u64 nwarps = ((u64)gridDim.x * blockDim.x) >> 5;
  const bool locked = true;  // phased tables keep the generic kernel
  for (u64 c = (blockIdx.x * (u64)blockDim.x + threadIdx.x) >> 5; c * 32 < n; c += nwarps) {
    const u64 i = c * 32 + lane;
    bool pending = i < n;
    const u64 key = pending ? __ldg(keys + i) : 0;
    const u64 val = pending ? __ldg(vals + i) : 0;
    const u64 b = d.nbm(mix64(key ^ d.seeds[0]) >> 16);
    bool held = false;
    u8 st = S_INSERTED;
    unsigned backoff = 64;
    while (__any_sync(0xFFFFFFFFu, pending)) {
      if (pending && locked && !held) held = try_lock_bucket(d.locks, b);
      const bool ready = pending && (!locked || held);
      if (ready) {
        u64 m = b + 1, tail = m, hm = 0, fm = 0, hv = 0;
        int hj = -1, fj = -1;
        for (;;) {
          const u64* nd = d.cells + 16 * m;
          u64 w[16];
#pragma unroll
          for (int q = 0; q < 4; q++)
            asm volatile("ld.relaxed.gpu.global.v4.u64 {%0,%1,%2,%3}, [%4];"
                         : "=l"(w[4 * q]), "=l"(w[4 * q + 1]), "=l"(w[4 * q + 2]), "=l"(w[4 * q + 3])
                         : "l"(nd + 4 * q) : "memory");
          bool stop = false;
#pragma unroll
          for (int j = 0; j < 7; j++) {
            if (stop) break;
            const u64 k = w[2 * j];
            if (k == key) { hm = m; hj = j; hv = w[2 * j + 1]; stop = true; }
            else if (k == EMPTY) { if (fj < 0) { fm = m; fj = j; } stop = true; }
            else if (k == TOMB && fj < 0) { fm = m; fj = j; }
          }
          tail = m;
          if (stop || !w[14]) break;
          m = w[14];
        }
        if (hj >= 0) {
          st_cell(d.cells + 16 * hm + 2 * hj, key, apply_merge(merge, hv, val));
          st = S_UPDATED;
        } else if (fj >= 0) {
          st_cell(d.cells + 16 * fm + 2 * fj, key, val);
          st = S_INSERTED;
        } else {
          const u64 m2 = atomicAdd(d.chain_next, 1ull);
          if (m2 >= d.chain_cap) {
            st_u32_relaxed(d.cs + 2, 1u);  // host grows the pool and re-runs this op
            st = S_RETRY;
          } else {
            st_cell(d.cells + 16 * m2, key, val);
            st_u64_release(d.cells + 16 * tail + 14, m2);
            st = S_INSERTED;
          }
        }
        pending = false;
      }
      if (locked) {
        __syncwarp();
        fence_acq_rel();
        if (ready && held) {
          asm volatile("red.relaxed.gpu.global.and.b32 [%0], %1;" ::"l"(d.locks + (b >> 5)), "r"(~(1u << (b & 31)))
                       : "memory");
          held = false;
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

static void chaining_ops(const OpsArgs& a, bool def) {
  const bool upsert_only = !a.ops && (a.uop & 15) == OP_UPSERT;
  if (def && upsert_only && a.status && !a.instr && !a.d.delay_ns && !a.serial && !a.redo && !a.d.phased && a.d.wpn == 16 &&
      a.d.tune_upsert == 4) {
    u64 g = (a.n + 255) / 256;
    const u64 lim = std::max<u64>((a.d.nb + 255) / 256, 4);  // <= ~1 op in flight per bucket
    g = std::max<u64>(std::min<u64>(std::min<u64>(g, (u64)kSMs * table_grid_per_sm(a.d)), lim), 1);
    k_upsert_chain_rounds<<<(unsigned)g, 256, 0, a.s>>>(a.d, a.keys, a.vals, a.n, a.uop >> 4, a.status, a.gated);
    return;
  }
  if (def) launch_ops_t<D_CHAINING, 7>(a); else launch_ops_t<D_CHAINING, 0>(a);
}
static void chaining_query(const QueryArgs& a, bool def) {
  if (def && !a.conc_erase && a.d.wpn == 16 && a.d.tune_qilp > 0) {
    const unsigned g = grid_for(a.n, kThreads, table_grid_per_sm(a.d));
    if (a.ro) k_query_chain_lines<true><<<g, kThreads, 0, a.s>>>(a.d, a.keys, a.n, a.vout, a.found, a.gated);
    else k_query_chain_lines<false><<<g, kThreads, 0, a.s>>>(a.d, a.keys, a.n, a.vout, a.found, a.gated);
    return;
  }
  if (def) launch_query_t<D_CHAINING, 7>(a); else launch_query_t<D_CHAINING, 0>(a);
}
static void chaining_locate(const LocateArgs& a, bool def) {
  if (def) launch_locate_t<D_CHAINING, 7>(a); else launch_locate_t<D_CHAINING, 0>(a);
}
static void chaining_preload(bool def) {
  if (!def) { preload_t<D_CHAINING, 0>(); return; }
  preload_t<D_CHAINING, 7>();
  preload_fn(k_query_chain_lines<false>);
  preload_fn(k_query_chain_lines<true>);
  preload_fn(k_upsert_chain_rounds);
}
Launchers launchers_chaining() { return Launchers{chaining_ops, chaining_query, chaining_locate, chaining_preload}; }

}  // namespace ws

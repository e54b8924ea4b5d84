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
  if (gated && (ld_u32_relaxed(d.state + 2) | ld_u32_relaxed(d.state + 3))) return;
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

static void chaining_ops(const OpsArgs& a, bool def) {
  if (def) launch_ops_t<D_CHAINING, 7>(a); else launch_ops_t<D_CHAINING, 0>(a);
}
static void chaining_query(const QueryArgs& a, bool def) {
  if (def && !a.conc_erase && a.d.wpn == 16 && a.d.tune_qilp > 0) {
    const unsigned g = grid_for(a.n);
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
}
Launchers launchers_chaining() { return Launchers{chaining_ops, chaining_query, chaining_locate, chaining_preload}; }

}  // namespace ws

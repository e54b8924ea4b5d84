// Kernel instantiations for the p2 design (see ws_kernels.cuh), plus a
// line-at-a-time lock-free query for the default 32-slot buckets.
#include "ws_kernels.cuh"
#include "ws_scan32.cuh"

namespace ws {

// P2 query (reference openaddr.py:433-447, Ctx::p2_find with the early exit):
// scan b0; stop if found, or if b0 holds an EMPTY cell, the table never
// tombstoned and b0 is below the shortcut threshold; else scan b1.
template <bool RO>
__global__ void __launch_bounds__(256) k_query_p2_lines(Dev d, const u64* __restrict__ keys, u64 n, u64* vout,
                                                        u8* found, int conc_erase, int gated) {
  if (gated && (ld_u32_relaxed(d.state + 2) | ld_u32_relaxed(d.state + 3))) return;
  const u32 te0 = ld_u32_relaxed(d.state);
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
    const u64 key = __ldg(keys + i);
    const u64 b0 = d.nbm(mix64(key ^ d.seeds[0]) >> 16);
    i64 idx, hint;
    u64 val = 0;
    int used;
    bool saw_empty;
    scan32_lines<RO>(d.cells, b0 * 32, key, idx, val, used, hint, saw_empty);
    if (idx < 0) {
      bool te = te0 != 0;
      if (conc_erase) { fence_acq_rel(); te = ld_u32_relaxed(d.state) != 0; }
      if (!(saw_empty && !te && used < d.shortcut)) {
        const u64 b1 = d.nbm(mix64(key ^ d.seeds[1]) >> 16);
        if (b1 != b0) scan32_lines<RO>(d.cells, b1 * 32, key, idx, val, used, hint, saw_empty);
      }
    }
    if (found) found[i] = idx >= 0;
    if (vout) vout[i] = idx >= 0 ? val : 0;
  }
}

static void p2_ops(const OpsArgs& a, bool def) {
  if (def) launch_ops_t<D_P2, 32>(a); else launch_ops_t<D_P2, 0>(a);
}
static void p2_query(const QueryArgs& a, bool def) {
  if (def && a.d.tune_qilp > 0) {
    const unsigned g = grid_for(a.n);
    if (a.ro) k_query_p2_lines<true><<<g, kThreads, 0, a.s>>>(a.d, a.keys, a.n, a.vout, a.found, a.conc_erase, a.gated);
    else k_query_p2_lines<false><<<g, kThreads, 0, a.s>>>(a.d, a.keys, a.n, a.vout, a.found, a.conc_erase, a.gated);
    return;
  }
  if (def) launch_query_t<D_P2, 32>(a); else launch_query_t<D_P2, 0>(a);
}
static void p2_locate(const LocateArgs& a, bool def) {
  if (def) launch_locate_t<D_P2, 32>(a); else launch_locate_t<D_P2, 0>(a);
}
static void p2_preload(bool def) {
  if (!def) { preload_t<D_P2, 0>(); return; }
  preload_t<D_P2, 32>();
  preload_fn(k_query_p2_lines<false>);
  preload_fn(k_query_p2_lines<true>);
}
Launchers launchers_p2() { return Launchers{p2_ops, p2_query, p2_locate, p2_preload}; }

}  // namespace ws

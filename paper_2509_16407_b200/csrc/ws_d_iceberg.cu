// Kernel instantiations for the iceberg design (see ws_kernels.cuh), plus a
// line-at-a-time lock-free query for the default 32-slot buckets.
#include "ws_kernels.cuh"
#include "ws_scan32.cuh"

namespace ws {

// Iceberg query (reference openaddr.py:589-609, Ctx::ice_find with the early
// exit): scan the front bucket; stop if found or if it holds an EMPTY cell;
// else scan the backyard pair.
template <bool RO>
__global__ void __launch_bounds__(256) k_query_ice_lines(Dev d, const u64* __restrict__ keys, u64 n, u64* vout,
                                                         u8* found, int gated) {
  if (gated && (ld_u32_relaxed(d.state + 2) | ld_u32_relaxed(d.state + 3))) return;
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
    const u64 key = __ldg(keys + i);
    const u64 b0 = d.frontm(mix64(key ^ d.seeds[0]) >> 16);
    i64 idx, hint;
    u64 val = 0;
    int used;
    bool saw_empty;
    scan32_lines<RO>(d.cells, b0 * 32, key, idx, val, used, hint, saw_empty);
    if (idx < 0 && !saw_empty) {
      const u64 b1 = d.front + d.backm(mix64(key ^ d.seeds[1]) >> 16);
      const u64 b2 = d.front + d.backm(mix64(key ^ d.seeds[2]) >> 16);
      scan32_lines<RO>(d.cells, b1 * 32, key, idx, val, used, hint, saw_empty);
      if (idx < 0 && b2 != b1) scan32_lines<RO>(d.cells, b2 * 32, key, idx, val, used, hint, saw_empty);
    }
    if (found) found[i] = idx >= 0;
    if (vout) vout[i] = idx >= 0 ? val : 0;
  }
}

static void iceberg_ops(const OpsArgs& a, bool def) {
  if (def) launch_ops_t<D_ICEBERG, 32>(a); else launch_ops_t<D_ICEBERG, 0>(a);
}
static void iceberg_query(const QueryArgs& a, bool def) {
  if (def && a.d.tune_qilp > 0) {
    const unsigned g = grid_for(a.n);
    if (a.ro) k_query_ice_lines<true><<<g, kThreads, 0, a.s>>>(a.d, a.keys, a.n, a.vout, a.found, a.gated);
    else k_query_ice_lines<false><<<g, kThreads, 0, a.s>>>(a.d, a.keys, a.n, a.vout, a.found, a.gated);
    return;
  }
  if (def) launch_query_t<D_ICEBERG, 32>(a); else launch_query_t<D_ICEBERG, 0>(a);
}
static void iceberg_locate(const LocateArgs& a, bool def) {
  if (def) launch_locate_t<D_ICEBERG, 32>(a); else launch_locate_t<D_ICEBERG, 0>(a);
}
static void iceberg_preload(bool def) {
  if (!def) { preload_t<D_ICEBERG, 0>(); return; }
  preload_t<D_ICEBERG, 32>();
  preload_fn(k_query_ice_lines<false>);
  preload_fn(k_query_ice_lines<true>);
}
Launchers launchers_iceberg() { return Launchers{iceberg_ops, iceberg_query, iceberg_locate, iceberg_preload}; }

}  // namespace ws

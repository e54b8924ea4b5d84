// Kernel instantiations for the p2_md design (the headline path): the
// generic kernels of ws_kernels.cuh plus the tuned kernels of ws_fast.cuh --
// the pair-cooperative query, the lock-round upsert and the fused mixed /
// erase kernel.  Knob values (ws_tune): upsert 4 = lock rounds + 64-byte L2
// fills + whole-sector cell writes (default), 3 = without the whole-sector
// writes, 2 = without the 64-byte fills, 0 = the generic kernel; query_ilp
// > 0 = the pair-cooperative query (default), 0 = the generic kernel.
#include "ws_fast.cuh"
#include "ws_kernels.cuh"

#include <algorithm>

namespace ws {

static void p2_md_ops(const OpsArgs& a, bool def) {
  const bool upsert_only = !a.ops && (a.uop & 15) == OP_UPSERT;
  // mixed launches (interleaved / small batches, the split's remainder) and
  // uniform erases: the fused lock-round kernel
  if (def && (a.ops || (a.uop & 15) == OP_ERASE) && !a.instr && !a.d.delay_ns && !a.serial && !a.redo &&
      !a.rlist && !a.d.phased && !a.d.lock_elided && a.d.tune_upsert == 4) {
    u64 g = (a.n + 255) / 256;
    const u64 lim = std::max<u64>((a.d.nb + 255) / 256, 4);  // <= ~1 op in flight per bucket
    g = std::max<u64>(std::min<u64>(std::min<u64>(g, (u64)kSMs * table_grid_per_sm(a.d)), lim), 1);
    k_mixed_p2md_rounds<3><<<(unsigned)g, 256, 0, a.s>>>(a.d, a.ops, a.uop, a.keys, a.vals, a.n, a.status, a.vout,
                                                          a.conc_erase, a.gated);
    return;
  }
  if (def && upsert_only && !a.instr && !a.d.delay_ns && !a.serial && !a.redo && !a.d.lock_elided &&
      a.d.tune_upsert >= 2) {
    u64 g = (a.n + 255) / 256;
    const u64 lim = std::max<u64>((a.d.nb + 255) / 256, 4);  // <= ~1 op in flight per bucket
    g = std::max<u64>(std::min<u64>(std::min<u64>(g, (u64)kSMs * table_grid_per_sm(a.d)), lim), 1);
#define WS_UR(F, PH, FI) k_upsert_p2md_rounds<F, 4, PH, FI><<<(unsigned)g, 256, 0, a.s>>>(a.d, a.keys, a.vals, \
                                                   a.n, a.uop >> 4, a.status, a.conc_erase, a.gated)
    if (a.d.phased) { if (a.d.tune_upsert >= 3) WS_UR(true, true, false); else WS_UR(false, true, false); }
    else if (a.d.tune_upsert >= 4) WS_UR(true, false, true);
    else if (a.d.tune_upsert == 3) WS_UR(true, false, false);
    else WS_UR(false, false, false);
#undef WS_UR
    return;
  }
  if (def) launch_ops_t<D_P2_MD, 32>(a); else launch_ops_t<D_P2_MD, 0>(a);
}
static void p2_md_query(const QueryArgs& a, bool def) {
  if (!def || a.d.tune_qilp <= 0) {
    if (def) launch_query_t<D_P2_MD, 32>(a); else launch_query_t<D_P2_MD, 0>(a);
    return;
  }
  // one thread per op, pair-cooperative tag fetches
  u64 g = (a.n + 255) / 256;
  g = std::min<u64>(std::max<u64>(g, 1), (u64)kSMs * table_grid_per_sm(a.d));
#define WS_QC(RO, F) k_query_p2md_coop<RO, F, 5><<<(unsigned)g, 256, 0, a.s>>>(a.d, a.keys, a.n, a.vout, a.found, \
                                                                              a.conc_erase, a.gated, a.check_keys)
  const bool f64 = a.d.tune_l2pol == 2;
  if (a.ro) { if (f64) WS_QC(true, true); else WS_QC(true, false); }
  else { if (f64) WS_QC(false, true); else WS_QC(false, false); }
#undef WS_QC
}
static void p2_md_locate(const LocateArgs& a, bool def) {
  if (def) launch_locate_t<D_P2_MD, 32>(a); else launch_locate_t<D_P2_MD, 0>(a);
}
static void p2_md_preload(bool def) {
  if (!def) { preload_t<D_P2_MD, 0>(); return; }
  preload_t<D_P2_MD, 32>();
  preload_fn(k_query_p2md_coop<false, true, 5>);
  preload_fn(k_query_p2md_coop<true, true, 5>);
  preload_fn(k_upsert_p2md_rounds<true, 4, false, true>);
  preload_fn(k_upsert_p2md_rounds<true, 4, true>);
  preload_fn(k_mixed_p2md_rounds<3>);
}

Launchers launchers_p2_md() { return Launchers{p2_md_ops, p2_md_query, p2_md_locate, p2_md_preload}; }

}  // namespace ws

// Kernel instantiations for the p2_md design (the headline path): the generic
// kernels of ws_kernels.cuh plus the tuned multi-lookup query of ws_fast.cuh.
#include "ws_fast.cuh"
#include "ws_kernels.cuh"

#include <algorithm>

namespace ws {

template <int Q, bool RO, int POL>
static void launch_fast_query(const QueryArgs& a) {
  u64 g = (a.n + 256ull * Q - 1) / (256ull * Q);
  if (g > (u64)kSMs * 8) g = (u64)kSMs * 8;
  if (!g) g = 1;
  k_query_p2md<Q, RO, POL><<<(unsigned)g, 256, 0, a.s>>>(a.d, a.keys, a.n, a.vout, a.found, a.conc_erase,
                                                         a.gated);
}

template <int Q>
static void fast_query_q(const QueryArgs& a) {
  const bool pol = a.d.tune_l2pol == 1;
  if (a.ro) { if (pol) launch_fast_query<Q, true, 1>(a); else launch_fast_query<Q, true, 0>(a); }
  else { if (pol) launch_fast_query<Q, false, 1>(a); else launch_fast_query<Q, false, 0>(a); }
}

static void p2_md_ops(const OpsArgs& a, bool def) {
  // lane-pair upsert: uniform-upsert launches on exclusive (locked) tables
  const bool upsert_only = !a.ops && (a.uop & 15) == OP_UPSERT;
  // mixed launches (interleaved / small batches, the split's remainder) and
  // uniform erases: the fused lock-round kernel
  if (def && (a.ops || (a.uop & 15) == OP_ERASE) && !a.instr && !a.d.delay_ns && !a.serial && !a.redo &&
      !a.rlist && !a.d.phased && !a.d.lock_elided && a.d.tune_upsert == 4) {
    u64 g = (a.n + 255) / 256;
    const u64 lim = std::max<u64>((a.d.nb + 255) / 256, 4);  // <= ~1 op in flight per bucket
    g = std::max<u64>(std::min<u64>(std::min<u64>(g, (u64)kSMs * 8), lim), 1);
    k_mixed_p2md_rounds<1><<<(unsigned)g, 256, 0, a.s>>>(a.d, a.ops, a.uop, a.keys, a.vals, a.n, a.status, a.vout,
                                                          a.conc_erase, a.gated);
    return;
  }
  if (def && upsert_only && !a.instr && !a.serial && !a.redo && !a.d.phased && !a.d.lock_elided &&
      a.d.tune_upsert == 1) {
    u64 g = (2 * a.n + 255) / 256;
    const u64 lim = std::max<u64>((2 * a.d.nb + 255) / 256, 4);  // <= ~1 op in flight per bucket
    g = std::min<u64>(std::min<u64>(g, (u64)kSMs * 8), lim);
    k_upsert_p2md_pair<<<(unsigned)std::max<u64>(g, 1), 256, 0, a.s>>>(a.d, a.keys, a.vals, a.n, a.uop >> 4,
                                                                       a.status, a.conc_erase, a.gated);
    return;
  }
  if (def && upsert_only && !a.instr && !a.d.delay_ns && !a.serial && !a.redo && !a.d.lock_elided && a.d.tune_upsert >= 2) {
    u64 g = (a.n + 255) / 256;
    const u64 lim = std::max<u64>((a.d.nb + 255) / 256, 4);  // <= ~1 op in flight per bucket
    g = std::max<u64>(std::min<u64>(std::min<u64>(g, (u64)kSMs * 8), lim), 1);
#define WS_UR(F, MB, PH) k_upsert_p2md_rounds<F, MB, PH><<<(unsigned)g, 256, 0, a.s>>>(a.d, a.keys, a.vals, \
                                                   a.n, a.uop >> 4, a.status, a.conc_erase, a.gated)
    const bool f64 = a.d.tune_upsert >= 3;
    if (a.d.tune_upsert == 5 && !a.d.phased) {
      k_upsert_p2md_rounds<true, 1, false, true, true><<<(unsigned)g, 256, 0, a.s>>>(
          a.d, a.keys, a.vals, a.n, a.uop >> 4, a.status, a.conc_erase, a.gated);
    } else if (a.d.tune_upsert == 4 && !a.d.phased && a.d.tune_occ == 4) {
      k_upsert_p2md_rounds<true, 4, false, true><<<(unsigned)g, 256, 0, a.s>>>(a.d, a.keys, a.vals, a.n,
                                                                                a.uop >> 4, a.status,
                                                                                a.conc_erase, a.gated);
    } else if (a.d.tune_upsert == 4 && !a.d.phased && a.d.tune_occ == 5) {
      k_upsert_p2md_rounds<true, 5, false, true><<<(unsigned)g, 256, 0, a.s>>>(a.d, a.keys, a.vals, a.n,
                                                                                a.uop >> 4, a.status,
                                                                                a.conc_erase, a.gated);
    } else if (a.d.tune_upsert == 4 && !a.d.phased) {
      k_upsert_p2md_rounds<true, 1, false, true><<<(unsigned)g, 256, 0, a.s>>>(a.d, a.keys, a.vals, a.n,
                                                                                a.uop >> 4, a.status,
                                                                                a.conc_erase, a.gated);
    } else if (a.d.phased) {
      if (f64) WS_UR(true, 1, true); else WS_UR(false, 1, true);
    } else {
      switch (a.d.tune_occ) {
        case 5: if (f64) WS_UR(true, 5, false); else WS_UR(false, 5, false); break;
        case 6: if (f64) WS_UR(true, 6, false); else WS_UR(false, 6, false); break;
        default: if (f64) WS_UR(true, 1, false); else WS_UR(false, 1, false); break;
      }
    }
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
  switch (a.d.tune_qilp) {
    case 3: {  // lane-pair tile (one line request per tag block)
      u64 g = (2 * a.n + 255) / 256;
      g = std::min<u64>(std::max<u64>(g, 1), (u64)kSMs * 8);
#define WS_QP(RO, F) k_query_p2md_pair<RO, F><<<(unsigned)g, 256, 0, a.s>>>(a.d, a.keys, a.n, a.vout, a.found, a.conc_erase, a.gated)
      const bool f64 = a.d.tune_l2pol == 2;
      if (a.ro) { if (f64) WS_QP(true, true); else WS_QP(true, false); }
      else { if (f64) WS_QP(false, true); else WS_QP(false, false); }
#undef WS_QP
      break;
    }
    case 5: {  // one thread per op, pair-cooperative tag fetches
      u64 g = (a.n + 255) / 256;
      g = std::min<u64>(std::max<u64>(g, 1), (u64)kSMs * 8);
#define WS_QC(RO, F, MB) k_query_p2md_coop<RO, F, MB><<<(unsigned)g, 256, 0, a.s>>>(a.d, a.keys, a.n, a.vout, a.found, a.conc_erase, a.gated)
#define WS_QC2(MB) \
  if (a.ro) { if (f64) WS_QC(true, true, MB); else WS_QC(true, false, MB); } \
  else { if (f64) WS_QC(false, true, MB); else WS_QC(false, false, MB); }
      const bool f64 = a.d.tune_l2pol == 2;
      if (a.d.tune_occ == 8) { WS_QC2(8) } else { WS_QC2(1) }
#undef WS_QC2
#undef WS_QC
      break;
    }
    case 1: fast_query_q<1>(a); break;
    case 2: fast_query_q<2>(a); break;
    case 8: fast_query_q<8>(a); break;
    default: fast_query_q<4>(a); break;
  }
}
static void p2_md_locate(const LocateArgs& a, bool def) {
  if (def) launch_locate_t<D_P2_MD, 32>(a); else launch_locate_t<D_P2_MD, 0>(a);
}
static void p2_md_preload(bool def) {
  if (!def) { preload_t<D_P2_MD, 0>(); return; }
  preload_t<D_P2_MD, 32>();
  preload_fn(k_query_p2md_coop<false, true, 1>);
  preload_fn(k_query_p2md_coop<true, true, 1>);
  preload_fn(k_upsert_p2md_rounds<true, 1, false, true>);
  preload_fn(k_upsert_p2md_rounds<true, 1, true>);
  preload_fn(k_mixed_p2md_rounds<1>);
}

Launchers launchers_p2_md() { return Launchers{p2_md_ops, p2_md_query, p2_md_locate, p2_md_preload}; }

}  // namespace ws

// Kernel instantiations for the double_md design (see ws_kernels.cuh), plus a
// lock-round upsert for uniform-upsert launches.
#include "ws_kernels.cuh"

#include <algorithm>

namespace ws {

// Double-hashing-MD upsert (reference openaddr.py:232-264 with the md
// find of :247) in warp-synchronous lock rounds: each lane try-locks its
// primary bucket (never blocks); holders run the generic body
// (Ctx::dbl_upsert_held: tag-filtered probe walk, CAS claim of the first
// reusable slot); then ONE fence per warp-round and relaxed releases of the
// finished lanes, instead of an acquire/release pair per op.
__global__ void __launch_bounds__(256) k_upsert_dblmd_rounds(Dev d, const u64* __restrict__ keys,
                                                             const u64* __restrict__ vals, u64 n, int merge,
                                                             u8* status, int conc_erase, int gated) {
  WS_PROLOGUE(d, gated, n);
  Ctx<D_DOUBLE_MD, 32, false, false> c{d, nullptr, conc_erase != 0, ld_u32_relaxed(d.state)};
  const int lane = threadIdx.x & 31;
  const u64 nwarps = ((u64)gridDim.x * blockDim.x) >> 5;
  for (u64 w = (blockIdx.x * (u64)blockDim.x + threadIdx.x) >> 5; w * 32 < n; w += nwarps) {
    const u64 i = w * 32 + lane;
    bool pending = i < n;
    const u64 key = pending ? __ldg(keys + i) : 0;
    const u64 val = pending ? __ldg(vals + i) : 0;
    const u64 b0 = d.nbm(mix64(key ^ d.seeds[0]) >> 16);
    bool held = false;
    u8 st = S_INSERTED;
    unsigned backoff = 64;
    while (__any_sync(0xFFFFFFFFu, pending)) {
      if (pending && !held) held = try_lock_bucket(d.locks, b0);
      if (pending && held) {
        st = c.dbl_upsert_held(key, val, merge);
        pending = false;
      }
      __syncwarp();
      fence_acq_rel();
      if (!pending && held) {
        asm volatile("red.relaxed.gpu.global.and.b32 [%0], %1;" ::"l"(d.locks + (b0 >> 5)), "r"(~(1u << (b0 & 31)))
                     : "memory");
        held = false;
      }
      if (pending) {
        __nanosleep(backoff + 8 * lane);
        if (backoff < 4096) backoff <<= 1;
      }
    }
    if (i < n && status) status[i] = st;
  }
}

static void double_md_ops(const OpsArgs& a, bool def) {
  const bool upsert_only = !a.ops && (a.uop & 15) == OP_UPSERT;
  if (def && upsert_only && !a.instr && !a.d.delay_ns && !a.serial && !a.redo && !a.d.phased && !a.d.lock_elided &&
      a.d.tune_upsert == 4) {
    u64 g = (a.n + 255) / 256;
    const u64 lim = std::max<u64>((a.d.nb + 255) / 256, 4);  // <= ~1 op in flight per bucket
    g = std::max<u64>(std::min<u64>(std::min<u64>(g, (u64)kSMs * 8), lim), 1);
    k_upsert_dblmd_rounds<<<(unsigned)g, 256, 0, a.s>>>(a.d, a.keys, a.vals, a.n, a.uop >> 4, a.status,
                                                        a.conc_erase, a.gated);
    return;
  }
  if (def) launch_ops_t<D_DOUBLE_MD, 32>(a); else launch_ops_t<D_DOUBLE_MD, 0>(a);
}
static void double_md_query(const QueryArgs& a, bool def) {
  if (def) launch_query_t<D_DOUBLE_MD, 32>(a); else launch_query_t<D_DOUBLE_MD, 0>(a);
}
static void double_md_locate(const LocateArgs& a, bool def) {
  if (def) launch_locate_t<D_DOUBLE_MD, 32>(a); else launch_locate_t<D_DOUBLE_MD, 0>(a);
}
static void double_md_preload(bool def) {
  if (!def) { preload_t<D_DOUBLE_MD, 0>(); return; }
  preload_t<D_DOUBLE_MD, 32>();
  preload_fn(k_upsert_dblmd_rounds);
}
Launchers launchers_double_md() {
  return Launchers{double_md_ops, double_md_query, double_md_locate, double_md_preload};
}

}  // namespace ws

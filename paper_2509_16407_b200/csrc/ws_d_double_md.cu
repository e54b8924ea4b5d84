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

// Mixed batches in ONE launch (interleaved / small mixed batches, the split's
// remainder) and uniform erases, for both double-hashing designs: the lock
// rounds above with erase lanes (primary lock held: Ctx::dbl_find, then
// Ctx::tombstone -- reference openaddr.py:300-318) and lock-free query lanes
// (Ctx::query, openaddr.py:266-298) that finish in the first round.  Op bytes
// of another kind run as queries (Ctx::run).
template <int DES, int BS>
__global__ void __launch_bounds__(256) k_mixed_dbl_rounds(Dev d, const u8* __restrict__ ops, u8 uop,
                                                          const u64* __restrict__ keys, const u64* __restrict__ vals,
                                                          u64 n, u8* status, u64* vout, int conc_erase, int gated) {
  WS_PROLOGUE(d, gated, n);
  const bool conc = conc_erase == 2 ? ld_u32_relaxed(d.cs + 3) != 0 : conc_erase != 0;
  Ctx<DES, BS, false, false> c{d, nullptr, conc, ld_u32_relaxed(d.state)};
  const int lane = threadIdx.x & 31;
  const u64 nwarps = ((u64)gridDim.x * blockDim.x) >> 5;
  for (u64 w = (blockIdx.x * (u64)blockDim.x + threadIdx.x) >> 5; w * 32 < n; w += nwarps) {
    const u64 i = w * 32 + lane;
    bool pending = i < n;
    int kind = OP_QUERY, merge = 0;
    u64 key = 0, val = 0;
    if (pending) {
      const u8 op = ops ? __ldg(ops + i) : uop;
      kind = op & 15;
      if (kind > OP_QUERY) kind = OP_QUERY;
      merge = op >> 4;
      key = __ldg(keys + i);
      val = vals ? __ldg(vals + i) : 0ull;
    }
    const u64 b0 = d.nbm(mix64(key ^ d.seeds[0]) >> 16);
    bool held = false;
    u8 st = 0;
    u64 qv = 0;
    unsigned backoff = 64;
    while (__any_sync(0xFFFFFFFFu, pending)) {
      if (pending && kind == OP_QUERY) {
        st = c.template query<DES>(key, qv) ? 1 : 0;
        pending = false;
      }
      if (pending && !held) held = try_lock_bucket(d.locks, b0);
      if (pending && held) {
        if (kind == OP_UPSERT) {
          st = c.dbl_upsert_held(key, val, merge);
        } else {
          u64 v;
          const i64 idx = c.dbl_find(key, v);
          if (idx >= 0) c.tombstone((u64)idx);
          st = idx >= 0;
        }
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
    if (i < n) {
      if (status) status[i] = st;
      if (vout) vout[i] = kind == OP_QUERY ? qv : 0;
    }
  }
}

void launch_mixed_dbl(const OpsArgs& a, bool md) {
  u64 g = (a.n + 255) / 256;
  const u64 lim = std::max<u64>((a.d.nb + 255) / 256, 4);  // <= ~1 op in flight per bucket
  g = std::max<u64>(std::min<u64>(std::min<u64>(g, (u64)kSMs * table_grid_per_sm(a.d)), lim), 1);
  if (md)
    k_mixed_dbl_rounds<D_DOUBLE_MD, 32><<<(unsigned)g, 256, 0, a.s>>>(a.d, a.ops, a.uop, a.keys, a.vals, a.n,
                                                                      a.status, a.vout, a.conc_erase, a.gated);
  else
    k_mixed_dbl_rounds<D_DOUBLE, 8><<<(unsigned)g, 256, 0, a.s>>>(a.d, a.ops, a.uop, a.keys, a.vals, a.n,
                                                                  a.status, a.vout, a.conc_erase, a.gated);
}

// mixed launches / uniform erases that the fused kernel serves (no
// instrumentation, serial replay, delay injection, redo lists or phased mode)
bool mixed_dbl_ok(const OpsArgs& a) {
  return (a.ops || (a.uop & 15) == OP_ERASE) && !a.instr && !a.d.delay_ns && !a.serial && !a.redo && !a.rlist &&
         !a.d.phased && !a.d.lock_elided && a.d.tune_upsert == 4;
}

static void double_md_ops(const OpsArgs& a, bool def) {
  if (def && mixed_dbl_ok(a)) {
    launch_mixed_dbl(a, true);
    return;
  }
  const bool upsert_only = !a.ops && (a.uop & 15) == OP_UPSERT;
  if (def && upsert_only && !a.instr && !a.d.delay_ns && !a.serial && !a.redo && !a.d.phased && !a.d.lock_elided &&
      a.d.tune_upsert == 4) {
    u64 g = (a.n + 255) / 256;
    const u64 lim = std::max<u64>((a.d.nb + 255) / 256, 4);  // <= ~1 op in flight per bucket
    g = std::max<u64>(std::min<u64>(std::min<u64>(g, (u64)kSMs * table_grid_per_sm(a.d)), lim), 1);
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
  preload_fn(k_mixed_dbl_rounds<D_DOUBLE_MD, 32>);
}
Launchers launchers_double_md() {
  return Launchers{double_md_ops, double_md_query, double_md_locate, double_md_preload};
}

}  // namespace ws

// Kernel instantiations for the cuckoo design (see ws_kernels.cuh), plus the
// tuned lock-round query for the default 8-slot buckets.
#include "ws_kernels.cuh"

#include <algorithm>

namespace ws {

// 32 bytes (two cells) in one LDG.E.ENL2.256
__device__ __forceinline__ void ld_cells2(const u64* p, u64& k0, u64& v0, u64& k1, u64& v1) {
  asm volatile("ld.relaxed.gpu.global.v4.u64 {%0,%1,%2,%3}, [%4];"
               : "=l"(k0), "=l"(v0), "=l"(k1), "=l"(v1) : "l"(p) : "memory");
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
__global__ void __launch_bounds__(256) k_query_cuckoo_rounds(Dev d, const u64* __restrict__ keys, u64 n,
                                                             u64* vout, u8* found, int gated) {
  if (gated && (ld_u32_relaxed(d.state + 2) | ld_u32_relaxed(d.state + 3))) return;
  const int lane = threadIdx.x & 31;
  const u64 nwarps = ((u64)gridDim.x * blockDim.x) >> 5;
  const bool locked = !d.phased;
  for (u64 c = (blockIdx.x * (u64)blockDim.x + threadIdx.x) >> 5; c * 32 < n; c += nwarps) {
    const u64 i = c * 32 + lane;
    bool pending = i < n;
    const u64 key = pending ? __ldg(keys + i) : 0;
    u64 uq[8], srt[8];
    int nu = 0;
    if (pending) {
      for (int w = 0; w < d.ways; w++) {  // dict.fromkeys(buckets): hash order, deduplicated
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
    bool hit = false;
    u64 val = 0;
    unsigned backoff = 64;
    while (__any_sync(0xFFFFFFFFu, pending)) {
      if (pending && locked)
        while (held < nu && try_lock_bucket(d.locks, srt[held])) held++;
      const bool ready = pending && (!locked || held == nu);
      if (ready) {
        for (int q = 0; q < nu && !hit; q++) {
          const u64* base = d.cells + 2 * (uq[q] * 8);
          bool empty = false;
#pragma unroll
          for (int h = 0; h < 4; h++) {
            if (empty || hit) break;
            u64 k0, v0, k1, v1;
            ld_cells2(base + 4 * h, k0, v0, k1, v1);
            if (k0 == key) { hit = true; val = v0; }
            else if (k0 == EMPTY) empty = true;
            else if (k1 == key) { hit = true; val = v1; }
            else if (k1 == EMPTY) empty = true;
          }
        }
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
    if (i < n) {
      if (found) found[i] = hit;
      if (vout) vout[i] = hit ? val : 0;
    }
  }
}

static void cuckoo_ops(const OpsArgs& a, bool def) {
  if (def) launch_ops_t<D_CUCKOO, 8>(a); else launch_ops_t<D_CUCKOO, 0>(a);
}
static void cuckoo_query(const QueryArgs& a, bool def) {
  if (def && a.d.ways <= 8 && a.d.tune_qilp > 0) {
    u64 g = (a.n + 255) / 256;
    g = std::max<u64>(std::min<u64>(g, (u64)kSMs * 8), 1);
    k_query_cuckoo_rounds<<<(unsigned)g, 256, 0, a.s>>>(a.d, a.keys, a.n, a.vout, a.found, a.gated);
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
  preload_fn(k_query_cuckoo_rounds);
}
Launchers launchers_cuckoo() { return Launchers{cuckoo_ops, cuckoo_query, cuckoo_locate, cuckoo_preload}; }

}  // namespace ws

// ws_shard.cu -- routing kernels of the hash-sharded multi-GPU table.
//
// A key's owner GPU is the top log2(G) bits of its primary hash
// h0 = mix64(k ^ seed0); the local table indexes bucket bits 16..16+log2(nb),
// so owner and bucket are independent.  A batch is split into
// per-owner contiguous segments (a two-pass counting partition: per-CTA
// histograms, one exclusive scan, per-CTA scatter), exchanged with one
// all-to-all, applied locally, and the results are returned by the reverse
// all-to-all and scattered back to the caller's order with the permutation.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>

#include <cub/cub.cuh>

#include "warpspeed.h"
#include "ws_ops.cuh"

using namespace ws;

namespace {

constexpr int kPartThreads = 256;
constexpr int kMaxParts = 64;

__device__ __forceinline__ u32 owner_of(u64 key, u64 seed0, int shift) {
  return shift >= 64 ? 0u : (u32)(mix64(key ^ seed0) >> shift);
}

__global__ void k_part_count(const u64* __restrict__ keys, u64 n, u64 chunk, u64 seed0, int shift, int parts,
                             u64* block_counts) {
  __shared__ u32 cnt[kMaxParts];
  for (int p = threadIdx.x; p < parts; p += blockDim.x) cnt[p] = 0;
  __syncthreads();
  const u64 lo = blockIdx.x * chunk, hi = lo + chunk < n ? lo + chunk : n;
  for (u64 i = lo + threadIdx.x; i < hi; i += blockDim.x) atomicAdd(&cnt[owner_of(__ldg(keys + i), seed0, shift)], 1u);
  __syncthreads();
  for (int p = threadIdx.x; p < parts; p += blockDim.x) block_counts[(u64)p * gridDim.x + blockIdx.x] = cnt[p];
}

__global__ void k_part_scatter(const u64* __restrict__ keys, const u64* __restrict__ vals, const u8* __restrict__ ops,
                               u64 n, u64 chunk, u64 seed0, int shift, int parts, const u64* offsets,
                               u64* out_keys, u64* out_vals, u8* out_ops, u32* perm) {
  __shared__ u64 base[kMaxParts];
  __shared__ u32 cur[kMaxParts];
  for (int p = threadIdx.x; p < parts; p += blockDim.x) {
    base[p] = offsets[(u64)p * gridDim.x + blockIdx.x];
    cur[p] = 0;
  }
  __syncthreads();
  const u64 lo = blockIdx.x * chunk, hi = lo + chunk < n ? lo + chunk : n;
  for (u64 i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    const u64 k = __ldg(keys + i);
    const u32 o = owner_of(k, seed0, shift);
    const u64 pos = base[o] + atomicAdd(&cur[o], 1u);
    out_keys[pos] = k;
    if (vals) out_vals[pos] = __ldg(vals + i);
    if (ops) out_ops[pos] = __ldg(ops + i);
    perm[pos] = (u32)i;
  }
}

__global__ void k_part_totals(const u64* offsets, int parts, int blocks, u64 n, u64* counts) {
  const int p = threadIdx.x;
  if (p < parts) {
    const u64 a = offsets[(u64)p * blocks];
    const u64 b = p + 1 < parts ? offsets[(u64)(p + 1) * blocks] : n;
    counts[p] = b - a;
  }
}

template <typename T>
__global__ void k_unpermute(const T* __restrict__ in, const u32* __restrict__ perm, u64 n, T* out) {
  for (u64 j = blockIdx.x * (u64)blockDim.x + threadIdx.x; j < n; j += (u64)gridDim.x * blockDim.x)
    out[__ldg(perm + j)] = in[j];
}

}  // namespace

extern "C" {

WS_API int ws_partition(const uint64_t* keys, const uint64_t* vals, const uint8_t* ops, uint64_t n,
                        uint64_t seed0, int log2_parts, uint64_t* out_keys, uint64_t* out_vals,
                        uint8_t* out_ops, uint32_t* perm, uint64_t* counts, void* stream) {
  if (log2_parts < 0 || log2_parts > 6 || n >= (1ull << 32) || (n && (!keys || !out_keys || !perm)) || !counts)
    return WS_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  const int parts = 1 << log2_parts;
  const int shift = log2_parts ? 64 - log2_parts : 64;
  if (!n) return cudaMemsetAsync(counts, 0, 8 * parts, s) == cudaSuccess ? WS_OK : WS_ERR_CUDA;
  int blocks = 148 * 8;
  u64 chunk = (n + blocks - 1) / blocks;
  if (chunk < 1024) {
    chunk = 1024;
    blocks = (int)((n + chunk - 1) / chunk);
  }
  const u64 nbc = (u64)parts * blocks;
  u64 *bc = nullptr, *off = nullptr;
  void* tmp = nullptr;
  size_t tb = 0;
  if (cudaMallocAsync((void**)&bc, 8 * nbc, s) != cudaSuccess) return WS_ERR_ALLOC;
  if (cudaMallocAsync((void**)&off, 8 * nbc, s) != cudaSuccess) return WS_ERR_ALLOC;
  k_part_count<<<blocks, kPartThreads, 0, s>>>((const u64*)keys, n, chunk, seed0, shift, parts, bc);
  cub::DeviceScan::ExclusiveSum(nullptr, tb, bc, off, (int64_t)nbc, s);
  if (cudaMallocAsync(&tmp, tb + 16, s) != cudaSuccess) return WS_ERR_ALLOC;
  cub::DeviceScan::ExclusiveSum(tmp, tb, bc, off, (int64_t)nbc, s);
  k_part_scatter<<<blocks, kPartThreads, 0, s>>>((const u64*)keys, (const u64*)vals, ops, n, chunk, seed0, shift,
                                                 parts, off, (u64*)out_keys, (u64*)out_vals, out_ops, perm);
  k_part_totals<<<1, 64, 0, s>>>(off, parts, blocks, n, (u64*)counts);
  cudaFreeAsync(tmp, s);
  cudaFreeAsync(bc, s);
  cudaFreeAsync(off, s);
  return cudaGetLastError() == cudaSuccess ? WS_OK : WS_ERR_CUDA;
}

WS_API int ws_unpermute(const void* in, const uint32_t* perm, uint64_t n, int elem_bytes, void* out,
                        void* stream) {
  if (!n) return WS_OK;
  if (!in || !perm || !out) return WS_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  u64 g = (n + 255) / 256;
  if (g > 148 * 8) g = 148 * 8;
  switch (elem_bytes) {
    case 1: k_unpermute<u8><<<(unsigned)g, 256, 0, s>>>((const u8*)in, perm, n, (u8*)out); break;
    case 4: k_unpermute<u32><<<(unsigned)g, 256, 0, s>>>((const u32*)in, perm, n, (u32*)out); break;
    case 8: k_unpermute<u64><<<(unsigned)g, 256, 0, s>>>((const u64*)in, perm, n, (u64*)out); break;
    default: return WS_ERR_ARG;
  }
  return cudaGetLastError() == cudaSuccess ? WS_OK : WS_ERR_CUDA;
}

}  // extern "C"

// ============================================================================
// Fused routing over NVLink peer memory ("xchg").
//
// Every rank owns one IPC-exported region:
//   inbox  keys / vals / src / ops   world x C entries  (segment s <- rank s)
//   incoming[world]                   entries rank s wrote into segment s
//   result  status / value            world x C (local results of the inbox)
//   reply   status / value            C          (results for MY ops, written by owners)
//   bar                               barrier counter (peers add, owner waits)
// A round moves up to C of this rank's ops:
//   1. k_xs_send: owner of each op, warp-aggregated position in the owner's
//      segment `rank` (local counters: the sender owns that segment), keys /
//      vals / op bytes / source index stored straight into the owner's inbox
//      over NVLink; the last CTA publishes the per-owner counts into the
//      owners' `incoming[rank]` and signals every owner's barrier
//      (fence.sc.sys + red.release.sys).
//   2. k_xs_wait: one thread spins (ld.acquire.sys) until world signals.
//   3. the owner applies each inbox segment with the ordinary table kernels.
//   4. k_xs_reply: results stored straight into the source rank's reply
//      buffer at the op's source index; last CTA signals, 5. wait.
// No partition buffer, no all-to-all call, no unpermute pass.
// ============================================================================

struct ws_table;
int ws_internal_run(ws_table* t, const u8* ops, u8 uop, const u64* keys, const u64* vals, u64 n, u8* status,
                    u64* vout, cudaStream_t s, u32 flags, bool has_erase, bool has_upsert, bool query_only);

namespace {

constexpr int kMaxWorld = 8;
constexpr u64 kWaitLimitNs = 60ull * 1000 * 1000 * 1000;  // a peer silent for 60 s is gone

struct XRegion {  // byte offsets inside a rank's region
  u64 keys, vals, src, ops, incoming, res_st, res_vo, rep_st, rep_vo, bar, total;
};

XRegion layout(int world, u64 C) {
  XRegion r{};
  u64 o = 0;
  auto take = [&](u64 bytes) { const u64 at = o; o += (bytes + 255) & ~255ull; return at; };
  const u64 E = (u64)world * C;
  r.keys = take(8 * E);
  r.vals = take(8 * E);
  r.src = take(4 * E);
  r.ops = take(E);
  r.incoming = take(8 * kMaxWorld);
  r.res_st = take(E);
  r.res_vo = take(8 * E);
  r.rep_st = take(C);
  r.rep_vo = take(8 * C);
  r.bar = take(8);
  r.total = o;
  return r;
}

struct XPeers {
  char* base[kMaxWorld];
};

__device__ __forceinline__ void red_add_release_sys(u64* p, u64 v) {
  asm volatile("red.release.sys.global.add.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ u64 ld_acquire_sys(const u64* p) {
  u64 r;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(r) : "l"(p) : "memory");
  return r;
}

// routing of this round's ops [lo, lo+m) of the local batch
__global__ void k_xs_send(XPeers peers, XRegion L, int world, int rank, int shift, u64 C, u64 seed0,
                          const u64* __restrict__ keys, const u64* __restrict__ vals, const u8* __restrict__ ops,
                          u8 uop, u64 lo, u64 m, u32* cnt, u32* done_ctas) {
  const int lane = threadIdx.x & 31;
  for (u64 base = blockIdx.x * (u64)blockDim.x; base < m; base += (u64)gridDim.x * blockDim.x) {
    const u64 j = base + threadIdx.x;
    const bool act = j < m;
    u64 key = 0;
    u32 o = 0;
    if (act) {
      key = __ldg(keys + lo + j);
      o = shift >= 64 ? 0u : (u32)(mix64(key ^ seed0) >> shift);
    }
    // warp-aggregated reservation in owner o's segment `rank`
    u32 pos = 0;
    for (int w = 0; w < world; w++) {
      const u32 mask = __ballot_sync(0xFFFFFFFFu, act && o == (u32)w);
      if (!mask) continue;
      const int leader = __ffs(mask) - 1;
      u32 b = 0;
      if (lane == leader) b = atomicAdd(cnt + w, (u32)__popc(mask));
      b = __shfl_sync(0xFFFFFFFFu, b, leader);
      if (act && o == (u32)w) pos = b + __popc(mask & ((1u << lane) - 1));
    }
    if (act) {
      char* R = peers.base[o];
      const u64 e = (u64)rank * C + pos;
      ((u64*)(R + L.keys))[e] = key;
      ((u64*)(R + L.vals))[e] = vals ? __ldg(vals + lo + j) : 0ull;
      ((u32*)(R + L.src))[e] = (u32)j;
      R[L.ops + e] = ops ? __ldg(ops + lo + j) : uop;
    }
  }
  // last CTA out: publish counts into every owner and signal its barrier.
  // Every thread fences its own peer stores before the CTA counts itself done.
  __threadfence_system();
  __syncthreads();
  __shared__ bool last;
  if (threadIdx.x == 0) last = atomicAdd(done_ctas, 1u) == gridDim.x - 1;
  __syncthreads();
  if (last && threadIdx.x < (unsigned)world) {
    const int w = threadIdx.x;
    __threadfence_system();
    char* R = peers.base[w];
    ((volatile u64*)(R + L.incoming))[rank] = cnt[w];
    __threadfence_system();
    red_add_release_sys((u64*)(R + L.bar), 1ull);
  }
}

// Bounded device-side wait: a rank that never arrives (crashed peer) must not
// hang the GPU; after `limit_ns` the kernel records a timeout and returns.
__device__ __forceinline__ u64 globaltimer_ns() {
  u64 t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__global__ void k_xs_wait(u64* bar, u64 target, u64 limit_ns, u32* timed_out) {
  unsigned ns = 32;
  const u64 t0 = globaltimer_ns();
  while (ld_acquire_sys(bar) < target) {
    __nanosleep(ns);
    if (ns < 1024) ns <<= 1;
    if (globaltimer_ns() - t0 > limit_ns) {
      atomicExch(timed_out, 1u);
      return;
    }
  }
}

// results of inbox segment s (n_s entries) back to rank s's reply buffer
__global__ void k_xs_reply(XPeers peers, XRegion L, int world, u64 C, const u64* incoming_counts,
                           char* self, u32* done_ctas, int with_vals) {
  const u64 E = (u64)world * C;
  const u32* src = (const u32*)(self + L.src);
  const u8* st = (const u8*)(self + L.res_st);
  const u64* vo = (const u64*)(self + L.res_vo);
  for (u64 e = blockIdx.x * (u64)blockDim.x + threadIdx.x; e < E; e += (u64)gridDim.x * blockDim.x) {
    const u64 s = e / C, j = e % C;
    if (j >= incoming_counts[s]) continue;
    char* R = peers.base[s];
    const u32 i = src[e];
    R[L.rep_st + i] = st[e];
    if (with_vals) ((u64*)(R + L.rep_vo))[i] = vo[e];
  }
  __threadfence_system();
  __syncthreads();
  __shared__ bool last;
  if (threadIdx.x == 0) last = atomicAdd(done_ctas, 1u) == gridDim.x - 1;
  __syncthreads();
  if (last && threadIdx.x < (unsigned)world) {
    __threadfence_system();
    red_add_release_sys((u64*)(peers.base[threadIdx.x] + L.bar), 1ull);
  }
}

}  // namespace

struct ws_xchg {
  int world, rank, device;
  u64 C;
  XRegion L;
  char* region;           // this rank's region (device memory, IPC-exported)
  XPeers peers;           // device-usable base of every rank's region (self included)
  bool opened[kMaxWorld];
  u32* scratch;           // [0..world) send counters, [8] send CTAs done, [9] reply CTAs done
  u64* h_counts;          // pinned
  u64 epoch;              // barrier target progression
};

extern "C" {

WS_API int ws_xchg_create(int world, int rank, uint64_t chunk_ops, int device, ws_xchg** out) {
  if (!out || world < 1 || world > kMaxWorld || (world & (world - 1)) || rank < 0 || rank >= world ||
      chunk_ops == 0 || chunk_ops >= (1ull << 31))
    return WS_ERR_ARG;
  if (cudaSetDevice(device) != cudaSuccess) return WS_ERR_CUDA;
  ws_xchg* x = new ws_xchg();
  x->world = world;
  x->rank = rank;
  x->device = device;
  x->C = chunk_ops;
  x->L = layout(world, chunk_ops);
  if (cudaMalloc((void**)&x->region, x->L.total) != cudaSuccess) { delete x; return WS_ERR_ALLOC; }
  cudaMemset(x->region, 0, x->L.total);
  if (cudaMalloc((void**)&x->scratch, 64 * 4) != cudaSuccess) { cudaFree(x->region); delete x; return WS_ERR_ALLOC; }
  cudaMallocHost((void**)&x->h_counts, 8 * (kMaxWorld + 1));
  for (int i = 0; i < kMaxWorld; i++) x->peers.base[i] = nullptr;
  x->peers.base[rank] = x->region;
  *out = x;
  return cudaDeviceSynchronize() == cudaSuccess ? WS_OK : WS_ERR_CUDA;
}

WS_API int ws_xchg_handle(ws_xchg* x, void* handle_out) {
  if (!x || !handle_out) return WS_ERR_ARG;
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, x->region) != cudaSuccess) return WS_ERR_CUDA;
  memcpy(handle_out, &h, sizeof(h));
  return WS_OK;
}

WS_API int ws_xchg_open(ws_xchg* x, const void* handles) {
  if (!x || !handles) return WS_ERR_ARG;
  cudaSetDevice(x->device);
  for (int r = 0; r < x->world; r++) {
    if (r == x->rank) continue;
    cudaIpcMemHandle_t h;
    memcpy(&h, (const char*)handles + r * sizeof(h), sizeof(h));
    void* p = nullptr;
    if (cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) return WS_ERR_CUDA;
    x->peers.base[r] = (char*)p;
    x->opened[r] = true;
  }
  return WS_OK;
}

WS_API int ws_xchg_destroy(ws_xchg* x) {
  if (!x) return WS_OK;
  cudaSetDevice(x->device);
  cudaDeviceSynchronize();
  for (int r = 0; r < x->world; r++)
    if (x->opened[r]) cudaIpcCloseMemHandle(x->peers.base[r]);
  cudaFree(x->region);
  cudaFree(x->scratch);
  cudaFreeHost(x->h_counts);
  delete x;
  return WS_OK;
}

// One batch through the sharded table: every rank calls it collectively with
// its own batch and the same `rounds` (= ceil(max_n / chunk) over ranks).
// op_kind: WS_OP_UPSERT / ERASE / QUERY for a uniform batch (merge in uop's
// high nibble), or ops != NULL for a mixed batch.  Device pointers only.
WS_API int ws_xchg_run(ws_xchg* x, ws_table* local, const uint8_t* ops, uint8_t uop, const uint64_t* keys,
                       const uint64_t* vals, uint64_t n, uint64_t rounds, uint64_t seed0, uint8_t* status,
                       uint64_t* vals_out, void* stream, uint32_t flags) {
  if (!x || !local || (n && !keys)) return WS_ERR_ARG;
  if (cudaSetDevice(x->device) != cudaSuccess) return WS_ERR_CUDA;
  cudaStream_t s = (cudaStream_t)stream;
  const int W = x->world, log2w = __builtin_ctz((unsigned)W);
  const int shift = log2w ? 64 - log2w : 64;
  const XRegion& L = x->L;
  const bool mixed = ops != nullptr;
  const int kind = uop & 15;
  const bool q_only = !mixed && kind == OP_QUERY;
  const bool has_erase = mixed || kind == OP_ERASE;
  const bool has_upsert = mixed || kind == OP_UPSERT;
  const bool want_vals = mixed || q_only;
  int rc = WS_OK;
  for (u64 r = 0; r < rounds && rc == WS_OK; r++) {
    const u64 lo = r * x->C;
    const u64 m = lo < n ? std::min<u64>(x->C, n - lo) : 0;
    // 1. route this round's ops into the owners' inboxes
    if (cudaMemsetAsync(x->scratch, 0, 64 * 4, s) != cudaSuccess) return WS_ERR_CUDA;
    u64 g = (m + 255) / 256;
    g = std::max<u64>(1, std::min<u64>(g, 148 * 4));
    k_xs_send<<<(unsigned)g, 256, 0, s>>>(x->peers, L, W, x->rank, shift, x->C, seed0, (const u64*)keys,
                                          (const u64*)vals, ops, uop, lo, m, x->scratch, x->scratch + 8);
    x->epoch += W;
    k_xs_wait<<<1, 1, 0, s>>>((u64*)(x->region + L.bar), x->epoch, kWaitLimitNs, x->scratch + 10);
    // 2. apply each source segment locally
    if (cudaMemcpyAsync(x->h_counts, x->region + L.incoming, 8 * W, cudaMemcpyDeviceToHost, s) != cudaSuccess)
      return WS_ERR_CUDA;
    if (cudaMemcpyAsync(x->h_counts + kMaxWorld, x->scratch + 10, 4, cudaMemcpyDeviceToHost, s) != cudaSuccess)
      return WS_ERR_CUDA;
    if (cudaStreamSynchronize(s) != cudaSuccess) return WS_ERR_CUDA;
    if (*(const u32*)(x->h_counts + kMaxWorld)) return WS_ERR_TIMEOUT;
    for (int src = 0; src < W && rc == WS_OK; src++) {
      const u64 ns = x->h_counts[src];
      if (!ns) continue;
      const u64 e = (u64)src * x->C;
      rc = ws_internal_run(local, mixed ? (const u8*)(x->region + L.ops) + e : nullptr, uop,
                           (const u64*)(x->region + L.keys) + e,
                           has_upsert ? (const u64*)(x->region + L.vals) + e : nullptr, ns,
                           (u8*)(x->region + L.res_st) + e, want_vals ? (u64*)(x->region + L.res_vo) + e : nullptr,
                           s, flags, has_erase, has_upsert, q_only);
    }
    if (rc) break;
    // 3. return results to their sources, 4. wait for mine
    k_xs_reply<<<148 * 4, 256, 0, s>>>(x->peers, L, W, x->C, (const u64*)(x->region + L.incoming), x->region,
                                       x->scratch + 9, want_vals ? 1 : 0);
    x->epoch += W;
    k_xs_wait<<<1, 1, 0, s>>>((u64*)(x->region + L.bar), x->epoch, kWaitLimitNs, x->scratch + 10);
    if (m) {
      if (status && cudaMemcpyAsync(status + lo, x->region + L.rep_st, m, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
        return WS_ERR_CUDA;
      if (vals_out && cudaMemcpyAsync(vals_out + lo, x->region + L.rep_vo, 8 * m, cudaMemcpyDeviceToDevice, s) !=
                          cudaSuccess)
        return WS_ERR_CUDA;
    }
  }
  if (rc == WS_OK && cudaGetLastError() != cudaSuccess) rc = WS_ERR_CUDA;
  if (rc == WS_OK) {
    if (cudaMemcpyAsync(x->h_counts + kMaxWorld, x->scratch + 10, 4, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
      return WS_ERR_CUDA;
    if (*(const u32*)(x->h_counts + kMaxWorld)) rc = WS_ERR_TIMEOUT;
  }
  return rc;
}

}  // extern "C"

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
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

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
// Fused routing over NVLink peer memory ("xchg"), double-buffered.
//
// Every rank owns one IPC-exported region holding TWO buffers b = 0, 1:
//   inbox[b]     keys / vals / src / ops, world x C entries (segment s <- rank s)
//   incoming[b]  entries rank s wrote into segment s of round r's inbox
//   result[b]    status / value of the inbox entries (applied locally)
//   reply[b]     status / value for MY ops of the round, written by owners
//   bar_send[b], bar_rep[b]   monotonic arrival counters (peers add, I wait)
// Round r uses buffer b = r & 1 and moves up to C of this rank's ops:
//   s_send: k_xs_send routes each op into its owner's inbox[b] segment
//           `rank` over NVLink (warp-aggregated LOCAL reservations: a sender
//           owns its segment in every inbox); the last CTA publishes the
//           per-owner counts and signals every owner's bar_send[b]
//           (fence.sc.sys + red.release.sys)
//   s:      k_xs_wait(bar_send[b]) -> one table launch per inbox segment with
//           the segment's count read ON THE DEVICE (Dev::dn) -> k_xs_reply
//           stores every result into its source's reply[b] and signals it
//   s_recv: k_xs_wait(bar_rep[b]) -> copy reply[b] to the caller's outputs
// No host synchronisation inside the loop.  The next round's routing runs on
// s_send (high priority) while this round's inbox is being applied on s:
// round r+1 only waits for the replies of round r-1 (buffer reuse), so the
// NVLink transfer of one round hides under the local apply of the previous.
// Waits are bounded by %globaltimer (a dead peer yields WS_ERR_TIMEOUT, never
// a hung GPU); the timeout flag is sticky for the whole call and every later
// wait returns at once once it is set.
// ============================================================================

struct ws_table;
int ws_internal_run(ws_table* t, const u8* ops, u8 uop, const u64* keys, const u64* vals, u64 n, u8* status,
                    u64* vout, cudaStream_t s, u32 flags, bool has_erase, bool has_upsert, bool query_only,
                    const u64* n_dev);

namespace {

constexpr int kMaxWorld = 8;
constexpr u64 kWaitLimitNs = 60ull * 1000 * 1000 * 1000;  // a peer silent for 60 s is gone

struct XBuf {  // byte offsets of one buffer inside a rank's region
  u64 keys, vals, src, ops, incoming, res_st, res_vo, rep_st, rep_vo, bar_send, bar_rep;
};
struct XRegion {
  XBuf b[2];
  u64 total;
};

XRegion layout(int world, u64 C) {
  XRegion r{};
  u64 o = 0;
  auto take = [&](u64 bytes) { const u64 at = o; o += (bytes + 255) & ~255ull; return at; };
  const u64 E = (u64)world * C;
  for (int b = 0; b < 2; b++) {
    XBuf& x = r.b[b];
    x.keys = take(8 * E);
    x.vals = take(8 * E);
    x.src = take(4 * E);
    x.ops = take(E);
    x.incoming = take(8 * kMaxWorld);
    x.res_st = take(E);
    x.res_vo = take(8 * E);
    x.rep_st = take(C);
    x.rep_vo = take(8 * C);
    x.bar_send = take(8);
    x.bar_rep = take(8);
  }
  r.total = o;
  return r;
}

struct XPeers {
  char* base[kMaxWorld];
};

// scratch words (u32) of a rank: per buffer b at 16*b: [0, world) send
// counters, [8] send CTAs done, [9] reply CTAs done; [32] sticky timeout flag
constexpr int kTimeoutWord = 32;

__device__ __forceinline__ void red_add_release_sys(u64* p, u64 v) {
  asm volatile("red.release.sys.global.add.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ u64 ld_acquire_sys(const u64* p) {
  u64 r;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(r) : "l"(p) : "memory");
  return r;
}

// routing of this round's ops [lo, lo+m) of the local batch into buffer B of the owners
__global__ void __launch_bounds__(256) k_xs_send(XPeers peers, XBuf B, int world, int rank, int shift, u64 C,
                                                 u64 seed0, const u64* __restrict__ keys,
                                                 const u64* __restrict__ vals, const u8* __restrict__ ops, u8 uop,
                                                 u64 lo, u64 m, u32* cnt, u32* done_ctas) {
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
      ((u64*)(R + B.keys))[e] = key;
      ((u64*)(R + B.vals))[e] = vals ? __ldg(vals + lo + j) : 0ull;
      ((u32*)(R + B.src))[e] = (u32)j;
      R[B.ops + e] = ops ? __ldg(ops + lo + j) : uop;
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
    ((volatile u64*)(R + B.incoming))[rank] = cnt[w];
    __threadfence_system();
    red_add_release_sys((u64*)(R + B.bar_send), 1ull);
  }
}

// Bounded device-side wait: a rank that never arrives (crashed peer) must not
// hang the GPU; after `limit_ns` the kernel records a timeout and returns.
// The flag is sticky for the call: once set, every later wait returns at once.
__device__ __forceinline__ u64 globaltimer_ns() {
  u64 t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__global__ void k_xs_wait(u64* bar, u64 target, u64 limit_ns, u32* timed_out) {
  unsigned ns = 32;
  const u64 t0 = globaltimer_ns();
  while (ld_acquire_sys(bar) < target) {
    if (*(volatile u32*)timed_out) return;
    __nanosleep(ns);
    if (ns < 1024) ns <<= 1;
    if (globaltimer_ns() - t0 > limit_ns) {
      atomicExch(timed_out, 1u);
      return;
    }
  }
}

// results of inbox segment s (incoming[s] entries) back to rank s's reply buffer
__global__ void __launch_bounds__(256) k_xs_reply(XPeers peers, XBuf B, int world, u64 C, const char* self,
                                                  u32* done_ctas, int with_vals) {
  const u64* incoming = (const u64*)(self + B.incoming);
  const u32* src = (const u32*)(self + B.src);
  const u8* st = (const u8*)(self + B.res_st);
  const u64* vo = (const u64*)(self + B.res_vo);
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (int s = 0; s < world; s++) {
    const u64 ns = incoming[s] < C ? incoming[s] : C;
    char* R = peers.base[s];
    for (u64 j = blockIdx.x * (u64)blockDim.x + threadIdx.x; j < ns; j += stride) {
      const u64 e = (u64)s * C + j;
      const u32 i = src[e];
      R[B.rep_st + i] = st[e];
      if (with_vals) ((u64*)(R + B.rep_vo))[i] = vo[e];
    }
  }
  __threadfence_system();
  __syncthreads();
  __shared__ bool last;
  if (threadIdx.x == 0) last = atomicAdd(done_ctas, 1u) == gridDim.x - 1;
  __syncthreads();
  if (last && threadIdx.x < (unsigned)world) {
    __threadfence_system();
    red_add_release_sys((u64*)(peers.base[threadIdx.x] + B.bar_rep), 1ull);
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
  u32* scratch;           // see kTimeoutWord
  u32* h_flag;            // pinned: timeout verdict
  u64 ep_send[2], ep_rep[2];  // barrier targets per buffer (monotonic across calls)
  cudaStream_t s_send, s_recv;
  cudaEvent_t ev_start, ev_free[2], ev_send_done, ev_recv_done;
  // WS_XCHG_TRACE=<file>: timing events around every phase of every round
  // (route on s_send, apply + reply on s, reply wait + copy-out on s_recv),
  // appended to <file> as "rank,round,phase,start_ms,end_ms" after each call
  // -- the evidence that round r+1's routing overlaps round r's apply
  const char* trace_path;
  std::vector<cudaEvent_t> tev;
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
  cudaMemset(x->scratch, 0, 64 * 4);
  cudaMallocHost((void**)&x->h_flag, 64);
  int lo_prio = 0, hi_prio = 0;
  cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio);
  // routing runs beside the previous round's table kernels: high priority,
  // so its CTAs are scheduled as soon as SM slots free up
  cudaStreamCreateWithPriority(&x->s_send, cudaStreamNonBlocking, hi_prio);
  cudaStreamCreateWithFlags(&x->s_recv, cudaStreamNonBlocking);
  for (cudaEvent_t* e : {&x->ev_start, &x->ev_free[0], &x->ev_free[1], &x->ev_send_done, &x->ev_recv_done})
    cudaEventCreateWithFlags(e, cudaEventDisableTiming);
  for (int i = 0; i < kMaxWorld; i++) x->peers.base[i] = nullptr;
  x->peers.base[rank] = x->region;
  x->trace_path = getenv("WS_XCHG_TRACE");
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
  cudaFreeHost(x->h_flag);
  for (cudaEvent_t e : {x->ev_start, x->ev_free[0], x->ev_free[1], x->ev_send_done, x->ev_recv_done})
    if (e) cudaEventDestroy(e);
  for (cudaStream_t st : {x->s_send, x->s_recv})
    if (st) cudaStreamDestroy(st);
  for (cudaEvent_t e : x->tev) cudaEventDestroy(e);
  delete x;
  return WS_OK;
}

// One batch through the sharded table: every rank calls it collectively with
// its own batch and the same `rounds` (= ceil(max_n / chunk) over ranks).
// op_kind: WS_OP_UPSERT / ERASE / QUERY for a uniform batch (merge in uop's
// high nibble), or ops != NULL for a mixed batch.  Device pointers only; the
// caller validated the batch group-wide (ShardedTable._validate), so the
// local launches run unchecked.
WS_API int ws_xchg_run(ws_xchg* x, ws_table* local, const uint8_t* ops, uint8_t uop, const uint64_t* keys,
                       const uint64_t* vals, uint64_t n, uint64_t rounds, uint64_t seed0, uint8_t* status,
                       uint64_t* vals_out, void* stream, uint32_t flags) {
  if (!x || !local || (n && !keys)) return WS_ERR_ARG;
  if (cudaSetDevice(x->device) != cudaSuccess) return WS_ERR_CUDA;
  cudaStream_t s = (cudaStream_t)stream;
  const int W = x->world, log2w = __builtin_ctz((unsigned)W);
  const int shift = log2w ? 64 - log2w : 64;
  const bool mixed = ops != nullptr;
  const int kind = uop & 15;
  const bool q_only = !mixed && kind == OP_QUERY;
  const bool has_erase = mixed || kind == OP_ERASE;
  const bool has_upsert = mixed || kind == OP_UPSERT;
  const bool want_vals = mixed || q_only;
  const u32 lflags = (flags & ~(WS_F_SYNC_CHECK | WS_F_COMBINE)) | WS_F_NO_CHECK;
  u32* tflag = x->scratch + kTimeoutWord;
#define XCK(call) do { if ((call) != cudaSuccess) return WS_ERR_CUDA; } while (0)
  // tracing: 6 timing events per round (send a/b, apply a/b, recv a/b) + t0
  const bool tr = x->trace_path != nullptr;
  if (tr) {
    while (x->tev.size() < 1 + 6 * rounds) {
      cudaEvent_t e;
      XCK(cudaEventCreate(&e));
      x->tev.push_back(e);
    }
    XCK(cudaEventRecord(x->tev[0], s));
  }
  auto mark = [&](u64 r, int k, cudaStream_t st) { if (tr) cudaEventRecord(x->tev[1 + 6 * r + k], st); };
  // the call starts after everything already queued on the caller's stream
  XCK(cudaMemsetAsync(tflag, 0, 4, s));
  XCK(cudaEventRecord(x->ev_start, s));
  XCK(cudaStreamWaitEvent(x->s_send, x->ev_start, 0));
  XCK(cudaStreamWaitEvent(x->s_recv, x->ev_start, 0));
  int rc = WS_OK;
  for (u64 r = 0; r < rounds && rc == WS_OK; r++) {
    const int b = (int)(r & 1);
    const XBuf& B = x->L.b[b];
    const u64 lo = r * x->C;
    const u64 m = lo < n ? std::min<u64>(x->C, n - lo) : 0;
    u32* sc = x->scratch + 16 * b;
    // 1. [s_send] route this round's ops once every owner has released buffer b
    //    (= my replies of round r-2 arrived, recorded on s_recv)
    if (r >= 2) XCK(cudaStreamWaitEvent(x->s_send, x->ev_free[b], 0));
    XCK(cudaMemsetAsync(sc, 0, 16 * 4, x->s_send));
    const u64 g = std::max<u64>(1, std::min<u64>((m + 255) / 256, 148 * 2));
    mark(r, 0, x->s_send);
    k_xs_send<<<(unsigned)g, 256, 0, x->s_send>>>(x->peers, B, W, x->rank, shift, x->C, seed0, (const u64*)keys,
                                                  (const u64*)vals, ops, uop, lo, m, sc, sc + 8);
    mark(r, 1, x->s_send);
    // 2. [s] wait for every source's segment, apply each segment with its
    //    device-resident count, return the results
    x->ep_send[b] += W;
    k_xs_wait<<<1, 1, 0, s>>>((u64*)(x->region + B.bar_send), x->ep_send[b], kWaitLimitNs, tflag);
    const u64* inc = (const u64*)(x->region + B.incoming);
    mark(r, 2, s);
    for (int src = 0; src < W && rc == WS_OK; src++) {
      const u64 e = (u64)src * x->C;
      rc = ws_internal_run(local, mixed ? (const u8*)(x->region + B.ops) + e : nullptr, uop,
                           (const u64*)(x->region + B.keys) + e,
                           has_upsert ? (const u64*)(x->region + B.vals) + e : nullptr, x->C,
                           (u8*)(x->region + B.res_st) + e, want_vals ? (u64*)(x->region + B.res_vo) + e : nullptr,
                           s, lflags, has_erase, has_upsert, q_only, inc + src);
    }
    if (rc) break;
    k_xs_reply<<<148 * 2, 256, 0, s>>>(x->peers, B, W, x->C, x->region, sc + 9, want_vals ? 1 : 0);
    mark(r, 3, s);
    // 3. [s_recv] wait for my replies, copy them out, release buffer b
    x->ep_rep[b] += W;
    mark(r, 4, x->s_recv);
    k_xs_wait<<<1, 1, 0, x->s_recv>>>((u64*)(x->region + B.bar_rep), x->ep_rep[b], kWaitLimitNs, tflag);
    if (m) {
      if (status) XCK(cudaMemcpyAsync(status + lo, x->region + B.rep_st, m, cudaMemcpyDeviceToDevice, x->s_recv));
      if (vals_out)
        XCK(cudaMemcpyAsync(vals_out + lo, x->region + B.rep_vo, 8 * m, cudaMemcpyDeviceToDevice, x->s_recv));
    }
    mark(r, 5, x->s_recv);
    XCK(cudaEventRecord(x->ev_free[b], x->s_recv));
  }
  // the caller's stream resumes after every route, apply and copy-out
  XCK(cudaEventRecord(x->ev_send_done, x->s_send));
  XCK(cudaEventRecord(x->ev_recv_done, x->s_recv));
  XCK(cudaStreamWaitEvent(s, x->ev_send_done, 0));
  XCK(cudaStreamWaitEvent(s, x->ev_recv_done, 0));
  if (rc == WS_OK && cudaGetLastError() != cudaSuccess) rc = WS_ERR_CUDA;
  XCK(cudaMemcpyAsync(x->h_flag, tflag, 4, cudaMemcpyDeviceToHost, s));
  XCK(cudaStreamSynchronize(s));
  if (rc == WS_OK && *x->h_flag) rc = WS_ERR_TIMEOUT;
  if (tr && rc == WS_OK) {
    if (FILE* f = fopen(x->trace_path, "a")) {
      static const char* names[3] = {"route", "apply+reply", "recv+copy"};
      for (u64 r = 0; r < rounds; r++)
        for (int k = 0; k < 3; k++) {
          float a = 0, e = 0;
          cudaEventElapsedTime(&a, x->tev[0], x->tev[1 + 6 * r + 2 * k]);
          cudaEventElapsedTime(&e, x->tev[0], x->tev[1 + 6 * r + 2 * k + 1]);
          fprintf(f, "%d,%llu,%s,%.4f,%.4f\n", x->rank, (unsigned long long)r, names[k], a, e);
        }
      fclose(f);
    }
  }
#undef XCK
  return rc;
}

}  // extern "C"

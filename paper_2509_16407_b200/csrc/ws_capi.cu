// ws_capi.cu -- kernels and the extern "C" ABI declared in include/warpspeed.h.
//
// Launch shape: one thread per operation, grid-stride, 256-thread CTAs, grid
// capped at 148 SMs x 8 resident CTAs.  Batch keys / values / op bytes are read
// with coalesced streaming loads (consecutive threads own consecutive ops);
// results are written coalesced the same way.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <atomic>
#include <map>
#include <mutex>
#include <new>
#include <shared_mutex>
#include <thread>
#include <vector>

#include <cub/cub.cuh>

#include "warpspeed.h"
#include "ws_kernels.cuh"

using namespace ws;

namespace {

constexpr u32 N_STATE = 16;  // [0] tomb_ever; [8..11] the default per-call words (Dev::cs)

Launchers launchers_for(int design) {
  switch (design) {
    case D_DOUBLE: return launchers_double();
    case D_DOUBLE_MD: return launchers_double_md();
    case D_P2: return launchers_p2();
    case D_P2_MD: return launchers_p2_md();
    case D_ICEBERG: return launchers_iceberg();
    case D_ICEBERG_MD: return launchers_iceberg_md();
    case D_CUCKOO: return launchers_cuckoo();
    case D_CHAINING: return launchers_chaining();
    default: return launchers_unsafe();
  }
}

// ------------------------------------------------------------------ kernels

// mixed batches: count erase ops so the op kernel enables the concurrent-erase
// (fenced tombstone-flag) path only when the batch really erases
__global__ void k_count_erases(const u8* __restrict__ ops, u64 n, u32* cs) {
  u32 c = 0;
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x)
    c += (__ldg(ops + i) & 15) == OP_ERASE;
  c = __reduce_add_sync(0xFFFFFFFFu, c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(cs + 3, c);
}

// Batch-wide sentinel / op-byte check, run before any mutation.  A pure
// streaming pass (8 B per key): 16-byte streaming loads, 4 per thread in
// flight, so the pass runs near the copy bandwidth (2^30 keys: ~1.2 ms).
__global__ void __launch_bounds__(256) k_validate(const u64* __restrict__ keys, const u8* __restrict__ ops, u64 n,
                                                  u32* cs) {
  u32 bad_k = 0, bad_o = 0;
  const u64 tid = blockIdx.x * (u64)blockDim.x + threadIdx.x, nt = (u64)gridDim.x * blockDim.x;
  const bool vec = ((uintptr_t)keys & 15) == 0;
  const u64 npair = vec ? n / 2 : 0;
  const ulonglong2* kp = (const ulonglong2*)keys;
  u64 j = tid;
  for (; j + 3 * nt < npair; j += 4 * nt) {
    ulonglong2 v[4];
#pragma unroll
    for (int r = 0; r < 4; r++) v[r] = __ldcs(kp + j + r * nt);
#pragma unroll
    for (int r = 0; r < 4; r++) bad_k += is_sentinel(v[r].x) + is_sentinel(v[r].y);
  }
  for (; j < npair; j += nt) {
    const ulonglong2 v = __ldcs(kp + j);
    bad_k += is_sentinel(v.x) + is_sentinel(v.y);
  }
  for (u64 i = 2 * npair + tid; i < n; i += nt) bad_k += is_sentinel(__ldg(keys + i));
  if (ops) {
    for (u64 i = tid; i < n; i += nt) {
      const u8 o = __ldg(ops + i);
      bad_o += ((o & 15) > OP_QUERY) | ((o >> 4) > M_MIN);
    }
  }
  bad_k = __reduce_add_sync(0xFFFFFFFFu, bad_k);
  bad_o = __reduce_add_sync(0xFFFFFFFFu, bad_o);
  if ((threadIdx.x & 31) == 0) {
    if (bad_k) atomicAdd(cs, bad_k);
    if (bad_o) atomicAdd(cs + 1, bad_o);
  }
}

// live pair i?  (chaining: only pair slots of allocated nodes)
__device__ __forceinline__ bool pair_live(const Dev& d, u64 i, u64 next_node, u64& k, u64& v) {
  if (d.design == D_CHAINING) {
    const u64 per = (u64)d.wpn / 2, m = i / per, j = i % per;
    if (m < 1 || m >= next_node || j >= (u64)d.bs) return false;
  }
  ld_cell(d.cells + 2 * i, k, v);
  return !is_sentinel(k);
}

__global__ void k_item_flags(Dev d, u64 npairs, u64 next_node, u8* flags) {
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < npairs; i += (u64)gridDim.x * blockDim.x) {
    u64 k, v;
    flags[i] = pair_live(d, i, next_node, k, v);
  }
}

__global__ void k_checksum(Dev d, u64 npairs, u64 next_node, u64* out) {
  u64 cnt = 0, sk = 0, sv = 0, x = 0;
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < npairs; i += (u64)gridDim.x * blockDim.x) {
    u64 k, v;
    if (pair_live(d, i, next_node, k, v)) {
      cnt++;
      sk += k;
      sv += v;
      x ^= mix64(k ^ mix64(v));
    }
  }
  for (int o = 16; o; o >>= 1) {
    cnt += __shfl_xor_sync(0xFFFFFFFFu, cnt, o);
    sk += __shfl_xor_sync(0xFFFFFFFFu, sk, o);
    sv += __shfl_xor_sync(0xFFFFFFFFu, sv, o);
    x ^= __shfl_xor_sync(0xFFFFFFFFu, x, o);
  }
  if ((threadIdx.x & 31) == 0 && cnt) {
    atomicAdd((unsigned long long*)out, (unsigned long long)cnt);
    atomicAdd((unsigned long long*)out + 1, (unsigned long long)sk);
    atomicAdd((unsigned long long*)out + 2, (unsigned long long)sv);
    atomicXor((unsigned long long*)out + 3, (unsigned long long)x);
  }
}

__global__ void k_split_pairs(const ulonglong2* pairs, u64 n, u64* keys, u64* vals) {
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
    const ulonglong2 p = pairs[i];
    if (keys) keys[i] = p.x;
    if (vals) vals[i] = p.y;
  }
}

__global__ void k_pair_keys(const ulonglong2* pairs, u64 n, u64* keys) {
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x)
    keys[i] = pairs[i].x;
}

// sorted keys -> (key, multiplicity) for every run longer than one
__global__ void k_dup_runs(const u64* sorted, u64 n, u64* dk, u64* dc, u64 cap, u64* ndup) {
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i + 1 < n; i += (u64)gridDim.x * blockDim.x) {
    if (sorted[i] != sorted[i + 1] || (i > 0 && sorted[i - 1] == sorted[i])) continue;
    u64 e = i + 1;
    while (e < n && sorted[e] == sorted[i]) e++;
    const u64 slot = atomicAdd((unsigned long long*)ndup, 1ull);
    if (slot < cap) { dk[slot] = sorted[i]; dc[slot] = e - i; }
  }
}

}  // namespace

// ====================================================================== table

struct ws_table {
  ws_config cfg;
  int device;
  Dev d;
  Launchers L;
  bool def_bs;
  u64 cell_words;
  u64 lock_words;
  // WS_TUNE_KERNEL_EVENTS: CUDA events bracket every table-kernel launch of
  // run_device_plain on its stream (bench.py's per-kernel roofline timing);
  // ws_kernel_times() reads and clears them
  bool time_kernels = false;
  std::mutex ev_mu;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> kev;
  // Concurrent calls (reference tables/base.py:5-7: every public op may be
  // called from many threads) hold `mu` shared for their whole host-side
  // duration; only a chaining pool growth (which moves the node arena) takes
  // it exclusively.  Per-call device state, pinned scratch and staging
  // streams are private to the call / calling thread (CallCtx, pin(),
  // staging()), so nothing else on the host side is shared.
  std::shared_mutex mu;
};

namespace {

thread_local char g_cuda_msg[256] = "CUDA error";

inline int note_cuda(cudaError_t e, int line) {
  snprintf(g_cuda_msg, sizeof g_cuda_msg, "CUDA error %s (%s) at ws_capi.cu:%d", cudaGetErrorName(e),
           cudaGetErrorString(e), line);
  return WS_ERR_CUDA;
}
inline int cuda_err_at(cudaError_t e, int line) { return e == cudaSuccess ? WS_OK : note_cuda(e, line); }
#define cuda_err(x) cuda_err_at((x), __LINE__)
#define WS_CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) return note_cuda(e_, __LINE__); } while (0)

inline cudaStream_t S(void* s) { return (cudaStream_t)s; }

// pinned host scratch of the calling thread (64 words) for stream-ordered
// device -> host reads of small results
u64* pin() {
  struct Pin {
    u64* p = nullptr;
    ~Pin() { if (p) cudaFreeHost(p); }
  };
  thread_local Pin tp;
  if (!tp.p && cudaMallocHost((void**)&tp.p, 64 * 8) != cudaSuccess) tp.p = nullptr;
  return tp.p;
}

// a second pinned block of the calling thread (512 words) for the bin starts
// of run_device_split, which outlive nested calls that use pin()
u64* pin_call() {
  struct Pin {
    u64* p = nullptr;
    ~Pin() { if (p) cudaFreeHost(p); }
  };
  thread_local Pin tp;
  if (!tp.p && cudaMallocHost((void**)&tp.p, 512 * 8) != cudaSuccess) tp.p = nullptr;
  return tp.p;
}

// H2D / D2H staging streams and events of the calling thread on one device
struct Staging {
  cudaStream_t s_in = nullptr, s_aux = nullptr;
  cudaEvent_t ev_a = nullptr, ev_b = nullptr, ev_in = nullptr;
  std::vector<cudaEvent_t> ev_chunk;  // per-chunk H2D completion (staged mutations)
  ~Staging() {
    for (cudaEvent_t e : ev_chunk) cudaEventDestroy(e);
    for (cudaEvent_t e : {ev_a, ev_b, ev_in}) if (e) cudaEventDestroy(e);
    for (cudaStream_t x : {s_in, s_aux}) if (x) cudaStreamDestroy(x);
  }
};

Staging* staging(int device) {
  thread_local std::map<int, Staging> per_dev;
  Staging& st = per_dev[device];
  if (!st.s_in) {
    if (cudaStreamCreateWithFlags(&st.s_in, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&st.s_aux, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&st.ev_a, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&st.ev_b, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&st.ev_in, cudaEventDisableTiming) != cudaSuccess) {
      per_dev.erase(device);
      return nullptr;
    }
  }
  return &st;
}

// One API call's private context: its 4 device state words (Dev::cs) and the
// shared hold on the table it keeps for its host-side duration.
struct CallCtx {
  u32* cs;
  std::shared_lock<std::shared_mutex>* lk;
  const u64* dn = nullptr;  // device-resident batch size (ws_internal_run from the exchange), n = upper bound
};

inline Dev dev_of(const ws_table* t, const CallCtx& cx) {
  Dev d = t->d;
  d.cs = cx.cs;
  d.dn = cx.dn;
  return d;
}

bool is_device_ptr(const void* p) {
  if (!p) return true;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

u64 next_pow2(u64 x) {
  u64 p = 1;
  while (p < x) p <<= 1;
  return p;
}

Mod make_mod(u64 d) {
  Mod m;
  m.d = d ? d : 1;
  m.mask = (d && !(d & (d - 1))) ? d - 1 : 0;
  return m;
}

// reset the invalid counters and count sentinel keys / bad op bytes
int validate(const u64* keys, const u8* ops, u64 n, cudaStream_t s, bool sync, u32 flags, const CallCtx& cx) {
  if (flags & WS_F_NO_CHECK) return WS_OK;
  WS_CK(cudaMemsetAsync(cx.cs, 0, 2 * sizeof(u32), s));
  if (n) k_validate<<<grid_for(n / 2 + 1, kThreads, 8), kThreads, 0, s>>>(keys, ops, n, cx.cs);
  WS_CK(cudaGetLastError());
  if (!sync) return WS_OK;
  u64* hp = pin();
  if (!hp) return WS_ERR_ALLOC;
  WS_CK(cudaMemcpyAsync(hp, cx.cs, 2 * sizeof(u32), cudaMemcpyDeviceToHost, s));
  WS_CK(cudaStreamSynchronize(s));
  const u32* c = (const u32*)hp;
  if (c[0]) return WS_ERR_INVALID_KEY;
  if (c[1]) return WS_ERR_INVALID_OP;
  return WS_OK;
}

// chaining: grow the node pool by 1.5x when a launch exhausted it.  The
// caller holds the table exclusively; every launch that may still read the
// old arena (other threads' calls return before their kernels finish) is
// drained by a device synchronisation before the arena moves.
int chain_grow(ws_table* t, cudaStream_t s) {
  WS_CK(cudaDeviceSynchronize());
  const u64 old = t->d.chain_cap;
  const u64 ncap = old + std::max<u64>(old / 2, 64);
  const u64 words = ncap * (u64)t->d.wpn;
  u64* nc = nullptr;
  WS_CK(cudaMallocAsync((void**)&nc, words * 8, s));
  WS_CK(cudaMemcpyAsync(nc, t->d.cells, old * t->d.wpn * 8, cudaMemcpyDeviceToDevice, s));
  WS_CK(cudaMemsetAsync(nc + old * t->d.wpn, 0, (ncap - old) * t->d.wpn * 8, s));
  WS_CK(cudaFreeAsync(t->d.cells, s));
  t->d.cells = nc;
  t->d.chain_cap = ncap;
  t->cell_words = words;
  // every index < old was handed out; failed bumps overshot past it
  u64* hp = pin();
  if (!hp) return WS_ERR_ALLOC;
  WS_CK(cudaMemcpyAsync(hp, t->d.chain_next, 8, cudaMemcpyDeviceToHost, s));
  WS_CK(cudaStreamSynchronize(s));
  if (hp[0] > old) hp[0] = old;
  WS_CK(cudaMemcpyAsync(t->d.chain_next, hp, 8, cudaMemcpyHostToDevice, s));
  WS_CK(cudaStreamSynchronize(s));
  return WS_OK;
}

__global__ void k_comb_iota(u64 n, u32* idx);

// internal flags of run_device_plain
constexpr u32 kF_VALIDATED = 1u << 30;  // the caller validated the batch; keep the kernels gated
constexpr u32 kF_NO_KIND_SORT = 1u << 29;
constexpr u32 kF_CONC_ERASE = 1u << 28;  // other launches of this call may erase concurrently

__global__ void k_kind_gather(const u32* __restrict__ perm, const u64* __restrict__ keys,
                              const u64* __restrict__ vals, u64 n, u64* kp, u64* vp) {
  for (u64 j = blockIdx.x * (u64)blockDim.x + threadIdx.x; j < n; j += (u64)gridDim.x * blockDim.x) {
    const u32 i = perm[j];
    kp[j] = keys[i];
    if (vals) vp[j] = vals[i];
  }
}
__global__ void k_kind_scatter(const u32* __restrict__ perm, const u8* __restrict__ sp, const u64* __restrict__ vop,
                               u64 n, u8* status, u64* vout) {
  for (u64 j = blockIdx.x * (u64)blockDim.x + threadIdx.x; j < n; j += (u64)gridDim.x * blockDim.x) {
    const u32 i = perm[j];
    if (status) status[i] = sp[j];
    if (vout) vout[i] = vop[j];
  }
}

int run_device_plain(ws_table* t, const u8* ops, u8 uop, const u64* keys, const u64* vals, u64 n,
                     u8* status, u64* vout, cudaStream_t s, u32 flags, bool has_erase, bool has_upsert,
                     bool query_only, const CallCtx& cx);

// first index of every op-byte value in the sorted op array (~0 when absent)
__global__ void k_seg_starts(const u8* __restrict__ op_sorted, u64 n, u64* start) {
  for (u64 j = blockIdx.x * (u64)blockDim.x + threadIdx.x; j < n; j += (u64)gridDim.x * blockDim.x)
    if (j == 0 || op_sorted[j] != op_sorted[j - 1]) start[op_sorted[j]] = j;
}

// Mixed batches: the generic op kernel carries every op kind's code path
// (~100 KB of SASS for a 32-slot md design); with kinds interleaved at random
// every warp walks all of them and the SMs stall on instruction fetch (ncu:
// 65% "no instruction" stalls in the iceberg aging batch).  Large mixed
// batches are therefore stably partitioned by op byte (kind | merge << 4) and
// each segment runs as its own uniform launch -- upserts of one merge through
// the design's upsert kernel (the tuned lock-round kernel for P2-MD), erases,
// queries through the lock-free query kernel -- one after another on the
// stream, then the results are scattered back.  Running the segments in
// sequence is one serial order of the concurrent batch.
int combine_uniform(ws_table* t, u8 uop, const u64* keys, const u64* vals, u64 n, u8* status, cudaStream_t s,
                    u32 flags, const CallCtx& cx, const u32* oidx, const u64* dn, u64 nbatch);

// ---- split by kind without a sort or a blocking read-back
// A counting partition by op byte (one histogram pass, a scan of the
// bin-major [256 x blocks] counts, one scatter pass; order within a bin is
// arbitrary, so every op carries its batch index) writes the erases and the
// queries into regions of their own, whose bases the host knows, and every
// other op byte into a third region ordered by op byte.  The erase and query
// segments are launched at once with their device-resident counts; the host
// waits only for the 257 bin starts (an event behind the partition) while
// the GPU runs them, then launches the upsert segments at known offsets.
constexpr int kKindTile = 256;

// per-block chunk, a multiple of 32 so every warp's lanes share one loop bound
__device__ __forceinline__ u32 kind_chunk(u64 n, u32 nblk) { return (u32)(((n + nblk - 1) / nblk + 31) & ~31ull); }

__global__ void __launch_bounds__(kKindTile) k_kind_hist(const u8* __restrict__ ops, u64 n, u32* H) {
  __shared__ u32 h[256];
  for (int b = threadIdx.x; b < 256; b += blockDim.x) h[b] = 0;
  __syncthreads();
  const u32 ch = kind_chunk(n, gridDim.x);
  const u64 lo = (u64)blockIdx.x * ch, hi = lo + ch < n ? lo + ch : n;
  for (u64 i = lo + threadIdx.x; i < ((hi + 31) & ~31ull) && lo < hi; i += blockDim.x) {
    const bool act = i < hi;
    const u32 b = act ? ops[i] : 256u;
    const unsigned peers = __match_any_sync(0xFFFFFFFFu, b);
    if (act && (threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&h[b], (u32)__popc(peers));
  }
  __syncthreads();
  for (int b = threadIdx.x; b < 256; b += blockDim.x) H[(u64)b * gridDim.x + blockIdx.x] = h[b];
}

struct KindOut {
  u64 *ke, *kq, *kr, *vr;
  u32 *ie, *iq, *ir;
  u8* opr;
};

// S: exclusive scan of H (bin-major).  Bin 1 (erase) and bin 2 (query) go to
// their own regions; every other bin to the rest region, shifted down by the
// erase and query counts when it sorts above them.
__global__ void __launch_bounds__(kKindTile) k_kind_split(const u8* __restrict__ ops, const u64* __restrict__ keys,
                                                          const u64* __restrict__ vals, u64 n, const u32* S,
                                                          KindOut o) {
  __shared__ u32 cur[256];
  const u32 nb = gridDim.x;
  for (int b = threadIdx.x; b < 256; b += blockDim.x) cur[b] = S[(u64)b * nb + blockIdx.x];
  const u32 s1 = S[1ull * nb], s2 = S[2ull * nb], s3 = S[3ull * nb];
  __syncthreads();
  const u32 ch = kind_chunk(n, nb);
  const u64 lo = (u64)blockIdx.x * ch, hi = lo + ch < n ? lo + ch : n;
  for (u64 i = lo + threadIdx.x; i < ((hi + 31) & ~31ull) && lo < hi; i += blockDim.x) {
    const bool act = i < hi;
    const u32 b = act ? ops[i] : 256u;
    const unsigned peers = __match_any_sync(0xFFFFFFFFu, b);
    const int lane = threadIdx.x & 31, first = __ffs(peers) - 1;
    u32 base = 0;
    if (act && lane == first) base = atomicAdd(&cur[b], (u32)__popc(peers));
    base = __shfl_sync(0xFFFFFFFFu, base, first);
    if (!act) continue;
    const u32 p = base + __popc(peers & ((1u << lane) - 1));
    const u64 k = keys[i];
    if (b == 1) {
      o.ke[p - s1] = k;
      o.ie[p - s1] = (u32)i;
    } else if (b == 2) {
      o.kq[p - s2] = k;
      o.iq[p - s2] = (u32)i;
    } else {
      const u32 r = b > 2 ? p - (s3 - s1) : p;
      o.kr[r] = k;
      o.vr[r] = vals[i];
      o.ir[r] = (u32)i;
      o.opr[r] = (u8)b;
    }
  }
}

// bin starts S[b][0] (b = 0..255) and n, plus the erase / query / rest counts
__global__ void k_kind_starts(const u32* S, u32 nb, u64 n, u64* starts, u64* cnt) {
  const int b = threadIdx.x;
  starts[b] = S[(u64)b * nb];
  if (b == 0) {
    starts[256] = n;
    const u64 s1 = S[1ull * nb], s2 = S[2ull * nb], s3 = S[3ull * nb];
    cnt[0] = s2 - s1;
    cnt[1] = s3 - s2;
    cnt[2] = n - (s3 - s1);
  }
}

// results back to batch order; region 0 erases, 1 queries, 2 the rest
__global__ void k_kind_unsplit(const u64* cnt, const u32* ie, const u8* ste, const u32* iq, const u8* stq,
                               const u64* voq, const u32* ir, const u8* str, const u64* vor, const u8* opr,
                               u8* status, u64* vout) {
  const int g = blockIdx.y;
  const u64 m = cnt[g];
  for (u64 j = blockIdx.x * (u64)blockDim.x + threadIdx.x; j < m; j += (u64)gridDim.x * blockDim.x) {
    if (g == 0) {
      const u32 i = ie[j];
      if (status) status[i] = ste[j];
      if (vout) vout[i] = 0;
    } else if (g == 1) {
      const u32 i = iq[j];
      if (status) status[i] = stq[j];
      if (vout) vout[i] = voq[j];
    } else {
      const u32 i = ir[j];
      if (status) status[i] = str[j];
      if (vout) vout[i] = (opr[j] & 15) == OP_QUERY ? vor[j] : 0;
    }
  }
}

int run_device_split(ws_table* t, const u8* ops, const u64* keys, const u64* vals, u64 n, u8* status, u64* vout,
                     cudaStream_t s, u32 flags, bool has_erase, bool has_upsert, const CallCtx& cx) {
  const u32 nblk = (u32)std::max<u64>(1, std::min<u64>((u64)kSMs * 8, (n + 2047) / 2048));
  const u64 nh = 256ull * nblk;
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, (u32*)nullptr, (u32*)nullptr, (int64_t)nh, s);
  // one scratch allocation, carved
  const u64 need = n * (8 + 4 + 1) + n * (8 + 4 + 1 + 8) + n * (8 + 8 + 4 + 1 + 1 + 8) + 8 * nh + 257 * 8 + 3 * 8 +
                   tb + 24 * 128;
  char* buf = nullptr;
  WS_CK(cudaMallocAsync((void**)&buf, need, s));
  char* p = buf;
  auto carve = [&](u64 bytes) { char* r = p; p += (bytes + 127) & ~127ull; return (void*)r; };
  KindOut o;
  o.ke = (u64*)carve(8 * n); o.ie = (u32*)carve(4 * n); u8* ste = (u8*)carve(n);
  o.kq = (u64*)carve(8 * n); o.iq = (u32*)carve(4 * n); u8* stq = (u8*)carve(n); u64* voq = (u64*)carve(8 * n);
  o.kr = (u64*)carve(8 * n); o.vr = (u64*)carve(8 * n); o.ir = (u32*)carve(4 * n); o.opr = (u8*)carve(n);
  u8* str = (u8*)carve(n); u64* vor = (u64*)carve(8 * n);
  u32* H = (u32*)carve(4 * nh); u32* S = (u32*)carve(4 * nh);
  u64* starts = (u64*)carve(257 * 8); u64* cnt = (u64*)carve(3 * 8);
  void* tmp = carve(tb + 16);
  // WS_F_CONCURRENT_KINDS: erases on se, queries on sq, upserts on s, all
  // concurrent; every segment launch then assumes concurrent erases (the
  // tombstone flag re-read behind a fence, as for multi_stream tables)
  const bool par = (flags & WS_F_CONCURRENT_KINDS) != 0;
  const u32 inner = (flags & ~(WS_F_SYNC_CHECK | WS_F_COMBINE | WS_F_CONCURRENT_KINDS)) | kF_NO_KIND_SORT |
                    ((flags & WS_F_NO_CHECK) ? 0u : (kF_VALIDATED | WS_F_NO_CHECK)) | (par ? kF_CONC_ERASE : 0u);
  const bool comb = (flags & WS_F_COMBINE) != 0;
  Staging* sg = par ? staging(t->device) : nullptr;
  if (par && !sg) { cudaFreeAsync(buf, s); return WS_ERR_ALLOC; }
  cudaStream_t se = par ? sg->s_in : s, sq = par ? sg->s_aux : s;
  cudaEvent_t ev_fork = nullptr, ev_e = nullptr, ev_q = nullptr;
  k_kind_hist<<<nblk, kKindTile, 0, s>>>(ops, n, H);
  cub::DeviceScan::ExclusiveSum(tmp, tb, H, S, (int64_t)nh, s);
  k_kind_split<<<nblk, kKindTile, 0, s>>>(ops, keys, vals, n, S, o);
  k_kind_starts<<<1, 256, 0, s>>>(S, nblk, n, starts, cnt);
  int rc = cuda_err(cudaGetLastError());
  u64* hst = pin_call();
  if (!hst) rc = WS_ERR_ALLOC;
  cudaEvent_t ev = nullptr;
  if (!rc) rc = cuda_err(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  if (!rc) rc = cuda_err(cudaMemcpyAsync(hst, starts, 257 * 8, cudaMemcpyDeviceToHost, s));
  if (!rc) rc = cuda_err(cudaEventRecord(ev, s));
  if (par && !rc) {
    for (cudaEvent_t* e : {&ev_fork, &ev_e, &ev_q})
      if (!rc) rc = cuda_err(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    if (!rc) rc = cuda_err(cudaEventRecord(ev_fork, s));
    if (!rc) rc = cuda_err(cudaStreamWaitEvent(se, ev_fork, 0));
    if (!rc) rc = cuda_err(cudaStreamWaitEvent(sq, ev_fork, 0));
  }
  // erases and queries at once, their counts read on the device
  if (!rc) {
    CallCtx ce = cx;
    ce.dn = cnt;
    rc = run_device_plain(t, nullptr, OP_ERASE, o.ke, nullptr, n, ste, nullptr, se, inner, true, false, false, ce);
  }
  if (!rc) {
    CallCtx cq = cx;
    cq.dn = cnt + 1;
    rc = run_device_plain(t, nullptr, OP_QUERY, o.kq, nullptr, n, stq, voq, sq, inner, par, false, true, cq);
  }
  if (par && !rc) rc = cuda_err(cudaEventRecord(ev_e, se));
  if (par && !rc) rc = cuda_err(cudaEventRecord(ev_q, sq));
  if (!rc) rc = cuda_err(cudaEventSynchronize(ev));
  std::vector<u64> st_h(257, 0);
  if (!rc) std::copy(hst, hst + 257, st_h.begin());
  const u64* hs = st_h.data();
  // the rest region, one segment per op byte present, in op-byte order
  const u64 c1 = hs[2] - hs[1], c2 = hs[3] - hs[2];
  for (int v = 0; v < 256 && !rc; v++) {
    if (v == 1 || v == 2) continue;
    const u64 lo = hs[v] - (v > 2 ? c1 + c2 : 0), m = hs[v + 1] - hs[v];
    if (!m) continue;
    const int kind = v & 15, merge = v >> 4;
    if (kind == OP_UPSERT && merge <= M_MIN) {
      rc = comb && m >= 2 ? combine_uniform(t, (u8)v, o.kr + lo, o.vr + lo, m, str + lo, s, inner, cx, o.ir + lo,
                                            nullptr, n)
                          : run_device_plain(t, nullptr, (u8)v, o.kr + lo, o.vr + lo, m, str + lo, nullptr, s, inner,
                                             par, true, false, cx);
    } else {  // erase / query bytes with stray merge bits, invalid bytes (gated): the generic kernel
      rc = run_device_plain(t, o.opr + lo, 0, o.kr + lo, o.vr + lo, m, str + lo, vor + lo, s, inner,
                            has_erase || par, has_upsert, false, cx);
    }
  }
  if (par) {  // join the side streams before the results are gathered (and before any error return)
    if (ev_e) cudaStreamWaitEvent(s, ev_e, 0);
    if (ev_q) cudaStreamWaitEvent(s, ev_q, 0);
  }
  if (!rc) {
    dim3 g(grid_for(n, kThreads, kTableGridPerSM), 3);
    k_kind_unsplit<<<g, kThreads, 0, s>>>(cnt, o.ie, ste, o.iq, stq, voq, o.ir, str, vor, o.opr, status, vout);
    rc = cuda_err(cudaGetLastError());
  }
  for (cudaEvent_t e : {ev, ev_fork, ev_e, ev_q})
    if (e) cudaEventDestroy(e);
  cudaFreeAsync(buf, s);
  return rc;
}

int run_device_by_kind(ws_table* t, const u8* ops, u8 uop, const u64* keys, const u64* vals, u64 n, u8* status,
                       u64* vout, cudaStream_t s, u32 flags, bool has_erase, bool has_upsert, const CallCtx& cx) {
  int rc = validate(keys, ops, n, s, (flags & WS_F_SYNC_CHECK) != 0, flags, cx);
  if (rc) return rc;
  if (vals && n < (1ull << 31)) return run_device_split(t, ops, keys, vals, n, status, vout, s, flags, has_erase,
                                                          has_upsert, cx);
  u8 *op_p = nullptr, *st_p = nullptr;
  u32 *idx = nullptr, *perm = nullptr;
  u64 *k_p = nullptr, *v_p = nullptr, *vo_p = nullptr, *starts = nullptr;
  void* tmp = nullptr;
  size_t tb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tb, ops, op_p, idx, perm, (int64_t)n, 0, 8, s);
  WS_CK(cudaMallocAsync((void**)&op_p, n, s));
  WS_CK(cudaMallocAsync((void**)&st_p, n, s));
  WS_CK(cudaMallocAsync((void**)&idx, 4 * n, s));
  WS_CK(cudaMallocAsync((void**)&perm, 4 * n, s));
  WS_CK(cudaMallocAsync((void**)&k_p, 8 * n, s));
  WS_CK(cudaMallocAsync((void**)&starts, 8 * 256, s));
  if (vals) WS_CK(cudaMallocAsync((void**)&v_p, 8 * n, s));
  if (vout) WS_CK(cudaMallocAsync((void**)&vo_p, 8 * n, s));
  WS_CK(cudaMallocAsync(&tmp, tb + 16, s));
  k_comb_iota<<<grid_for(n), kThreads, 0, s>>>(n, idx);
  cub::DeviceRadixSort::SortPairs(tmp, tb, ops, op_p, idx, perm, (int64_t)n, 0, 8, s);
  k_kind_gather<<<grid_for(n), kThreads, 0, s>>>(perm, keys, vals, n, k_p, v_p);
  WS_CK(cudaMemsetAsync(starts, 0xFF, 8 * 256, s));
  k_seg_starts<<<grid_for(n), kThreads, 0, s>>>(op_p, n, starts);
  rc = cuda_err(cudaGetLastError());
  std::vector<u64> st_h(256);
  if (!rc) rc = cuda_err(cudaMemcpyAsync(st_h.data(), starts, 8 * 256, cudaMemcpyDeviceToHost, s));
  if (!rc) rc = cuda_err(cudaStreamSynchronize(s));
  const bool comb = (flags & WS_F_COMBINE) != 0;
  const u32 inner = (flags & ~(WS_F_SYNC_CHECK | WS_F_COMBINE)) | kF_NO_KIND_SORT |
                    ((flags & WS_F_NO_CHECK) ? 0u : (kF_VALIDATED | WS_F_NO_CHECK));
  // segments in op-byte order
  std::vector<std::pair<u64, int>> seg;
  for (int v = 0; v < 256; v++)
    if (st_h[v] != ~0ull) seg.push_back({st_h[v], v});
  std::sort(seg.begin(), seg.end());
  for (size_t q = 0; q < seg.size() && !rc; q++) {
    const u64 lo = seg[q].first, hi = q + 1 < seg.size() ? seg[q + 1].first : n;
    const u8 v = (u8)seg[q].second;
    const int kind = v & 15, merge = v >> 4;
    const u64 m = hi - lo;
    if (kind == OP_UPSERT && merge <= M_MIN && v_p) {
      rc = comb && m >= 2 ? combine_uniform(t, v, k_p + lo, v_p + lo, m, st_p + lo, s, inner, cx, nullptr, nullptr, 0)
                          : run_device_plain(t, nullptr, v, k_p + lo, v_p + lo, m, st_p + lo, nullptr, s, inner,
                                             false, true, false, cx);
      if (vo_p && !rc) rc = cuda_err(cudaMemsetAsync(vo_p + lo, 0, 8 * m, s));
    } else if (kind == OP_ERASE && merge == 0) {
      rc = run_device_plain(t, nullptr, v, k_p + lo, nullptr, m, st_p + lo, nullptr, s, inner, true, false, false,
                            cx);
      if (vo_p && !rc) rc = cuda_err(cudaMemsetAsync(vo_p + lo, 0, 8 * m, s));
    } else if (kind == OP_QUERY && merge == 0) {
      rc = run_device_plain(t, nullptr, v, k_p + lo, nullptr, m, st_p + lo, vo_p ? vo_p + lo : nullptr, s, inner,
                            false, false, true, cx);
    } else {  // value-less upserts or invalid op bytes (gated): the generic kernel handles them
      rc = run_device_plain(t, op_p + lo, 0, k_p + lo, v_p ? v_p + lo : nullptr, m, st_p + lo,
                            vo_p ? vo_p + lo : nullptr, s, inner, has_erase, has_upsert, false, cx);
    }
  }
  if (!rc) {
    k_kind_scatter<<<grid_for(n), kThreads, 0, s>>>(perm, st_p, vo_p, n, status, vout);
    rc = cuda_err(cudaGetLastError());
  }
  for (void* p : {(void*)op_p, (void*)st_p, (void*)idx, (void*)perm, (void*)k_p, (void*)v_p, (void*)vo_p,
                  (void*)starts, tmp})
    if (p) cudaFreeAsync(p, s);
  return rc;
}

// open / close a kernel-timing bracket (WS_TUNE_KERNEL_EVENTS)
cudaEvent_t kev_begin(ws_table* t, cudaStream_t s) {
  if (!t->time_kernels) return nullptr;
  cudaEvent_t e = nullptr;
  if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
  cudaEventRecord(e, s);
  return e;
}
void kev_end(ws_table* t, cudaStream_t s, cudaEvent_t b) {
  if (!b) return;
  cudaEvent_t e = nullptr;
  if (cudaEventCreate(&e) != cudaSuccess) { cudaEventDestroy(b); return; }
  cudaEventRecord(e, s);
  std::lock_guard<std::mutex> g(t->ev_mu);
  t->kev.push_back({b, e});
}

int run_device_plain(ws_table* t, const u8* ops, u8 uop, const u64* keys, const u64* vals, u64 n,
                     u8* status, u64* vout, cudaStream_t s, u32 flags, bool has_erase, bool has_upsert,
                     bool query_only, const CallCtx& cx) {
  if (ops && !query_only && n >= (1u << 16) && n < (1ull << 32) && !t->d.delay_ns && !cx.dn &&
      !(flags & (WS_F_SERIAL | WS_F_INTERLEAVED | kF_NO_KIND_SORT)))
    return run_device_by_kind(t, ops, uop, keys, vals, n, status, vout, s, flags, has_erase, has_upsert, cx);
  const bool sync = (flags & WS_F_SYNC_CHECK) != 0;
  int rc = validate(keys, ops, n, s, sync, flags, cx);
  if (rc) return rc;
  if (!n) return WS_OK;
  const int gated = (flags & kF_VALIDATED) ? 1 : (flags & WS_F_NO_CHECK) ? 0 : 1;
  int conc = (has_erase || t->cfg.multi_stream || (flags & kF_CONC_ERASE)) ? 1 : 0;
  if (ops && !t->cfg.multi_stream && !(flags & (WS_F_SERIAL | kF_CONC_ERASE))) {
    // let the device decide: conc_erase = 2 reads the erase count at launch
    WS_CK(cudaMemsetAsync(cx.cs + 3, 0, sizeof(u32), s));
    k_count_erases<<<grid_for(n, kThreads, 4), kThreads, 0, s>>>(ops, n, cx.cs);
    conc = 2;
  }
  if (query_only && !(flags & WS_F_SERIAL)) {
    QueryArgs qa{dev_of(t, cx), keys, n, vout, status, conc, gated, t->cfg.phased ? 1 : 0, s};
    cudaEvent_t kb = kev_begin(t, s);
    t->L.query(qa, t->def_bs);
    kev_end(t, s, kb);
    return cuda_err(cudaGetLastError());
  }
  const bool chain_up = t->cfg.design == D_CHAINING && has_upsert;
  u8* st = status;
  if (chain_up && !st) {  // the grow-and-redo protocol needs per-op statuses
    WS_CK(cudaMallocAsync((void**)&st, n, s));
  }
  if (chain_up) WS_CK(cudaMemsetAsync(cx.cs + 2, 0, sizeof(u32), s));
  OpsArgs lo{dev_of(t, cx), ops, uop, keys, vals, n, st, vout, nullptr, nullptr, nullptr, conc, gated, 0,
             (flags & WS_F_SERIAL) ? 1 : 0, s};
  cudaEvent_t kb = kev_begin(t, s);
  t->L.ops(lo, t->def_bs);
  kev_end(t, s, kb);
  rc = cuda_err(cudaGetLastError());
  while (rc == WS_OK && chain_up) {
    u64* hp = pin();
    if (!hp) { rc = WS_ERR_ALLOC; break; }
    WS_CK(cudaMemcpyAsync(hp, cx.cs + 2, sizeof(u32), cudaMemcpyDeviceToHost, s));
    WS_CK(cudaStreamSynchronize(s));
    if (!*(const u32*)hp) break;
    // the pool is exhausted: grow it exclusively (unless a concurrent call
    // already did), then redo this launch's deferred ops
    const u64 seen = lo.d.chain_cap;
    cx.lk->unlock();
    {
      std::unique_lock<std::shared_mutex> ex(t->mu);
      if (t->d.chain_cap == seen) rc = chain_grow(t, s);
    }
    cx.lk->lock();
    if (rc) break;
    WS_CK(cudaMemsetAsync(cx.cs + 2, 0, sizeof(u32), s));
    lo.redo = st;
    lo.d = dev_of(t, cx);  // the pool moved
    t->L.ops(lo, t->def_bs);
    rc = cuda_err(cudaGetLastError());
  }
  if (st != status) cudaFreeAsync(st, s);
  return rc;
}

// ------------------------------------------------------------------ combining
// WS_F_COMBINE: same-key upserts of one batch are reduced before they touch
// the table; one op per (key, merge) group is applied and the statuses are
// expanded: the group leader gets the real status, the other members
// UPDATED (FULL if the leader was).  Equivalent to a serial order of the
// batch in which each group's upserts run back to back, in batch-index order;
// the point is Zipf hot keys, whose ops would otherwise serialise on one
// bucket lock.
//   * mixed batches are first split by op byte (run_device_by_kind); every
//     upsert segment (one merge) is then combined on its own;
//   * every merge uses hash aggregation into an L2-resident open-addressing
//     table (claim by CAS): ADD / MAX / MIN fold the values with one atomic
//     per warp group; REPLACE keeps the value of the group's HIGHEST batch
//     index (atomicMax on index+1: the last write of the serial order), KEEP
//     the value of its LOWEST (the first write; later KEEPs keep it).  The
//     leader -- the op reporting INSERTED for a new key -- is the lowest batch
//     index.  Compaction of the leaders, then the apply, with the group count
//     read on the device: no sort and no host synchronisation.
//   * `oidx` (optional) maps a segment position to its batch index when the
//     segment was gathered out of order (run_device_by_kind); `dn` (optional)
//     is the segment's device-resident length (n = its upper bound).
__global__ void k_comb_iota(u64 n, u32* idx) {
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) idx[i] = (u32)i;
}

__device__ __forceinline__ u64 merge_of(int merge, u64 a, u64 b) {
  return merge == M_ADD ? a + b : merge == M_MAX ? (a > b ? a : b) : (a < b ? a : b);
}
__device__ __forceinline__ u64 dev_n(u64 n, const u64* dn) { return dn && *dn < n ? *dn : n; }

// one slot of the scratch aggregation table: key, folded value (REPLACE: the
// group's highest batch index + 1), leader (lowest batch index) and group
// number share one 32-byte sector, so an op touches one DRAM line
struct __align__(32) AggSlot {
  u64 key;
  u64 val;
  u32 leader;
  u32 slot2g;
  u64 pad;
};
__global__ void k_agg_init(AggSlot* tab, u64 cap, u64 ident) {
  for (u64 h = blockIdx.x * (u64)blockDim.x + threadIdx.x; h < cap; h += (u64)gridDim.x * blockDim.x)
    tab[h] = AggSlot{0ull, ident, 0xFFFFFFFFu, 0u, 0ull};
}

// Lanes of a warp holding the same key fold first (__match_any_sync), so a
// Zipf hot key costs one table atomic per warp instead of one per op.
__global__ void __launch_bounds__(256) k_agg_insert(const u64* __restrict__ keys, const u64* __restrict__ vals,
                                                    const u32* __restrict__ oidx, u64 n, const u64* dn, int merge,
                                                    AggSlot* tab, u64 mask, u32* grp) {
  n = dev_n(n, dn);
  const int lane = threadIdx.x & 31;
  const bool fold = merge == M_ADD || merge == M_MAX || merge == M_MIN;
  for (u64 base = (blockIdx.x * (u64)blockDim.x + threadIdx.x) & ~31ull; base < n;
       base += (u64)gridDim.x * blockDim.x) {
    const u64 i = base + lane;
    const bool act = i < n;
    const u64 key = act ? __ldg(keys + i) : 0ull;
    const u64 v0 = act && fold ? __ldg(vals + i) : 0ull;
    u64 v = v0;
    const u32 bi = act ? (oidx ? __ldg(oidx + i) : (u32)i) : 0xFFFFFFFFu;  // batch index
    const unsigned act_m = __ballot_sync(0xFFFFFFFFu, act);
    const unsigned same = __match_any_sync(0xFFFFFFFFu, key) & act_m;
    // the group's lowest and highest batch index, and (fold) its folded value,
    // gathered into every member lane (all lanes take part in every shuffle)
    u32 lo = bi, hi = act ? bi : 0u;
    for (int j = 0; j < 32; j++) {
      const u64 vj = __shfl_sync(0xFFFFFFFFu, v0, j);  // members' own values, not partial folds
      const u32 bj = __shfl_sync(0xFFFFFFFFu, bi, j);
      if (act && j != lane && ((same >> j) & 1u)) {
        if (fold && j < lane) v = merge_of(merge, v, vj);
        lo = bj < lo ? bj : lo;
        hi = bj > hi ? bj : hi;
      }
    }
    // one lane per warp group talks to the table: the group's last lane,
    // which (fold) now holds the fold of every member
    const int last = same ? 31 - __clz(same) : -1;
    u64 h = 0;
    if (act && lane == last) {
      h = mix64(key ^ 0x9E3779B97F4A7C15ull) & mask;
      while (true) {
        const u64 cur = *(volatile const u64*)&tab[h].key;
        if (cur == key) break;
        if (cur == 0) {
          const u64 prev = atomicCAS((unsigned long long*)&tab[h].key, 0ull, (unsigned long long)key);
          if (prev == 0 || prev == key) break;
        }
        h = (h + 1) & mask;
      }
      // key, value and leader share the slot's 32-byte sector: one DRAM line
      // per op.  The leader and the MAX / MIN / REPLACE values only ever move
      // one way, so an atomic is issued only when the current value (a plain
      // read; a stale one only costs an extra atomic) would change: a hot
      // key's group then takes ~ln(m) of them instead of one per warp
      AggSlot& e = tab[h];
      if (*(volatile const u32*)&e.leader > lo) atomicMin(&e.leader, lo);
      unsigned long long* tv = (unsigned long long*)&e.val;
      const u64 cur = merge == M_ADD ? 0ull : *(volatile const u64*)&e.val;
      if (merge == M_ADD) atomicAdd(tv, (unsigned long long)v);
      else if (merge == M_MAX) { if (cur < v) atomicMax(tv, (unsigned long long)v); }
      else if (merge == M_MIN) { if (cur > v) atomicMin(tv, (unsigned long long)v); }
      else if (merge == M_REPLACE) { if (cur < (u64)hi + 1) atomicMax(tv, (unsigned long long)hi + 1); }
    }
    h = __shfl_sync(0xFFFFFFFFu, h, last < 0 ? 0 : last);
    if (act) grp[i] = (u32)h;
  }
}

// one group per leader op (ops, not table slots, are scanned).  REPLACE /
// KEEP: the winning op's value is read back through a batch-index -> segment
// position map (pos), the identity when the segment is in batch order.
__global__ void __launch_bounds__(256) k_agg_compact(const u64* __restrict__ keys, const u64* __restrict__ vals,
                                                     const u32* __restrict__ oidx, const u32* __restrict__ grp,
                                                     AggSlot* tab, const u32* pos, u64 n,
                                                     const u64* dn, int merge, u64* gkey, u64* gval,
                                                     u64* ng) {
  n = dev_n(n, dn);
  const int lane = threadIdx.x & 31;
  for (u64 base = (blockIdx.x * (u64)blockDim.x + threadIdx.x) & ~31ull; base < n;
       base += (u64)gridDim.x * blockDim.x) {
    const u64 i = base + lane;
    const u32 h = i < n ? grp[i] : 0u;
    const u32 bi = i < n ? (oidx ? oidx[i] : (u32)i) : 0u;
    const bool lead = i < n && tab[h].leader == bi;
    const u32 m = __ballot_sync(0xFFFFFFFFu, lead);
    if (!m) continue;
    u64 at = 0;
    if (lane == 0) at = atomicAdd((unsigned long long*)ng, (unsigned long long)__popc(m));
    at = __shfl_sync(0xFFFFFFFFu, at, 0);
    if (lead) {
      const u64 g = at + __popc(m & ((1u << lane) - 1));
      gkey[g] = __ldg(keys + i);
      u64 v;
      if (merge == M_KEEP) v = __ldg(vals + i);  // the leader is the first write
      else if (merge == M_REPLACE) {
        const u32 w = (u32)(tab[h].val - 1);  // highest batch index of the group
        v = __ldg(vals + (pos ? pos[w] : w));
      } else v = tab[h].val;
      gval[g] = v;
      tab[h].slot2g = (u32)g;
    }
  }
}

__global__ void k_pos_of(const u32* __restrict__ oidx, u64 n, const u64* dn, u32* pos) {
  n = dev_n(n, dn);
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x)
    pos[oidx[i]] = (u32)i;
}

__global__ void k_agg_expand(const u32* grp, const AggSlot* tab, const u32* __restrict__ oidx,
                             u64 n, const u64* dn, const u8* gst, u8* status) {
  n = dev_n(n, dn);
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
    const u32 h = grp[i];
    const u8 gs = gst[tab[h].slot2g];
    const u32 bi = oidx ? oidx[i] : (u32)i;
    status[i] = tab[h].leader == bi ? gs : (gs == S_FULL ? (u8)S_FULL : (u8)S_UPDATED);
  }
}

// one uniform upsert batch (merge = uop >> 4), combined; see above.  oidx /
// dn / nbatch: a gathered segment (positions -> batch indices < nbatch, the
// device-resident length dn); all null / 0 for a plain batch.
int combine_uniform(ws_table* t, u8 uop, const u64* keys, const u64* vals, u64 n, u8* status, cudaStream_t s,
                    u32 flags, const CallCtx& cx, const u32* oidx, const u64* dn, u64 nbatch) {
  int rc = dn ? WS_OK : validate(keys, nullptr, n, s, (flags & WS_F_SYNC_CHECK) != 0, flags, cx);
  if (rc) return rc;
  // the folded batch keeps the kernels gated on this call's validation verdict
  // (an asynchronous check is not read back here, but a batch holding a
  // sentinel key still mutates nothing)
  const u32 inner = (flags & ~(WS_F_COMBINE | WS_F_SYNC_CHECK)) | WS_F_NO_CHECK |
                    ((flags & WS_F_NO_CHECK) && !(flags & kF_VALIDATED) ? 0u : kF_VALIDATED);
  const int m = uop >> 4;
  std::vector<void*> mem;
  auto alloc = [&](size_t bytes) -> void* {
    void* p = nullptr;
    if (cudaMallocAsync(&p, bytes ? bytes : 16, s) != cudaSuccess) return nullptr;
    mem.push_back(p);
    return p;
  };
  auto release = [&]() { for (void* p : mem) cudaFreeAsync(p, s); };
  const u64 cap = next_pow2(n + n / 2);  // load <= 2/3; 32 B/slot, L2-resident up to ~2M ops
  u8* gst = (u8*)alloc(n);
  u64* gkey = (u64*)alloc(8 * n);
  u64* gval = (u64*)alloc(8 * n);
  u64* ng = (u64*)alloc(8);
  AggSlot* tab = (AggSlot*)alloc(sizeof(AggSlot) * cap);
  u32* grp = (u32*)alloc(4 * n);
  u32* pos = (oidx && m == M_REPLACE) ? (u32*)alloc(4 * std::max<u64>(nbatch, 1)) : nullptr;
  if (!gst || !gkey || !gval || !ng || !tab || !grp || (oidx && m == M_REPLACE && !pos)) {
    release();
    return WS_ERR_ALLOC;
  }
  k_agg_init<<<grid_for(cap), kThreads, 0, s>>>(tab, cap, m == M_MIN ? ~0ull : 0ull);  // merge identity
  WS_CK(cudaMemsetAsync(ng, 0, 8, s));
  if (pos) k_pos_of<<<grid_for(n), kThreads, 0, s>>>(oidx, n, dn, pos);
  // random table accesses: the table kernels' launch shape (ws_kernels.cuh kTableGridPerSM)
  k_agg_insert<<<grid_for(n, 256, kTableGridPerSM), 256, 0, s>>>(keys, vals, oidx, n, dn, m, tab, cap - 1, grp);
  k_agg_compact<<<grid_for(n, 256, kTableGridPerSM), 256, 0, s>>>(keys, vals, oidx, grp, tab, pos, n, dn, m, gkey,
                                                                   gval, ng);
  rc = cuda_err(cudaGetLastError());
  CallCtx gcx = cx;
  gcx.dn = ng;  // the group count stays on the device
  if (!rc) rc = run_device_plain(t, nullptr, uop, gkey, gval, n, gst, nullptr, s, inner, false, true, false, gcx);
  if (!rc && status) {
    k_agg_expand<<<grid_for(n, kThreads, kTableGridPerSM), kThreads, 0, s>>>(grp, tab, oidx, n, dn, gst, status);
    rc = cuda_err(cudaGetLastError());
  }
  release();
  return rc;
}

int run_device(ws_table* t, const u8* ops, u8 uop, const u64* keys, const u64* vals, u64 n,
               u8* status, u64* vout, cudaStream_t s, u32 flags, bool has_erase, bool has_upsert,
               bool query_only, const CallCtx& cx) {
  const bool comb = (flags & WS_F_COMBINE) && !query_only && has_upsert && n >= 2 && n < (1ull << 32) &&
                    !(flags & (WS_F_SERIAL | WS_F_INTERLEAVED)) && !cx.dn && !t->d.delay_ns && vals;
  if (!comb)
    return run_device_plain(t, ops, uop, keys, vals, n, status, vout, s, flags & ~WS_F_COMBINE, has_erase,
                            has_upsert, query_only, cx);
  if (ops)  // split by op byte; each upsert segment is combined (run_device_by_kind)
    return run_device_by_kind(t, ops, uop, keys, vals, n, status, vout, s, flags, has_erase, has_upsert, cx);
  if (vout) WS_CK(cudaMemsetAsync(vout, 0, 8 * n, s));
  return combine_uniform(t, uop, keys, vals, n, status, s, flags, cx, nullptr, nullptr, 0);
}

// Host-buffer batches: staged through device memory in 4M-op chunks on three
// streams -- H2D on s_in, validation + kernels on the caller's stream, D2H on
// s_aux -- so copies in both directions overlap compute.  Queries never
// mutate, so each chunk is queried as soon as it lands and an invalid key is
// reported after the fact.  Mutating batches must be validated in full before
// the first mutation: all chunks are copied and validated (overlapped), one
// sync reads the verdict, then compute and D2H overlap chunk by chunk.
// Sentinel / op-byte scan of host-resident batch inputs on all host cores
// (same rule as k_validate): WS_OK, WS_ERR_INVALID_KEY or WS_ERR_INVALID_OP.
int host_validate(const u64* keys, const u8* ops, u64 n) {
  unsigned nt = std::thread::hardware_concurrency();
  nt = std::max(1u, std::min(nt, 16u));
  if (n < ((u64)1 << 20)) nt = 1;
  std::vector<int> res(nt, WS_OK);
  auto work = [&](unsigned w) {
    const u64 lo = n * w / nt, hi = n * (w + 1) / nt;
    for (u64 b = lo; b < hi; b += 4096) {
      const u64 e = std::min(hi, b + 4096);
      u64 bad = 0;
      for (u64 i = b; i < e; i++) bad |= (u64)(keys[i] - 1 >= 0xFFFFFFFFFFFFFFFDull);  // 0, 2^64-2, 2^64-1
      if (bad) { res[w] = WS_ERR_INVALID_KEY; return; }
      if (ops) {
        u32 bo = 0;
        for (u64 i = b; i < e; i++) bo |= (u32)((ops[i] & 15) > OP_QUERY) | (u32)((ops[i] >> 4) > M_MIN);
        if (bo) res[w] = WS_ERR_INVALID_OP;  // keep scanning: a bad key anywhere wins
      }
    }
  };
  if (nt == 1) {
    work(0);
  } else {
    std::vector<std::thread> th;
    for (unsigned w = 1; w < nt; w++) th.emplace_back(work, w);
    work(0);
    for (auto& x : th) x.join();
  }
  int rc = WS_OK;
  for (int r : res) {
    if (r == WS_ERR_INVALID_KEY) return r;
    if (r) rc = r;
  }
  return rc;
}

int run_staged(ws_table* t, const u8* ops, u8 uop, const u64* keys, const u64* vals, u64 n,
               u8* status, u64* vout, cudaStream_t s, u32 flags, bool has_erase, bool has_upsert,
               bool query_only, const CallCtx& cx) {
  if (!n) return WS_OK;
  Staging* sg = staging(t->device);
  u64* hp = pin();
  if (!sg || !hp) return WS_ERR_ALLOC;
  const bool k_dev = is_device_ptr(keys), v_dev = is_device_ptr(vals), o_dev = is_device_ptr(ops);
  const bool st_dev = is_device_ptr(status), vo_dev = is_device_ptr(vout);
  const bool hk = !k_dev, hv = vals && !v_dev, ho = ops && !o_dev;
  const bool hst = status && !st_dev, hvo = vout && !vo_dev;
  char* buf = nullptr;
  const u64 need = n * (8 * hk + 8 * hv + ho + hst + 8 * hvo) + 6 * 128;
  WS_CK(cudaMallocAsync((void**)&buf, need, s));
  char* p = buf;
  auto carve = [&](u64 bytes) { char* r = p; p += (bytes + 127) & ~127ull; return r; };
  const u64* dk = hk ? (const u64*)carve(8 * n) : keys;
  const u64* dv = hv ? (const u64*)carve(8 * n) : vals;
  const u8* dops = ho ? (const u8*)carve(n) : ops;
  u8* dst = hst ? (u8*)carve(n) : status;
  u64* dvo = hvo ? (u64*)carve(8 * n) : vout;
  const bool check = !(flags & WS_F_NO_CHECK);
  if (check) WS_CK(cudaMemsetAsync(cx.cs, 0, 2 * sizeof(u32), s));
  WS_CK(cudaEventRecord(sg->ev_b, s));  // staging allocation visible to s_in / s_aux
  WS_CK(cudaStreamWaitEvent(sg->s_in, sg->ev_b, 0));
  WS_CK(cudaStreamWaitEvent(sg->s_aux, sg->ev_b, 0));
  const bool chain_up = t->cfg.design == D_CHAINING && has_upsert;
  const u64 chunk = chain_up ? n : (u64)1 << 22;
  const u32 sub = WS_F_NO_CHECK | (flags & (WS_F_SERIAL | WS_F_COMBINE));
  int rc = WS_OK;
  auto h2d = [&](u64 off, u64 m) -> int {
    if (hk) WS_CK(cudaMemcpyAsync((void*)(dk + off), keys + off, 8 * m, cudaMemcpyHostToDevice, sg->s_in));
    if (hv) WS_CK(cudaMemcpyAsync((void*)(dv + off), vals + off, 8 * m, cudaMemcpyHostToDevice, sg->s_in));
    if (ho) WS_CK(cudaMemcpyAsync((void*)(dops + off), ops + off, m, cudaMemcpyHostToDevice, sg->s_in));
    WS_CK(cudaEventRecord(sg->ev_in, sg->s_in));
    WS_CK(cudaStreamWaitEvent(s, sg->ev_in, 0));
    if (check) k_validate<<<grid_for(m / 2 + 1, kThreads, 8), kThreads, 0, s>>>(dk + off, dops ? dops + off : nullptr, m,
                                                                         cx.cs);
    return cuda_err(cudaGetLastError());
  };
  auto d2h = [&](u64 off, u64 m) -> int {
    if (!hst && !hvo) return WS_OK;
    WS_CK(cudaEventRecord(sg->ev_a, s));
    WS_CK(cudaStreamWaitEvent(sg->s_aux, sg->ev_a, 0));
    if (hst) WS_CK(cudaMemcpyAsync(status + off, dst + off, m, cudaMemcpyDeviceToHost, sg->s_aux));
    if (hvo) WS_CK(cudaMemcpyAsync(vout + off, dvo + off, 8 * m, cudaMemcpyDeviceToHost, sg->s_aux));
    return WS_OK;
  };
  auto compute = [&](u64 off, u64 m) -> int {
    return run_device(t, dops ? dops + off : nullptr, uop, dk + off, dv ? dv + off : nullptr, m,
                      dst ? dst + off : nullptr, dvo ? dvo + off : nullptr, s, sub, has_erase, has_upsert,
                      query_only, cx);
  };
  if (query_only) {
    for (u64 off = 0; off < n && rc == WS_OK; off += chunk) {
      const u64 m = std::min(chunk, n - off);
      rc = h2d(off, m);
      if (!rc) rc = compute(off, m);
      if (!rc) rc = d2h(off, m);
    }
  } else {
    // A mutation may not start before the WHOLE batch is validated (the
    // reference rejects a batch with a sentinel key before any op runs).
    // Host-resident inputs are validated on the host, by all cores, WHILE
    // the copy engine streams them in; each chunk's compute then starts as
    // soon as its own copy lands, so the kernels hide under the H2D stream.
    const u64 nch = (n + chunk - 1) / chunk;
    while (sg->ev_chunk.size() < nch) {
      cudaEvent_t e;
      WS_CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      sg->ev_chunk.push_back(e);
    }
    for (u64 c = 0; c < nch; c++) {
      const u64 off = c * chunk, m = std::min(chunk, n - off);
      if (hk) WS_CK(cudaMemcpyAsync((void*)(dk + off), keys + off, 8 * m, cudaMemcpyHostToDevice, sg->s_in));
      if (hv) WS_CK(cudaMemcpyAsync((void*)(dv + off), vals + off, 8 * m, cudaMemcpyHostToDevice, sg->s_in));
      if (ho) WS_CK(cudaMemcpyAsync((void*)(dops + off), ops + off, m, cudaMemcpyHostToDevice, sg->s_in));
      WS_CK(cudaEventRecord(sg->ev_chunk[c], sg->s_in));
    }
    if (check && hk && (!ops || ho)) {
      rc = host_validate(keys, ho ? ops : nullptr, n);
    } else if (check) {
      for (u64 c = 0; c < nch; c++) {
        const u64 off = c * chunk, m = std::min(chunk, n - off);
        WS_CK(cudaStreamWaitEvent(s, sg->ev_chunk[c], 0));
        k_validate<<<grid_for(m / 2 + 1, kThreads, 8), kThreads, 0, s>>>(dk + off, dops ? dops + off : nullptr, m,
                                                                 cx.cs);
      }
      WS_CK(cudaGetLastError());
      WS_CK(cudaMemcpyAsync(hp, cx.cs, 2 * sizeof(u32), cudaMemcpyDeviceToHost, s));
      WS_CK(cudaStreamSynchronize(s));
      const u32* c = (const u32*)hp;
      if (c[0]) rc = WS_ERR_INVALID_KEY;
      else if (c[1]) rc = WS_ERR_INVALID_OP;
    }
    for (u64 c = 0; c < nch && rc == WS_OK; c++) {
      const u64 off = c * chunk, m = std::min(chunk, n - off);
      WS_CK(cudaStreamWaitEvent(s, sg->ev_chunk[c], 0));
      rc = compute(off, m);
      if (!rc) rc = d2h(off, m);
    }
  }
  WS_CK(cudaEventRecord(sg->ev_b, sg->s_aux));
  WS_CK(cudaStreamWaitEvent(s, sg->ev_b, 0));
  WS_CK(cudaEventRecord(sg->ev_in, sg->s_in));
  WS_CK(cudaStreamWaitEvent(s, sg->ev_in, 0));
  cudaFreeAsync(buf, s);
  if (query_only && check && rc == WS_OK) {
    WS_CK(cudaMemcpyAsync(hp, cx.cs, 2 * sizeof(u32), cudaMemcpyDeviceToHost, s));
    WS_CK(cudaStreamSynchronize(s));
    const u32* c = (const u32*)hp;
    if (c[0]) rc = WS_ERR_INVALID_KEY;
  }
  WS_CK(cudaStreamSynchronize(s));
  return rc;
}

int run_batch(ws_table* t, const u8* ops, u8 uop, const u64* keys, const u64* vals, u64 n,
              u8* status, u64* vout, void* stream, u32 flags, bool has_erase, bool has_upsert,
              bool query_only) {
  if (!t || (!keys && n)) return WS_ERR_ARG;
  if (cudaSetDevice(t->device) != cudaSuccess) return WS_ERR_CUDA;
  cudaGetLastError();  // drop any stale error from an earlier, unrelated call
  cudaStream_t s = S(stream);
  const bool all_dev = is_device_ptr(keys) && is_device_ptr(vals) && is_device_ptr(ops) &&
                       is_device_ptr(status) && is_device_ptr(vout);
  std::shared_lock<std::shared_mutex> lk(t->mu);
  CallCtx cx{nullptr, &lk};
  WS_CK(cudaMallocAsync((void**)&cx.cs, 4 * sizeof(u32), s));
  int rc = cuda_err(cudaMemsetAsync(cx.cs, 0, 4 * sizeof(u32), s));
  if (!rc)
    rc = all_dev ? run_device(t, ops, uop, keys, vals, n, status, vout, s, flags, has_erase, has_upsert, query_only, cx)
                 : run_staged(t, ops, uop, keys, vals, n, status, vout, s, flags, has_erase, has_upsert, query_only,
                              cx);
  cudaFreeAsync(cx.cs, s);
  return rc;
}

u64 npairs_of(const ws_table* t) { return t->cell_words / 2; }

int next_node_of(ws_table* t, cudaStream_t s, u64& nn) {
  nn = 0;
  if (t->cfg.design != D_CHAINING) return WS_OK;
  u64* hp = pin();
  if (!hp) return WS_ERR_ALLOC;
  WS_CK(cudaMemcpyAsync(hp, t->d.chain_next, 8, cudaMemcpyDeviceToHost, s));
  WS_CK(cudaStreamSynchronize(s));
  nn = hp[0];
  if (nn > t->d.chain_cap) nn = t->d.chain_cap;
  return WS_OK;
}

// live pairs compacted (in slot order) into a fresh device buffer
int compact_items(ws_table* t, cudaStream_t s, ulonglong2** out, u64* count) {
  u64 nn;
  int rc = next_node_of(t, s, nn);
  if (rc) return rc;
  const u64 np = npairs_of(t);
  u8* flags = nullptr;
  ulonglong2* sel = nullptr;
  u64* nsel = nullptr;
  WS_CK(cudaMallocAsync((void**)&flags, np, s));
  WS_CK(cudaMallocAsync((void**)&sel, np * sizeof(ulonglong2), s));
  WS_CK(cudaMallocAsync((void**)&nsel, 8, s));
  k_item_flags<<<grid_for(np), kThreads, 0, s>>>(t->d, np, nn, flags);
  size_t tmp_bytes = 0;
  const ulonglong2* in = (const ulonglong2*)t->d.cells;
  cub::DeviceSelect::Flagged(nullptr, tmp_bytes, in, flags, sel, nsel, (int64_t)np, s);
  void* tmp = nullptr;
  WS_CK(cudaMallocAsync(&tmp, tmp_bytes + 16, s));
  cub::DeviceSelect::Flagged(tmp, tmp_bytes, in, flags, sel, nsel, (int64_t)np, s);
  u64* hp = pin();
  if (!hp) return WS_ERR_ALLOC;
  WS_CK(cudaMemcpyAsync(hp, nsel, 8, cudaMemcpyDeviceToHost, s));
  cudaFreeAsync(tmp, s);
  cudaFreeAsync(flags, s);
  cudaFreeAsync(nsel, s);
  WS_CK(cudaStreamSynchronize(s));
  *count = hp[0];
  *out = sel;
  return cuda_err(cudaGetLastError());
}

}  // namespace

// internal (not exported): device-pointer batch execution for ws_shard.cu
// n_dev != nullptr: the batch size lives on the device (an exchange inbox
// count); n is its upper bound.  Such batches run unvalidated, uncombined and
// without the per-kind split (all of which need n on the host).
int ws_internal_run(ws_table* t, const u8* ops, u8 uop, const u64* keys, const u64* vals, u64 n, u8* status,
                    u64* vout, cudaStream_t s, u32 flags, bool has_erase, bool has_upsert, bool query_only,
                    const u64* n_dev) {
  if (cudaSetDevice(t->device) != cudaSuccess) return WS_ERR_CUDA;
  if (n_dev) flags = (flags & ~(WS_F_SYNC_CHECK | WS_F_COMBINE)) | WS_F_NO_CHECK;
  std::shared_lock<std::shared_mutex> lk(t->mu);
  CallCtx cx{nullptr, &lk, n_dev};
  WS_CK(cudaMallocAsync((void**)&cx.cs, 4 * sizeof(u32), s));
  int rc = cuda_err(cudaMemsetAsync(cx.cs, 0, 4 * sizeof(u32), s));
  if (!rc) rc = run_device(t, ops, uop, keys, vals, n, status, vout, s, flags, has_erase, has_upsert, query_only, cx);
  cudaFreeAsync(cx.cs, s);
  return rc;
}
int ws_internal_device(ws_table* t) { return t->device; }

// ===================================================================== C ABI

extern "C" {

const char* ws_strerror(int code) {
  switch (code) {
    case WS_OK: return "ok";
    case WS_ERR_INVALID_KEY: return "batch contains a reserved sentinel key (0, 2^64-1 or 2^64-2)";
    case WS_ERR_CONFIG: return "invalid table configuration";
    case WS_ERR_CUDA: return g_cuda_msg;
    case WS_ERR_ALLOC: return "device allocation failed";
    case WS_ERR_ARG: return "invalid argument";
    case WS_ERR_INVALID_OP: return "invalid op byte (kind > 2 or merge > 4)";
    case WS_ERR_TIMEOUT: return "a peer rank never reached the exchange barrier (60 s)";
    default: return "unknown error";
  }
}

int ws_create(const ws_config* cfg, int device, ws_table** out) {
  if (!cfg || !out) return WS_ERR_ARG;
  *out = nullptr;
  const ws_config& c = *cfg;
  if (c.design < 0 || c.design > D_UNSAFE || c.bucket_size <= 0 || c.capacity_slots == 0 ||
      c.capacity_slots % (u64)c.bucket_size || c.n_seeds < 1 || c.line_bytes < 16 ||
      c.ways < 2 || c.ways > 8 || c.path_depth < 1 || c.probe_cap < 1)
    return WS_ERR_CONFIG;
  const u64 nb = c.capacity_slots / (u64)c.bucket_size;
  const bool ice = c.design == D_ICEBERG || c.design == D_ICEBERG_MD;
  if (ice && (c.front_buckets < 1 || c.front_buckets >= nb)) return WS_ERR_CONFIG;
  if (c.design == D_CHAINING && (2 * c.bucket_size + 2) * 8 > 2 * c.line_bytes) return WS_ERR_CONFIG;
  if (cudaSetDevice(device) != cudaSuccess) return WS_ERR_CUDA;

  ws_table* t = new (std::nothrow) ws_table();
  if (!t) return WS_ERR_ALLOC;
  t->cfg = c;
  t->device = device;
  t->L = launchers_for(c.design);
  t->def_bs = c.bucket_size == default_bs(c.design);
  Dev& d = t->d;
  d.design = c.design;
  d.bs = c.bucket_size;
  d.md = c.design == D_DOUBLE_MD || c.design == D_P2_MD || c.design == D_ICEBERG_MD;
  d.cap = c.capacity_slots;
  d.nb = nb;
  d.front = ice ? c.front_buckets : nb;
  d.back = ice ? nb - c.front_buckets : 0;
  d.nbm = make_mod(nb);
  d.frontm = make_mod(d.front);
  d.backm = make_mod(d.back ? d.back : 1);
  for (int i = 0; i < 8; i++) d.seeds[i] = i < c.n_seeds ? c.seeds[i] : 0;
  d.shortcut = c.shortcut_slots;
  d.zcc = c.zero_count_cap;
  d.probe_cap = c.probe_cap;
  d.ways = c.ways;
  d.depth = c.path_depth;
  d.phased = c.phased;
  d.lock_elided = c.design == D_UNSAFE;
  d.line_bytes = c.line_bytes;
  d.wpn = 2 * c.bucket_size + 2;
  d.tune_qilp = 5;
  d.tune_l2pol = 2;
  d.tune_upsert = 4;
  d.ck_resume = 0;

  auto fail = [&](int code) { ws_destroy(t); return code; };
  if (c.design == D_CHAINING) {
    const u64 heads = nb + 1;
    u64 pool = c.chain_pool_nodes ? c.chain_pool_nodes : heads + std::max<u64>(64, heads / 2);
    if (pool < heads + 1) pool = heads + 1;
    d.chain_cap = pool;
    t->cell_words = pool * (u64)d.wpn;
    if (cudaMalloc((void**)&d.chain_next, 8) != cudaSuccess) return fail(WS_ERR_ALLOC);
  } else {
    t->cell_words = 2 * c.capacity_slots;
  }
  if (cudaMalloc((void**)&d.cells, t->cell_words * 8) != cudaSuccess) return fail(WS_ERR_ALLOC);
  if (cudaMemset(d.cells, 0, t->cell_words * 8) != cudaSuccess) return fail(WS_ERR_CUDA);
  if (d.md) {
    if (cudaMalloc((void**)&d.tags, c.capacity_slots * 2) != cudaSuccess) return fail(WS_ERR_ALLOC);
    if (cudaMemset(d.tags, 0, c.capacity_slots * 2) != cudaSuccess) return fail(WS_ERR_CUDA);
  }
  t->lock_words = (nb + 31) / 32;
  if (cudaMalloc((void**)&d.locks, t->lock_words * 4) != cudaSuccess) return fail(WS_ERR_ALLOC);
  if (cudaMemset(d.locks, 0, t->lock_words * 4) != cudaSuccess) return fail(WS_ERR_CUDA);
  if (cudaMalloc((void**)&d.state, N_STATE * 4) != cudaSuccess) return fail(WS_ERR_ALLOC);
  if (cudaMemset(d.state, 0, N_STATE * 4) != cudaSuccess) return fail(WS_ERR_CUDA);
  d.cs = d.state + 8;  // only internal launches outside any API call use the default words
  if (c.design == D_CHAINING) {
    const u64 nn = nb + 1;
    if (cudaMemcpy(d.chain_next, &nn, 8, cudaMemcpyHostToDevice) != cudaSuccess) return fail(WS_ERR_CUDA);
  }
  if (c.design == D_CUCKOO) {
    // BFS workspace: every visited entry is a distinct bucket, and one
    // expansion adds at most bucket_size * ways entries (cuckoo.py:107-156)
    const u64 E = std::min<u64>(nb + 8, 8 + (u64)BFS_BUDGET * c.bucket_size * c.ways) + c.path_depth + 80;
    const u64 SC = next_pow2(2 * E + 16);
    d.bfs_entries = E;
    d.bfs_seen_cap = SC;
    d.bfs_stride = 4 * E + SC + SC / 2 + 2;
    d.n_bfs = 64;
    const u64 bytes = d.bfs_stride * 8 * d.n_bfs;
    if (cudaMalloc((void**)&d.bfs_mem, bytes) != cudaSuccess) return fail(WS_ERR_ALLOC);
    if (cudaMemset(d.bfs_mem, 0, bytes) != cudaSuccess) return fail(WS_ERR_CUDA);
    if (cudaMalloc((void**)&d.bfs_busy, 4 * d.n_bfs) != cudaSuccess) return fail(WS_ERR_ALLOC);
    if (cudaMemset(d.bfs_busy, 0, 4 * d.n_bfs) != cudaSuccess) return fail(WS_ERR_CUDA);
  }
  {
    // keep staging / scratch allocations of the stream-ordered pool mapped
    // between calls instead of returning them to the driver at every sync
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      u64 thr = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  }
  t->L.preload(t->def_bs);
  preload_fn(k_validate);
  preload_fn(k_checksum);
  cudaGetLastError();
  if (cudaDeviceSynchronize() != cudaSuccess) return fail(WS_ERR_CUDA);
  *out = t;
  return WS_OK;
}

int ws_destroy(ws_table* t) {
  if (!t) return WS_OK;
  cudaSetDevice(t->device);
  cudaDeviceSynchronize();
  Dev& d = t->d;
  if (d.cells) cudaFree(d.cells);
  if (d.tags) cudaFree(d.tags);
  if (d.locks) cudaFree(d.locks);
  if (d.state) cudaFree(d.state);
  if (d.chain_next) cudaFree(d.chain_next);
  if (d.bfs_mem) cudaFree(d.bfs_mem);
  if (d.bfs_busy) cudaFree(d.bfs_busy);
  delete t;
  return WS_OK;
}

int ws_clear(ws_table* t, void* stream) {
  if (!t) return WS_ERR_ARG;
  cudaSetDevice(t->device);
  cudaStream_t s = S(stream);
  Dev& d = t->d;
  WS_CK(cudaMemsetAsync(d.cells, 0, t->cell_words * 8, s));
  if (d.tags) WS_CK(cudaMemsetAsync(d.tags, 0, d.cap * 2, s));
  WS_CK(cudaMemsetAsync(d.locks, 0, t->lock_words * 4, s));
  WS_CK(cudaMemsetAsync(d.state, 0, N_STATE * 4, s));
  if (t->cfg.design == D_CHAINING) {
    u64* hp = pin();
    if (!hp) return WS_ERR_ALLOC;
    hp[0] = d.nb + 1;
    WS_CK(cudaMemcpyAsync(d.chain_next, hp, 8, cudaMemcpyHostToDevice, s));
    WS_CK(cudaStreamSynchronize(s));
  }
  return WS_OK;
}

int ws_upsert(ws_table* t, const uint64_t* keys, const uint64_t* vals, uint64_t n, uint32_t merge,
              uint8_t* status, void* stream, uint32_t flags) {
  if (merge > WS_MERGE_MIN || (!vals && n)) return WS_ERR_ARG;
  return run_batch(t, nullptr, (u8)(OP_UPSERT | (merge << 4)), (const u64*)keys, (const u64*)vals, n,
                   status, nullptr, stream, flags, false, true, false);
}

int ws_query(ws_table* t, const uint64_t* keys, uint64_t n, uint64_t* vals_out, uint8_t* found,
             void* stream, uint32_t flags) {
  return run_batch(t, nullptr, OP_QUERY, (const u64*)keys, nullptr, n, found, (u64*)vals_out, stream,
                   flags, false, false, true);
}

int ws_erase(ws_table* t, const uint64_t* keys, uint64_t n, uint8_t* found, void* stream,
             uint32_t flags) {
  return run_batch(t, nullptr, OP_ERASE, (const u64*)keys, nullptr, n, found, nullptr, stream, flags,
                   true, false, false);
}

int ws_mixed(ws_table* t, const uint8_t* ops, const uint64_t* keys, const uint64_t* vals, uint64_t n,
             uint8_t* status, uint64_t* vals_out, void* stream, uint32_t flags) {
  if (!ops && n) return WS_ERR_ARG;
  // a zero-filled value array is substituted when none is given
  return run_batch(t, ops, 0, (const u64*)keys, (const u64*)vals, n, status, (u64*)vals_out, stream,
                   flags, true, true, false);
}

int ws_locate(ws_table* t, const uint64_t* keys, uint64_t n, int64_t* slot_out, void* stream) {
  if (!t || (!keys && n) || (!slot_out && n)) return WS_ERR_ARG;
  if (!n) return WS_OK;
  cudaSetDevice(t->device);
  cudaStream_t s = S(stream);
  const bool kd = is_device_ptr(keys), od = is_device_ptr(slot_out);
  u64* dk = (u64*)keys;
  i64* dout = (i64*)slot_out;
  if (!kd) { WS_CK(cudaMallocAsync((void**)&dk, 8 * n, s)); WS_CK(cudaMemcpyAsync(dk, keys, 8 * n, cudaMemcpyHostToDevice, s)); }
  if (!od) WS_CK(cudaMallocAsync((void**)&dout, 8 * n, s));
  LocateArgs la{t->d, dk, n, dout, s};
  t->L.locate(la, t->def_bs);
  int rc = cuda_err(cudaGetLastError());
  if (!od) WS_CK(cudaMemcpyAsync(slot_out, dout, 8 * n, cudaMemcpyDeviceToHost, s));
  if (!kd) cudaFreeAsync(dk, s);
  if (!od) cudaFreeAsync(dout, s);
  WS_CK(cudaStreamSynchronize(s));
  return rc;
}

int ws_probe_counts(ws_table* t, const uint8_t* ops, const uint64_t* keys, const uint64_t* vals,
                    uint64_t n, uint8_t* status, uint64_t* vals_out, uint32_t* probes,
                    uint64_t* lock_touches, void* stream, uint32_t flags) {
  if (!t || !ops || !keys || !probes) return WS_ERR_ARG;
  cudaSetDevice(t->device);
  cudaStream_t s = S(stream);
  if (!n) { if (lock_touches) *lock_touches = 0; return WS_OK; }
  // stage everything (instrumented runs are measurement passes, not hot)
  char* buf = nullptr;
  const u64 need = n * (1 + 8 + 8 + 1 + 8 + 4) + 2048;
  WS_CK(cudaMallocAsync((void**)&buf, need, s));
  char* p = buf;
  auto carve = [&](u64 bytes) { char* r = p; p += (bytes + 127) & ~127ull; return r; };
  u8* dops = (u8*)carve(n);
  u64* dk = (u64*)carve(8 * n);
  u64* dv = (u64*)carve(8 * n);
  u8* dst = (u8*)carve(n);
  u64* dvo = (u64*)carve(8 * n);
  u32* dpr = (u32*)carve(4 * n);
  u64* dlock = (u64*)carve(8);
  WS_CK(cudaMemcpyAsync(dops, ops, n, cudaMemcpyDefault, s));
  WS_CK(cudaMemcpyAsync(dk, keys, 8 * n, cudaMemcpyDefault, s));
  if (vals) WS_CK(cudaMemcpyAsync(dv, vals, 8 * n, cudaMemcpyDefault, s));
  else WS_CK(cudaMemsetAsync(dv, 0, 8 * n, s));
  WS_CK(cudaMemsetAsync(dlock, 0, 8, s));
  u32* cs = (u32*)carve(16);
  WS_CK(cudaMemsetAsync(cs, 0, 16, s));
  std::shared_lock<std::shared_mutex> lk(t->mu);
  const CallCtx cx{cs, &lk};
  u64* hp = pin();
  if (!hp) { cudaFreeAsync(buf, s); cudaStreamSynchronize(s); return WS_ERR_ALLOC; }
  int rc = validate(dk, dops, n, s, true, 0, cx);
  if (rc) { cudaFreeAsync(buf, s); cudaStreamSynchronize(s); return rc; }
  OpsArgs lo{dev_of(t, cx), dops, 0, dk, dv, n, dst, dvo, nullptr, dpr, dlock, 1, 0, 1,
             (flags & WS_F_SERIAL) ? 1 : 0, s};
  t->L.ops(lo, t->def_bs);
  rc = cuda_err(cudaGetLastError());
  if (!rc && status) WS_CK(cudaMemcpyAsync(status, dst, n, cudaMemcpyDefault, s));
  if (!rc && vals_out) WS_CK(cudaMemcpyAsync(vals_out, dvo, 8 * n, cudaMemcpyDefault, s));
  if (!rc) WS_CK(cudaMemcpyAsync(probes, dpr, 4 * n, cudaMemcpyDefault, s));
  if (!rc) WS_CK(cudaMemcpyAsync(hp, dlock, 8, cudaMemcpyDeviceToHost, s));
  cudaFreeAsync(buf, s);
  WS_CK(cudaStreamSynchronize(s));
  if (!rc && lock_touches) *lock_touches = hp[0];
  return rc;
}

int ws_occupied(ws_table* t, uint64_t* count_out, void* stream) {
  uint64_t cs[4];
  int rc = ws_checksum(t, cs, stream);
  if (!rc && count_out) *count_out = cs[0];
  return rc;
}

int ws_checksum(ws_table* t, uint64_t out[4], void* stream) {
  if (!t || !out) return WS_ERR_ARG;
  cudaSetDevice(t->device);
  cudaStream_t s = S(stream);
  u64 nn;
  int rc = next_node_of(t, s, nn);
  if (rc) return rc;
  u64* dout = nullptr;
  WS_CK(cudaMallocAsync((void**)&dout, 32, s));
  WS_CK(cudaMemsetAsync(dout, 0, 32, s));
  const u64 np = npairs_of(t);
  k_checksum<<<grid_for(np), kThreads, 0, s>>>(t->d, np, nn, dout);
  u64* hp = pin();
  if (!hp) return WS_ERR_ALLOC;
  WS_CK(cudaMemcpyAsync(hp, dout, 32, cudaMemcpyDeviceToHost, s));
  cudaFreeAsync(dout, s);
  WS_CK(cudaStreamSynchronize(s));
  memcpy(out, hp, 32);
  return cuda_err(cudaGetLastError());
}

int ws_export_items(ws_table* t, uint64_t* keys, uint64_t* vals, uint64_t cap, uint64_t* n_out,
                    void* stream) {
  if (!t) return WS_ERR_ARG;
  cudaSetDevice(t->device);
  cudaStream_t s = S(stream);
  ulonglong2* sel = nullptr;
  u64 cnt = 0;
  int rc = compact_items(t, s, &sel, &cnt);
  if (rc) return rc;
  if (n_out) *n_out = cnt;
  const u64 m = std::min<u64>(cap, cnt);
  if (m && (keys || vals)) {
    u64* tmp = nullptr;
    WS_CK(cudaMallocAsync((void**)&tmp, 16 * m, s));
    k_split_pairs<<<grid_for(m), kThreads, 0, s>>>(sel, m, keys ? tmp : nullptr, vals ? tmp + m : nullptr);
    if (keys) WS_CK(cudaMemcpyAsync(keys, tmp, 8 * m, cudaMemcpyDefault, s));
    if (vals) WS_CK(cudaMemcpyAsync(vals, tmp + m, 8 * m, cudaMemcpyDefault, s));
    cudaFreeAsync(tmp, s);
  }
  cudaFreeAsync(sel, s);
  WS_CK(cudaStreamSynchronize(s));
  return cuda_err(cudaGetLastError());
}

int ws_duplicate_scan(ws_table* t, uint64_t* dup_keys, uint64_t* dup_counts, uint64_t cap,
                      uint64_t* n_dup_out, void* stream) {
  if (!t) return WS_ERR_ARG;
  cudaSetDevice(t->device);
  cudaStream_t s = S(stream);
  ulonglong2* sel = nullptr;
  u64 cnt = 0;
  int rc = compact_items(t, s, &sel, &cnt);
  if (rc) return rc;
  u64 ndup = 0;
  if (cnt > 1) {
    u64 *k_in = nullptr, *k_out = nullptr, *dk = nullptr, *dc = nullptr, *dn = nullptr;
    const u64 cap_d = std::max<u64>(cap, 1);
    WS_CK(cudaMallocAsync((void**)&k_in, 8 * cnt, s));
    WS_CK(cudaMallocAsync((void**)&k_out, 8 * cnt, s));
    WS_CK(cudaMallocAsync((void**)&dk, 8 * cap_d, s));
    WS_CK(cudaMallocAsync((void**)&dc, 8 * cap_d, s));
    WS_CK(cudaMallocAsync((void**)&dn, 8, s));
    WS_CK(cudaMemsetAsync(dn, 0, 8, s));
    k_pair_keys<<<grid_for(cnt), kThreads, 0, s>>>(sel, cnt, k_in);
    size_t tb = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, tb, k_in, k_out, (int64_t)cnt, 0, 64, s);
    void* tmp = nullptr;
    WS_CK(cudaMallocAsync(&tmp, tb + 16, s));
    cub::DeviceRadixSort::SortKeys(tmp, tb, k_in, k_out, (int64_t)cnt, 0, 64, s);
    k_dup_runs<<<grid_for(cnt), kThreads, 0, s>>>(k_out, cnt, dk, dc, cap_d, dn);
    u64* hp = pin();
    if (!hp) return WS_ERR_ALLOC;
    WS_CK(cudaMemcpyAsync(hp, dn, 8, cudaMemcpyDeviceToHost, s));
    WS_CK(cudaStreamSynchronize(s));
    ndup = hp[0];
    const u64 m = std::min<u64>(ndup, cap);
    if (m && dup_keys) WS_CK(cudaMemcpyAsync(dup_keys, dk, 8 * m, cudaMemcpyDefault, s));
    if (m && dup_counts) WS_CK(cudaMemcpyAsync(dup_counts, dc, 8 * m, cudaMemcpyDefault, s));
    cudaFreeAsync(tmp, s);
    cudaFreeAsync(k_in, s);
    cudaFreeAsync(k_out, s);
    cudaFreeAsync(dk, s);
    cudaFreeAsync(dc, s);
    cudaFreeAsync(dn, s);
  }
  cudaFreeAsync(sel, s);
  WS_CK(cudaStreamSynchronize(s));
  if (n_dup_out) *n_dup_out = ndup;
  return cuda_err(cudaGetLastError());
}

int ws_export_raw(ws_table* t, uint64_t* words, uint64_t nwords, uint16_t* tags, void* stream) {
  if (!t) return WS_ERR_ARG;
  cudaSetDevice(t->device);
  cudaStream_t s = S(stream);
  const u64 m = std::min<u64>(nwords, t->cell_words);
  if (words && m) WS_CK(cudaMemcpyAsync(words, t->d.cells, 8 * m, cudaMemcpyDefault, s));
  if (tags) {
    if (t->d.tags) WS_CK(cudaMemcpyAsync(tags, t->d.tags, 2 * t->d.cap, cudaMemcpyDefault, s));
    else WS_CK(cudaMemsetAsync(tags, 0, 0, s));
  }
  WS_CK(cudaStreamSynchronize(s));
  return WS_OK;
}

int ws_read_range(ws_table* t, uint64_t first_word, uint64_t nwords, uint64_t* words, uint64_t first_tag,
                  uint64_t ntags, uint16_t* tags, void* stream) {
  if (!t || (nwords && !words) || (ntags && !tags)) return WS_ERR_ARG;
  cudaSetDevice(t->device);
  std::shared_lock<std::shared_mutex> lk(t->mu);
  if (first_word > t->cell_words || nwords > t->cell_words - first_word) return WS_ERR_ARG;
  const u64 ncap_tags = t->d.tags ? t->d.cap : 0;
  if (first_tag > ncap_tags || ntags > ncap_tags - first_tag) return WS_ERR_ARG;
  cudaStream_t s = S(stream);
  if (nwords) WS_CK(cudaMemcpyAsync(words, t->d.cells + first_word, 8 * nwords, cudaMemcpyDefault, s));
  if (ntags) WS_CK(cudaMemcpyAsync(tags, t->d.tags + first_tag, 2 * ntags, cudaMemcpyDefault, s));
  WS_CK(cudaStreamSynchronize(s));
  return WS_OK;
}

int ws_tune(ws_table* t, int knob, int value) {
  if (!t) return WS_ERR_ARG;
  switch (knob) {
    case WS_TUNE_QUERY_ILP:
      if (value < -1 || value > 8) return WS_ERR_ARG;
      t->d.tune_qilp = value;
      return WS_OK;
    case WS_TUNE_L2_POLICY:
      if (value < 0 || value > 2) return WS_ERR_ARG;
      t->d.tune_l2pol = value;
      return WS_OK;
    case WS_TUNE_OCCUPANCY:  // retired in round 2 (every forced occupancy measured slower): accepted, no effect
      return value < 0 ? WS_ERR_ARG : WS_OK;
    case WS_TUNE_DELAY_NS:
      if (value < 0) return WS_ERR_ARG;
      t->d.delay_ns = (u32)value;
      return WS_OK;
    case WS_TUNE_DELAY_P16:
      if (value < 0 || value > 65536) return WS_ERR_ARG;
      t->d.delay_p16 = (u32)value;
      return WS_OK;
    case WS_TUNE_DELAY_SEED:
      t->d.delay_seed = mix64((u64)(unsigned)value);
      return WS_OK;
    case WS_TUNE_PREFETCH:  // retired in round 2 (L2 prefetch measured slower): accepted, no effect
      return value < 0 || value > 4 ? WS_ERR_ARG : WS_OK;
    case WS_TUNE_KERNEL_EVENTS:
      t->time_kernels = value != 0;
      return WS_OK;
    case WS_TUNE_UPSERT:
      if (value < 0 || value > 6) return WS_ERR_ARG;
      // 1 / 5 (removed P2-MD variants) and 6 outside cuckoo select the default
      if (value == 1 || value == 5 || (value == 6 && t->cfg.design != D_CUCKOO)) value = 4;
      t->d.tune_upsert = value;
      return WS_OK;
    default: return WS_ERR_ARG;
  }
}

int ws_kernel_times(ws_table* t, float* ms_out, uint64_t cap, uint64_t* count) {
  if (!t || !count) return WS_ERR_ARG;
  cudaSetDevice(t->device);
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;
  {
    std::lock_guard<std::mutex> g(t->ev_mu);
    ev.swap(t->kev);
  }
  *count = ev.size();
  int rc = WS_OK;
  for (u64 i = 0; i < ev.size(); i++) {
    float ms = 0.f;
    if (cudaEventSynchronize(ev[i].second) != cudaSuccess ||
        cudaEventElapsedTime(&ms, ev[i].first, ev[i].second) != cudaSuccess)
      rc = WS_ERR_CUDA;
    if (ms_out && i < cap) ms_out[i] = ms;
    cudaEventDestroy(ev[i].first);
    cudaEventDestroy(ev[i].second);
  }
  return rc;
}

int ws_info(ws_table* t, ws_info_t* info) {
  if (!t || !info) return WS_ERR_ARG;
  cudaSetDevice(t->device);
  memset(info, 0, sizeof(*info));
  info->capacity_slots = t->d.cap;
  info->num_buckets = t->d.nb;
  info->primary_buckets = t->d.front;
  info->lock_bytes = t->lock_words * 4;
  info->device = t->device;
  if (t->cfg.design == D_CHAINING) {
    info->node_bytes = t->cell_words * 8;
    info->pool_nodes = t->d.chain_cap;
  } else {
    info->slot_bytes = t->cell_words * 8;
  }
  info->tag_bytes = t->d.tags ? t->d.cap * 2 : 0;
  u32 st[2] = {0, 0};
  WS_CK(cudaMemcpy(st, t->d.state, 8, cudaMemcpyDeviceToHost));
  info->tombstones_ever = (int32_t)st[0];
  if (t->cfg.design == D_CHAINING) {
    u64 nn = 0;
    WS_CK(cudaMemcpy(&nn, t->d.chain_next, 8, cudaMemcpyDeviceToHost));
    info->next_node = std::min<u64>(nn, t->d.chain_cap);
  }
  return WS_OK;
}

}  // extern "C"

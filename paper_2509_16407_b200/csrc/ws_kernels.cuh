// ws_kernels.cuh -- batch kernels (one thread per op) and their per-design
// launchers.  Each design's instantiations live in their own translation unit
// (ws_d_<design>.cu) so the library builds in parallel.
#pragma once
#include <cuda_runtime.h>

#include "ws_ops.cuh"

namespace ws {

constexpr int kThreads = 256;
constexpr int kSMs = 148;

__host__ __device__ constexpr int default_bs(int design) {
  return design == D_DOUBLE ? 8 : design == D_CUCKOO ? 8 : design == D_CHAINING ? 7 : 32;
}

// Table kernels (one op per thread or lane group, random DRAM accesses,
// lock rounds) are launched with up to kTableGridPerSM CTAs per SM instead of
// a few resident waves walking the batch grid-stride: the block scheduler
// then keeps every SM full to the last op.  Measured on P2-MD (2^28 / 2^30,
// profiles/grid_size_r02.log): 8 -> 256 CTAs/SM takes the query 11.75 ->
// 10.29 ms / 54.5 -> 43.6 ms and the insert 25.5 -> 24.2 ms / 101.2 -> 94.8
// ms; the plateau starts near 96.
constexpr int kTableGridPerSM = 256;
// A launch whose batch size lives on the device (Dev::dn: the split's erase /
// query segments, the multi-GPU exchange's per-source inbox segments) is
// sized for its host-side UPPER bound, so much of a 256-per-SM grid would be
// CTAs that read the count and exit; such launches keep 32 per SM and walk
// their segment grid-stride (same-box A/B: aging and YCSB equal or better
// than with the full grid, profiles/grid_size_r02.log).
constexpr int kTableGridPerSMDev = 32;
__host__ __device__ inline int table_grid_per_sm(const Dev& d) {
  return d.dn ? kTableGridPerSMDev : kTableGridPerSM;
}

inline unsigned grid_for(u64 n, int threads = kThreads, int per_sm = 8) {
  u64 g = (n + threads - 1) / threads;
  const u64 cap = (u64)kSMs * per_sm;
  if (g > cap) g = cap;
  return (unsigned)(g ? g : 1);
}

// Grid for a mutating launch: besides the SM-count cap, keep the number of
// ops in flight at most ~one per bucket.  Routing decisions (P2 shortcut /
// least-loaded, iceberg backyard choice) read bucket occupancy; when a whole
// batch of a small table runs at once, thousands of decisions see the same
// stale counts and pile into the same buckets.  Large tables (2^28 slots =
// 2^23 buckets vs ~300K resident threads) are unaffected.
inline unsigned grid_for_table(u64 n, u64 nb, int threads = kThreads, int per_sm = 8) {
  const unsigned g = grid_for(n, threads, per_sm);
  u64 lim = (nb + threads - 1) / threads;
  if (lim < 4) lim = 4;
  return (unsigned)(g < lim ? g : lim);
}

__device__ __forceinline__ bool gate_closed(const Dev& d, int gated) {
  return gated && (ld_u32_relaxed(d.cs) | ld_u32_relaxed(d.cs + 1));
}

template <int DES, int BS, bool INSTR>
__global__ void __launch_bounds__(kThreads) k_ops(Dev d, const u8* __restrict__ ops, u8 uop,
                                                  const u64* __restrict__ keys,
                                                  const u64* __restrict__ vals, u64 n, u8* status,
                                                  u64* vout, const u8* redo, u32* probes,
                                                  u64* lock_acc, int conc_erase, int gated,
                                                  const u32* __restrict__ rlist = nullptr,
                                                  const u32* __restrict__ rcount = nullptr) {
  WS_PROLOGUE(d, gated, n);
  Probe* pp = nullptr;
  Probe pr;
  if constexpr (INSTR) pp = &pr;
  // conc_erase 2: the launch's erase count (k_count_erases) decides
  const bool conc = conc_erase == 2 ? ld_u32_relaxed(d.cs + 3) != 0 : conc_erase != 0;
  Ctx<DES, BS, false, INSTR> c{d, pp, conc, ld_u32_relaxed(d.state)};
  // rlist: a compacted list of the batch indices to run (*rcount of them),
  // so every lane of a warp has work (k_compact_retry)
  const u64 nn = rcount ? *rcount : n;
  for (u64 t = blockIdx.x * (u64)blockDim.x + threadIdx.x; t < nn; t += (u64)gridDim.x * blockDim.x) {
    const u64 i = rlist ? rlist[t] : t;
    if (redo && !rlist && redo[i] != S_RETRY) continue;
    const u8 op = ops ? __ldg(ops + i) : uop;
    const u64 key = __ldg(keys + i);
    const u64 val = vals ? __ldg(vals + i) : 0ull;
    if constexpr (INSTR) pr.reset((u32)d.line_bytes);
    const OpOut o = c.template run<DES>(op & 15, op >> 4, key, val);
    if (status) status[i] = o.status;
    if (vout) vout[i] = o.val;
    if constexpr (INSTR) {
      probes[i] = pr.count();
      if (pr.locks) atomicAdd((unsigned long long*)lock_acc, (unsigned long long)pr.locks);
    }
  }
}

template <int DES, int BS, bool RO>
__global__ void __launch_bounds__(kThreads) k_query(Dev d, const u64* __restrict__ keys, u64 n,
                                                    u64* vout, u8* found, int conc_erase, int gated) {
  WS_PROLOGUE(d, gated, n);
  Ctx<DES, BS, RO, false> c{d, nullptr, conc_erase != 0, ld_u32_relaxed(d.state)};
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
    u64 v = 0;
    const bool f = c.template query<DES>(__ldg(keys + i), v);
    if (found) found[i] = f;
    if (vout) vout[i] = v;
  }
}

template <int DES, int BS>
__global__ void k_locate(Dev d, const u64* __restrict__ keys, u64 n, i64* out) {
  Ctx<DES, BS, false, false> c{d, nullptr, false, ld_u32_relaxed(d.state)};
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x)
    out[i] = c.template locate<DES>(__ldg(keys + i));
}


struct OpsArgs {
  Dev d;
  const u8* ops;
  u8 uop;
  const u64* keys;
  const u64* vals;
  u64 n;
  u8* status;
  u64* vout;
  const u8* redo;
  u32* probes;
  u64* lock_acc;
  int conc_erase, gated, instr, serial;
  cudaStream_t s;
  const u32* rlist = nullptr;   // optional compacted index list (k_ops; batches < 2^32)
  const u32* rcount = nullptr;
};

struct QueryArgs {
  Dev d;
  const u64* keys;
  u64 n;
  u64* vout;
  u8* found;
  int conc_erase, gated, ro;
  cudaStream_t s;
  int check_keys = 0;  // count sentinel keys into d.cs[0] (kernels that support it: P2-MD's tuned query)
};

struct LocateArgs {
  Dev d;
  const u64* keys;
  u64 n;
  i64* out;
  cudaStream_t s;
};

template <int DES, int BS>
void launch_ops_t(const OpsArgs& a) {
  // serial: one thread walks the batch in index order (exact sequential
  // semantics, used to replay reference op streams)
  if (a.instr)
    k_ops<DES, BS, true><<<a.serial ? 1 : grid_for_table(a.n, a.d.nb, 128, 4), a.serial ? 1 : 128, 0, a.s>>>(a.d, a.ops, a.uop, a.keys, a.vals, a.n, a.status,
                                                                  a.vout, a.redo, a.probes, a.lock_acc,
                                                                  a.conc_erase, a.gated);
  else
    k_ops<DES, BS, false><<<a.serial ? 1 : grid_for_table(a.n, a.d.nb, kThreads, table_grid_per_sm(a.d)), a.serial ? 1 : kThreads, 0, a.s>>>(a.d, a.ops, a.uop, a.keys, a.vals, a.n, a.status,
                                                                a.vout, a.redo, a.probes, a.lock_acc,
                                                                a.conc_erase, a.gated, a.rlist, a.rcount);
}

template <int DES, int BS>
void launch_query_t(const QueryArgs& a) {
  if (a.ro)
    k_query<DES, BS, true><<<grid_for(a.n, kThreads, table_grid_per_sm(a.d)), kThreads, 0, a.s>>>(a.d, a.keys, a.n, a.vout, a.found, a.conc_erase,
                                                                 a.gated);
  else
    k_query<DES, BS, false><<<grid_for(a.n, kThreads, table_grid_per_sm(a.d)), kThreads, 0, a.s>>>(a.d, a.keys, a.n, a.vout, a.found,
                                                                  a.conc_erase, a.gated);
}

template <int DES, int BS>
void launch_locate_t(const LocateArgs& a) {
  k_locate<DES, BS><<<grid_for(a.n), kThreads, 0, a.s>>>(a.d, a.keys, a.n, a.out);
}

// per-design entry points, defined in ws_d_<design>.cu
struct Launchers {
  void (*ops)(const OpsArgs&, bool default_bs);
  void (*query)(const QueryArgs&, bool default_bs);
  void (*locate)(const LocateArgs&, bool default_bs);
  void (*preload)(bool default_bs);  // load every kernel now, not lazily inside a timed launch
};

template <class K>
inline void preload_fn(K kernel) {
  cudaFuncAttributes a;
  if (cudaFuncGetAttributes(&a, kernel) != cudaSuccess) return;
  // reserve the per-thread local memory now: growing the context's local
  // pool later happens synchronously inside some unrelated timed launch
  size_t cur = 0;
  if (cudaDeviceGetLimit(&cur, cudaLimitStackSize) == cudaSuccess && cur < a.localSizeBytes)
    cudaDeviceSetLimit(cudaLimitStackSize, a.localSizeBytes);
}

template <int DES, int BS>
void preload_t() {
  preload_fn(k_ops<DES, BS, false>);
  preload_fn(k_ops<DES, BS, true>);
  preload_fn(k_query<DES, BS, false>);
  preload_fn(k_query<DES, BS, true>);
  preload_fn(k_locate<DES, BS>);
}

#define WS_DEFINE_DESIGN(DES, NAME)                                                       \
  namespace ws {                                                                          \
  static void NAME##_ops(const OpsArgs& a, bool def) {                                    \
    if (def) launch_ops_t<DES, default_bs(DES)>(a); else launch_ops_t<DES, 0>(a);         \
  }                                                                                       \
  static void NAME##_query(const QueryArgs& a, bool def) {                                \
    if (def) launch_query_t<DES, default_bs(DES)>(a); else launch_query_t<DES, 0>(a);     \
  }                                                                                       \
  static void NAME##_locate(const LocateArgs& a, bool def) {                              \
    if (def) launch_locate_t<DES, default_bs(DES)>(a); else launch_locate_t<DES, 0>(a);   \
  }                                                                                       \
  static void NAME##_preload(bool def) {                                                   \
    if (def) preload_t<DES, default_bs(DES)>(); else preload_t<DES, 0>();                 \
  }                                                                                       \
  Launchers launchers_##NAME() {                                                          \
    return Launchers{NAME##_ops, NAME##_query, NAME##_locate, NAME##_preload};            \
  }                                                                                       \
  }

Launchers launchers_double();
Launchers launchers_double_md();
Launchers launchers_p2();
Launchers launchers_p2_md();
Launchers launchers_iceberg();
Launchers launchers_iceberg_md();
Launchers launchers_cuckoo();
Launchers launchers_chaining();
Launchers launchers_unsafe();

}  // namespace ws

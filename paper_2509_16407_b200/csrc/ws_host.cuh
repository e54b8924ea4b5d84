// ws_host.cuh -- host-side internals shared by the ABI translation unit
// (ws_capi.cu: table lifecycle, single-kind batches, host staging,
// introspection) and the mixed-batch machinery (ws_batch.cu: the split by
// op kind and same-key combining).  Not part of the public ABI.
#pragma once
#include <cuda_runtime.h>

#include <map>
#include <mutex>
#include <shared_mutex>
#include <utility>
#include <vector>

#include "warpspeed.h"
#include "ws_kernels.cuh"

using ws::u8;
using ws::u32;
using ws::u64;

// ====================================================================== table

struct ws_table {
  using Dev = ws::Dev;
  using Launchers = ws::Launchers;
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


namespace ws_host {
using namespace ws;

// CUDA error bookkeeping: the message of the calling thread's last failure
// (ws_strerror) and the file:line it came from
extern thread_local char g_cuda_msg[256];
int note_cuda_at(cudaError_t e, const char* file, int line);
inline int cuda_err_at(cudaError_t e, const char* file, int line) {
  return e == cudaSuccess ? WS_OK : note_cuda_at(e, file, line);
}
#define cuda_err(x) cuda_err_at((x), __FILE__, __LINE__)
#define WS_CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) return note_cuda_at(e_, __FILE__, __LINE__); } while (0)

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


// internal flags of run_device_plain
constexpr u32 kF_VALIDATED = 1u << 30;   // the caller validated the batch; keep the kernels gated
constexpr u32 kF_NO_KIND_SORT = 1u << 29;
constexpr u32 kF_CONC_ERASE = 1u << 28;  // other launches of this call may erase concurrently

Staging* staging(int device);
u64* pin();
u64* pin_call();
u64 next_pow2(u64 x);
int validate(const u64* keys, const u8* ops, u64 n, cudaStream_t s, bool sync, u32 flags, const CallCtx& cx);

// one launch (or the chaining grow-and-redo sequence) of the design's kernel
// for a uniform or mixed device batch (ws_capi.cu)
int run_device_plain(ws_table* t, const u8* ops, u8 uop, const u64* keys, const u64* vals, u64 n,
                     u8* status, u64* vout, cudaStream_t s, u32 flags, bool has_erase, bool has_upsert,
                     bool query_only, const CallCtx& cx);
// a large mixed batch as per-kind segments (ws_batch.cu)
int run_device_by_kind(ws_table* t, const u8* ops, u8 uop, const u64* keys, const u64* vals, u64 n, u8* status,
                       u64* vout, cudaStream_t s, u32 flags, bool has_erase, bool has_upsert, const CallCtx& cx);
// one uniform upsert batch with same-key combining (ws_batch.cu)
int combine_uniform(ws_table* t, u8 uop, const u64* keys, const u64* vals, u64 n, u8* status, cudaStream_t s,
                    u32 flags, const CallCtx& cx, const u32* oidx, const u64* dn, u64 nbatch);

}  // namespace ws_host

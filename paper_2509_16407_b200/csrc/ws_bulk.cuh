// ws_bulk.cuh -- bucket-partitioned bulk upsert for P2-MD (see ws_bulk.cu).
#pragma once
#include <cuda_runtime.h>

#include "ws_ops.cuh"

namespace ws {

struct BulkPlan {
  int gb_log2;   // buckets per group = 2^gb_log2 (one CTA owns a group)
  u64 groups;    // ceil(nb / 2^gb_log2)
  int passes;    // LSD partition passes over the group id
  int radix;     // bits per pass
  bool skip_b;   // diagnostics: run phase A only (deferred ops are dropped)
  int cap;       // phase A claims slots only below this occupancy (<= shortcut; see ws_bulk.cu)
};

// Group size and partition shape for a batch of n upserts into nb buckets.
BulkPlan bulk_plan(u64 n, u64 nb, int gb_log2 = -1);

// Phase A (partition + owner-applied shortcut inserts) and phase B (the
// locked per-op kernel over the deferred ops), stream-ordered on s.  Requires
// a P2-MD table with 32-slot buckets, not lock-elided, not phased, and no
// concurrent mutation from other streams; n < 2^32.
cudaError_t bulk_upsert_p2md(const Dev& d, const u64* keys, const u64* vals, u64 n, int merge, u8* status,
                             int gated, cudaStream_t s, const BulkPlan& plan);

void bulk_preload();

// Phase B launcher (defined beside the rounds kernel in ws_d_p2_md.cu): the
// locked per-op upsert over the batch ops whose bit is set in dmask (one bit
// per batch index), in batch order; statuses written at those indices.
void bulk_phase_b(const Dev& d, const u64* keys, const u64* vals, u64 n, int merge, u8* status, int gated,
                  const u32* dmask, unsigned grid, cudaStream_t s);

// 16-byte aligned key / value arrays (the cp.async staging needs them)
bool bulk_aligned(const void* keys, const void* vals);

}  // namespace ws

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

#include <cub/cub.cuh>

#include "warpspeed.h"
#include "ws_device.cuh"

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

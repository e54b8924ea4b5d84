// tlb_bench.cu -- is the footprint dependence of the random-access plateau
// (dependent chains 53.8 G/s at 2^28, 48.5 at 2^30,
// 44.0 at 2^32) a TLB-reach effect, and does the allocation method change it?
//
// Independent random 32-byte reads (.nc .L2::64B, 8 per thread in flight,
// the scripts/gather_bench.cu 'g' shape) over a
// buffer of `gb` GiB, launched as 148 x 256 CTAs of 256 threads.  Addresses
// are drawn from (a) every 2 MiB page of the buffer, (b) a subset of P pages
// spread evenly over it (same DRAM spread, fewer translations), (c) the first
// P pages only.  Allocations: cudaMalloc vs cuMemCreate mapped at a 1 GiB
// aligned reservation.
//
// build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o scripts/tlb_bench scripts/tlb_bench.cu -lcuda
// run:   scripts/tlb_bench 16   (a power of two GiB: page selections are masks)
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>

typedef unsigned long long u64;

__device__ __forceinline__ u64 mix(u64 x) {
  x ^= x >> 30; x *= 0xBF58476D1CE4E5B9ull; x ^= x >> 27; x *= 0x94D049BB133111EBull; return x ^ (x >> 31);
}

// page_sel: number of pages addresses may fall in; page_stride: distance (in
// pages) between selected pages
__global__ void __launch_bounds__(256) k_reads(const char* base, u64 npages, u64 page_sel, u64 page_stride,
                                               u64 seed, unsigned* sink) {
  const u64 t = blockIdx.x * (u64)blockDim.x + threadIdx.x;
  unsigned acc = 0;
  u64 p[8];
#pragma unroll
  for (int r = 0; r < 8; r++) {
    const u64 h = mix(t * 8 + r + seed);
    const u64 page = (h & (page_sel - 1)) * page_stride;  // page_sel: a power of two
    const u64 off = (h >> 40) & ((1ull << 21) - 1) & ~31ull;
    p[r] = (u64)(base + page * (1ull << 21) + off);
  }
  u64 w[8][4];
#pragma unroll
  for (int r = 0; r < 8; r++)
    asm volatile("ld.global.nc.L1::no_allocate.L2::64B.v4.u64 {%0,%1,%2,%3}, [%4];"
                 : "=l"(w[r][0]), "=l"(w[r][1]), "=l"(w[r][2]), "=l"(w[r][3]) : "l"(p[r]));
#pragma unroll
  for (int r = 0; r < 8; r++) acc += (unsigned)(w[r][0] ^ w[r][3]);
  if (acc == 0x12345678u) sink[0] = acc;
}

static double run(const char* base, u64 npages, u64 sel, u64 stride, unsigned* sink) {
  const unsigned grid = 148 * 256;
  const u64 reads = (u64)grid * 256 * 8;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int w = 0; w < 3; w++) k_reads<<<grid, 256>>>(base, npages, sel, stride, 1000 + w, sink);
  const int reps = 20;
  cudaEventRecord(a);
  for (int r = 0; r < reps; r++) k_reads<<<grid, 256>>>(base, npages, sel, stride, 77 * r, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  if (cudaGetLastError() != cudaSuccess) { printf("kernel error\n"); exit(1); }
  return reads * reps / (ms * 1e-3) / 1e9;
}

static void sweep(const char* what, const char* base, u64 bytes, unsigned* sink) {
  const u64 npages = bytes >> 21;
  printf("%s: %.1f GiB, %llu pages of 2 MiB\n", what, bytes / 1073741824.0, npages);
  printf("  all pages            : %6.2f G reads/s\n", run(base, npages, npages, 1, sink));
  const u64 sels[] = {256, 1024, 2048, 4096, 8192, 16384};
  for (u64 s : sels) {
    if (s >= npages) continue;
    printf("  %5llu pages spread   : %6.2f G reads/s\n", s, run(base, npages, s, npages / s, sink));
    printf("  %5llu pages leading  : %6.2f G reads/s\n", s, run(base, npages, s, 1, sink));
  }
}

int main(int argc, char** argv) {
  const u64 gb = argc > 1 ? strtoull(argv[1], 0, 10) : 16;
  const u64 bytes = gb << 30;
  unsigned* sink;
  cudaMalloc(&sink, 4);
  {
    char* p;
    if (cudaMalloc(&p, bytes) != cudaSuccess) { printf("cudaMalloc failed\n"); return 1; }
    cudaMemset(p, 1, bytes);
    sweep("cudaMalloc", p, bytes, sink);
    cudaFree(p);
  }
  {
    cuInit(0);
    CUdevice dev;
    cuDeviceGet(&dev, 0);
    CUmemAllocationProp prop = {};
    prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    prop.location.id = 0;
    size_t gmin = 0, grec = 0;
    cuMemGetAllocationGranularity(&gmin, &prop, CU_MEM_ALLOC_GRANULARITY_MINIMUM);
    cuMemGetAllocationGranularity(&grec, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED);
    printf("VMM granularity: minimum %zu, recommended %zu\n", gmin, grec);
    CUmemGenericAllocationHandle h;
    if (cuMemCreate(&h, bytes, &prop, 0) != CUDA_SUCCESS) { printf("cuMemCreate failed\n"); return 1; }
    CUdeviceptr va;
    if (cuMemAddressReserve(&va, bytes, 1ull << 30, 0, 0) != CUDA_SUCCESS) { printf("reserve failed\n"); return 1; }
    cuMemMap(va, bytes, 0, h, 0);
    CUmemAccessDesc acc = {};
    acc.location = prop.location;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    cuMemSetAccess(va, bytes, &acc, 1);
    cudaMemset((void*)va, 1, bytes);
    sweep("cuMemCreate (one handle, 1 GiB aligned)", (const char*)va, bytes, sink);
    cuMemUnmap(va, bytes);
    cuMemAddressFree(va, bytes);
    cuMemRelease(h);
  }
  return 0;
}

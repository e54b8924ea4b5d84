// gather_bench.cu -- B200 random-access ceilings for the hash-table roofline.
//
// Each thread performs R independent random reads of W bytes (W = 16, 32, 64,
// 128) at W-aligned positions of a large buffer (>> L2), addresses from a
// splitmix64 hash masked to the (power-of-two) buffer -- no index array and
// no 64-bit division, so the kernel is not issue-bound -- and XOR-folds the
// data.  Mode 'm' sweeps memory-level parallelism (CTAs/SM x loads in flight)
// and the cooperative one-instruction block reads of gather_coop.  Variants:
//   flavor 0: weak loads (ld.global, L1 allocate)
//   flavor 1: ld.global.nc.L1::no_allocate
//   flavor 2: ld.relaxed.gpu (coherent, what mutating kernels use)
//   flavor 3: ld.global.L2::64B hint (nc)
// Prints useful GB/s and G accesses/s; run under ncu for DRAM sectors/access.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_bench gather_bench.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

typedef unsigned long long u64;

__device__ __forceinline__ u64 mix64(u64 x) {
  x ^= x >> 30; x *= 0xBF58476D1CE4E5B9ull; x ^= x >> 27; x *= 0x94D049BB133111EBull; x ^= x >> 31;
  return x;
}

template <int FL>
__device__ __forceinline__ void ld16(const void* p, u64& a, u64& b) {
  if (FL == 0) asm volatile("ld.global.v2.u64 {%0,%1}, [%2];" : "=l"(a), "=l"(b) : "l"(p));
  else if (FL == 1) asm volatile("ld.global.nc.L1::no_allocate.v2.u64 {%0,%1}, [%2];" : "=l"(a), "=l"(b) : "l"(p));
  else if (FL == 2) asm volatile("ld.relaxed.gpu.global.v2.u64 {%0,%1}, [%2];" : "=l"(a), "=l"(b) : "l"(p));
  else asm volatile("ld.global.nc.L1::no_allocate.L2::64B.v2.u64 {%0,%1}, [%2];" : "=l"(a), "=l"(b) : "l"(p));
}
template <int FL>
__device__ __forceinline__ void ld32(const void* p, u64& a, u64& b, u64& c, u64& d) {
  if (FL == 0) asm volatile("ld.global.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
  else if (FL == 1) asm volatile("ld.global.nc.L1::no_allocate.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
  else if (FL == 2) asm volatile("ld.relaxed.gpu.global.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
  else asm volatile("ld.global.nc.L1::no_allocate.L2::64B.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
}

template <int W, int FL, int R>
__global__ void __launch_bounds__(256) gather(const char* buf, u64 nunits, u64 seed, u64* out, int iters) {
  u64 acc = 0;
  const u64 tid = blockIdx.x * (u64)blockDim.x + threadIdx.x;
  for (int it = 0; it < iters; it++) {
    u64 idx[R];
#pragma unroll
    for (int r = 0; r < R; r++) idx[r] = mix64(seed ^ (tid * R + r) ^ ((u64)it << 40)) & (nunits - 1);
#pragma unroll
    for (int r = 0; r < R; r++) {
      const char* p = buf + idx[r] * W;
      if (W == 16) { u64 a, b; ld16<FL>(p, a, b); acc ^= a ^ b; }
      else {
#pragma unroll
        for (int o = 0; o < W; o += 32) { u64 a, b, c, d; ld32<FL>(p + o, a, b, c, d); acc ^= a ^ b ^ c ^ d; }
      }
    }
  }
  if (acc == 0x123456789ull) out[0] = acc;
}

// Cooperative form: a group of G consecutive lanes reads one random
// (32*G)-byte block with ONE load instruction (lane l of the group takes the
// l-th 32-byte sector), the access pattern of the pair-cooperative tag fetch.
// Counts blocks/s, i.e. random DRAM line accesses of 32*G bytes.
template <int G, int R>
__global__ void __launch_bounds__(256) gather_coop(const char* buf, u64 nblocks, u64 seed, u64* out, int iters) {
  u64 acc = 0;
  const u64 tid = blockIdx.x * (u64)blockDim.x + threadIdx.x;
  const u64 grp = tid / G;
  const int sub = (int)(tid % G);
  for (int it = 0; it < iters; it++) {
    u64 idx[R];
#pragma unroll
    for (int r = 0; r < R; r++) idx[r] = mix64(seed ^ (grp * R + r) ^ ((u64)it << 40)) & (nblocks - 1);
#pragma unroll
    for (int r = 0; r < R; r++) {
      u64 a, b, c, d;
      ld32<3>(buf + idx[r] * (32 * G) + 32 * sub, a, b, c, d);
      acc ^= a ^ b ^ c ^ d;
    }
  }
  if (acc == 0x123456789ull) out[0] = acc;
}

template <int G, int R>
void run_coop(const char* buf, u64 bytes, u64* out, int blocks, int iters, const char* name) {
  const u64 nb = bytes / (32 * G);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  gather_coop<G, R><<<blocks, 256>>>(buf, nb, 1, out, 1);
  cudaEventRecord(a);
  gather_coop<G, R><<<blocks, 256>>>(buf, nb, 7, out, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double acc = (double)blocks * 256 / G * R * iters;
  printf("%-28s W=%4d R=%d  %8.2f G blocks/s  %8.1f GB/s useful\n", name, 32 * G, R, acc / ms / 1e6,
         acc * 32 * G / ms / 1e6);
}

// random stores of W bytes (2, 16 or 32) at W-aligned positions
template <int W, int R>
__global__ void __launch_bounds__(256) scatter(char* buf, u64 nunits, u64 seed, int iters) {
  const u64 tid = blockIdx.x * (u64)blockDim.x + threadIdx.x;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int r = 0; r < R; r++) {
      const u64 idx = mix64(seed ^ (tid * R + r) ^ ((u64)it << 40)) & (nunits - 1);
      char* p = buf + idx * W;
      if (W == 2) asm volatile("st.global.u16 [%0], %1;" :: "l"(p), "h"((unsigned short)tid) : "memory");
      else if (W == 16) asm volatile("st.global.v2.u64 [%0], {%1, %2};" :: "l"(p), "l"(tid), "l"(idx) : "memory");
      else asm volatile("st.global.v4.u64 [%0], {%1, %2, %3, %4};" :: "l"(p), "l"(tid), "l"(idx), "l"(tid), "l"(idx) : "memory");
    }
  }
}

// random 64-byte read, then a write into the sector just read: MODE 0 none,
// 1 a 2-byte store, 2 a full 32-byte sector store
template <int MODE, int R>
__global__ void __launch_bounds__(256) readwrite(char* buf, u64 nunits, u64 seed, int iters, u64* out) {
  const u64 tid = blockIdx.x * (u64)blockDim.x + threadIdx.x;
  u64 acc = 0;
  for (int it = 0; it < iters; it++) {
    u64 a[R][4];
    char* p[R];
#pragma unroll
    for (int r = 0; r < R; r++) {
      p[r] = buf + (mix64(seed ^ (tid * R + r) ^ ((u64)it << 40)) & (nunits - 1)) * 64;
      asm volatile("ld.relaxed.gpu.global.L2::64B.v4.u64 {%0,%1,%2,%3}, [%4];"
                   : "=l"(a[r][0]), "=l"(a[r][1]), "=l"(a[r][2]), "=l"(a[r][3]) : "l"(p[r]) : "memory");
    }
#pragma unroll
    for (int r = 0; r < R; r++) {
      acc ^= a[r][0];
      if (MODE == 1) asm volatile("st.global.u16 [%0], %1;" :: "l"(p[r] + 6), "h"((unsigned short)a[r][1]) : "memory");
      if (MODE == 2) asm volatile("st.global.v4.u64 [%0], {%1, %2, %3, %4};" :: "l"(p[r]), "l"(a[r][0] + 1), "l"(a[r][1]), "l"(a[r][2]), "l"(a[r][3]) : "memory");
    }
  }
  if (acc == 7) out[0] = acc;
}

template <int MODE, int R>
void run_rw(char* buf, u64 bytes, u64* out, int blocks, int iters, const char* name) {
  const u64 nunits = bytes / 64;
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  readwrite<MODE, R><<<blocks, 256>>>(buf, nunits, 1, 1, out);
  cudaEventRecord(a);
  readwrite<MODE, R><<<blocks, 256>>>(buf, nunits, 7, iters, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double acc = (double)blocks * 256 * R * iters;
  printf("%-36s R=%d  %8.2f G ops/s\n", name, R, acc / ms / 1e6);
}

template <int W, int R>
void run_st(char* buf, u64 bytes, int blocks, int iters, const char* name) {
  const u64 nunits = bytes / W;
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  scatter<W, R><<<blocks, 256>>>(buf, nunits, 1, 1);
  cudaEventRecord(a);
  scatter<W, R><<<blocks, 256>>>(buf, nunits, 7, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double acc = (double)blocks * 256 * R * iters;
  printf("%-28s W=%4d R=%d  %8.2f G st/s  %8.1f GB/s useful\n", name, W, R, acc / ms / 1e6, acc * W / ms / 1e6);
}

template <int W, int FL, int R>
void run(const char* buf, u64 bytes, u64* out, int blocks, int iters, const char* name) {
  const u64 nunits = bytes / W;
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  gather<W, FL, R><<<blocks, 256>>>(buf, nunits, 1, out, 1);
  cudaEventRecord(a);
  gather<W, FL, R><<<blocks, 256>>>(buf, nunits, 7, out, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double acc = (double)blocks * 256 * R * iters;
  printf("%-28s W=%4d R=%d  %8.2f G acc/s  %8.1f GB/s useful\n", name, W, R, acc / ms / 1e6, acc * W / ms / 1e6);
}

// query-shaped dependent chains: a random 32 B tag-block read in T (1/8 of
// the footprint, as the tag array is to the cells) and then a dependent random
// 16 B cell read in C, R chains per thread.  Mode 'q' runs it over the whole
// buffer split 1:8 (powers of two), so 4608 MiB ~ the 2^28-slot table, 18432 MiB ~ 2^30:
// does the rate fall with the footprint (TLB reach) as the query's does?
template <int R>
__global__ void __launch_bounds__(256) chain(const char* tags, u64 ntag, const char* cells, u64 ncell, u64 seed,
                                             u64* out, int iters) {
  u64 acc = 0;
  const u64 tid = blockIdx.x * (u64)blockDim.x + threadIdx.x;
  for (int it = 0; it < iters; it++) {
    u64 h[R], a[R];
#pragma unroll
    for (int r = 0; r < R; r++) {
      h[r] = mix64(seed ^ (tid * R + r) ^ ((u64)it << 40));
      u64 x, y, z, w;
      ld32<3>(tags + (h[r] & (ntag - 1)) * 64, x, y, z, w);
      a[r] = x ^ y ^ z ^ w;
    }
#pragma unroll
    for (int r = 0; r < R; r++) {
      u64 x, y;
      ld16<3>(cells + (((h[r] >> 20) ^ (a[r] & 1)) & (ncell - 1)) * 16, x, y);
      acc ^= x ^ y;
    }
  }
  if (acc == 0x123456789ull) out[0] = acc;
}

// the same chains over a bucket-interleaved layout: bucket b = 64 B of tags
// then 512 B of cells at b * 576, so a bucket's tag block and its cells share
// one 2 MiB page (one TLB entry per chain instead of two)
template <int R>
__global__ void __launch_bounds__(256) chain_colo(const char* buf, u64 nb, u64 seed, u64* out, int iters) {
  u64 acc = 0;
  const u64 tid = blockIdx.x * (u64)blockDim.x + threadIdx.x;
  for (int it = 0; it < iters; it++) {
    u64 h[R], a[R];
#pragma unroll
    for (int r = 0; r < R; r++) {
      h[r] = mix64(seed ^ (tid * R + r) ^ ((u64)it << 40));
      u64 x, y, z, w;
      ld32<3>(buf + (h[r] & (nb - 1)) * 576, x, y, z, w);
      a[r] = x ^ y ^ z ^ w;
    }
#pragma unroll
    for (int r = 0; r < R; r++) {
      u64 x, y;
      ld16<3>(buf + (h[r] & (nb - 1)) * 576 + 64 + (((h[r] >> 40) ^ (a[r] & 1)) & 31) * 16, x, y);
      acc ^= x ^ y;
    }
  }
  if (acc == 0x123456789ull) out[0] = acc;
}

int main(int argc, char** argv) {
  const u64 mb = argc > 1 ? strtoull(argv[1], 0, 10) : 4096;  // a power of two (index masks)
  const u64 bytes = mb << 20;
  printf("buffer %llu MiB\n", mb);
  char* buf; u64* out;
  cudaMalloc(&buf, bytes); cudaMalloc(&out, 64);
  cudaMemset(buf, 1, bytes);
  const int blocks = 148 * 8, iters = 16;
  if (argc > 2 && argv[2][0] == 'm') {  // memory-level-parallelism sweep: is ~45 G/s a plateau?
    for (int bps : {1, 2, 4, 8}) {
      printf("-- %d CTAs/SM x 256 threads\n", bps);
      const int bl = 148 * bps;
      run<32, 3, 1>(buf, bytes, out, bl, iters, "nc L2::64B 32B");
      run<32, 3, 2>(buf, bytes, out, bl, iters, "nc L2::64B 32B");
      run<32, 3, 4>(buf, bytes, out, bl, iters, "nc L2::64B 32B");
      run<32, 3, 8>(buf, bytes, out, bl, iters, "nc L2::64B 32B");
      run<32, 3, 16>(buf, bytes, out, bl, iters, "nc L2::64B 32B");
      run<32, 3, 32>(buf, bytes, out, bl, iters, "nc L2::64B 32B");
      run<32, 1, 16>(buf, bytes, out, bl, iters, "nc (128B fill) 32B");
      run<64, 3, 16>(buf, bytes, out, bl, iters, "nc L2::64B 64B");
      run<128, 1, 8>(buf, bytes, out, bl, iters, "nc 128B");
      run_coop<2, 8>(buf, bytes, out, bl, iters, "coop 2 lanes (1 instr)");
      run_coop<2, 16>(buf, bytes, out, bl, iters, "coop 2 lanes (1 instr)");
      run_coop<4, 8>(buf, bytes, out, bl, iters, "coop 4 lanes (1 instr)");
      run_coop<4, 16>(buf, bytes, out, bl, iters, "coop 4 lanes (1 instr)");
    }
    cudaDeviceSynchronize();
    return 0;
  }
  if (argc > 2 && argv[2][0] == 'g') {  // independent random reads: resident waves vs a 148x256-CTA grid
    run<32, 3, 8>(buf, bytes, out, 148 * 8, iters, "nc L2::64B 32B, 8 CTAs/SM x16 it");
    run<32, 3, 8>(buf, bytes, out, 148 * 256, 1, "nc L2::64B 32B, 148x256 CTAs x1 it");
    run<32, 3, 2>(buf, bytes, out, 148 * 256, 1, "nc L2::64B 32B, 148x256 CTAs x1 it");
    run_coop<2, 8>(buf, bytes, out, 148 * 8, iters, "coop 2 lanes, 8 CTAs/SM x16 it");
    run_coop<2, 8>(buf, bytes, out, 148 * 256, 1, "coop 2 lanes, 148x256 CTAs x1 it");
    cudaDeviceSynchronize();
    return 0;
  }
  if (argc > 2 && argv[2][0] == 'q') {
    const u64 tb = bytes / 9 & ~63ull, ntag = 1ull << (63 - __builtin_clzll(tb / 64));
    const char* cells = buf + ntag * 64;
    const u64 ncell = 1ull << (63 - __builtin_clzll((bytes - ntag * 64) / 16));
    // resident waves walking the work (bps = 4, 8 CTAs per SM, 16 iterations
    // each) vs a grid of 148 x 256 CTAs of one iteration each, the launch
    // shape of the table kernels (ws_kernels.cuh kTableGridPerSM)
    for (int bps : {4, 8, -256}) {
      cudaEvent_t a, b;
      cudaEventCreate(&a); cudaEventCreate(&b);
      if (bps < 0) {
        const int nb_ = 148 * -bps;
        chain<2><<<nb_, 256>>>(buf, ntag, cells, ncell, 1, out, 1);
        cudaEventRecord(a);
        for (int rep = 0; rep < 16; rep++) chain<2><<<nb_, 256>>>(buf, ntag, cells, ncell, 7 + rep, out, 1);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        const double ch = (double)nb_ * 256 * 2 * 16;
        printf("chain tags %6llu MiB + cells %6llu MiB, grid 148x256 CTAs: %6.2f G chains/s = %6.2f G acc/s\n",
               ntag * 64 >> 20, ncell * 16 >> 20, ch / ms / 1e6, 2 * ch / ms / 1e6);
        continue;
      }
      chain<2><<<148 * bps, 256>>>(buf, ntag, cells, ncell, 1, out, 1);
      cudaEventRecord(a);
      chain<2><<<148 * bps, 256>>>(buf, ntag, cells, ncell, 7, out, iters);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      const double ch = (double)148 * bps * 256 * 2 * iters;
      printf("chain tags %6llu MiB + cells %6llu MiB, %d CTAs/SM: %6.2f G chains/s = %6.2f G acc/s\n",
             ntag * 64 >> 20, ncell * 16 >> 20, bps, ch / ms / 1e6, 2 * ch / ms / 1e6);
    }
    const u64 nb = 1ull << (63 - __builtin_clzll(bytes / 576));
    for (int bps : {4, 8}) {
      cudaEvent_t a, b;
      cudaEventCreate(&a); cudaEventCreate(&b);
      chain_colo<2><<<148 * bps, 256>>>(buf, nb, 1, out, 1);
      cudaEventRecord(a);
      chain_colo<2><<<148 * bps, 256>>>(buf, nb, 7, out, iters);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      const double ch = (double)148 * bps * 256 * 2 * iters;
      printf("colocated %8llu buckets x 576 B = %6llu MiB, %d CTAs/SM: %6.2f G chains/s = %6.2f G acc/s\n",
             nb, nb * 576 >> 20, bps, ch / ms / 1e6, 2 * ch / ms / 1e6);
    }
    cudaDeviceSynchronize();
    return 0;
  }
  if (argc > 2 && argv[2][0] == 'r') {  // read-then-write-same-sector
    run_rw<0, 4>(buf, bytes, out, blocks, iters, "read 32B only");
    run_rw<1, 4>(buf, bytes, out, blocks, iters, "read 32B + 2B store same sector");
    run_rw<2, 4>(buf, bytes, out, blocks, iters, "read 32B + 32B store same sector");
    cudaDeviceSynchronize();
    return 0;
  }
  if (argc > 2 && argv[2][0] == 'w') {  // random-store ceilings
    run_st<2, 8>(buf, bytes, blocks, iters, "store 2B");
    run_st<16, 8>(buf, bytes, blocks, iters, "store 16B");
    run_st<32, 8>(buf, bytes, blocks, iters, "store 32B (full sector)");
    cudaDeviceSynchronize();
    return 0;
  }
  if (argc > 2) {  // short sweep
    run<32, 1, 8>(buf, bytes, out, blocks, iters, "nc 32B");
    run<32, 3, 8>(buf, bytes, out, blocks, iters, "nc L2::64B 32B");
    run<16, 1, 8>(buf, bytes, out, blocks, iters, "nc 16B");
    cudaDeviceSynchronize();
    return 0;
  }
  run<16, 0, 8>(buf, bytes, out, blocks, iters, "weak 16B");
  run<16, 1, 8>(buf, bytes, out, blocks, iters, "nc 16B");
  run<16, 2, 8>(buf, bytes, out, blocks, iters, "relaxed 16B");
  run<16, 3, 8>(buf, bytes, out, blocks, iters, "nc L2::64B 16B");
  run<32, 0, 8>(buf, bytes, out, blocks, iters, "weak 32B");
  run<32, 1, 8>(buf, bytes, out, blocks, iters, "nc 32B");
  run<32, 2, 8>(buf, bytes, out, blocks, iters, "relaxed 32B");
  run<32, 3, 8>(buf, bytes, out, blocks, iters, "nc L2::64B 32B");
  run<64, 1, 8>(buf, bytes, out, blocks, iters, "nc 64B");
  run<64, 2, 8>(buf, bytes, out, blocks, iters, "relaxed 64B");
  run<128, 1, 4>(buf, bytes, out, blocks, iters, "nc 128B");
  run<128, 2, 4>(buf, bytes, out, blocks, iters, "relaxed 128B");
  run<16, 1, 2>(buf, bytes, out, blocks, iters, "nc 16B low-MLP");
  run<16, 1, 16>(buf, bytes, out, blocks, iters, "nc 16B high-MLP");
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}

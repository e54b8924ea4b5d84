// locality_bench.cu -- does placing a bucket's tag block next to its cells pay
// on B200 HBM3e?  Each "op" touches a random 128-byte-aligned line A (a 64-byte
// read, the tag block) and then, dependent on that read, a second address
// A + OFF (OFF < 0: an independent random line, today's separate tag / cell
// arrays).  MODE 0: the second access is a 32-byte read (positive query);
// MODE 1: a 32-byte store (insert's cell write) plus a 2-byte store back into
// line A (insert's tag write).  Prints G ops/s per (MODE, OFF).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o locality_bench locality_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

typedef unsigned long long u64;

__device__ __forceinline__ u64 mix64(u64 x) {
  x ^= x >> 30; x *= 0xBF58476D1CE4E5B9ull; x ^= x >> 27; x *= 0x94D049BB133111EBull; x ^= x >> 31;
  return x;
}

template <int MODE, int R>
__global__ void __launch_bounds__(256) pairs(char* buf, u64 nlines, long long off, u64 seed, int iters, u64* out) {
  const u64 tid = blockIdx.x * (u64)blockDim.x + threadIdx.x;
  u64 acc = 0;
  for (int it = 0; it < iters; it++) {
    u64 a[R], x[R];
#pragma unroll
    for (int r = 0; r < R; r++) {
      const u64 h = mix64(seed ^ (tid * R + r) ^ ((u64)it << 40));
      a[r] = (h % (nlines - 1024)) * 128;
      u64 p0, p1, p2, p3;
      asm volatile("ld.relaxed.gpu.global.v4.u64 {%0,%1,%2,%3}, [%4];"
                   : "=l"(p0), "=l"(p1), "=l"(p2), "=l"(p3) : "l"(buf + a[r]) : "memory");
      u64 q0, q1, q2, q3;
      asm volatile("ld.relaxed.gpu.global.v4.u64 {%0,%1,%2,%3}, [%4];"
                   : "=l"(q0), "=l"(q1), "=l"(q2), "=l"(q3) : "l"(buf + a[r] + 32) : "memory");
      x[r] = p0 ^ p1 ^ p2 ^ p3 ^ q0 ^ q1 ^ q2 ^ q3;  // buffer is zero: dependency only
    }
#pragma unroll
    for (int r = 0; r < R; r++) {
      const u64 b = off < 0 ? (mix64(a[r] ^ 0x9E3779B97F4A7C15ull) % (nlines - 1024)) * 128 + x[r]
                            : a[r] + (u64)off + x[r];
      if (MODE == 0) {
        u64 c0, c1, c2, c3;
        asm volatile("ld.relaxed.gpu.global.v4.u64 {%0,%1,%2,%3}, [%4];"
                     : "=l"(c0), "=l"(c1), "=l"(c2), "=l"(c3) : "l"(buf + b) : "memory");
        acc ^= c0 ^ c1 ^ c2 ^ c3;
      } else {
        asm volatile("st.global.v4.u64 [%0], {%1, %1, %1, %1};" ::"l"(buf + b), "l"(x[r]) : "memory");
        asm volatile("st.global.u16 [%0], %1;" ::"l"(buf + a[r] + 6), "h"((unsigned short)x[r]) : "memory");
      }
    }
  }
  if (acc == 0x123456789ull) out[0] = acc;
}

// blocks x iters: 148*8 CTAs walking 16 iterations (round 1) or 148*256 CTAs
// of one iteration (the launch shape of the table kernels since round 2)
template <int MODE>
static float run(char* buf, u64 nlines, long long off, u64* out, int blocks = 148 * 8, int iters = 16) {
  const int R = 4;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  pairs<MODE, R><<<blocks, 256>>>(buf, nlines, off, 1, iters, out);
  cudaEventRecord(e0);
  for (int rep = 0; rep < 5; rep++) pairs<MODE, R><<<blocks, 256>>>(buf, nlines, off, 2 + rep, iters, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double ops = 5.0 * blocks * 256.0 * R * iters;
  return (float)(ops / (ms * 1e-3) / 1e9);
}

int main() {
  const u64 bytes = 8ull << 30, nlines = bytes / 128;
  char* buf;
  u64* out;
  printf("start\n"); fflush(stdout);
  if (cudaMalloc(&buf, bytes) != cudaSuccess) { printf("malloc failed\n"); return 1; }
  cudaMalloc(&out, 8);
  cudaMemset(buf, 0, bytes);
  const long long offs[] = {-1, 128, 256, 512, 1024, 2048, 4096, 8192, 65536};
  for (int mode = 0; mode < 2; mode++)
    for (long long off : offs) {
      const float g = mode == 0 ? run<0>(buf, nlines, off, out) : run<1>(buf, nlines, off, out);
      printf("mode %d (%s) off %6lld : %.2f G ops/s [%s]\n", mode, mode ? "read+2 stores" : "read+read", off, g,
             cudaGetErrorString(cudaGetLastError()));
      fflush(stdout);
    }
  for (int mode = 0; mode < 2; mode++) {
    const float g = mode == 0 ? run<0>(buf, nlines, -1, out, 148 * 256, 1) : run<1>(buf, nlines, -1, out, 148 * 256, 1);
    printf("mode %d (%s) off     -1, grid 148x256 CTAs x 1 iteration: %.2f G ops/s [%s]\n", mode,
           mode ? "read+2 stores" : "read+read", g, cudaGetErrorString(cudaGetLastError()));
  }
  printf("err: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}

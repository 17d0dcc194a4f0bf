// TMEM load / store throughput per SM on sm_100a, without register arrays spilled to local memory (measurement tool,
// not part of the product; supersedes the load figures of tmem_micro.cu, whose dynamically indexed register arrays
// put part of each load's destination in local memory).  One CTA per SM, W warps, warp w on TMEM lanes
// 32*(w%4)..+31, each iteration = 128 fp32 columns per thread (16 KB per warp) in chunks of X columns, then
// tcgen05.wait; the destination registers are consumed only after the loop (asm volatile keeps every load).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/tmem_bw tools/tmem_bw.cu && build/tmem_bw
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2505_18875_b200/csrc/ptx.cuh"

using namespace svg2;
constexpr int kIters = 4000;

#define R4(i) "=r"(r[i]), "=r"(r[i + 1]), "=r"(r[i + 2]), "=r"(r[i + 3])
__device__ __forceinline__ void ld_x8(uint32_t t, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : R4(0), R4(4) : "r"(t));
}
__device__ __forceinline__ void ld_x16(uint32_t t, uint32_t (&r)[16]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
               : R4(0), R4(4), R4(8), R4(12) : "r"(t));
}
// 16x256b: a warp reads 16 lanes x 256 bits (8 columns) per repetition; lane l holds 4 registers of row l/4
__device__ __forceinline__ void ld_16x256_x4(uint32_t t, uint32_t (&r)[16]) {
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x4.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
               : R4(0), R4(4), R4(8), R4(12) : "r"(t));
}

template <int kMode>
__global__ void k_bw(long long* cyc, uint32_t* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t base = tmem + (uint32_t((warp & 3) * 32) << 16) + uint32_t((warp >> 2) & 3) * 128u;
  uint32_t a[32], b[32], c[32], d[32];
#pragma unroll
  for (int e = 0; e < 32; ++e) a[e] = b[e] = c[e] = d[e] = e + threadIdx.x;
  if (kMode == 9) {  // initialise the columns read below
    tmem_st32(base, a);
    tmem_st32(base + 32, a);
    tmem_st32(base + 64, a);
    tmem_st32(base + 96, a);
    tmem_wait_st();
  }
  __syncthreads();
  uint32_t x = 0;
  const long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < kIters; ++i) {
    // one register of every load instruction feeds x, so no load is dead (static indices: no local memory)
#define FOLD8(r) x ^= r[0] ^ r[8] ^ r[16] ^ r[24]
#define FOLD16(r) x ^= r[0] ^ r[16]
    if (kMode == 0) {  // 4 x 32x32b.x32
      tmem_ld32(base + 0, a);
      tmem_ld32(base + 32, b);
      tmem_ld32(base + 64, c);
      tmem_ld32(base + 96, d);
      tmem_wait_ld();
      x ^= a[1] ^ b[2] ^ c[3] ^ d[4];
    } else if (kMode == 1) {  // 8 x 32x32b.x16
      uint32_t* rr[4] = {a, b, c, d};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        ld_x16(base + 32 * q, *reinterpret_cast<uint32_t(*)[16]>(rr[q]));
        ld_x16(base + 32 * q + 16, *reinterpret_cast<uint32_t(*)[16]>(rr[q] + 16));
      }
      tmem_wait_ld();
      FOLD16(a);
      FOLD16(b);
      FOLD16(c);
      FOLD16(d);
    } else if (kMode == 2) {  // 16 x 32x32b.x8
      uint32_t* rr[4] = {a, b, c, d};
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int h = 0; h < 4; ++h) ld_x8(base + 32 * q + 8 * h, *reinterpret_cast<uint32_t(*)[8]>(rr[q] + 8 * h));
      tmem_wait_ld();
      FOLD8(a);
      FOLD8(b);
      FOLD8(c);
      FOLD8(d);
    } else if (kMode == 3) {  // 2 x (2 x x32) with a wait in between (half-tile granularity)
      tmem_ld32(base + 0, a);
      tmem_ld32(base + 32, b);
      tmem_wait_ld();
      tmem_ld32(base + 64, c);
      tmem_ld32(base + 96, d);
      tmem_wait_ld();
      x ^= a[1] ^ b[2] ^ c[3] ^ d[4];
    } else if (kMode == 4) {  // 16x256b.x4 over lanes 0-15 and 16-31 of the warp's quarter: 16 KB per warp
      uint32_t* rr[4] = {a, b, c, d};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        ld_16x256_x4(base + 32 * q, *reinterpret_cast<uint32_t(*)[16]>(rr[q]));
        ld_16x256_x4(base + (16u << 16) + 32 * q, *reinterpret_cast<uint32_t(*)[16]>(rr[q] + 16));
      }
      tmem_wait_ld();
      FOLD16(a);
      FOLD16(b);
      FOLD16(c);
      FOLD16(d);
    } else if (kMode == 5) {  // stores 4 x 32x32b.x32
      tmem_st32(base + 0, a);
      tmem_st32(base + 32, b);
      tmem_st32(base + 64, c);
      tmem_st32(base + 96, d);
      tmem_wait_st();
    } else if (kMode == 6) {  // stores of P: 4 x 32x32b.x16 (bf16 P of 128 keys = 64 columns)
      tmem_st16(base + 0, *reinterpret_cast<uint32_t(*)[16]>(a));
      tmem_st16(base + 16, *reinterpret_cast<uint32_t(*)[16]>(b));
      tmem_st16(base + 32, *reinterpret_cast<uint32_t(*)[16]>(c));
      tmem_st16(base + 48, *reinterpret_cast<uint32_t(*)[16]>(d));
      tmem_wait_st();
    } else {  // kMode 9: a single x32 load + wait (latency)
      tmem_ld32(base + 0 + (x & 0u), a);
      tmem_wait_ld();
      x ^= a[31];
    }
  }
  const long long t1 = clock64();
  sink[blockIdx.x * blockDim.x + threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

template <int kMode>
void run(const char* name, int warps, double bytes_per_warp_iter) {
  long long* cyc;
  uint32_t* sink;
  cudaMalloc(&cyc, 148 * 8);
  cudaMalloc(&sink, 148 * 1024 * 4);
  k_bw<kMode><<<148, warps * 32>>>(cyc, sink);
  k_bw<kMode><<<148, warps * 32>>>(cyc, sink);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double c = 0;
  for (int i = 0; i < 148; ++i) c += h[i];
  c /= 148;
  printf("%-34s warps %2d  cycles/iter %7.1f  TMEM bytes/clk/SM %7.1f  %s\n", name, warps, c / kIters,
         warps * kIters * bytes_per_warp_iter / c, cudaGetErrorString(e));
  cudaFree(cyc);
  cudaFree(sink);
}

int main() {
  for (int w : {4, 8}) {
    run<0>("ld 4 x 32x32b.x32 + wait", w, 16384);
    run<1>("ld 8 x 32x32b.x16 + wait", w, 16384);
    run<2>("ld 16 x 32x32b.x8 + wait", w, 16384);
    run<3>("ld 2 x (2 x x32 + wait)", w, 16384);
    run<4>("ld 8 x 16x256b.x4 + wait", w, 16384);
    run<5>("st 4 x 32x32b.x32 + wait", w, 16384);
    run<6>("st 4 x 32x32b.x16 + wait (P)", w, 8192);
  }
  run<9>("ld 1 x 32x32b.x32 + wait (latency)", 4, 4096);
  return 0;
}

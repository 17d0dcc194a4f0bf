// Does the bf16 pack (F2FP) share a pipe with MUFU.EX2?  Throughput probe with independent operations (no loop-carried
// dependency through the exponentials): per thread, 32 independent ex2 per iteration, packed in pairs by
//   mode 0: no pack (sum the results)          mode 1: F2FP.BF16.PACK_AB (cvt.rn.bf16x2.f32)
//   mode 2: PRMT of the high halves (truncate)  mode 3: FMUL2 by (1 + 2^-9) then PRMT (round-half-up-ish)
// 4 warps per block (one per SMSP), 2 blocks per SM.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kIters = 2048, kN = 32;

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t f2fp(float a, float b) {
  uint32_t r;
  asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b), "f"(a));
  return r;
}
__device__ __forceinline__ uint32_t prmt_hi(float a, float b) { return __byte_perm(__float_as_uint(a), __float_as_uint(b), 0x7632); }
__device__ __forceinline__ uint64_t fmul2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm volatile("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

template <int kMode>
__global__ void k(uint32_t* out, long long* cyc, float seed) {
  float base = seed * threadIdx.x * 1e-4f;
  uint32_t acc = 0;
  float facc = 0.f;
  const uint64_t one = (uint64_t(__float_as_uint(1.001953125f)) << 32) | __float_as_uint(1.001953125f);
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < kIters; ++it) {
    float p[kN];
#pragma unroll
    for (int i = 0; i < kN; ++i) p[i] = ex2(base - 0.03125f * i);
#pragma unroll
    for (int i = 0; i < kN; i += 2) {
      if (kMode == 0) facc += p[i] + p[i + 1];
      if (kMode == 1) acc ^= f2fp(p[i], p[i + 1]);
      if (kMode == 2) acc ^= prmt_hi(p[i], p[i + 1]);
      if (kMode == 3) {
        uint64_t v = (uint64_t(__float_as_uint(p[i + 1])) << 32) | __float_as_uint(p[i]);
        v = fmul2(v, one);
        acc ^= __byte_perm(uint32_t(v), uint32_t(v >> 32), 0x7632);
      }
    }
    base += 1e-6f * float(acc & 1u);
  }
  const long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc + __float_as_uint(facc) + __float_as_uint(base);
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int kMode>
void run(const char* name, int per_sm = 2) {
  uint32_t* out;
  long long* cyc;
  const int blocks = 148 * per_sm, threads = 128;
  cudaMalloc(&out, blocks * threads * 4);
  cudaMalloc(&cyc, blocks * 8);
  k<kMode><<<blocks, threads>>>(out, cyc, 1.0f);
  k<kMode><<<blocks, threads>>>(out, cyc, 1.0f);
  cudaDeviceSynchronize();
  long long h[296 * 2];
  cudaMemcpy(h, cyc, blocks * sizeof(long long), cudaMemcpyDeviceToHost);
  double c = 0;
  for (int i = 0; i < blocks; ++i) c += h[i];
  c /= blocks;
  // per_sm blocks per SM run concurrently (one warp per SMSP each): lanes per SM per clock
  printf("%-34s %d warp(s)/SMSP: ex2 lanes/clk/SM %6.2f\n", name, per_sm, double(per_sm) * threads * kIters * kN / c);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  for (int w = 1; w <= 4; w *= 2) {
    run<0>("ex2 only (fadd)", w);
    run<1>("ex2 + F2FP pack per pair", w);
    run<3>("ex2 + FMUL2 + PRMT per pair", w);
  }
  return 0;
}

// One softmax exponential phase of k_varblock_attn<128> in isolation: 80 scores per thread -> FFMA2 (scale, -max) ->
// 80 x ex2 -> FADD2 row sum + bf16x2 packs, the next phase depending on this phase's sum (as the kernel's next tile
// depends on its row state).  Cycles per phase per warp, 1 or 2 warps per SMSP, for schedules of the same work:
//   0 "compiler"   : the kernel's loop as written (ex2 asm non-volatile; nvcc schedules)
//   1 "two-phase"  : all 80 ex2 issued first (volatile asm keeps their order), then the sums and packs
//   2 "4 acc"      : compiler schedule with 4 independent FADD2 accumulators (no single serial sum chain)
//   3 "lag 8"      : ex2 of pair group k+1 (8 pairs) issued before the sums/packs of group k (volatile asm)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/epm tools/exp_phase_micro.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kN = 80, kIters = 512;

__device__ __forceinline__ uint64_t f2(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void f2_split(uint64_t v, float& lo, float& hi) { asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v)); }
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float ex2v(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t pack(float a, float b) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b), "f"(a));
  return r;
}
__device__ __forceinline__ uint32_t packv(float a, float b) {
  uint32_t r;
  asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b), "f"(a));
  return r;
}

template <int kMode>
__global__ void __launch_bounds__(256, 1) k(uint32_t* out, long long* cyc, float seed) {
  float s[kN];
#pragma unroll
  for (int e = 0; e < kN; ++e) s[e] = seed * float((threadIdx.x * 7 + e * 13) & 63) * 0.125f;
  const float sl2 = 0.127f;
  float l = 0.f;
  uint32_t acc = 0;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < kIters; ++it) {
    const float negm = -8.f - l * 1e-30f;  // depends on the previous phase
    const uint64_t sl2x2 = f2(sl2, sl2), negm2 = f2(negm, negm);
    uint32_t pk[kN / 2];
    if constexpr (kMode == 0 || kMode == 2) {
      uint64_t ls[4] = {f2(0.f, 0.f), f2(0.f, 0.f), f2(0.f, 0.f), f2(0.f, 0.f)};
#pragma unroll
      for (int e = 0; e < kN / 2; ++e) {
        float x0, x1;
        f2_split(ffma2(f2(s[2 * e], s[2 * e + 1]), sl2x2, negm2), x0, x1);
        const float p0 = ex2(x0), p1 = ex2(x1);
        const int a = kMode == 2 ? (e & 3) : 0;
        ls[a] = fadd2(ls[a], f2(p0, p1));
        pk[e] = pack(p0, p1);
      }
      float a0, a1, b0, b1;
      f2_split(fadd2(fadd2(ls[0], ls[1]), fadd2(ls[2], ls[3])), a0, a1);
      (void)b0;
      (void)b1;
      l += a0 + a1;
    } else if constexpr (kMode == 1) {
      float p[kN];
#pragma unroll
      for (int e = 0; e < kN / 2; ++e) {
        float x0, x1;
        f2_split(ffma2(f2(s[2 * e], s[2 * e + 1]), sl2x2, negm2), x0, x1);
        p[2 * e] = ex2v(x0);
        p[2 * e + 1] = ex2v(x1);
      }
      uint64_t ls[4] = {f2(0.f, 0.f), f2(0.f, 0.f), f2(0.f, 0.f), f2(0.f, 0.f)};
#pragma unroll
      for (int e = 0; e < kN / 2; ++e) {
        ls[e & 3] = fadd2(ls[e & 3], f2(p[2 * e], p[2 * e + 1]));
        pk[e] = packv(p[2 * e], p[2 * e + 1]);
      }
      float a0, a1;
      f2_split(fadd2(fadd2(ls[0], ls[1]), fadd2(ls[2], ls[3])), a0, a1);
      l += a0 + a1;
    } else {
      float p[kN];
      uint64_t ls[4] = {f2(0.f, 0.f), f2(0.f, 0.f), f2(0.f, 0.f), f2(0.f, 0.f)};
      constexpr int G = 8;  // pairs per group
#pragma unroll
      for (int g = 0; g <= kN / 2 / G; ++g) {
        if (g < kN / 2 / G) {
#pragma unroll
          for (int e = g * G; e < (g + 1) * G; ++e) {
            float x0, x1;
            f2_split(ffma2(f2(s[2 * e], s[2 * e + 1]), sl2x2, negm2), x0, x1);
            p[2 * e] = ex2v(x0);
            p[2 * e + 1] = ex2v(x1);
          }
        }
        if (g > 0) {
#pragma unroll
          for (int e = (g - 1) * G; e < g * G; ++e) {
            ls[e & 3] = fadd2(ls[e & 3], f2(p[2 * e], p[2 * e + 1]));
            pk[e] = packv(p[2 * e], p[2 * e + 1]);
          }
        }
      }
      float a0, a1;
      f2_split(fadd2(fadd2(ls[0], ls[1]), fadd2(ls[2], ls[3])), a0, a1);
      l += a0 + a1;
    }
#pragma unroll
    for (int e = 0; e < kN / 2; ++e) acc ^= pk[e];
  }
  const long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc + __float_as_uint(l);
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int kMode>
void run(const char* name, int threads) {
  uint32_t* out;
  long long* cyc;
  const int blocks = 148;
  cudaMalloc(&out, blocks * threads * 4);
  cudaMalloc(&cyc, blocks * 8);
  k<kMode><<<blocks, threads>>>(out, cyc, 1.0f);
  k<kMode><<<blocks, threads>>>(out, cyc, 1.0f);
  cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double c = 0;
  for (int i = 0; i < blocks; ++i) c += h[i];
  c /= blocks;
  const int wps = threads / 128;
  printf("%-12s %d warp(s)/SMSP: %7.1f cycles per 80-exp phase per warp, %5.2f ex2 lanes/clk/SM\n", name, wps,
         c / kIters, double(threads) * kIters * kN / c);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  for (int t : {128, 256}) {
    run<0>("compiler", t);
    run<1>("two-phase", t);
    run<2>("4 acc", t);
    run<3>("lag 8", t);
  }
  return 0;
}

// Per-SM issue throughput of the softmax instruction mix on sm_100a (measurement tool, not part of the product).
// Each kernel runs 4 warps per block (one per SM sub-partition), 8 independent chains per thread, 1 block per SM.
// Prints lanes-per-clock-per-SM for: MUFU.EX2, F2FP.BF16 pack, FFMA2, FMNMX3, and mixes.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/xu_micro tools/xu_micro.cu && build/xu_micro
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kIters = 4096, kChains = 8;

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t pack(float a, float b) {
  uint32_t r;
  asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b), "f"(a));
  return r;
}
__device__ __forceinline__ uint32_t pack_alu(float a, float b) {  // round-half-up via integer add + byte permute
  const uint32_t ua = __float_as_uint(a) + 0x8000u, ub = __float_as_uint(b) + 0x8000u;
  return __byte_perm(ua, ub, 0x7632);
}

__device__ __forceinline__ uint32_t ex2_bf16x2(uint32_t x) {
  uint32_t y;
  asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}

__device__ __forceinline__ uint32_t ex2_f16x2(uint32_t x) {
  uint32_t y;
  asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}
__device__ __forceinline__ uint32_t pack_f16(float a, float b) {
  uint32_t r;
  asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b), "f"(a));
  return r;
}
__device__ __forceinline__ uint32_t hadd2(uint32_t a, uint32_t b) {
  uint32_t r;
  asm volatile("add.rn.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}

template <int kMode>
__global__ void k_bench(float* out, long long* cyc, float seed) {
  float v[kChains];
  uint32_t acc = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) v[c] = seed * (threadIdx.x + c) * 1e-3f;
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
      if (kMode == 0) v[c] = ex2(v[c]);                                  // MUFU only
      if (kMode == 1) acc += pack(v[c], v[(c + 1) % kChains]), v[c] += 1e-7f * float(acc & 1u);  // F2FP
      if (kMode == 2) { v[c] = ex2(v[c]); if (c & 1) acc ^= pack(v[c - 1], v[c]); }  // softmax ratio 2 ex2 : 1 pack
      if (kMode == 3) { v[c] = ex2(v[c]); if (c & 1) acc ^= pack_alu(v[c - 1], v[c]); }  // same with ALU pack
      if (kMode == 4) { v[c] = ex2(v[c]); if (c & 1) acc ^= __float_as_uint(v[c - 1] + v[c]); }  // no pack (FADD)
      if (kMode == 8) {  // packed bf16x2 exp2: two results per MUFU op?
        uint32_t u = __float_as_uint(v[c]);
        u = ex2_bf16x2(u & 0xBFFFBFFFu);
        v[c] = __uint_as_float(u & 0x3F7F3F7Fu);
      }
      if (kMode == 9) {  // packed f16x2 exp2 on a dependent chain (2 results per op?)
        uint32_t u = __float_as_uint(v[c]);
        u = ex2_f16x2(u & 0xBBFFBBFFu);
        v[c] = __uint_as_float(u & 0x3BFF3BFFu);
      }
      if (kMode == 10) acc += pack_f16(v[c], v[(c + 1) % kChains]), v[c] += 1e-7f * float(acc & 1u);  // F2FP.F16
      if (kMode == 11) {  // the f16 softmax shape: x = s*c - m (FFMA2), cvt to f16x2, ex2.f16x2, HADD2 row sum
        const float x0 = fmaf(v[c], 1.4427f, -float(i & 7)), x1 = fmaf(v[(c + 1) % kChains], 1.4427f, -float(i & 3));
        const uint32_t p = ex2_f16x2(pack_f16(x0, x1));
        acc = hadd2(acc, p);
        v[c] += 1e-9f * float(p & 1u);
      }
      if (kMode >= 5 && kMode <= 7) {  // independent inputs: the real softmax shape (x = s*c - m; p = ex2(x); sum; pack)
        const float x0 = fmaf(v[c], 1.4427f, -float(i & 7)), x1 = fmaf(v[(c + 1) % kChains], 1.4427f, -float(i & 3));
        const float p0 = ex2(x0), p1 = ex2(x1);
        v[c] += 1e-9f * (p0 + p1);
        if (kMode == 6) acc ^= pack(p0, p1);
        if (kMode == 7) acc ^= pack_alu(p0, p1);
      }
    }
  }
  const long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += v[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + float(acc);
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int kMode>
void run(const char* name, int ops_per_chain_iter_ex2, int packs_per_iter) {
  float* out;
  long long* cyc;
  const int blocks = 148, threads = 128;
  cudaMalloc(&out, blocks * threads * 4);
  cudaMalloc(&cyc, blocks * 8);
  k_bench<kMode><<<blocks, threads>>>(out, cyc, 1.0f);
  k_bench<kMode><<<blocks, threads>>>(out, cyc, 1.0f);
  cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double c = 0;
  for (int i = 0; i < blocks; ++i) c += h[i];
  c /= blocks;
  const double lanes_ex2 = double(threads) * kIters * ops_per_chain_iter_ex2;
  const double lanes_pack = double(threads) * kIters * packs_per_iter;
  printf("%-28s cycles %10.0f  ex2 lanes/clk/SM %6.2f  pack lanes/clk/SM %6.2f\n", name, c, lanes_ex2 / c,
         lanes_pack / c);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  run<0>("MUFU.EX2 only", kChains, 0);
  run<1>("F2FP pack only", 0, kChains);
  run<2>("2 ex2 : 1 F2FP", kChains, kChains / 2);
  run<3>("2 ex2 : 1 ALU pack", kChains, kChains / 2);
  run<4>("2 ex2 : 1 FADD", kChains, 0);
  run<5>("indep: ffma ex2 fadd", 2 * kChains, 0);
  run<6>("indep: + F2FP", 2 * kChains, kChains);
  run<7>("indep: + ALU pack", 2 * kChains, kChains);
  run<8>("ex2.bf16x2 (2 per op)", 2 * kChains, 0);
  run<9>("ex2.f16x2 (2 per op)", 2 * kChains, 0);
  run<10>("F2FP.F16 pack only", 0, kChains);
  run<11>("indep f16: ffma cvt ex2x2 hadd2", 2 * kChains, kChains);
  return 0;
}

// Single-warp exponential-phase probe (measurement tool): one warp per SMSP (the product's alternation leaves one
// softmax warp per SMSP in its exponential phase) runs the softmax's exp loop -- 40 pairs: FFMA2 argument, ex2 (MUFU)
// or the FMA-pipe polynomial for kPoly pairs of every 8, FADD2 row sum, F2FP bf16 pack -- on independent inputs.
// Prints cycles per 80 exponentials.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2505_18875_b200/csrc
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "ptx.cuh"

using namespace svg2;
constexpr int kIters = 1024;

template <int kPoly>
__global__ void k(uint32_t* out, long long* cyc, float seed) {
  float s[80];
#pragma unroll
  for (int i = 0; i < 80; ++i) s[i] = seed * (threadIdx.x + i) * 1e-3f;
  uint32_t acc = 0;
  float lsum = 0.f;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < kIters; ++it) {
    const float m = -float(it & 7);
    const uint64_t sl2x2 = f2(0.125f, 0.125f), negm2 = f2(m, m);
    uint64_t lsum2 = f2(0.f, 0.f);
    uint32_t pk[40];
#pragma unroll
    for (int e = 0; e < 40; ++e) {
      float x0, x1;
      f2_split(ffma2(f2(s[2 * e], s[2 * e + 1]), sl2x2, negm2), x0, x1);
      float p0, p1;
      if ((e % 8) < kPoly) {
        f2_split(ex2_poly2(f2(x0, x1)), p0, p1);
      } else {
        p0 = ex2_approx(x0);
        p1 = ex2_approx(x1);
      }
      lsum2 = fadd2(lsum2, f2(p0, p1));
      pk[e] = pack_bf16x2(p0, p1);
    }
#pragma unroll
    for (int e = 0; e < 40; ++e) acc ^= pk[e];
    float a, b;
    f2_split(lsum2, a, b);
    lsum += a + b;
    s[it % 80] += 1e-7f * float(acc & 1u);
  }
  const long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc ^ __float_as_uint(lsum);
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int kPoly>
void run(int warps_per_smsp) {
  uint32_t* out;
  long long* cyc;
  const int blocks = 148 * warps_per_smsp, threads = 128;
  cudaMalloc(&out, blocks * threads * 4);
  cudaMalloc(&cyc, blocks * 8);
  k<kPoly><<<blocks, threads>>>(out, cyc, 1.0f);
  k<kPoly><<<blocks, threads>>>(out, cyc, 1.0f);
  cudaDeviceSynchronize();
  long long h[148 * 4];
  cudaMemcpy(h, cyc, blocks * 8, cudaMemcpyDeviceToHost);
  double c = 0;
  for (int i = 0; i < blocks; ++i) c += h[i];
  c /= blocks;
  printf("poly pairs %d of 8, %d warp(s)/SMSP: %7.1f cycles per 80 exponentials per warp\n", kPoly, warps_per_smsp,
         c / kIters);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  for (int w = 1; w <= 2; ++w) {
    run<0>(w);
    run<1>(w);
    run<2>(w);
    run<3>(w);
    run<4>(w);
  }
  return 0;
}

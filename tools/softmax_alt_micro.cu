// The two softmax warpgroups of k_varblock_attn<128> without the MMAs: per iteration each warp loads its 80 S columns
// from TMEM, takes the row max, waits for its exponential turn (named barriers, strict a/b alternation per SMSP as in
// the kernel), runs the 80-exp phase, hands the turn over and stores 40 packed P columns to TMEM.  Cycles per period
// and per exponential phase, to see what the kernel's 883-cycle phase (646 alone, tools/exp_phase_micro.cu) loses to
// the partner warp's TMEM traffic.
//   mode 0: as the kernel (TMEM ld + st, alternation)     mode 1: no TMEM (S from registers), alternation
//   mode 2: TMEM, no alternation                            mode 3: TMEM ld only (P kept in registers), alternation
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2505_18875_b200/csrc -o /tmp/sam tools/softmax_alt_micro.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "ptx.cuh"

using namespace svg2;
template <int N>
__device__ __forceinline__ uint32_t (&sub32(uint32_t (&a)[N], int off))[32] { return *reinterpret_cast<uint32_t(*)[32]>(a + off); }
template <int N>
__device__ __forceinline__ uint32_t (&sub16(uint32_t (&a)[N], int off))[16] { return *reinterpret_cast<uint32_t(*)[16]>(a + off); }
template <int N>
__device__ __forceinline__ uint32_t (&sub8(uint32_t (&a)[N], int off))[8] { return *reinterpret_cast<uint32_t(*)[8]>(a + off); }
constexpr int kN = 80, kIters = 256;
#define R4(i) "=r"(r[i]), "=r"(r[i + 1]), "=r"(r[i + 2]), "=r"(r[i + 3])
__device__ __forceinline__ void ld_x8(uint32_t t, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : R4(0), R4(4) : "r"(t));
}
__device__ __forceinline__ void ld_x4(uint32_t t, uint32_t (&r)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];" : R4(0) : "r"(t));
}
template <int N>
__device__ __forceinline__ uint32_t (&sub4(uint32_t (&a)[N], int off))[4] { return *reinterpret_cast<uint32_t(*)[4]>(a + off); }

// kMode bits: 1 = S from TMEM, 2 = exponential turns, 4 = P stored to TMEM, 8 = launder S through FADDs before the
// barrier, 16 = warpgroup b idles (one softmax warp per SMSP)
template <int kMode, int kPoly = 0>
__global__ void __launch_bounds__(256, 1) k(uint32_t* out, long long* cyc) {
  constexpr bool kTmem = kMode & 1, kTurns = kMode & 2, kStore = kMode & 4, kLaunder = kMode & 8, kSolo = kMode & 16;
  constexpr bool kLdInTurn = kMode & 32;
  constexpr bool kLd8 = kMode & 64, kLd4 = kMode & 128;  // S loaded as 10 x8 / 20 x4 loads instead of x32, x32, x16  // the S load waits for the turn (its address depends on a load after it)
  __shared__ uint32_t tmem_slot;
  __shared__ float zero_slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = warp >> 2;
  if (warp == 0) tmem_alloc<512>(&tmem_slot);
  if (threadIdx.x == 0) zero_slot = 0.f;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot + (uint32_t((warp & 3) * 32) << 16);
  const uint32_t tS = tmem + (g ? 128u : 0u), tP = tmem + (g ? 208u : 80u);
  {
    uint32_t z[32];
#pragma unroll
    for (int e = 0; e < 32; ++e) z[e] = __float_as_uint(float((lane * 5 + e * 3) & 31) * 0.5f);
    tmem_st32(tS, z);
    tmem_st32(tS + 32, z);
    tmem_st32(tS + 64, z);
    tmem_wait_st();
  }
  __syncthreads();
  const bool turns = kTurns && !kSolo;
  const int bar_mine = (g == 0 ? 2 : 6) + (warp & 3), bar_other = (g == 0 ? 6 : 2) + (warp & 3);
  if (turns && g == 1) named_bar_arrive(bar_other, 64);
  const float sl2 = 0.127f;
  float l = 0.f, m_used = 0.f;
  uint32_t acc = 0;
  uint32_t sreg[kN];
#pragma unroll
  for (int e = 0; e < kN; ++e) sreg[e] = __float_as_uint(float((lane * 7 + e * 13) & 63) * 0.125f);
  long long exp_cyc = 0;
  const long long t0 = clock64();
  for (int it = 0; it < kIters; ++it) {
    uint32_t s[kN];
    if (kSolo && g == 1) break;
    float zsync = 0.f;
    if (kLdInTurn && turns) {
      named_bar_sync(bar_mine, 64);
      zsync = ld_shared_volatile(&zero_slot);
    }
    const uint32_t tSx = tS + __float_as_uint(zsync);
    if (!kTmem) {
#pragma unroll
      for (int e = 0; e < kN; ++e) s[e] = sreg[e] ^ (uint32_t(it) & 1u);
    } else {
      if (kLd8) {
#pragma unroll
        for (int c = 0; c < kN / 8; ++c) ld_x8(tSx + 8 * c, sub8(s, 8 * c));
      } else if (kLd4) {
#pragma unroll
        for (int c = 0; c < kN / 4; ++c) ld_x4(tSx + 4 * c, sub4(s, 4 * c));
      } else {
        tmem_ld32(tSx, sub32(s, 0));
        tmem_ld32(tSx + 32, sub32(s, 32));
        tmem_ld16(tSx + 64, sub16(s, 64));
      }
      tmem_wait_ld();
      if (kLaunder) {
#pragma unroll
        for (int e = 0; e < kN; ++e) asm volatile("add.f32 %0, %0, 0f00000000;" : "+f"(*reinterpret_cast<float*>(&s[e])));
      }
    }
    float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
    for (int e = 0; e < kN; e += 4) {
      mx0 = fmaxf(mx0, fmaxf(__uint_as_float(s[e]), __uint_as_float(s[e + 2])));
      mx1 = fmaxf(mx1, fmaxf(__uint_as_float(s[e + 1]), __uint_as_float(s[e + 3])));
    }
    m_used = fmaxf(m_used, fmaxf(mx0, mx1) * sl2);
    float negm = -m_used;
    if (turns && !kLdInTurn) {
      named_bar_sync(bar_mine, 64);
      negm += ld_shared_volatile(&zero_slot);
    }
    const long long e0 = clock64();
    const uint64_t sl2x2 = f2(sl2, sl2), negm2 = f2(negm, negm);
    uint64_t lsum2 = f2(0.f, 0.f);
    uint32_t pk[kN / 2];
#pragma unroll
    for (int e = 0; e < kN / 2; ++e) {
      float x0, x1;
      f2_split(ffma2(f2(__uint_as_float(s[2 * e]), __uint_as_float(s[2 * e + 1])), sl2x2, negm2), x0, x1);
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
    if (turns) named_bar_arrive_after(bar_other, 64, lsum2);
    float a0, a1;
    f2_split(lsum2, a0, a1);
    exp_cyc += clock64() - e0;
    if (kStore) {
      tmem_st16(tP, sub16(pk, 0));
      tmem_st16(tP + 16, sub16(pk, 16));
      tmem_st8(tP + 32, sub8(pk, 32));
      tmem_wait_st();
    } else {
#pragma unroll
      for (int e = 0; e < kN / 2; ++e) acc ^= pk[e];
    }
    l += a0 + a1;
  }
  const long long t1 = clock64();
  if (turns && g == 0) named_bar_sync(bar_mine, 64);  // b's last hand-over
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc + __float_as_uint(l);
  if (lane == 0) {
    cyc[(blockIdx.x * 8 + warp) * 2] = t1 - t0;
    cyc[(blockIdx.x * 8 + warp) * 2 + 1] = exp_cyc;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem_slot);
}

template <int kMode, int kPoly = 0>
void run(const char* name) {
  uint32_t* out;
  long long* cyc;
  const int blocks = 148, threads = 256;
  cudaMalloc(&out, blocks * threads * 4);
  cudaMalloc(&cyc, blocks * 8 * 2 * 8);
  k<kMode, kPoly><<<blocks, threads>>>(out, cyc);
  k<kMode, kPoly><<<blocks, threads>>>(out, cyc);
  cudaError_t err = cudaDeviceSynchronize();
  static long long h[148 * 16];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double per = 0, ex = 0;
  const int nw = (kMode & 16) ? 4 : 8;
  for (int b = 0; b < blocks; ++b)
    for (int w = 0; w < nw; ++w) {
      per += h[2 * (b * 8 + w)];
      ex += h[2 * (b * 8 + w) + 1];
    }
  per /= blocks * double(nw) * kIters;
  ex /= blocks * double(nw) * kIters;
  printf("%-28s period %7.1f cycles per tile (both warps of an SMSP), exp phase %6.1f cycles  %s\n", name, per, ex,
         cudaGetErrorString(err));
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  run<1 | 2 | 4>("TMEM ld+st, turns");
  run<2>("no TMEM, turns");
  run<1 | 4>("TMEM ld+st, no turns");
  run<1 | 2>("TMEM ld only, turns");
  run<1 | 2 | 4 | 8>("TMEM ld+st, laundered, turns");
  run<1 | 4 | 16>("TMEM ld+st, solo");
  run<16>("no TMEM, solo");
  run<1 | 4 | 8 | 16>("TMEM ld+st, laundered, solo");
  run<1 | 2 | 4 | 32>("TMEM ld+st, ld in turn");
  run<1 | 2 | 32>("TMEM ld only, ld in turn");
  run<1 | 2 | 4 | 64>("TMEM ld(x8)+st, turns");
  run<1 | 2 | 4 | 128>("TMEM ld(x4)+st, turns");
  run<1 | 4 | 64>("TMEM ld(x8)+st, no turns");
  run<1 | 2 | 4, 1>("TMEM ld+st, turns, poly 1/8");
  run<1 | 2 | 4, 2>("TMEM ld+st, turns, poly 2/8");
  run<1 | 2 | 4, 3>("TMEM ld+st, turns, poly 3/8");
  run<2, 2>("no TMEM, turns, poly 2/8");
  run<1 | 4, 2>("TMEM ld+st, no turns, poly 2/8");
  return 0;
}

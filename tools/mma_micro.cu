// tcgen05.mma issue/execution rate per SM on sm_100a (measurement tool, not part of the product).
// One CTA per SM; one convergent warp issues R back-to-back kind::f16 MMAs (M = 128, K = 16, bf16 -> f32) with
// operands in shared memory (SS) or A in TMEM (TS), then commits and waits.  Operand contents are irrelevant.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o build/mma_micro tools/mma_micro.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2505_18875_b200/csrc/ptx.cuh"

using namespace svg2;
constexpr int kReps = 512;

template <int N, bool kTS>
__global__ void k_mma(long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (warp == 0) {
    const uint64_t da = desc_kmajor_sw128(smem_u32(smem)), db = desc_kmajor_sw128(smem_u32(smem + 65536));
    const uint32_t idesc = idesc_bf16_f32(128, N, false);
    const long long t0 = clock64();
    for (int r = 0; r < kReps; ++r) {
      const uint64_t off = uint64_t(((r & 3) * 32) >> 4);
      if (kTS)
        mma_ts_warp(tmem, tmem + 256 + 8 * (r & 7), db + off, idesc, 1u);
      else
        mma_ss_warp(tmem, da + off, db + off, idesc, r > 0);
    }
    const long long t1 = clock64();
    mma_commit_warp(&bar);
    mbar_wait_warp(&bar, 0);
    const long long t2 = clock64();
    if (threadIdx.x == 0) {
      cyc[2 * blockIdx.x] = t1 - t0;
      cyc[2 * blockIdx.x + 1] = t2 - t0;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

template <int N, bool kTS>
void run(const char* name) {
  long long* cyc;
  cudaMalloc(&cyc, 148 * 16);
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(k_mma<N, kTS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_mma<N, kTS><<<148, 128, smem>>>(cyc);
  k_mma<N, kTS><<<148, 128, smem>>>(cyc);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[296];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double issue = 0, done = 0;
  for (int i = 0; i < 148; ++i) issue += h[2 * i], done += h[2 * i + 1];
  issue /= 148.0 * kReps;
  done /= 148.0 * kReps;
  printf("%-6s N=%3d  issue %6.1f cyc/mma  complete %6.1f cyc/mma  floor %5.1f  %s\n", name, N, issue, done,
         128.0 * N / 256.0, cudaGetErrorString(e));
  cudaFree(cyc);
}

int main() {
  run<64, false>("SS");
  run<128, false>("SS");
  run<256, false>("SS");
  run<64, true>("TS");
  run<128, true>("TS");
  run<256, true>("TS");
  return 0;
}

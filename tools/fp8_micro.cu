// fp8_micro.cu — does tcgen05.mma kind::f8f6f4 take P (e4m3) from TMEM and V (e4m3) as an MN-major 128B-swizzled
// shared-memory operand?  (Feasibility test for an FP8 PV, not part of the product.)
//   O[128 x 128] = P[128 x 128 keys] * V[128 keys x 128 d], fp32 accumulate, 4 MMAs of K = 32.
// P and V are rounded to e4m3 on the device (cvt.rn.satfinite.e4m3x2.f32); the host decodes those bytes and
// computes the reference in double.  Prints max |O - ref| and PASS/FAIL.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o build/fp8_micro tools/fp8_micro.cu
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#include "../paper_2505_18875_b200/csrc/ptx.cuh"

using namespace svg2;

__device__ __forceinline__ uint16_t e4m3x2(float lo, float hi) {
  uint16_t r;
  asm("{\n\t.reg .b16 t;\n\tcvt.rn.satfinite.e4m3x2.f32 t, %1, %2;\n\tmov.b16 %0, t;\n\t}" : "=h"(r) : "f"(hi), "f"(lo));
  return r;
}

__global__ void k_quant(const float* x, uint8_t* q, int n) {
  const int i = 2 * (blockIdx.x * blockDim.x + threadIdx.x);
  if (i + 1 < n) {
    const uint16_t v = e4m3x2(x[i], x[i + 1]);
    q[i] = uint8_t(v & 0xFF);
    q[i + 1] = uint8_t(v >> 8);
  }
}

__device__ __forceinline__ void mma_ts_f8(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

// Pq [128 rows][128 keys] e4m3, Vq [128 keys][128 d] e4m3 (d contiguous), O [128][128] f32
__global__ void __launch_bounds__(128, 1) k_pv(const uint8_t* Pq, const uint8_t* Vq, float* O) {
  __shared__ __align__(1024) uint8_t sV[128 * 128];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, row = threadIdx.x;
  if (warp == 0) tmem_alloc<512>(&slot);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  // V -> shared memory, MN-major 128B swizzle: key k, 16-byte chunk c of its 128-byte row at
  // atom (k / 8) * 1024 + (k % 8) * 128 + ((c ^ (k % 8)) * 16)
  for (int e = threadIdx.x; e < 128 * 8; e += 128) {
    const int k = e / 8, c = e % 8;
    const uint4 v = *reinterpret_cast<const uint4*>(Vq + k * 128 + c * 16);
    *reinterpret_cast<uint4*>(sV + (k / 8) * 1024 + (k % 8) * 128 + ((c ^ (k % 8)) * 16)) = v;
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t lane_off = uint32_t(warp * 32) << 16;
  // P row -> TMEM columns [256, 288): 4 e4m3 per 32-bit column, key 4c + j in byte j
  uint32_t r[32];
  for (int c = 0; c < 32; ++c) r[c] = *reinterpret_cast<const uint32_t*>(Pq + row * 128 + 4 * c);
  tmem_st32(tmem + lane_off + 256, r);
  tmem_wait_st();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    // kind::f8f6f4: D f32 (bit 4), A e4m3 (0), B e4m3 (0), B MN-major (bit 16), N = 128, M = 128
    const uint32_t idesc = (1u << 4) | (1u << 16) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
    for (int k = 0; k < 4; ++k) {  // K = 32 keys per MMA: 8 TMEM columns of A, 32 key rows (4 KB) of B
      const uint64_t b = desc_mnmajor_sw128(smem_u32(sV) + k * 32 * 128, 128 * 128);
      mma_ts_f8(tmem, tmem + 256 + 8 * k, b, idesc, k > 0);
    }
    mma_commit(&bar);
  }
  __syncwarp();
  mbar_wait(&bar, 0);
  tc_fence_after();
  for (int c0 = 0; c0 < 128; c0 += 32) {
    tmem_ld32(tmem + lane_off + c0, r);
    tmem_wait_ld();
    for (int j = 0; j < 32; ++j) O[row * 128 + c0 + j] = __uint_as_float(r[j]);
  }
  (void)lane;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

static double e4m3_decode(uint8_t b) {
  const int s = b >> 7, e = (b >> 3) & 15, m = b & 7;
  double v;
  if (e == 0) v = std::ldexp(m / 8.0, -6);
  else if (e == 15 && m == 7) v = NAN;
  else v = std::ldexp(1.0 + m / 8.0, e - 7);
  return s ? -v : v;
}

int main() {
  const int n = 128 * 128;
  std::vector<float> P(n), V(n);
  srand(7);
  for (int i = 0; i < n; ++i) P[i] = float(rand() % 1000) / 400.f;          // [0, 2.5): softmax P scale
  for (int i = 0; i < n; ++i) V[i] = float(rand() % 2001 - 1000) / 250.f;   // [-4, 4]
  float *dP, *dV, *dO;
  uint8_t *qP, *qV;
  cudaMalloc(&dP, n * 4);
  cudaMalloc(&dV, n * 4);
  cudaMalloc(&dO, n * 4);
  cudaMalloc(&qP, n);
  cudaMalloc(&qV, n);
  cudaMemcpy(dP, P.data(), n * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dV, V.data(), n * 4, cudaMemcpyHostToDevice);
  k_quant<<<n / 2 / 256, 256>>>(dP, qP, n);
  k_quant<<<n / 2 / 256, 256>>>(dV, qV, n);
  k_pv<<<1, 128>>>(qP, qV, dO);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<uint8_t> hP(n), hV(n);
  std::vector<float> O(n);
  cudaMemcpy(hP.data(), qP, n, cudaMemcpyDeviceToHost);
  cudaMemcpy(hV.data(), qV, n, cudaMemcpyDeviceToHost);
  cudaMemcpy(O.data(), dO, n * 4, cudaMemcpyDeviceToHost);
  double maxerr = 0, maxref = 0, maxq = 0;
  for (int i = 0; i < 128; ++i)
    for (int j = 0; j < 128; ++j) {
      double ref = 0;
      for (int k = 0; k < 128; ++k) ref += e4m3_decode(hP[i * 128 + k]) * e4m3_decode(hV[k * 128 + j]);
      maxerr = std::fmax(maxerr, std::fabs(ref - O[i * 128 + j]));
      maxref = std::fmax(maxref, std::fabs(ref));
    }
  for (int i = 0; i < n; ++i) maxq = std::fmax(maxq, std::fabs(e4m3_decode(hV[i]) - V[i]) / std::fmax(1e-3, std::fabs(V[i])));
  printf("fp8 TS MMA (P e4m3 in TMEM, V e4m3 MN-major SW128 smem): %s  max|O-ref| = %.3e (max|ref| %.2f), "
         "V e4m3 max rel rounding %.3f  -> %s\n",
         cudaGetErrorString(e), maxerr, maxref, maxq, (e == cudaSuccess && maxerr < 1e-3 * maxref) ? "PASS" : "FAIL");
  return 0;
}

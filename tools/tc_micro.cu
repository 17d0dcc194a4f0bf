// tc_micro.cu — standalone GPU self-test of the tcgen05 / TMA encodings in csrc/ptx.cuh.
// Not part of the product; run once on a B200 to pin descriptor bit layouts before the kernels use them.
//   T1: SS  MMA  C = A * B^T   (both K-major SW128, TMA box loads)             N = 128 and 64
//   T2: TS  MMA  O = P * V     (P bf16 in TMEM, V MN-major SW128)              N = 128 and 64
//   T3: SS  MMA  with B assembled from 16 scattered 8-row TMA boxes
//   T4: SS  MMA  with B assembled from 32 TMA gather4 loads (arbitrary rows)
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include "../paper_2505_18875_b200/csrc/ptx.cuh"

using namespace svg2;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

static CUtensorMap make_map(const void* ptr, uint64_t rows, uint64_t cols, uint32_t box_cols, uint32_t box_rows) {
  CUtensorMap m;
  cuuint64_t gdim[2] = {cols, rows};
  cuuint64_t gstr[1] = {cols * 2};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = g_encode(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), gdim, gstr, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) printf("encode failed %d (box %u x %u)\n", int(r), box_cols, box_rows);
  return m;
}

// mode 0: B via two 128|64-row boxes; mode 1: 8-row groups at rows[g]; mode 2: gather4 rows[]
__global__ void __launch_bounds__(128, 1) k_ss(const __grid_constant__ CUtensorMap mA,
                                               const __grid_constant__ CUtensorMap mB,
                                               const int* rows, int n, int mode, float* C) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;             // 2 x 16 KB
  uint8_t* sB = smem + 32768;     // 2 x (n*128) B
  __shared__ uint64_t bar_load, bar_mma;
  __shared__ uint32_t tmem_slot;
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc<512>(&tmem_slot);
  if (threadIdx.x == 0) {
    mbar_init(&bar_load, 1);
    mbar_init(&bar_mma, 1);
    fence_mbar_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  const uint32_t bblk = uint32_t(n) * 128u;
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&bar_load, 32768u + 2u * bblk);
    tma_load_2d(sA, &mA, &bar_load, 0, 0);
    tma_load_2d(sA + 16384, &mA, &bar_load, 64, 0);
    if (mode == 0) {
      tma_load_2d(sB, &mB, &bar_load, 0, 0);
      tma_load_2d(sB + bblk, &mB, &bar_load, 64, 0);
    } else if (mode == 1) {
      for (int g = 0; g < n / 8; ++g) {
        tma_load_2d(sB + g * 1024, &mB, &bar_load, 0, rows[g]);
        tma_load_2d(sB + bblk + g * 1024, &mB, &bar_load, 64, rows[g]);
      }
    } else {
      for (int g = 0; g < n / 4; ++g) {
        tma_gather4(sB + g * 512, &mB, &bar_load, 0, rows[4 * g], rows[4 * g + 1], rows[4 * g + 2], rows[4 * g + 3]);
        tma_gather4(sB + bblk + g * 512, &mB, &bar_load, 64, rows[4 * g], rows[4 * g + 1], rows[4 * g + 2],
                    rows[4 * g + 3]);
      }
    }
    mbar_wait(&bar_load, 0);
    tc_fence_after();
    const uint32_t idesc = idesc_bf16_f32(128, n, false);
    for (int k = 0; k < 8; ++k) {
      const uint32_t kb = k / 4, ko = (k % 4) * 32;
      uint64_t a = desc_kmajor_sw128(smem_u32(sA) + kb * 16384 + ko);
      uint64_t b = desc_kmajor_sw128(smem_u32(sB) + kb * bblk + ko);
      mma_ss(tmem, a, b, idesc, k > 0);
    }
    mma_commit(&bar_mma);
  }
  __syncwarp();
  mbar_wait(&bar_mma, 0);
  tc_fence_after();
  const int row = warp * 32 + lane_id();
  for (int c0 = 0; c0 < n; c0 += 32) {
    uint32_t r[32];
    tmem_ld32(tmem + ((uint32_t(warp) * 32u) << 16) + c0, r);
    tmem_wait_ld();
    for (int j = 0; j < 32; ++j) C[row * n + c0 + j] = __uint_as_float(r[j]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

// O[128 x dv] = P[128 x 128] * V[128 x dv];  P from global f32 -> bf16 -> TMEM via tcgen05.st
__global__ void __launch_bounds__(128, 1) k_ts(const float* P, const __grid_constant__ CUtensorMap mV, int dv,
                                               float* O) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sV = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar_load, bar_mma;
  __shared__ uint32_t tmem_slot;
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc<512>(&tmem_slot);
  if (threadIdx.x == 0) {
    mbar_init(&bar_load, 1);
    mbar_init(&bar_mma, 1);
    fence_mbar_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  const int row = warp * 32 + lane_id();
  const uint32_t lane_off = (uint32_t(warp) * 32u) << 16;
  // P row -> TMEM columns [256, 320) as packed bf16x2 (element 2c in the low half)
  for (int c0 = 0; c0 < 64; c0 += 16) {
    uint32_t r[16];
    for (int j = 0; j < 16; ++j) r[j] = pack_bf16x2(P[row * 128 + 2 * (c0 + j)], P[row * 128 + 2 * (c0 + j) + 1]);
    tmem_st16(tmem + lane_off + 256 + c0, r);
  }
  tmem_wait_st();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t vblk = 128u * 128u;  // one 64-column block of 128 key rows
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&bar_load, uint32_t(dv) * 128u * 2u);
    for (int b = 0; b < dv / 64; ++b) tma_load_2d(sV + b * vblk, &mV, &bar_load, 64 * b, 0);
    mbar_wait(&bar_load, 0);
    tc_fence_after();
    const uint32_t idesc = idesc_bf16_f32(128, dv, true);
    for (int k = 0; k < 8; ++k) {
      uint64_t b = desc_mnmajor_sw128(smem_u32(sV) + k * 16 * 128, vblk);
      mma_ts(tmem, tmem + 256 + 8 * k, b, idesc, k > 0);
    }
    mma_commit(&bar_mma);
  }
  __syncwarp();
  mbar_wait(&bar_mma, 0);
  tc_fence_after();
  for (int c0 = 0; c0 < dv; c0 += 32) {
    uint32_t r[32];
    tmem_ld32(tmem + lane_off + c0, r);
    tmem_wait_ld();
    for (int j = 0; j < 32; ++j) O[row * dv + c0 + j] = __uint_as_float(r[j]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

static float bf(float x) { return __bfloat162float(__float2bfloat16(x)); }

int main() {
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&g_encode), cudaEnableDefault, &q));
  const int RB = 1024;  // rows in the B source matrix
  std::vector<__nv_bfloat16> hA(128 * 128), hB(RB * 128);
  std::vector<float> fA(128 * 128), fB(RB * 128);
  srand(1);
  for (int i = 0; i < 128 * 128; ++i) { fA[i] = bf((rand() % 2001 - 1000) / 500.f); hA[i] = __float2bfloat16(fA[i]); }
  for (int i = 0; i < RB * 128; ++i) { fB[i] = bf((rand() % 2001 - 1000) / 500.f); hB[i] = __float2bfloat16(fB[i]); }
  __nv_bfloat16 *dA, *dB; float* dC; int* drows;
  CK(cudaMalloc(&dA, hA.size() * 2)); CK(cudaMalloc(&dB, hB.size() * 2));
  CK(cudaMalloc(&dC, 128 * 128 * 4)); CK(cudaMalloc(&drows, 128 * 4));
  CK(cudaMemcpy(dA, hA.data(), hA.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, hB.data(), hB.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaFuncSetAttribute(k_ss, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000));
  CK(cudaFuncSetAttribute(k_ts, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000));
  int fails = 0;
  auto check_ss = [&](const char* name, int n, const std::vector<int>& rowsel) {
    std::vector<float> hC(128 * n);
    CK(cudaMemcpy(hC.data(), dC, hC.size() * 4, cudaMemcpyDeviceToHost));
    double maxerr = 0;
    for (int i = 0; i < 128; ++i)
      for (int j = 0; j < n; ++j) {
        double s = 0;
        for (int k = 0; k < 128; ++k) s += double(fA[i * 128 + k]) * fB[rowsel[j] * 128 + k];
        maxerr = fmax(maxerr, fabs(s - hC[i * n + j]));
      }
    printf("%-28s n=%3d max_abs_err=%.3e %s\n", name, n, maxerr, maxerr < 1e-2 ? "OK" : "FAIL");
    if (!(maxerr < 1e-2)) ++fails;
  };
  // T1
  for (int n : {128, 64}) {
    CUtensorMap mA = make_map(dA, 128, 128, 64, 128), mB = make_map(dB, RB, 128, 64, n);
    k_ss<<<1, 128, 100000>>>(mA, mB, drows, n, 0, dC);
    CK(cudaGetLastError()); CK(cudaDeviceSynchronize());
    std::vector<int> rs(n); for (int j = 0; j < n; ++j) rs[j] = j;
    check_ss("T1 SS K-major box", n, rs);
  }
  // T3: 8-row groups at scattered starts
  {
    int n = 128; std::vector<int> starts(16), rs(n);
    for (int g = 0; g < 16; ++g) starts[g] = (g * 61 + 7) % (RB - 8);
    for (int g = 0; g < 16; ++g) for (int r = 0; r < 8; ++r) rs[g * 8 + r] = starts[g] + r;
    CK(cudaMemcpy(drows, starts.data(), 16 * 4, cudaMemcpyHostToDevice));
    CUtensorMap mA = make_map(dA, 128, 128, 64, 128), mB = make_map(dB, RB, 128, 64, 8);
    k_ss<<<1, 128, 100000>>>(mA, mB, drows, n, 1, dC);
    CK(cudaGetLastError()); CK(cudaDeviceSynchronize());
    check_ss("T3 SS 8-row groups", n, rs);
  }
  // T4: gather4 with arbitrary rows; try box rows 1 and 4
  for (int br : {1}) {
    int n = 128; std::vector<int> rs(n);
    for (int j = 0; j < n; ++j) rs[j] = (j * 397 + 11) % RB;
    CK(cudaMemcpy(drows, rs.data(), n * 4, cudaMemcpyHostToDevice));
    CUtensorMap mA = make_map(dA, 128, 128, 64, 128), mB = make_map(dB, RB, 128, 64, br);
    k_ss<<<1, 128, 100000>>>(mA, mB, drows, n, 2, dC);
    cudaError_t e = cudaGetLastError(); if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("T4 gather4 box_rows=%d: CUDA error %s\n", br, cudaGetErrorString(e)); ++fails; break; }
    char nm[64]; snprintf(nm, sizeof nm, "T4 SS gather4 box_rows=%d", br);
    check_ss(nm, n, rs);
  }
  // T2: TS
  for (int dv : {128, 64}) {
    std::vector<float> hP(128 * 128);
    for (int i = 0; i < 128 * 128; ++i) hP[i] = bf((rand() % 1001) / 1000.f);
    float* dP; CK(cudaMalloc(&dP, hP.size() * 4));
    CK(cudaMemcpy(dP, hP.data(), hP.size() * 4, cudaMemcpyHostToDevice));
    // V = rows 0..127 of B restricted to first dv columns: use a map with cols=128 but boxes of 64 cols
    CUtensorMap mV = make_map(dB, RB, 128, 64, 128);
    k_ts<<<1, 128, 100000>>>(dP, mV, dv, dC);
    CK(cudaGetLastError()); CK(cudaDeviceSynchronize());
    std::vector<float> hO(128 * dv);
    CK(cudaMemcpy(hO.data(), dC, hO.size() * 4, cudaMemcpyDeviceToHost));
    double maxerr = 0;
    for (int i = 0; i < 128; ++i)
      for (int j = 0; j < dv; ++j) {
        double s = 0;
        for (int k = 0; k < 128; ++k) s += double(hP[i * 128 + k]) * fB[k * 128 + j];
        maxerr = fmax(maxerr, fabs(s - hO[i * dv + j]));
      }
    printf("%-28s n=%3d max_abs_err=%.3e %s\n", "T2 TS P(tmem) x V(MN)", dv, maxerr, maxerr < 1e-2 ? "OK" : "FAIL");
    if (!(maxerr < 1e-2)) ++fails;
    cudaFree(dP);
  }
  printf("tc_micro: %s (%d failures)\n", fails ? "FAILED" : "ALL OK", fails);
  return fails ? 1 : 0;
}

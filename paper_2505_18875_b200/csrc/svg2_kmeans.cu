// svg2_kmeans.cu — A1/A2/A5: Lloyd k-means per (b,h) on one role, warm-started from the caller's
// centroid cache or from the deterministic strided cold init c_j = x[floor(j*N/C)] (DESIGN R2).
//
// One iteration = assign (argmin_j ||c_j||^2 - 2 x.c_j, f32; ties -> lowest j) -> stable sort of the labels
// (svg2_permute.cu) -> centroid update c_j = (sum of its rows, fp64) / |cluster|, stored f32; empty clusters keep
// their centroid (R6).  Sums of bf16 values in fp64 are exact at these magnitudes, so the update is order-free
// and bit-identical to a sequential fp64 sum.
#include <cuda_bf16.h>
#include "internal.h"

namespace svg2 {
namespace {

constexpr int kAssignRows = 128;  // rows per block (one row per thread, the row lives in registers)
constexpr int kCentChunk = 64;    // centroids staged in shared memory per pass

template <int D>
__global__ void __launch_bounds__(kAssignRows) k_assign(const __nv_bfloat16* __restrict__ X, int N, int C,
                                                        const float* __restrict__ cent, int32_t* __restrict__ labels) {
  __shared__ __align__(16) float sc[kCentChunk * D];
  __shared__ float sn[kCentChunk];
  const int bh = blockIdx.y;
  const int n = blockIdx.x * kAssignRows + threadIdx.x;
  float x[D];
  {
    const uint4* src = reinterpret_cast<const uint4*>(X + (size_t(bh) * N + min(n, N - 1)) * D);
#pragma unroll
    for (int v = 0; v < D / 8; ++v) {
      uint4 u = __ldg(src + v);
      const __nv_bfloat162* p = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float2 f = __bfloat1622float2(p[e]);
        x[8 * v + 2 * e] = f.x;
        x[8 * v + 2 * e + 1] = f.y;
      }
    }
  }
  const float* cb = cent + size_t(bh) * C * D;
  float best = INFINITY;
  int bj = 0;
  for (int j0 = 0; j0 < C; j0 += kCentChunk) {
    const int cnt = min(kCentChunk, C - j0);
    __syncthreads();
    for (int t = threadIdx.x; t < cnt * D / 4; t += kAssignRows)
      reinterpret_cast<float4*>(sc)[t] = __ldg(reinterpret_cast<const float4*>(cb + size_t(j0) * D) + t);
    __syncthreads();
    if (threadIdx.x < cnt) {
      float s = 0.f;
      for (int k = 0; k < D; ++k) s = fmaf(sc[threadIdx.x * D + k], sc[threadIdx.x * D + k], s);
      sn[threadIdx.x] = s;
    }
    __syncthreads();
    for (int jj = 0; jj < cnt; ++jj) {
      const float4* c4 = reinterpret_cast<const float4*>(sc + jj * D);
      float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll
      for (int k4 = 0; k4 < D / 4; ++k4) {
        const float4 c = c4[k4];
        a0 = fmaf(x[4 * k4 + 0], c.x, a0);
        a1 = fmaf(x[4 * k4 + 1], c.y, a1);
        a2 = fmaf(x[4 * k4 + 2], c.z, a2);
        a3 = fmaf(x[4 * k4 + 3], c.w, a3);
      }
      const float dist = fmaf(-2.f, (a0 + a1) + (a2 + a3), sn[jj]);
      if (dist < best) {  // strict: ties keep the lower index
        best = dist;
        bj = j0 + jj;
      }
    }
  }
  if (n < N) labels[size_t(bh) * N + n] = bj;
}

template <int D>
__global__ void __launch_bounds__(D / 2) k_update(const __nv_bfloat16* __restrict__ X, int N, int C,
                                                  const int32_t* __restrict__ perm, const int32_t* __restrict__ offsets,
                                                  float* __restrict__ cent) {
  const int j = blockIdx.x, bh = blockIdx.y, t = threadIdx.x;
  const int o0 = offsets[size_t(bh) * (C + 1) + j], o1 = offsets[size_t(bh) * (C + 1) + j + 1];
  if (o1 <= o0) return;  // empty cluster keeps its centroid (R6)
  const __nv_bfloat162* Xb = reinterpret_cast<const __nv_bfloat162*>(X) + size_t(bh) * N * (D / 2);
  const int32_t* pm = perm + size_t(bh) * N;
  double s0[4] = {0, 0, 0, 0}, s1[4] = {0, 0, 0, 0};
  int p = o0;
  for (; p + 4 <= o1; p += 4) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const float2 f = __bfloat1622float2(__ldg(Xb + size_t(__ldg(pm + p + u)) * (D / 2) + t));
      s0[u] += double(f.x);
      s1[u] += double(f.y);
    }
  }
  for (; p < o1; ++p) {
    const float2 f = __bfloat1622float2(__ldg(Xb + size_t(__ldg(pm + p)) * (D / 2) + t));
    s0[0] += double(f.x);
    s1[0] += double(f.y);
  }
  const double cntd = double(o1 - o0);
  const double m0 = ((s0[0] + s0[1]) + (s0[2] + s0[3])) / cntd;
  const double m1 = ((s1[0] + s1[1]) + (s1[2] + s1[3])) / cntd;
  float* c = cent + (size_t(bh) * C + j) * D;
  c[2 * t] = float(m0);
  c[2 * t + 1] = float(m1);
}

template <int D>
__global__ void k_init_cold(const __nv_bfloat16* __restrict__ X, int N, int C, float* __restrict__ cent) {
  const int j = blockIdx.x, bh = blockIdx.y;
  const long long src = (long long)j * N / C;  // floor(j N / C)
  cent[(size_t(bh) * C + j) * D + threadIdx.x] = __bfloat162float(X[(size_t(bh) * N + src) * D + threadIdx.x]);
}

template <int D>
cudaError_t run_kmeans(const void* Xv, int BH, int N, int C, int iters, bool warm, float* cent, int32_t* labels,
                       int32_t* sizes, int32_t* perm, int32_t* offsets, KmeansWs ws, cudaStream_t s) {
  const __nv_bfloat16* X = static_cast<const __nv_bfloat16*>(Xv);
  if (!warm) k_init_cold<D><<<dim3(C, BH), D, 0, s>>>(X, N, C, cent);
  for (int it = 0; it < iters; ++it) {
    k_assign<D><<<dim3((N + kAssignRows - 1) / kAssignRows, BH), kAssignRows, 0, s>>>(X, N, C, cent, labels);
    cudaError_t e = launch_stable_sort(labels, BH, N, C, ws.sort, perm, offsets, sizes, s);
    if (e != cudaSuccess) return e;
    k_update<D><<<dim3(C, BH), D / 2, 0, s>>>(X, N, C, perm, offsets, cent);
  }
  return cudaGetLastError();
}

}  // namespace

int kmeans_launch_count(int iters, bool warm) { return (warm ? 0 : 1) + iters * (2 + kSortLaunches); }

cudaError_t launch_kmeans(const void* X, int BH, int N, int d, int C, int iters, bool warm, float* centroids,
                          int32_t* labels, int32_t* sizes, int32_t* perm, int32_t* offsets, KmeansWs ws,
                          cudaStream_t s, int* launches) {
  if (!perm) perm = ws.perm;
  if (!offsets) offsets = ws.offsets;
  if (launches) *launches += kmeans_launch_count(iters, warm);
  if (d == 128) return run_kmeans<128>(X, BH, N, C, iters, warm, centroids, labels, sizes, perm, offsets, ws, s);
  return run_kmeans<64>(X, BH, N, C, iters, warm, centroids, labels, sizes, perm, offsets, ws, s);
}

}  // namespace svg2

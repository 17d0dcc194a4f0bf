// svg2_permute.cu — A3/A4/A6/A10: cluster histogram, exclusive scan, stable index scatter (the semantic-aware
// permutation pi of PAPER.md:275), and the bf16 row gather / scatter through it (Q' = pi_q Q, K' = pi_k K,
// V' = pi_k V; O = pi_q^T O').
//
// Stable counting sort in three coalesced passes per (b,h):
//   k_hist    : per 2048-label tile, shared-memory histogram -> tile_counts[bh][tile][C]
//   k_scan    : totals per cluster -> exclusive scan -> offsets; tile_counts becomes each (tile, cluster) base
//   k_scatter : one warp walks its tile in order; __match_any_sync groups equal labels, popc(lanemask_lt)
//               gives the stable rank, a shared cursor per cluster advances by the group size.
// All integer: bit-exact and deterministic.
#include <cuda_bf16.h>
#include "internal.h"
#include "ptx.cuh"

namespace svg2 {
namespace {

__global__ void k_hist(const int32_t* __restrict__ labels, int N, int C, int T, int32_t* __restrict__ counts) {
  extern __shared__ int32_t h[];
  const int bh = blockIdx.y, tile = blockIdx.x;
  for (int j = threadIdx.x; j < C; j += blockDim.x) h[j] = 0;
  __syncthreads();
  const int32_t* lab = labels + size_t(bh) * N;
  const int n0 = tile * kSortTile, n1 = min(N, n0 + kSortTile);
  for (int n = n0 + threadIdx.x; n < n1; n += blockDim.x) {
    int l = __ldg(lab + n);
    l = min(max(l, 0), C - 1);  // labels outside [0, C) are a caller contract violation; clamp for memory safety
    atomicAdd(&h[l], 1);
  }
  __syncthreads();
  int32_t* out = counts + (size_t(bh) * T + tile) * C;
  for (int j = threadIdx.x; j < C; j += blockDim.x) out[j] = h[j];
}

// block-wide exclusive scan of v (one value per thread); returns the exclusive prefix, *total = block sum
template <int kThreads>
__device__ int block_exclusive_scan(int v, int* total) {
  __shared__ int warp_sums[kThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_sums[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int w = lane < kThreads / 32 ? warp_sums[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < kThreads / 32) warp_sums[lane] = w;  // inclusive warp prefix
  }
  __syncthreads();
  const int warp_prefix = warp > 0 ? warp_sums[warp - 1] : 0;
  *total = warp_sums[kThreads / 32 - 1];
  __syncthreads();
  return warp_prefix + x - v;
}

constexpr int kScanThreads = 1024;

// One CTA per (b,h).  Bin j = b * kScanThreads + threadIdx.x (consecutive threads own consecutive clusters, so all
// threads work for any C); the loops over the T tiles keep 8 loads in flight.  Round b scans its kScanThreads bins
// and carries the running total into round b + 1.
__global__ void __launch_bounds__(kScanThreads) k_scan(int N, int C, int T, int32_t* __restrict__ counts,
                                                       int32_t* __restrict__ offsets, int32_t* __restrict__ sizes) {
  const int bh = blockIdx.x;
  int32_t* cnt = counts + size_t(bh) * T * C;
  int carry = 0;
  for (int b = 0; b * kScanThreads < C; ++b) {
    const int bin = b * kScanThreads + threadIdx.x;
    int tot = 0;
    if (bin < C) {
      int t = 0;
      for (; t + 8 <= T; t += 8) {
        int v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = cnt[size_t(t + u) * C + bin];
#pragma unroll
        for (int u = 0; u < 8; ++u) tot += v[u];
      }
      for (; t < T; ++t) tot += cnt[size_t(t) * C + bin];
    }
    int total;
    const int run = carry + block_exclusive_scan<kScanThreads>(tot, &total);
    if (bin < C) {
      offsets[size_t(bh) * (C + 1) + bin] = run;
      if (sizes) sizes[size_t(bh) * C + bin] = tot;
      int base = run;
      int t = 0;
      for (; t + 8 <= T; t += 8) {
        int v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = cnt[size_t(t + u) * C + bin];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          cnt[size_t(t + u) * C + bin] = base;  // becomes the first output position of (tile t + u, cluster bin)
          base += v[u];
        }
      }
      for (; t < T; ++t) {
        const int c = cnt[size_t(t) * C + bin];
        cnt[size_t(t) * C + bin] = base;
        base += c;
      }
    }
    carry += total;
    __syncthreads();  // block_exclusive_scan's shared scratch is reused by the next round
  }
  if (threadIdx.x == 0) offsets[size_t(bh) * (C + 1) + C] = N;
}

__global__ void __launch_bounds__(32) k_scatter(const int32_t* __restrict__ labels, int N, int C, int T,
                                                const int32_t* __restrict__ bases, int32_t* __restrict__ perm) {
  extern __shared__ int32_t cursor[];
  const int bh = blockIdx.y, tile = blockIdx.x, lane = threadIdx.x;
  const int32_t* base = bases + (size_t(bh) * T + tile) * C;
  for (int j = lane; j < C; j += 32) cursor[j] = base[j];
  __syncwarp();
  const int32_t* lab = labels + size_t(bh) * N;
  int32_t* out = perm + size_t(bh) * N;
  const int n0 = tile * kSortTile, n1 = min(N, n0 + kSortTile);
  const unsigned lt = (1u << lane) - 1u;
  for (int c0 = n0; c0 < n1; c0 += 32) {
    const int n = c0 + lane;
    const bool valid = n < n1;
    const int l = valid ? min(max(__ldg(lab + n), 0), C - 1) : -1 - lane;  // unique dummies never match
    const unsigned grp = __match_any_sync(0xffffffffu, l);
    const int rank = __popc(grp & lt);
    int pos = 0;
    if (valid) pos = cursor[l] + rank;
    __syncwarp();
    if (valid && rank == 0) cursor[l] += __popc(grp);
    __syncwarp();
    if (valid) out[pos] = n;
  }
}

// one (b,h,p) row of d bf16 per (d/8) lanes, 16-byte vectors
__global__ void k_gather_rows(const int32_t* __restrict__ perm, long long rows, int N, int vec_per_row,
                              const uint4* __restrict__ X0, uint4* __restrict__ X0p, const uint4* __restrict__ X1,
                              uint4* __restrict__ X1p) {
  const long long total = rows * vec_per_row;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const long long r = t / vec_per_row;
    const int v = int(t - r * vec_per_row);
    const long long bh = r / N;
    const long long src = bh * N + __ldg(perm + r);
    if (X0) X0p[r * vec_per_row + v] = __ldg(X0 + src * vec_per_row + v);
    if (X1) X1p[r * vec_per_row + v] = __ldg(X1 + src * vec_per_row + v);
  }
}

__global__ void k_scatter_rows(const uint4* __restrict__ Op, const int32_t* __restrict__ perm, long long rows, int N,
                               int vec_per_row, uint4* __restrict__ O) {
  const long long total = rows * vec_per_row;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const long long r = t / vec_per_row;
    const int v = int(t - r * vec_per_row);
    const long long bh = r / N;
    const long long dst = bh * N + __ldg(perm + r);
    O[dst * vec_per_row + v] = __ldg(Op + r * vec_per_row + v);
  }
}

// FP8 PV path: per (b,h) and channel c the largest |x_c| (bf16 -> f32, as float bits: non-negative floats order like
// uints).  Grid (blocks per head, B*H); 32-bit indices within a head (N * d/8 < 2^31), vec_per_row = 1 << lg; the
// stride is a multiple of the vectors per row, so a thread always reads the same 8 channels; four loads in flight.
__global__ void k_absmax(const XView X, int vec_per_bh, int lg, uint32_t* __restrict__ amax) {
  const int bh = blockIdx.y, vpr = 1 << lg;
  const uint16_t* xb = X.row(bh, 0);
  const int t0 = blockIdx.x * blockDim.x + threadIdx.x, S = gridDim.x * blockDim.x, v = t0 & (vpr - 1);
  float m[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) m[e] = 0.f;
  auto fold = [&](const uint4& u) {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 f = __bfloat1622float2(h[e]);
      m[2 * e] = fmaxf(m[2 * e], fabsf(f.x));
      m[2 * e + 1] = fmaxf(m[2 * e + 1], fabsf(f.y));
    }
  };
  auto load = [&](int t) { return __ldg(reinterpret_cast<const uint4*>(xb + (long long)(t >> lg) * X.sN) + v); };
  int t = t0;
  for (; t + 3 * S < vec_per_bh; t += 4 * S) {
    const uint4 u0 = load(t), u1 = load(t + S), u2 = load(t + 2 * S), u3 = load(t + 3 * S);
    fold(u0);
    fold(u1);
    fold(u2);
    fold(u3);
  }
  for (; t < vec_per_bh; t += S) fold(load(t));
  // lanes l and l ^ o (o >= vec_per_row) hold the same channels
  for (int o = 16; o >= vpr; o >>= 1)
#pragma unroll
    for (int e = 0; e < 8; ++e) m[e] = fmaxf(m[e], __shfl_xor_sync(0xffffffffu, m[e], o));
  if ((threadIdx.x & 31) < vpr) {
#pragma unroll
    for (int e = 0; e < 8; ++e) atomicMax(amax + size_t(bh) * vpr * 8 + v * 8 + e, __float_as_uint(m[e]));
  }
}

// FP8 PV path: V' = V[perm] rounded to e4m3, channel c scaled by 448 / amax_c of its head (448 = largest finite e4m3);
// the attention epilogue multiplies output channel c by amax_c / 448.  Same grid as k_absmax: a thread keeps its head
// and its 8 channels, so the scales are computed once; four rows in flight per thread.
__global__ void k_gather_rows_e4m3(const int32_t* __restrict__ perm, int N, int lg, const XView X,
                                   uint2* __restrict__ Xq, const uint32_t* __restrict__ amax) {
  const int bh = blockIdx.y, vpr = 1 << lg, total = N << lg;
  const int t0 = blockIdx.x * blockDim.x + threadIdx.x, S = gridDim.x * blockDim.x, v = t0 & (vpr - 1);
  float sc[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const float a = __uint_as_float(__ldg(amax + (size_t(bh) * vpr + v) * 8 + e));
    sc[e] = a > 0.f ? 448.f / a : 1.f;
  }
  const int32_t* pb = perm + size_t(bh) * N;
  uint2* qb = Xq + size_t(bh) * total;
  auto quant = [&](int t, const uint4& u) {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
    uint32_t q[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 f = __bfloat1622float2(h[e]);
      q[e] = pack_e4m3x2(f.x * sc[2 * e], f.y * sc[2 * e + 1]);
    }
    qb[t] = make_uint2(q[0] | (q[1] << 16), q[2] | (q[3] << 16));
  };
  auto src = [&](int t) { return reinterpret_cast<const uint4*>(X.row(bh, __ldg(pb + (t >> lg)))) + v; };
  int t = t0;
  for (; t + 3 * S < total; t += 4 * S) {
    const uint4* p0 = src(t);
    const uint4* p1 = src(t + S);
    const uint4* p2 = src(t + 2 * S);
    const uint4* p3 = src(t + 3 * S);
    const uint4 u0 = __ldg(p0), u1 = __ldg(p1), u2 = __ldg(p2), u3 = __ldg(p3);
    quant(t, u0);
    quant(t + S, u1);
    quant(t + 2 * S, u2);
    quant(t + 3 * S, u3);
  }
  for (; t < total; t += S) quant(t, __ldg(src(t)));
}

int copy_grid(long long work) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  long long blocks = (work + 255) / 256;
  long long cap = (long long)sms * 8;
  return int(blocks < cap ? (blocks > 0 ? blocks : 1) : cap);
}

}  // namespace

cudaError_t launch_stable_sort(const int32_t* labels, int BH, int N, int C, SortWs ws, int32_t* perm,
                               int32_t* offsets, int32_t* sizes, cudaStream_t s) {
  const int T = sort_tiles(N);
  const size_t smem = size_t(C) * sizeof(int32_t);
  k_hist<<<dim3(T, BH), 256, smem, s>>>(labels, N, C, T, ws.tile_counts);
  k_scan<<<BH, kScanThreads, 0, s>>>(N, C, T, ws.tile_counts, offsets, sizes);
  k_scatter<<<dim3(T, BH), 32, smem, s>>>(labels, N, C, T, ws.tile_counts, perm);
  return cudaGetLastError();
}

cudaError_t launch_gather_rows(const int32_t* perm, int BH, int N, int d, const void* X0, void* X0p, const void* X1,
                               void* X1p, cudaStream_t s) {
  const long long rows = (long long)BH * N;
  const int vpr = d / 8;
  k_gather_rows<<<copy_grid(rows * vpr), 256, 0, s>>>(perm, rows, N, vpr, static_cast<const uint4*>(X0),
                                                      static_cast<uint4*>(X0p), static_cast<const uint4*>(X1),
                                                      static_cast<uint4*>(X1p));
  return cudaGetLastError();
}

cudaError_t launch_absmax(int BH, int N, int d, XView X, uint32_t* amax, cudaStream_t s) {
  const int vpr = d / 8;
  cudaMemsetAsync(amax, 0, size_t(BH) * d * sizeof(uint32_t), s);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int per_bh = (sms * 8 + BH - 1) / BH;
  const int lg = 31 - __builtin_clz(unsigned(vpr));  // d / 8 = 8 or 16
  k_absmax<<<dim3(per_bh, BH), 256, 0, s>>>(X, N * vpr, lg, amax);
  return cudaGetLastError();
}

cudaError_t launch_gather_rows_e4m3(const int32_t* perm, int BH, int N, int d, XView X, void* Xq,
                                    const uint32_t* amax, cudaStream_t s) {
  const int vpr = d / 8;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int per_bh = (sms * 8 + BH - 1) / BH;
  const int lg = 31 - __builtin_clz(unsigned(vpr));
  k_gather_rows_e4m3<<<dim3(per_bh, BH), 256, 0, s>>>(perm, N, lg, X, static_cast<uint2*>(Xq), amax);
  return cudaGetLastError();
}

cudaError_t launch_scatter_rows(const void* Op, const int32_t* perm, int BH, int N, int d, void* O, cudaStream_t s) {
  const long long rows = (long long)BH * N;
  const int vpr = d / 8;
  k_scatter_rows<<<copy_grid(rows * vpr), 256, 0, s>>>(static_cast<const uint4*>(Op), perm, rows, N, vpr,
                                                       static_cast<uint4*>(O));
  return cudaGetLastError();
}

}  // namespace svg2

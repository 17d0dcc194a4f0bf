// svg2_kmeans.cu — A1/A2/A5: Lloyd k-means per (b,h) on one role, warm-started from the caller's
// centroid cache or from the deterministic strided cold init c_j = x[floor(j*N/C)] (DESIGN R2).
//
// One iteration:
//   k_centroid_split : c (f32) -> hi = bf16(c), lo = bf16(c - hi), ||c||^2 (f32); padded to 128-centroid chunks
//   k_assign_tc      : the distance GEMM on tcgen05 — X tile (bf16, exact) x [hi | lo]^T accumulated in fp32 in TMEM
//                      (K = 2d, so x.c carries ~16 mantissa bits of c), argmin_j ||c_j||^2 - 2 x.c_j read back with
//                      tcgen05.ld (ties -> lowest j).  Persistent (one CTA per SM over 128-row units); X and the
//                      centroid chunks are double-buffered in smem (TMA), accumulators four-deep in TMEM.
//   stable sort of the labels (svg2_permute.cu)
//   k_update         : c_j = (sum of its rows, fp64) / |cluster|, stored f32; empty clusters keep their centroid (R6).
//                      Sums of bf16 values in fp64 are exact at these magnitudes, so the update is order-free and
//                      bit-identical to the oracle's sequential sum.
#include <cuda_bf16.h>
#include <type_traits>
#include "internal.h"
#include "ptx.cuh"
#include "tmap.h"

namespace svg2 {
namespace {

constexpr int kAsgThreads = 192;  // warp 0 TMA, warp 1 MMA, warps 2-5 argmin epilogue (one TMEM lane quarter each)
constexpr int kAsgRows = 128;     // rows per work unit (one M = 128 tile)
constexpr int kAccStages = 4;     // TMEM accumulator stages of 128 columns

template <int D>
struct AsgCfg {
  static constexpr int kBlocks = D / 64;
  static constexpr uint32_t kBlockBytes = 128 * 128;            // 128 rows x 64 bf16
  static constexpr uint32_t kTileBytes = kBlocks * kBlockBytes;  // 128 rows x D bf16
  static constexpr uint32_t kNormBytes = kMaxClusters * 4;
  // X: 2 buffers | centroid chunk stages: 2 x (hi tile + lo tile) | norms
  static constexpr uint32_t kSmem = 2 * kTileBytes + 4 * kTileBytes + kNormBytes + 1024;
};

template <int D>
__global__ void __launch_bounds__(D) k_centroid_split(const float* __restrict__ cent, int C, int Cpad,
                                                      __nv_bfloat16* __restrict__ hi, __nv_bfloat16* __restrict__ lo,
                                                      float* __restrict__ norm) {
  __shared__ float red[D / 32];
  const int j = blockIdx.x, bh = blockIdx.y, k = threadIdx.x;
  const float c = j < C ? cent[(size_t(bh) * C + j) * D + k] : 0.f;
  const __nv_bfloat16 h = __float2bfloat16_rn(c);
  const __nv_bfloat16 l = __float2bfloat16_rn(c - __bfloat162float(h));
  hi[(size_t(bh) * Cpad + j) * D + k] = h;
  lo[(size_t(bh) * Cpad + j) * D + k] = l;
  float s = c * c;
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((k & 31) == 0) red[k >> 5] = s;
  __syncthreads();
  if (k == 0) {
    float t = 0.f;
    for (int w = 0; w < D / 32; ++w) t += red[w];
    norm[size_t(bh) * Cpad + j] = j < C ? t : INFINITY;
  }
}

struct AsgBars {
  uint64_t x_full[2], x_empty[2], c_full[2], c_empty[2], acc_full[kAccStages], acc_empty[kAccStages];
};

// Persistent assignment: one CTA per SM walks a contiguous range of 128-row work units (row tiles of one (b,h); the
// range is mostly one head).  Per unit the producer loads X (double-buffered) and streams the centroid chunks (two
// stages, hi and lo tiles); the MMA warp accumulates X [hi | lo]^T per chunk into one of four TMEM stages; the
// epilogue warps read each stage back and keep the running argmin.  Loads, MMAs and TMEM reads of consecutive
// units overlap, and TMEM allocation / barrier setup happen once per CTA instead of once per tile.
template <int D>
__global__ void __launch_bounds__(kAsgThreads, 1)
    k_assign_tc(const __grid_constant__ CUtensorMap mapX, const __grid_constant__ CUtensorMap mapHi,
                const __grid_constant__ CUtensorMap mapLo, const float* __restrict__ c_norm, int N, int Cpad,
                int BH, int32_t* __restrict__ labels) {
  using C = AsgCfg<D>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sX = smem;                       // [2 buffers]
  uint8_t* sH = smem + 2 * C::kTileBytes;   // [2 stages]
  uint8_t* sL = sH + 2 * C::kTileBytes;     // [2 stages]
  float* sNorm = reinterpret_cast<float*>(sL + 2 * C::kTileBytes);  // [Cpad] of the epilogue's current head
  __shared__ AsgBars bars;
  __shared__ uint32_t tmem_slot;

  const int warp = __shfl_sync(0xffffffffu, int(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const int upb = (N + kAsgRows - 1) / kAsgRows;  // units per (b,h)
  const long long total = (long long)BH * upb;
  const int u0 = int(total * blockIdx.x / gridDim.x), u1 = int(total * (blockIdx.x + 1) / gridDim.x);
  const int nchunks = Cpad / kCentChunk;
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&mapX);
    tma_prefetch_desc(&mapHi);
    tma_prefetch_desc(&mapLo);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&bars.x_full[s], 1);
      mbar_init(&bars.x_empty[s], 1);
      mbar_init(&bars.c_full[s], 1);
      mbar_init(&bars.c_empty[s], 1);
    }
    for (int s = 0; s < kAccStages; ++s) {
      mbar_init(&bars.acc_full[s], 1);
      mbar_init(&bars.acc_empty[s], 4);
    }
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<512>(&tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = __shfl_sync(0xffffffffu, tmem_slot, 0);

  if (warp == 0) {
    if (lane == 0) {
      uint32_t cc = 0;
      for (int u = u0, i = 0; u < u1; ++u, ++i) {
        const int bh = u / upb, row0 = (u - bh * upb) * kAsgRows;
        const int xs = i & 1;
        mbar_wait(&bars.x_empty[xs], ((i >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&bars.x_full[xs], C::kTileBytes);
        for (int b = 0; b < C::kBlocks; ++b)
          tma_load_2d(sX + xs * C::kTileBytes + b * C::kBlockBytes, &mapX, &bars.x_full[xs], 64 * b, bh * N + row0);
        for (int c = 0; c < nchunks; ++c, ++cc) {
          const int s = cc & 1;
          mbar_wait(&bars.c_empty[s], ((cc >> 1) & 1) ^ 1);
          mbar_arrive_expect_tx(&bars.c_full[s], 2 * C::kTileBytes);
          const int crow = bh * Cpad + c * kCentChunk;
          for (int b = 0; b < C::kBlocks; ++b) {
            tma_load_2d(sH + s * C::kTileBytes + b * C::kBlockBytes, &mapHi, &bars.c_full[s], 64 * b, crow);
            tma_load_2d(sL + s * C::kTileBytes + b * C::kBlockBytes, &mapLo, &bars.c_full[s], 64 * b, crow);
          }
        }
      }
    }
  } else if (warp == 1) {
    // whole warp, convergent: elect.sync inside the MMA asm -> back-to-back UTCHMMA on uniform registers
    const uint32_t idesc = idesc_bf16_f32(128, kCentChunk, false);
    uint32_t cc = 0, ac = 0;
    for (int u = u0, i = 0; u < u1; ++u, ++i) {
      const int xs = i & 1;
      mbar_wait_warp(&bars.x_full[xs], (i >> 1) & 1);
      const uint32_t x = smem_u32(sX + xs * C::kTileBytes);
      for (int c = 0; c < nchunks; ++c, ++cc, ++ac) {
        const int s = cc & 1, as = ac % kAccStages;
        mbar_wait_warp(&bars.c_full[s], (cc >> 1) & 1);
        mbar_wait_warp(&bars.acc_empty[as], ((ac / kAccStages) & 1) ^ 1);
        tc_fence_after();
        const uint32_t h = smem_u32(sH + s * C::kTileBytes), l = smem_u32(sL + s * C::kTileBytes);
        const uint32_t dcol = tmem + as * 128;
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const uint32_t off = (k >> 2) * C::kBlockBytes + (k & 3) * 32;
          mma_ss_warp(dcol, desc_kmajor_sw128(x + off), desc_kmajor_sw128(h + off), idesc, k > 0);
        }
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const uint32_t off = (k >> 2) * C::kBlockBytes + (k & 3) * 32;
          mma_ss_warp(dcol, desc_kmajor_sw128(x + off), desc_kmajor_sw128(l + off), idesc, 1u);
        }
        mma_commit_warp(&bars.c_empty[s]);
        mma_commit_warp(&bars.acc_full[as]);
      }
      mma_commit_warp(&bars.x_empty[xs]);
    }
  } else {
    const int quarter = warp & 3;  // warps 2..5 -> TMEM lane quarters 2, 3, 0, 1
    const uint32_t lane_addr = uint32_t(quarter * 32) << 16;
    uint32_t ac = 0;
    int cur_bh = -1;
    for (int u = u0; u < u1; ++u) {
      const int bh = u / upb, row0 = (u - bh * upb) * kAsgRows;
      if (bh != cur_bh) {  // stage this head's ||c||^2 (all four epilogue warps, named barrier 1)
        named_bar_sync(1, 128);
        for (int j = threadIdx.x - 64; j < Cpad; j += 128) sNorm[j] = __ldg(c_norm + size_t(bh) * Cpad + j);
        named_bar_sync(1, 128);
        cur_bh = bh;
      }
      float best = INFINITY;
      int bj = 0;
      for (int c = 0; c < nchunks; ++c, ++ac) {
        const int as = ac % kAccStages;
        mbar_wait(&bars.acc_full[as], (ac / kAccStages) & 1);
        tc_fence_after();
        // all four 32-column loads of the stage in flight before one wait (one TMEM round trip per chunk, not four)
        uint32_t r4[kCentChunk / 32][32];
#pragma unroll
        for (int q = 0; q < kCentChunk / 32; ++q) tmem_ld32(tmem + lane_addr + as * 128 + 32 * q, r4[q]);
        tmem_wait_ld();
#pragma unroll
        for (int q = 0; q < kCentChunk / 32; ++q) {
          const int j0 = c * kCentChunk + 32 * q;
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            const float dist = fmaf(-2.f, __uint_as_float(r4[q][e]), sNorm[j0 + e]);
            if (dist < best) {  // strict: ties keep the lower index
              best = dist;
              bj = j0 + e;
            }
          }
        }
        // released after the argmin (releasing right after the loads measured slower: 594 vs 574 us per K launch)
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars.acc_empty[as]);
      }
      const int row = row0 + quarter * 32 + lane;
      if (row < N) labels[size_t(bh) * N + row] = bj;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

// Centroid update, pass 1: each warp sums a contiguous chunk of kSumRows permuted positions (rows gathered through
// perm; lane l holds D/32 consecutive columns, so one row is one coalesced D*2-byte read) and flushes one fp64
// partial per cluster the chunk touches with atomicAdd.  kSumUnroll rows are loaded before any is accumulated, so
// each warp keeps several row reads in flight (the loop is latency-bound otherwise).  Sums of bf16 values in fp64
// are exact at these magnitudes, so the result does not depend on the order of the atomics: deterministic and
// bit-identical to a sequential fp64 sum.
// On the last iteration the same pass also writes the permuted copy X' = pi X (A6) and optionally Y' = pi Y (V,
// which shares pi_k), so the fused call reads Q and K once less (no separate gather launches).
constexpr int kSumRows = 64, kSumUnroll = 8, kSumWarps = 4;

template <int D, bool kGather>
__global__ void __launch_bounds__(32 * kSumWarps) k_update_sum(const __nv_bfloat16* __restrict__ X, int N, int C,
                                                             const int32_t* __restrict__ perm,
                                                             const int32_t* __restrict__ offsets,
                                                             double* __restrict__ sum, __nv_bfloat16* __restrict__ Xp,
                                                             const __nv_bfloat16* __restrict__ Y,
                                                             __nv_bfloat16* __restrict__ Yp) {
  constexpr int kCols = D / 32;  // 4 (d = 128) or 2 (d = 64) bf16 per lane
  using Vec = typename std::conditional<kCols == 4, uint2, uint32_t>::type;
  const int bh = blockIdx.y, lane = threadIdx.x & 31;
  const int p0 = (blockIdx.x * kSumWarps + (threadIdx.x >> 5)) * kSumRows;
  if (p0 >= N) return;
  const int p1 = min(N, p0 + kSumRows);
  const int32_t* off = offsets + size_t(bh) * (C + 1);
  int lo = 0, hi = C - 1;  // cluster of position p0: last j with off[j] <= p0
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (__ldg(off + mid) <= p0) lo = mid; else hi = mid - 1;
  }
  int j = lo, next = __ldg(off + j + 1);
  const Vec* Xv = reinterpret_cast<const Vec*>(X) + size_t(bh) * N * 32;  // 32 Vec per row
  Vec* Xpv = kGather ? reinterpret_cast<Vec*>(Xp) + size_t(bh) * N * 32 : nullptr;
  const Vec* Yv = kGather && Y ? reinterpret_cast<const Vec*>(Y) + size_t(bh) * N * 32 : nullptr;
  Vec* Ypv = kGather && Yp ? reinterpret_cast<Vec*>(Yp) + size_t(bh) * N * 32 : nullptr;
  const int32_t* pm = perm + size_t(bh) * N;
  double* sb = sum + size_t(bh) * C * D;
  double acc[kCols];
#pragma unroll
  for (int c = 0; c < kCols; ++c) acc[c] = 0.0;
  bool any = false;
  auto flush = [&] {
    if (any) {
#pragma unroll
      for (int c = 0; c < kCols; ++c) atomicAdd(sb + size_t(j) * D + kCols * lane + c, acc[c]);
    }
#pragma unroll
    for (int c = 0; c < kCols; ++c) acc[c] = 0.0;
    any = false;
  };
  for (int pb = p0; pb < p1; pb += kSumUnroll) {
    const int src_l = pb + (lane & (kSumUnroll - 1)) < p1 ? __ldg(pm + pb + (lane & (kSumUnroll - 1))) : 0;
    Vec v[kSumUnroll];
#pragma unroll
    for (int u = 0; u < kSumUnroll; ++u) {
      const int src = __shfl_sync(0xffffffffu, src_l, u);
      if (pb + u < p1) v[u] = __ldg(Xv + size_t(src) * 32 + lane);
    }
    if (kGather) {
      if (Ypv) {  // the gather-only tensor (V' = pi_k V): loads in flight together with X's
        Vec y[kSumUnroll];
#pragma unroll
        for (int u = 0; u < kSumUnroll; ++u) {
          const int src = __shfl_sync(0xffffffffu, src_l, u);
          if (pb + u < p1) y[u] = __ldg(Yv + size_t(src) * 32 + lane);
        }
#pragma unroll
        for (int u = 0; u < kSumUnroll; ++u)
          if (pb + u < p1) Ypv[size_t(pb + u) * 32 + lane] = y[u];
      }
#pragma unroll
      for (int u = 0; u < kSumUnroll; ++u)
        if (pb + u < p1) Xpv[size_t(pb + u) * 32 + lane] = v[u];
    }
#pragma unroll
    for (int u = 0; u < kSumUnroll; ++u) {
      const int pos = pb + u;
      if (pos >= p1) break;
      while (pos >= next) {  // crossed into the next cluster: flush the partial sum
        flush();
        ++j;
        next = __ldg(off + j + 1);
      }
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v[u]);
#pragma unroll
      for (int c = 0; c < kCols / 2; ++c) {
        const float2 f = __bfloat1622float2(h[c]);
        acc[2 * c] += double(f.x);
        acc[2 * c + 1] += double(f.y);
      }
      any = true;
    }
  }
  flush();
}

// The last (gather) iteration's pass with the row gathers as asynchronous copies (cp.async, 16 B per
// lane-instruction): a warp puts all kAsyncRows rows of its chunk (X and Y) in flight at once through shared memory
// instead of kSumUnroll rows through registers, and the permuted copies leave shared memory as one bulk copy per
// tensor (the chunk's rows are contiguous in X').  Measured (ncu, HunyuanVideo): K' + V' 0.69 -> 0.48 ms, Q' equal;
// for the plain update the register-staged kernel stays faster (0.20 vs 0.33 ms).
constexpr int kAsyncWarps = 4;
template <bool kGather>
constexpr int kAsyncRows = kGather ? 32 : 64;  // <= 64: two perm registers per lane
template <int D, bool kGather>
__global__ void __launch_bounds__(32 * kAsyncWarps) k_update_sum_async(
    const __nv_bfloat16* __restrict__ X, int N, int C, const int32_t* __restrict__ perm,
    const int32_t* __restrict__ offsets, double* __restrict__ sum, __nv_bfloat16* __restrict__ Xp,
    const __nv_bfloat16* __restrict__ Y, __nv_bfloat16* __restrict__ Yp) {
  constexpr int kCols = D / 32;           // bf16 per lane in the accumulation
  constexpr int kRowBytes = D * 2;        // 256 (d = 128) or 128 (d = 64)
  constexpr int kVecPerRow = kRowBytes / 16;
  constexpr int kTensors = kGather ? 2 : 1;
  constexpr int kRows = kAsyncRows<kGather>;  // rows per warp (the gather pass holds two tensors per row)
  extern __shared__ __align__(128) uint8_t sm_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, bh = blockIdx.y;
  uint8_t* sx = sm_raw + size_t(warp) * kTensors * kRows * kRowBytes;  // [kRows][row] X rows of this warp
  uint8_t* sy = sx + kRows * kRowBytes;                                 // [kRows][row] Y rows (kGather)
  const int p0 = (blockIdx.x * kAsyncWarps + warp) * kRows;
  if (p0 >= N) return;
  const int nrow = min(N - p0, kRows);
  const bool with_y = kGather && Y != nullptr;
  const int32_t* pm = perm + size_t(bh) * N + p0;
  const int src0 = lane < nrow ? __ldg(pm + lane) : 0, src1 = kRows > 32 && lane + 32 < nrow ? __ldg(pm + 32 + lane) : 0;
  const uint8_t* xb = reinterpret_cast<const uint8_t*>(X) + size_t(bh) * N * kRowBytes;
  const uint8_t* yb = with_y ? reinterpret_cast<const uint8_t*>(Y) + size_t(bh) * N * kRowBytes : nullptr;
  // issue: 32 lanes cover 32 / kVecPerRow rows per step, one 16-byte piece each
  constexpr int kRowsPerStep = 32 / kVecPerRow;
  const int piece = lane % kVecPerRow, rsub = lane / kVecPerRow;
  for (int r0 = 0; r0 < nrow; r0 += kRowsPerStep) {
    const int r = r0 + rsub;
    const int src = __shfl_sync(0xffffffffu, r < 32 ? src0 : src1, r & 31);
    if (r < nrow) {
      const uint32_t dst = smem_u32(sx + r * kRowBytes + piece * 16);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(xb + size_t(src) * kRowBytes + piece * 16)
                   : "memory");
      if (with_y) {
        const uint32_t dy = smem_u32(sy + r * kRowBytes + piece * 16);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dy), "l"(yb + size_t(src) * kRowBytes + piece * 16)
                     : "memory");
      }
    }
  }
  // cluster of the first position while the copies fly: last j with off[j] <= p0
  const int32_t* off = offsets + size_t(bh) * (C + 1);
  int lo = 0, hi = C - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (__ldg(off + mid) <= p0) lo = mid; else hi = mid - 1;
  }
  int j = lo, next = __ldg(off + j + 1) - p0;  // positions relative to p0
  asm volatile("cp.async.wait_all;" ::: "memory");
  // every lane's cp.async writes into shared memory are made visible to the async proxy (the bulk store below) by
  // that lane's own proxy fence before the warp barrier
  if (kGather) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  if (kGather) {  // X' (and Y') rows p0 .. p0 + nrow - 1 are contiguous: one bulk store each, issued by lane 0
    if (lane == 0) {
      uint8_t* gx = reinterpret_cast<uint8_t*>(Xp) + (size_t(bh) * N + p0) * kRowBytes;
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gx), "r"(smem_u32(sx)),
                   "r"(nrow * kRowBytes)
                   : "memory");
      if (with_y) {
        uint8_t* gy = reinterpret_cast<uint8_t*>(Yp) + (size_t(bh) * N + p0) * kRowBytes;
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gy), "r"(smem_u32(sy)),
                     "r"(nrow * kRowBytes)
                     : "memory");
      }
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  double* sb = sum + size_t(bh) * C * D;
  double acc[kCols];
#pragma unroll
  for (int c = 0; c < kCols; ++c) acc[c] = 0.0;
  bool any = false;
  for (int r = 0; r < nrow; ++r) {
    while (r >= next) {  // crossed into the next cluster: flush the partial sum
      if (any) {
#pragma unroll
        for (int c = 0; c < kCols; ++c) atomicAdd(sb + size_t(j) * D + kCols * lane + c, acc[c]);
      }
#pragma unroll
      for (int c = 0; c < kCols; ++c) acc[c] = 0.0;
      any = false;
      ++j;
      next = __ldg(off + j + 1) - p0;
    }
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(sx + r * kRowBytes + lane * kCols * 2);
#pragma unroll
    for (int c = 0; c < kCols / 2; ++c) {
      const float2 f = __bfloat1622float2(h[c]);
      acc[2 * c] += double(f.x);
      acc[2 * c + 1] += double(f.y);
    }
    any = true;
  }
  if (any) {
#pragma unroll
    for (int c = 0; c < kCols; ++c) atomicAdd(sb + size_t(j) * D + kCols * lane + c, acc[c]);
  }
  if (kGather && lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // smem stays live
  __syncwarp();
}

// Pass 2: c_j = sum_j / |cluster j| (fp64, rounded to f32); empty clusters keep their centroid (R6).  The sums are
// zeroed for the next iteration.
template <int D>
__global__ void __launch_bounds__(D) k_update_mean(int C, const int32_t* __restrict__ offsets,
                                                   double* __restrict__ sum, float* __restrict__ cent) {
  const int j = blockIdx.x, bh = blockIdx.y, k = threadIdx.x;
  const int cnt = offsets[size_t(bh) * (C + 1) + j + 1] - offsets[size_t(bh) * (C + 1) + j];
  double* s = sum + (size_t(bh) * C + j) * D + k;
  if (cnt > 0) cent[(size_t(bh) * C + j) * D + k] = float(*s / double(cnt));
  *s = 0.0;
}

template <int D>
__global__ void k_init_cold(const __nv_bfloat16* __restrict__ X, int N, int C, float* __restrict__ cent) {
  const int j = blockIdx.x, bh = blockIdx.y;
  const long long src = (long long)j * N / C;  // floor(j N / C)
  cent[(size_t(bh) * C + j) * D + threadIdx.x] = __bfloat162float(X[(size_t(bh) * N + src) * D + threadIdx.x]);
}

template <int D>
cudaError_t run_kmeans(const void* Xv, int BH, int N, int C, int iters, bool warm, const KmeansInit& init,
                       float* cent, int32_t* labels,
                       int32_t* sizes, int32_t* perm, int32_t* offsets, KmeansWs ws, cudaStream_t s,
                       const KmeansGather& g) {
  const __nv_bfloat16* X = static_cast<const __nv_bfloat16*>(Xv);
  const int Cpad = cent_pad(C);
  CUtensorMap mx, mh, ml;
  if (!make_tmap_bf16(&mx, Xv, uint64_t(BH) * N, D, 128) || !make_tmap_bf16(&mh, ws.c_hi, uint64_t(BH) * Cpad, D, 128) ||
      !make_tmap_bf16(&ml, ws.c_lo, uint64_t(BH) * Cpad, D, 128))
    return cudaErrorInvalidValue;
  cudaFuncSetAttribute(k_assign_tc<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, AsgCfg<D>::kSmem);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long units = (long long)BH * ((N + kAsgRows - 1) / kAsgRows);
  const int grid_asg = int(units < sms ? units : sms);  // persistent: one CTA per SM
  if (!warm && init.kmeanspp) {
    cudaError_t e = launch_kmeanspp(Xv, BH, N, D, C, init.seed, init.role, init.bh_base, cent, ws.pp, s);
    if (e != cudaSuccess) return e;
  } else if (!warm) {
    k_init_cold<D><<<dim3(C, BH), D, 0, s>>>(X, N, C, cent);
  }
  cudaMemsetAsync(ws.c_sum, 0, size_t(BH) * C * D * sizeof(double), s);
  __nv_bfloat16* hi = reinterpret_cast<__nv_bfloat16*>(ws.c_hi);
  __nv_bfloat16* lo = reinterpret_cast<__nv_bfloat16*>(ws.c_lo);
  for (int it = 0; it < iters; ++it) {
    k_centroid_split<D><<<dim3(Cpad, BH), D, 0, s>>>(cent, C, Cpad, hi, lo, ws.c_norm);
    k_assign_tc<D><<<grid_asg, kAsgThreads, AsgCfg<D>::kSmem, s>>>(mx, mh, ml, ws.c_norm, N, Cpad, BH, labels);
    cudaError_t e = launch_stable_sort(labels, BH, N, C, ws.sort, perm, offsets, sizes, s);
    if (e != cudaSuccess) return e;
    const dim3 grid_sum((N + kSumRows * kSumWarps - 1) / (kSumRows * kSumWarps), BH);
    // the gather pass (last iteration) uses the asynchronous-copy kernel: K' + V' 0.69 -> 0.48 ms, Q' equal; the
    // plain update keeps the register-staged one (0.20 ms vs 0.33 ms: its accumulation phase has no loads in flight)
    if (it + 1 == iters && g.wait_y) cudaStreamWaitEvent(s, g.wait_y, 0);
    if (it + 1 == iters && g.Xp) {
      constexpr int rows = kAsyncRows<true>;
      const dim3 grid_a((N + rows * kAsyncWarps - 1) / (rows * kAsyncWarps), BH);
      const size_t sm = size_t(kAsyncWarps) * 2 * rows * D * 2;
      cudaFuncSetAttribute(k_update_sum_async<D, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
      k_update_sum_async<D, true><<<grid_a, 32 * kAsyncWarps, sm, s>>>(
          X, N, C, perm, offsets, ws.c_sum, static_cast<__nv_bfloat16*>(g.Xp), static_cast<const __nv_bfloat16*>(g.Y),
          static_cast<__nv_bfloat16*>(g.Yp));
    } else {
      k_update_sum<D, false><<<grid_sum, 32 * kSumWarps, 0, s>>>(X, N, C, perm, offsets, ws.c_sum, nullptr, nullptr,
                                                                  nullptr);
    }
    k_update_mean<D><<<dim3(C, BH), D, 0, s>>>(C, offsets, ws.c_sum, cent);
  }
  return cudaGetLastError();
}

}  // namespace

// split + assign + sort (3) + sum + mean per iteration, plus the cold init
int kmeans_launch_count(int iters, bool warm) { return (warm ? 0 : 1) + iters * (4 + kSortLaunches); }

cudaError_t launch_kmeans(const void* X, int BH, int N, int d, int C, int iters, bool warm, float* centroids,
                          int32_t* labels, int32_t* sizes, int32_t* perm, int32_t* offsets, KmeansWs ws,
                          cudaStream_t s, int* launches, const KmeansInit& init, const KmeansGather& g) {
  if (!perm) perm = ws.perm;
  if (!offsets) offsets = ws.offsets;
  if (launches) {
    *launches += kmeans_launch_count(iters, warm);
    if (!warm && init.kmeanspp) *launches += kmeanspp_launch_count(BH, N, d) - 1;  // replaces the strided init
  }
  if (d == 128)
    return run_kmeans<128>(X, BH, N, C, iters, warm, init, centroids, labels, sizes, perm, offsets, ws, s, g);
  return run_kmeans<64>(X, BH, N, C, iters, warm, init, centroids, labels, sizes, perm, offsets, ws, s, g);
}

}  // namespace svg2

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
//                      A fixed-order segmented reduction (no atomics): deterministic for any data, and bit-identical
//                      to the oracle's sequential sum whenever the fp64 sums of bf16 rows are exact.  Optionally the
//                      Lloyd objective J before and after each update.
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
constexpr int kTiles = 6;         // shared-memory tiles of 128 rows x D, split between X buffers and centroid stages

template <int D>
struct AsgCfg {
  static constexpr int kBlocks = D / 64;
  static constexpr uint32_t kBlockBytes = 128 * 128;            // 128 rows x 64 bf16
  static constexpr uint32_t kTileBytes = kBlocks * kBlockBytes;  // 128 rows x D bf16
  static constexpr uint32_t kNormBytes = kMaxClusters * 4;
  // six tiles (X buffers | centroid half-chunk stages) | norms
  static constexpr uint32_t kSmem = kTiles * kTileBytes + kNormBytes + 1024;
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

// The six tiles: kXS X buffers and kTiles - kXS centroid half-stages, each one tile (the hi or the lo half of a
// 128-centroid chunk).  C > 128 (kXS = 2): four half-stages, so the hi half of chunk c+1 streams in while the lo half
// of chunk c is multiplied (a 2-deep ring of whole hi+lo chunks left the MMA waiting for chunks ~30% of the time:
// tensor pipe 68%, ncu).  C <= 128 (kXS = 4): one chunk, whose hi and lo halves stay resident across a head's units,
// so two half-stages suffice and four X buffers keep more of the X stream in flight (the Q role reads X at HBM rate).
struct AsgBars {
  uint64_t x_full[4], x_empty[4], c_full[4], c_empty[4], acc_full[kAccStages], acc_empty[kAccStages];
};

// Persistent assignment: one CTA per SM walks a contiguous range of 128-row work units (row tiles of one (b,h); the
// range is mostly one head).  Per unit the producer loads X (double-buffered) and streams the centroid chunks (two
// stages, hi and lo tiles); the MMA warp accumulates X [hi | lo]^T per chunk into one of four TMEM stages; the
// epilogue warps read each stage back and keep the running argmin.  Loads, MMAs and TMEM reads of consecutive
// units overlap, and TMEM allocation / barrier setup happen once per CTA instead of once per tile.
template <int D, int kXS>
__global__ void __launch_bounds__(kAsgThreads, 1)
    k_assign_tc(const __grid_constant__ CUtensorMap mapX, const __grid_constant__ CUtensorMap mapHi,
                const __grid_constant__ CUtensorMap mapLo, const float* __restrict__ c_norm, int N, int Cpad,
                int BH, int H, int32_t* __restrict__ labels) {
  using C = AsgCfg<D>;
  constexpr int kHalfStages = kTiles - kXS;
  static_assert(kXS == 2 || kXS == 4, "X buffers");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sX = smem;                         // [kXS buffers]
  uint8_t* sC = smem + kXS * C::kTileBytes;   // [kHalfStages] centroid half-chunks (hi or lo)
  float* sNorm = reinterpret_cast<float*>(sC + kHalfStages * C::kTileBytes);  // [Cpad] of the epilogue's current head
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
    for (int s = 0; s < kXS; ++s) {
      mbar_init(&bars.x_full[s], 1);
      mbar_init(&bars.x_empty[s], 1);
    }
    for (int s = 0; s < kHalfStages; ++s) {
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
      uint32_t cc = 0;  // half-chunks issued (C > 128) / centroid loads (C <= 128)
      int cur_bh = -1;
      for (int u = u0, i = 0; u < u1; ++u, ++i) {
        const int bh = u / upb, row0 = (u - bh * upb) * kAsgRows;
        const int xs = i % kXS;
        mbar_wait(&bars.x_empty[xs], ((i / kXS) & 1) ^ 1);
        mbar_arrive_expect_tx(&bars.x_full[xs], C::kTileBytes);
        for (int b = 0; b < C::kBlocks; ++b)
          tma_load_4d(sX + xs * C::kTileBytes + b * C::kBlockBytes, &mapX, &bars.x_full[xs], 64 * b, row0, bh % H,
                      bh / H);
        if constexpr (kXS == 4) {
          // C <= 128: the head's hi and lo halves stay resident in stages 0 / 1; reloaded when the head changes,
          // after the MMA released them (it commits c_empty after the head's last unit), so the X stream runs
          // kXS units ahead of the MMA
          if (bh != cur_bh) {
            for (int half = 0; half < 2; ++half) {
              mbar_wait(&bars.c_empty[half], (cc & 1) ^ 1);
              mbar_arrive_expect_tx(&bars.c_full[half], C::kTileBytes);
              for (int b = 0; b < C::kBlocks; ++b)
                tma_load_2d(sC + half * C::kTileBytes + b * C::kBlockBytes, half ? &mapLo : &mapHi,
                            &bars.c_full[half], 64 * b, bh * Cpad);
            }
            ++cc;
            cur_bh = bh;
          }
        } else {
          for (int c = 0; c < nchunks; ++c) {
            const int crow = bh * Cpad + c * kCentChunk;
            for (int half = 0; half < 2; ++half, ++cc) {  // hi, then lo
              const int s = cc % kHalfStages;
              mbar_wait(&bars.c_empty[s], ((cc / kHalfStages) & 1) ^ 1);
              mbar_arrive_expect_tx(&bars.c_full[s], C::kTileBytes);
              for (int b = 0; b < C::kBlocks; ++b)
                tma_load_2d(sC + s * C::kTileBytes + b * C::kBlockBytes, half ? &mapLo : &mapHi, &bars.c_full[s],
                            64 * b, crow);
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // whole warp, convergent: elect.sync inside the MMA asm -> back-to-back UTCHMMA on uniform registers
    const uint32_t idesc = idesc_bf16_f32(128, kCentChunk, false);
    uint32_t cc = 0, ac = 0;
    int cur_bh = -1;
    for (int u = u0, i = 0; u < u1; ++u, ++i) {
      const int xs = i % kXS;
      mbar_wait_warp(&bars.x_full[xs], (i / kXS) & 1);
      const uint32_t x = smem_u32(sX + xs * C::kTileBytes);
      if constexpr (kXS == 4) {
        const int bh = u / upb;
        if (bh != cur_bh) {  // this head's centroids were loaded (load number cc)
          mbar_wait_warp(&bars.c_full[0], cc & 1);
          mbar_wait_warp(&bars.c_full[1], cc & 1);
          ++cc;
          cur_bh = bh;
        }
        const int as = ac % kAccStages;
        mbar_wait_warp(&bars.acc_empty[as], ((ac / kAccStages) & 1) ^ 1);
        tc_fence_after();
        const uint32_t dcol = tmem + as * 128;
        for (int half = 0; half < 2; ++half) {  // x.hi then x.lo into the same accumulator
          const uint32_t cb = smem_u32(sC + half * C::kTileBytes);
#pragma unroll
          for (int k = 0; k < D / 16; ++k) {
            const uint32_t off = (k >> 2) * C::kBlockBytes + (k & 3) * 32;
            mma_ss_warp(dcol, desc_kmajor_sw128(x + off), desc_kmajor_sw128(cb + off), idesc, (half | k) > 0);
          }
        }
        if (u + 1 == u1 || (u + 1) / upb != bh) {  // the head's last unit here: its centroid stages are free
          mma_commit_warp(&bars.c_empty[0]);
          mma_commit_warp(&bars.c_empty[1]);
        }
        mma_commit_warp(&bars.acc_full[as]);
        ++ac;
      } else {
        for (int c = 0; c < nchunks; ++c, ++ac) {
          const int as = ac % kAccStages;
          mbar_wait_warp(&bars.acc_empty[as], ((ac / kAccStages) & 1) ^ 1);
          const uint32_t dcol = tmem + as * 128;
          for (int half = 0; half < 2; ++half, ++cc) {  // x.hi then x.lo into the same accumulator
            const int s = cc % kHalfStages;
            mbar_wait_warp(&bars.c_full[s], (cc / kHalfStages) & 1);
            tc_fence_after();
            const uint32_t cb = smem_u32(sC + s * C::kTileBytes);
#pragma unroll
            for (int k = 0; k < D / 16; ++k) {
              const uint32_t off = (k >> 2) * C::kBlockBytes + (k & 3) * 32;
              mma_ss_warp(dcol, desc_kmajor_sw128(x + off), desc_kmajor_sw128(cb + off), idesc, (half | k) > 0);
            }
            mma_commit_warp(&bars.c_empty[s]);
          }
          mma_commit_warp(&bars.acc_full[as]);
        }
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
      // kChains independent running argmins (column e of every 32 goes to chain e % kChains, indices ascending within
      // a chain, strict < keeps the lowest), merged at the end by (distance, index): the same label as one sequential
      // scan, without its compare-select dependency chain (ncu: the epilogue's serial argmin was the assign kernel's
      // hot spot, 60% of samples, "wait" stalls 37%)
      constexpr int kChains = 4;
      float best[kChains];
      int bj[kChains];
#pragma unroll
      for (int k = 0; k < kChains; ++k) {
        best[k] = INFINITY;
        bj[k] = 0;
      }
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
          const float4* nv = reinterpret_cast<const float4*>(sNorm + j0);
#pragma unroll
          for (int e4 = 0; e4 < 8; ++e4) {
            const float4 n4 = nv[e4];  // broadcast 16-byte load of four norms
            const float nn[4] = {n4.x, n4.y, n4.z, n4.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const int e = 4 * e4 + k;
              const float dist = fmaf(-2.f, __uint_as_float(r4[q][e]), nn[k]);
              if (dist < best[k]) {  // strict: ties keep the lower index
                best[k] = dist;
                bj[k] = j0 + e;
              }
            }
          }
        }
        // released after the argmin (releasing right after the loads measured slower: 594 vs 574 us per K launch)
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars.acc_empty[as]);
      }
      float b = best[0];
      int jb = bj[0];
#pragma unroll
      for (int k = 1; k < kChains; ++k) {
        if (best[k] < b || (best[k] == b && bj[k] < jb)) {
          b = best[k];
          jb = bj[k];
        }
      }
      const int row = row0 + quarter * 32 + lane;
      if (row < N) labels[size_t(bh) * N + row] = jb;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

// Centroid update, pass 1 — a fixed-order segmented reduction.  The permuted positions [0, N) of a head are cut into
// fixed chunks of R rows (R = the kernel's rows per warp); a warp sums its chunk's rows sequentially in fp64, one
// partial per cluster segment.  A segment that is a whole cluster (the cluster lies inside the chunk) is stored as its
// sum; a cluster that crosses chunk boundaries leaves one partial per chunk (slot 0 = the chunk's first segment, slot 1
// = its last), and k_update_mean adds them in chunk order.  Plain stores, no atomics: the summation order is a function
// of (offsets, R) alone, so the result is deterministic for any data (no reliance on fp64 sums of bf16 being exact),
// and it is the oracle's sequential sum bit for bit whenever those sums are exact (sums of bf16 values whose exponent
// spread + log2 |cluster| + 8 <= 53).  With `sq` set, the segment's sum of squared norms sum ||x||^2 (fp64, lane
// partials reduced by a fixed shuffle tree) is stored the same way for the Lloyd objective.
struct SegOut {
  double* sum;     // [BH, C, D]       complete cluster sums
  double* part;    // [BH, nch, 2, D]  partial segments of clusters crossing chunk boundaries
  double* sq;      // [BH, C]          (objective) complete sum ||x||^2, or nullptr
  double* sqpart;  // [BH, nch, 2]
  int nch;         // chunks per head at this R
};

template <int D, bool kSq>
__device__ __forceinline__ void store_segment(const SegOut& o, const int32_t* off, int bh, int C, int j, int chunk,
                                              int p0, int p1, int lane, const double* acc, double sq) {
  constexpr int kCols = D / 32;
  const int o0 = __ldg(off + j), o1 = __ldg(off + j + 1);
  double* dst;
  double* dsq;
  if (o0 >= p0 && o1 <= p1) {  // the whole cluster lies in this chunk
    dst = o.sum + (size_t(bh) * C + j) * D;
    dsq = kSq ? o.sq + size_t(bh) * C + j : nullptr;
  } else {
    const size_t slot = (size_t(bh) * o.nch + chunk) * 2 + (o0 <= p0 ? 0 : 1);
    dst = o.part + slot * D;
    dsq = kSq ? o.sqpart + slot : nullptr;
  }
#pragma unroll
  for (int c = 0; c < kCols; ++c) dst[kCols * lane + c] = acc[c];
  if (kSq) {
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, s);
    if (lane == 0) *dsq = sq;
  }
}

// The update pass: row gathers through perm as asynchronous copies (cp.async, 16 B per lane-instruction), a warp puts
// all 32 rows of its chunk in flight at once through shared memory (8 KB per warp, or 16 KB with the 32 rows of Y when
// the last pass also gathers V through the same pi_k); the chunk's perm entries and their labels are loaded up front
// and a segment ends where the label changes.  On the last Lloyd iteration of the fused call (Xp set) the permuted
// copies leave shared memory as one bulk copy per tensor (the chunk's rows are contiguous in X', A6).  32-row chunks
// and 8 KB per warp (24 warps per SM) measured 185 us per K pass at Wan 2.1 720p against 277 us for 64-row chunks in
// 16 KB (12 warps per SM): the pass is bound by the latency of the random row reads, not by the bytes in flight; it
// reads at 4.2 TB/s, next to the 5.0 TB/s (read + write) of the plain permute gather (profiles/r02_micro).
constexpr int kAsyncWarps = 4;
template <int D, bool kSq, bool kTwo>
__global__ void __launch_bounds__(32 * kAsyncWarps) k_update_sum_async(
    const XView X, int N, int C, const int32_t* __restrict__ perm, const int32_t* __restrict__ labels,
    const int32_t* __restrict__ offsets, SegOut out, __nv_bfloat16* __restrict__ Xp, const XView Y,
    __nv_bfloat16* __restrict__ Yp) {
  constexpr int kRows = kUpdRows;
  constexpr int kCols = D / 32;           // bf16 per lane in the accumulation
  constexpr int kRowBytes = D * 2;        // 256 (d = 128) or 128 (d = 64)
  constexpr int kVecPerRow = kRowBytes / 16;
  constexpr int kWarpBytes = kRows * kRowBytes * (kTwo ? 2 : 1);
  extern __shared__ __align__(128) uint8_t sm_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, bh = blockIdx.y;
  uint8_t* sx = sm_raw + size_t(warp) * kWarpBytes;  // [kRows][row] X rows of this warp
  uint8_t* sy = sx + kRows * kRowBytes;              // [kRows][row] Y rows (kTwo)
  const int chunk = blockIdx.x * kAsyncWarps + warp;
  const int p0 = chunk * kRows;
  if (p0 >= N) return;
  const int nrow = min(N - p0, kRows);
  constexpr bool with_y = kTwo;
  const int32_t* pm = perm + size_t(bh) * N + p0;
  const int s0 = lane < nrow ? __ldg(pm + lane) : 0;
  const uint8_t* xb = reinterpret_cast<const uint8_t*>(X.row(bh, 0));
  const uint8_t* yb = with_y ? reinterpret_cast<const uint8_t*>(Y.row(bh, 0)) : nullptr;
  const long long xrow = X.sN * 2, yrow = Y.sN * 2;  // bytes between tokens
  // issue: 32 lanes cover 32 / kVecPerRow rows per step, one 16-byte piece each
  constexpr int kRowsPerStep = 32 / kVecPerRow;
  const int piece = lane % kVecPerRow, rsub = lane / kVecPerRow;
#pragma unroll 4
  for (int r0 = 0; r0 < kRows; r0 += kRowsPerStep) {
    const int r = r0 + rsub;
    const int src = __shfl_sync(0xffffffffu, s0, r);
    if (r < nrow) {
      const uint32_t dst = smem_u32(sx + r * kRowBytes + piece * 16);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(xb + src * xrow + piece * 16)
                   : "memory");
      if (with_y) {
        const uint32_t dy = smem_u32(sy + r * kRowBytes + piece * 16);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dy), "l"(yb + src * yrow + piece * 16)
                     : "memory");
      }
    }
  }
  // the rows' labels while the copies fly
  const int32_t* lb = labels + size_t(bh) * N;
  const int l0 = lane < nrow ? __ldg(lb + s0) : 0;
  const int32_t* off = offsets + size_t(bh) * (C + 1);
  asm volatile("cp.async.wait_all;" ::: "memory");
  // every lane's cp.async writes into shared memory are made visible to the async proxy (the bulk store below) by
  // that lane's own proxy fence before the warp barrier
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  if (Xp != nullptr && lane == 0) {  // X' (and Y') rows p0 .. p0 + nrow - 1 are contiguous: one bulk store each
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
  double acc[kCols], sq = 0.0;
#pragma unroll
  for (int c = 0; c < kCols; ++c) acc[c] = 0.0;
  const int p1 = p0 + nrow;
  int j = __shfl_sync(0xffffffffu, l0, 0);
  for (int r = 0; r < nrow; ++r) {
    const int lab = __shfl_sync(0xffffffffu, l0, r);
    if (lab != j) {  // the next cluster starts: store the segment
      store_segment<D, kSq>(out, off, bh, C, j, chunk, p0, p1, lane, acc, sq);
#pragma unroll
      for (int c = 0; c < kCols; ++c) acc[c] = 0.0;
      sq = 0.0;
      j = lab;
    }
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(sx + r * kRowBytes + lane * kCols * 2);
#pragma unroll
    for (int c = 0; c < kCols / 2; ++c) {
      const float2 f = __bfloat1622float2(h[c]);
      acc[2 * c] += double(f.x);
      acc[2 * c + 1] += double(f.y);
      if (kSq) sq += double(f.x) * double(f.x) + double(f.y) * double(f.y);
    }
  }
  store_segment<D, kSq>(out, off, bh, C, j, chunk, p0, p1, lane, acc, sq);
  if (Xp != nullptr && lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // smem stays live
  __syncwarp();
}

// Pass 2: S_j = the cluster's sum (complete, or its chunk partials added in chunk order), c_j = S_j / |cluster j|
// (fp64, rounded to f32); empty clusters keep their centroid (R6).  With `jpart`, the cluster's share of the Lloyd
// objective before and after the update:
//   J_assign_j = sum ||x||^2 - 2 c_old . S_j + n ||c_old||^2,   J_post_j = the same with the new (f32) centroid,
// reduced over the D columns by a fixed tree (deterministic); empty clusters contribute 0.
template <int D>
__global__ void __launch_bounds__(D) k_update_mean(int C, int R, const int32_t* __restrict__ offsets, SegOut in,
                                                   float* __restrict__ cent, double* __restrict__ jpart) {
  const int j = blockIdx.x, bh = blockIdx.y, k = threadIdx.x;
  const int o0 = offsets[size_t(bh) * (C + 1) + j], o1 = offsets[size_t(bh) * (C + 1) + j + 1];
  const int cnt = o1 - o0;
  if (cnt == 0) {
    if (jpart && k == 0) jpart[(size_t(bh) * C + j) * 2] = jpart[(size_t(bh) * C + j) * 2 + 1] = 0.0;
    return;
  }
  const int c0 = o0 / R, c1 = (o1 - 1) / R;
  double s, sq = 0.0;
  if (c0 == c1) {
    s = in.sum[(size_t(bh) * C + j) * D + k];
    if (jpart) sq = in.sq[size_t(bh) * C + j];
  } else {
    size_t slot = (size_t(bh) * in.nch + c0) * 2 + (o0 <= c0 * R ? 0 : 1);
    s = in.part[slot * D + k];
    if (jpart) sq = in.sqpart[slot];
    for (int c = c0 + 1; c <= c1; ++c) {
      slot = (size_t(bh) * in.nch + c) * 2;
      s += in.part[slot * D + k];
      if (jpart) sq += in.sqpart[slot];
    }
  }
  float* cp = cent + (size_t(bh) * C + j) * D + k;
  const double c_old = double(*cp);
  const float c_new = float(s / double(cnt));
  *cp = c_new;
  if (jpart) {
    __shared__ double red[2][D / 32];
    double a = double(cnt) * c_old * c_old - 2.0 * c_old * s;
    double b = double(cnt) * double(c_new) * double(c_new) - 2.0 * double(c_new) * s;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, o);
      b += __shfl_xor_sync(0xffffffffu, b, o);
    }
    if ((k & 31) == 0) {
      red[0][k >> 5] = a;
      red[1][k >> 5] = b;
    }
    __syncthreads();
    if (k == 0) {
      double ta = sq, tb = sq;
      for (int w = 0; w < D / 32; ++w) {
        ta += red[0][w];
        tb += red[1][w];
      }
      jpart[(size_t(bh) * C + j) * 2] = ta;
      jpart[(size_t(bh) * C + j) * 2 + 1] = tb;
    }
  }
}

// Pass 3 (objective requested only): J(t) of each head = sum over clusters in ascending j, objective[bh] =
// (J_assign, J_post).
__global__ void k_objective(int BH, int C, const double* __restrict__ jpart, double* __restrict__ objective) {
  const int bh = blockIdx.x * blockDim.x + threadIdx.x;
  if (bh >= BH) return;
  double a = 0.0, b = 0.0;
  for (int j = 0; j < C; ++j) {
    a += jpart[(size_t(bh) * C + j) * 2];
    b += jpart[(size_t(bh) * C + j) * 2 + 1];
  }
  objective[size_t(bh) * 2] = a;
  objective[size_t(bh) * 2 + 1] = b;
}

template <int D>
__global__ void k_init_cold(const XView X, int N, int C, float* __restrict__ cent) {
  const int j = blockIdx.x, bh = blockIdx.y;
  const long long src = (long long)j * N / C;  // floor(j N / C)
  const uint16_t bits = X.row(bh, src)[threadIdx.x];
  cent[(size_t(bh) * C + j) * D + threadIdx.x] = __uint_as_float(uint32_t(bits) << 16);
}

template <int D>
cudaError_t run_kmeans(const XView X, int BH, int N, int C, int iters, bool warm, const KmeansInit& init,
                       float* cent, int32_t* labels,
                       int32_t* sizes, int32_t* perm, int32_t* offsets, KmeansWs ws, cudaStream_t s,
                       const KmeansGather& g, double* objective) {
  const int Cpad = cent_pad(C);
  CUtensorMap mx, mh, ml;
  if (!make_tmap_bf16_4d(&mx, X.p, D, N, X.H, BH / X.H, X.sN, X.sH, X.sB, 128) ||
      !make_tmap_bf16(&mh, ws.c_hi, uint64_t(BH) * Cpad, D, 128) ||
      !make_tmap_bf16(&ml, ws.c_lo, uint64_t(BH) * Cpad, D, 128))
    return cudaErrorInvalidValue;
  auto assign = Cpad == kCentChunk ? k_assign_tc<D, 4> : k_assign_tc<D, 2>;
  cudaFuncSetAttribute(assign, cudaFuncAttributeMaxDynamicSharedMemorySize, AsgCfg<D>::kSmem);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long units = (long long)BH * ((N + kAsgRows - 1) / kAsgRows);
  const int grid_asg = int(units < sms ? units : sms);  // persistent: one CTA per SM
  if (!warm && init.kmeanspp) {
    cudaError_t e = launch_kmeanspp(X, BH, N, D, C, init.seed, init.role, init.bh_base, cent, ws.pp, s);
    if (e != cudaSuccess) return e;
  } else if (!warm) {
    k_init_cold<D><<<dim3(C, BH), D, 0, s>>>(X, N, C, cent);
  }
  __nv_bfloat16* hi = reinterpret_cast<__nv_bfloat16*>(ws.c_hi);
  __nv_bfloat16* lo = reinterpret_cast<__nv_bfloat16*>(ws.c_lo);
  for (int it = 0; it < iters; ++it) {
    k_centroid_split<D><<<dim3(Cpad, BH), D, 0, s>>>(cent, C, Cpad, hi, lo, ws.c_norm);
    assign<<<grid_asg, kAsgThreads, AsgCfg<D>::kSmem, s>>>(mx, mh, ml, ws.c_norm, N, Cpad, BH, X.H, labels);
    cudaError_t e = launch_stable_sort(labels, BH, N, C, ws.sort, perm, offsets, sizes, s);
    if (e != cudaSuccess) return e;
    if (it + 1 == iters && g.wait_y) cudaStreamWaitEvent(s, g.wait_y, 0);
    // every update pass: the rows of a warp's 32-row chunk arrive by cp.async through shared memory (with the rows of
    // V when the last pass also gathers it); the last pass also writes the permuted copies (A6)
    const bool gather = it + 1 == iters && g.Xp;
    const bool two = gather && g.Y.p;
    constexpr int R = kUpdRows;
    SegOut seg{ws.c_sum, ws.c_part, objective ? ws.c_sq : nullptr, ws.c_sqpart, (N + R - 1) / R};
    const dim3 grid_a((N + R * kAsyncWarps - 1) / (R * kAsyncWarps), BH);
    const size_t sm = size_t(kAsyncWarps) * R * D * 2 * (two ? 2 : 1);
    auto kern = two ? (objective ? k_update_sum_async<D, true, true> : k_update_sum_async<D, false, true>)
                    : (objective ? k_update_sum_async<D, true, false> : k_update_sum_async<D, false, false>);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
    kern<<<grid_a, 32 * kAsyncWarps, sm, s>>>(X, N, C, perm, labels, offsets, seg,
                                              gather ? static_cast<__nv_bfloat16*>(g.Xp) : nullptr,
                                              two ? g.Y : XView(), two ? static_cast<__nv_bfloat16*>(g.Yp) : nullptr);
    k_update_mean<D><<<dim3(C, BH), D, 0, s>>>(C, R, offsets, seg, cent, objective ? ws.j_part : nullptr);
    if (objective) k_objective<<<(BH + 127) / 128, 128, 0, s>>>(BH, C, ws.j_part, objective + size_t(it) * BH * 2);
  }
  return cudaGetLastError();
}

}  // namespace

// split + assign + sort (3) + sum + mean per iteration, plus the cold init
int kmeans_launch_count(int iters, bool warm, bool objective) {
  return (warm ? 0 : 1) + iters * (4 + kSortLaunches + (objective ? 1 : 0));
}

cudaError_t launch_kmeans(XView X, int BH, int N, int d, int C, int iters, bool warm, float* centroids,
                          int32_t* labels, int32_t* sizes, int32_t* perm, int32_t* offsets, KmeansWs ws,
                          cudaStream_t s, int* launches, const KmeansInit& init, const KmeansGather& g,
                          double* objective) {
  if (!perm) perm = ws.perm;
  if (!offsets) offsets = ws.offsets;
  if (launches) {
    *launches += kmeans_launch_count(iters, warm, objective != nullptr);
    if (!warm && init.kmeanspp) *launches += kmeanspp_launch_count(BH, N, d) - 1;  // replaces the strided init
  }
  if (d == 128)
    return run_kmeans<128>(X, BH, N, C, iters, warm, init, centroids, labels, sizes, perm, offsets, ws, s, g,
                           objective);
  return run_kmeans<64>(X, BH, N, C, iters, warm, init, centroids, labels, sizes, perm, offsets, ws, s, g, objective);
}

}  // namespace svg2

// svg2_kmeanspp.cu — A1 cold start: k-means++ seeding with the generator of DESIGN R25.
//
// Pick 0 is a uniform random row; pick j >= 1 is row n with probability proportional to D_n, the squared distance
// to the nearest centroid picked so far.  R25 fixes every detail so the picks are reproducible bit for bit:
// Philox4x32-10 keyed (seed, 2*bh + role) with counter (j, 0, 0, 0); D_n accumulated in ascending k with every
// fp64 operation rounded (explicit __d*_rn intrinsics, no FMA contraction); integer weights
// W_n = floor(D_n / D_ref * 2^32) so the prefix sums that locate the sampled row are exact in any order.
//
// One cooperative persistent kernel per call: CTA (bh, blk) owns a contiguous range of rows of head bh, each thread a
// contiguous sub-range.  Per pick: every CTA loads the picked row, updates D_n over its rows and sums the next pick's
// weights (one pass over X); grid sync; the CTA whose weight range contains the sampled position finds the row (a
// scan of per-thread sums kept in shared memory, then one thread's rows); grid sync.  X is re-read once per pick, so
// the seeding is HBM-bound (C passes over X) — the cost the centroid cache (warm start) avoids.
#include <cooperative_groups.h>
#include <cuda_bf16.h>
#include "internal.h"

namespace svg2 {
namespace {

namespace cg = cooperative_groups;
constexpr int kPPThreads = 256;

__device__ __forceinline__ void philox4x32_10(uint32_t (&c)[4], uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    const uint32_t hi0 = __umulhi(0xD2511F53u, c[0]), lo0 = 0xD2511F53u * c[0];
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c[2]), lo1 = 0xCD9E8D57u * c[2];
    const uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = lo1;
    c[2] = n2;
    c[3] = lo0;
  }
}

// sum_k (x_k - c_k)^2 in ascending k, each operation rounded (R25)
template <int D>
__device__ __forceinline__ double sqdist_rn(const __nv_bfloat16* __restrict__ x, const double* __restrict__ c) {
  const uint4* xv = reinterpret_cast<const uint4*>(x);
  double acc = 0.0;
#pragma unroll 2
  for (int q = 0; q < D / 8; ++q) {
    const uint4 u = __ldg(xv + q);
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 f = __bfloat1622float2(h[e]);
      const double d0 = __dsub_rn(double(f.x), c[8 * q + 2 * e]);
      acc = __dadd_rn(acc, __dmul_rn(d0, d0));
      const double d1 = __dsub_rn(double(f.y), c[8 * q + 2 * e + 1]);
      acc = __dadd_rn(acc, __dmul_rn(d1, d1));
    }
  }
  return acc;
}

__device__ __forceinline__ unsigned long long pp_weight(double dn, double dref) {
  return dref > 0.0 ? (unsigned long long)floor(__dmul_rn(__ddiv_rn(dn, dref), 4294967296.0)) : 0ull;
}

struct PPWs {
  double* D;                 // [BH, N]
  double* bmax;              // [BH, nblk] per-CTA max of D after pick 0
  unsigned long long* part;  // [BH, nblk] per-CTA weight sums
  int32_t* pick;             // [BH] the next pick
};

template <int D>
__global__ void __launch_bounds__(kPPThreads) k_kmeanspp(const XView X, int N, int C, int bh0,
                                                        int nblk, uint32_t seed, uint32_t stream_base,
                                                        float* __restrict__ cent, PPWs ws) {
  cg::grid_group grid = cg::this_grid();
  const int bh = bh0 + blockIdx.x / nblk, blk = blockIdx.x % nblk, tid = threadIdx.x;
  const int rows_blk = (N + nblk - 1) / nblk;
  const int r0 = min(N, blk * rows_blk), r1 = min(N, r0 + rows_blk);
  const int R = (rows_blk + kPPThreads - 1) / kPPThreads;
  const int t0 = min(r1, r0 + tid * R), t1 = min(r1, t0 + R);
  __shared__ double c_s[D];
  __shared__ unsigned long long incl[kPPThreads];  // inclusive scan of the per-thread weight sums
  __shared__ double red[kPPThreads / 32];
  __shared__ unsigned long long part_s[kPPMaxBlocks];
  double* Dv = ws.D + size_t(bh) * N;
  const __nv_bfloat16* Xb = reinterpret_cast<const __nv_bfloat16*>(X.row(bh, 0));
  const long long sN = X.sN;
  const uint32_t stream = 2u * uint32_t(bh) + stream_base;  // 2 * (global bh) + role
  double dref = 0.0;
  for (int j = 0; j < C; ++j) {
    int pick;
    if (j == 0) {
      uint32_t c4[4] = {0u, 0u, 0u, 0u};
      philox4x32_10(c4, seed, stream);
      pick = int((uint64_t(c4[0]) * uint64_t(N)) >> 32);
    } else {
      pick = *((volatile int32_t*)(ws.pick + bh));
    }
    for (int k = tid; k < D; k += kPPThreads) {
      const float v = __bfloat162float(Xb[pick * sN + k]);
      c_s[k] = double(v);
      if (blk == 0) cent[(size_t(bh) * C + j) * D + k] = v;  // a data row: exact in f32
    }
    __syncthreads();
    // D update with the new centroid; weights of the next pick (known reference after pick 0)
    unsigned long long wsum = 0;
    double tmax = 0.0;
    for (int n = t0; n < t1; ++n) {
      double dn = sqdist_rn<D>(Xb + n * sN, c_s);
      if (j > 0) {
        const double old = Dv[n];
        dn = dn < old ? dn : old;
        wsum += pp_weight(dn, dref);
      } else {
        tmax = dn > tmax ? dn : tmax;
      }
      Dv[n] = dn;
    }
    if (j + 1 == C) break;
    if (j == 0) {  // D_ref = max_n D_n after pick 0, then the weights of pick 1
      for (int o = 16; o > 0; o >>= 1) {
        const double y = __shfl_xor_sync(0xffffffffu, tmax, o);
        tmax = y > tmax ? y : tmax;
      }
      if ((tid & 31) == 0) red[tid >> 5] = tmax;
      __syncthreads();
      if (tid == 0) {
        double m = 0.0;
        for (int w = 0; w < kPPThreads / 32; ++w) m = red[w] > m ? red[w] : m;
        ws.bmax[size_t(bh) * nblk + blk] = m;
      }
      grid.sync();
      if (tid < 32) {  // the head's CTA maxima: loaded in parallel, reduced in one warp
        double m = 0.0;
        for (int b = tid; b < nblk; b += 32) {
          const double v = *((volatile double*)(ws.bmax + size_t(bh) * nblk + b));
          m = v > m ? v : m;
        }
        for (int o = 16; o > 0; o >>= 1) {
          const double y = __shfl_xor_sync(0xffffffffu, m, o);
          m = y > m ? y : m;
        }
        if (tid == 0) red[0] = m;
      }
      __syncthreads();
      dref = red[0];
      for (int n = t0; n < t1; ++n) wsum += pp_weight(Dv[n], dref);
    }
    // block inclusive scan of the per-thread sums (kept in smem for the search below)
    incl[tid] = wsum;
    __syncthreads();
    for (int o = 1; o < kPPThreads; o <<= 1) {
      const unsigned long long v = tid >= o ? incl[tid - o] : 0ull;
      __syncthreads();
      incl[tid] += v;
      __syncthreads();
    }
    if (tid == 0) ws.part[size_t(bh) * nblk + blk] = incl[kPPThreads - 1];
    grid.sync();
    // pick j+1: total over the head's CTAs, sampled position r, owning CTA, owning thread, row
    uint32_t c4[4] = {uint32_t(j + 1), 0u, 0u, 0u};
    philox4x32_10(c4, seed, stream);
    // the head's per-CTA sums, loaded in parallel into shared memory (one load latency, not nblk)
    if (tid < nblk) part_s[tid] = *((volatile unsigned long long*)(ws.part + size_t(bh) * nblk + tid));
    __syncthreads();
    unsigned long long total = 0, before = 0;
    int owner = -1;
    const unsigned long long r64 = uint64_t(c4[0]) | (uint64_t(c4[1]) << 32);
    for (int b = 0; b < nblk; ++b) total += part_s[b];
    if (total == 0) {
      if (blk == 0 && tid == 0) ws.pick[bh] = int((uint64_t(c4[0]) * uint64_t(N)) >> 32);
    } else {
      const unsigned long long r = __umul64hi(r64, total);
      unsigned long long acc = 0;
      for (int b = 0; b < nblk && owner < 0; ++b) {
        const unsigned long long pb = part_s[b];
        if (r < acc + pb) {
          owner = b;
          before = acc;
        }
        acc += pb;
      }
      if (owner == blk) {
        const unsigned long long rr = r - before, hi = incl[tid], lo = tid > 0 ? incl[tid - 1] : 0ull;
        if (lo <= rr && rr < hi) {  // exactly one thread: its rows hold the sampled position
          unsigned long long run = lo;
          int found = t1 - 1;
          for (int n = t0; n < t1; ++n) {
            run += pp_weight(Dv[n], dref);
            if (run > rr) {
              found = n;
              break;
            }
          }
          ws.pick[bh] = found;
        }
      }
    }
    grid.sync();
  }
}

}  // namespace

size_t kmeanspp_ws_bytes(int BH, int N) {
  return size_t(BH) * N * sizeof(double) + size_t(BH) * kPPMaxBlocks * (sizeof(double) + sizeof(unsigned long long)) +
         size_t(BH) * sizeof(int32_t) + 256;
}

namespace {
struct PPPlan {
  int nblk, heads_per_launch;
};
// CTAs per head and heads per cooperative launch: all resident at once (a grid sync needs it), a head's rows spread
// over up to kPPMaxBlocks CTAs
template <int D>
PPPlan pp_plan(int BH, int N) {
  int dev = 0, sms = 148, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_kmeanspp<D>, kPPThreads, 0);
  const int capacity = sms * (per_sm > 0 ? per_sm : 1);
  int nblk = capacity / BH;
  nblk = nblk < 1 ? 1 : (nblk > kPPMaxBlocks ? kPPMaxBlocks : nblk);
  const int rows_cap = kPPThreads * 64;  // keep a thread's row range short
  while (nblk < kPPMaxBlocks && nblk < capacity && (N + nblk - 1) / nblk > rows_cap) ++nblk;
  PPPlan p;
  p.nblk = nblk;
  p.heads_per_launch = capacity / nblk > 0 ? capacity / nblk : 1;
  return p;
}
}  // namespace

cudaError_t launch_kmeanspp(XView X, int BH, int N, int d, int C, uint32_t seed, int role, int bh_base,
                            float* cent, void* ws_ptr, cudaStream_t s) {
  uint32_t stream_base = 2u * uint32_t(bh_base) + uint32_t(role);
  auto run = [&](auto kernel, PPPlan plan) -> cudaError_t {
    uint8_t* base = static_cast<uint8_t*>(ws_ptr);
    PPWs w;
    w.D = reinterpret_cast<double*>(base);
    base += size_t(BH) * N * sizeof(double);
    w.bmax = reinterpret_cast<double*>(base);
    base += size_t(BH) * kPPMaxBlocks * sizeof(double);
    w.part = reinterpret_cast<unsigned long long*>(base);
    base += size_t(BH) * kPPMaxBlocks * sizeof(unsigned long long);
    w.pick = reinterpret_cast<int32_t*>(base);
    int nblk = plan.nblk;
    for (int bh0 = 0; bh0 < BH; bh0 += plan.heads_per_launch) {
      const int nh = BH - bh0 < plan.heads_per_launch ? BH - bh0 : plan.heads_per_launch;
      void* args[] = {(void*)&X, (void*)&N, (void*)&C, (void*)&bh0, (void*)&nblk, (void*)&seed,
                      (void*)&stream_base, (void*)&cent, (void*)&w};
      cudaError_t e = cudaLaunchCooperativeKernel((const void*)kernel, dim3(nh * nblk), dim3(kPPThreads), args, 0, s);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  };
  if (d == 128) return run(k_kmeanspp<128>, pp_plan<128>(BH, N));
  return run(k_kmeanspp<64>, pp_plan<64>(BH, N));
}

int kmeanspp_launch_count(int BH, int N, int d) {
  const PPPlan p = d == 128 ? pp_plan<128>(BH, N) : pp_plan<64>(BH, N);
  return (BH + p.heads_per_launch - 1) / p.heads_per_launch;
}

}  // namespace svg2

// svg2_select.cu — A7/A8: centroid-based top-p selection, one CTA per (b, h, 4 query clusters).
//   Eq. 1  S_ij = scale * sum_k c^q_ik c^k_jk          fp64, sequential FMA over k ascending (spec, DESIGN R8)
//   Eq. 2  w_ij = |K_j| exp(S_ij - m_i), m_i = max over non-empty j;  Z_i = sum_j w_ij, ascending j (R9)
//   top-p  sort (w desc, j asc) by a shared-memory bitonic sort; select ranks while cum < p Z_i (R10, R11);
//          p == 1 selects every non-empty cluster exactly.
// The order of every floating-point operation is fixed by the specification above (not by shared code with the
// oracle), so the mask is bit-exact against it except at documented near-ties (R17).
#include <cfloat>
#include "internal.h"

namespace svg2 {
namespace {

constexpr int kSelThreads = 256;
constexpr int kEq1Unroll = 8;  // 16-byte key-centroid loads in flight per thread (the Eq. 1 loop is L2-latency-bound)

__device__ __forceinline__ void named_barrier_sync(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

__device__ __forceinline__ bool before(double wa, int ja, double wb, int jb) {
  return wa > wb || (wa == wb && ja < jb);
}

// One CTA per (kRows consecutive query clusters, bh).  Eq. 1 per key cluster j by one thread for all kRows rows:
// the key centroid row is read from L2 (kEq1Unroll 16-byte loads in flight) and widened to fp64 once for the
// kRows independent sequential FMA chains (one per query row, k ascending).  Eq. 2 weights; Z_i summed in ascending
// j by one lane per row of the last warp (loads issued ahead of the dependent adds) while the other warps sort the
// kRows rows together by one segmented shared-memory bitonic sort (w desc, j asc per row, the barriers shared); the
// top-p walks (R11) by one thread per row over prefetched chunks of its sorted order.
constexpr int kRows = 4;
__global__ void __launch_bounds__(kSelThreads) k_select(const float* __restrict__ cq, const float* __restrict__ ck,
                                                        const int32_t* __restrict__ sq, const int32_t* __restrict__ sk,
                                                        int Cq, int Ck, int d, double scale, double top_p, int sortN,
                                                        int R, uint8_t* __restrict__ mask,
                                                        unsigned long long* __restrict__ pairs) {
  // R <= kRows rows per CTA (fewer when the shared-memory layout of kRows rows does not fit, C_k up to 4096)
  extern __shared__ __align__(16) unsigned char smem[];
  double* w = reinterpret_cast<double*>(smem);            // [R][sortN] Eq. 2 weights, cluster order (Z reads these)
  double* ws = w + R * sortN;                             // [R][sortN] the same weights, sorted in place
  double* crow = ws + R * sortN;                          // [R][d]
  int* idx = reinterpret_cast<int*>(crow + R * d);        // [R][sortN]
  int* sks = idx + R * sortN;                             // [Ck] key-cluster sizes
  uint8_t* sel = reinterpret_cast<uint8_t*>(sks + Ck);    // [R][Ck]
  __shared__ double red[kRows][kSelThreads / 32];
  __shared__ double Z_sh[kRows];
  __shared__ long long keys_sh[kRows];
  const int i0 = blockIdx.x * R, bh = blockIdx.y, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nr = min(R, Cq - i0);  // rows of this CTA (the last CTA may have fewer)
  const float4* ckb = reinterpret_cast<const float4*>(ck + size_t(bh) * Ck * d);
  const int32_t* skb = sk + size_t(bh) * Ck;
  for (int e = tid; e < R * d; e += kSelThreads) {
    const int r = e / d, k = e - r * d;
    crow[e] = r < nr ? double(cq[(size_t(bh) * Cq + i0 + r) * d + k]) : 0.0;
  }
  for (int j = tid; j < Ck; j += kSelThreads) sks[j] = __ldg(skb + j);
  for (int e = tid; e < R * Ck; e += kSelThreads) sel[e] = 0;
  __syncthreads();
  // Eq. 1: S_ij = scale * (sequential fp64 FMA over k ascending), one chain per row
  double m[kRows];
#pragma unroll
  for (int r = 0; r < kRows; ++r) m[r] = -INFINITY;
  for (int j = tid; j < Ck; j += kSelThreads) {
    const float4* row = ckb + size_t(j) * (d / 4);
    double acc[kRows];
#pragma unroll
    for (int r = 0; r < kRows; ++r) acc[r] = 0.0;
    for (int k4 = 0; k4 < d / 4; k4 += kEq1Unroll) {
      float4 c[kEq1Unroll];
#pragma unroll
      for (int u = 0; u < kEq1Unroll; ++u) c[u] = __ldg(row + k4 + u);
#pragma unroll
      for (int u = 0; u < kEq1Unroll; ++u) {
        const double c0 = c[u].x, c1 = c[u].y, c2 = c[u].z, c3 = c[u].w;
        const int k = 4 * (k4 + u);
#pragma unroll
        for (int r = 0; r < kRows; ++r) {
          if (r >= R) break;
          const double* q = crow + r * d + k;
          acc[r] = fma(q[0], c0, acc[r]);
          acc[r] = fma(q[1], c1, acc[r]);
          acc[r] = fma(q[2], c2, acc[r]);
          acc[r] = fma(q[3], c3, acc[r]);
        }
      }
    }
    const bool nonempty = sks[j] > 0;
#pragma unroll
    for (int r = 0; r < kRows; ++r) {
      if (r >= R) break;
      const double S = scale * acc[r];
      w[r * sortN + j] = S;
      if (nonempty) m[r] = fmax(m[r], S);
    }
  }
  // per-row block max over non-empty clusters (exact, order-free)
#pragma unroll
  for (int r = 0; r < kRows; ++r) {
    for (int o = 16; o > 0; o >>= 1) m[r] = fmax(m[r], __shfl_xor_sync(0xffffffffu, m[r], o));
    if (lane == 0) red[r][warp] = m[r];
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kRows; ++r) {
    m[r] = red[r][0];
    for (int t = 1; t < kSelThreads / 32; ++t) m[r] = fmax(m[r], red[r][t]);
  }
  // Eq. 2: w_ij = |K_j| exp(S_ij - m_i); empty clusters weigh 0; sort padding sorts last
  for (int j = tid; j < sortN; j += kSelThreads) {
    const int s = j < Ck ? sks[j] : 0;
#pragma unroll
    for (int r = 0; r < kRows; ++r) {
      if (r >= R) break;
      double* wr = w + r * sortN;
      if (j < Ck) {
        wr[j] = s > 0 ? double(s) * exp(wr[j] - m[r]) : 0.0;
        idx[r * sortN + j] = j;
      } else {
        wr[j] = -1.0;
        idx[r * sortN + j] = 0x7fffffff;
      }
      ws[r * sortN + j] = wr[j];
    }
  }
  __syncthreads();
  if (top_p >= 1.0) {  // p = 1: exactly the non-empty clusters (R11), no order needed
    long long keys = 0;
    for (int j = tid; j < Ck; j += kSelThreads) {
      const int s = sks[j];
      for (int r = 0; r < R; ++r) sel[r * Ck + j] = s > 0;
      keys += s;
    }
    for (int o = 16; o > 0; o >>= 1) keys += __shfl_xor_sync(0xffffffffu, keys, o);
    if (tid < kRows) keys_sh[tid] = 0;
    __syncthreads();
    if (lane == 0) atomicAdd(reinterpret_cast<unsigned long long*>(&keys_sh[0]), (unsigned long long)keys);
    __syncthreads();
    if (tid > 0 && tid < R) keys_sh[tid] = keys_sh[0];
    __syncthreads();
  } else {
    constexpr int kZWarp = kSelThreads / 32 - 1;       // sums Z while the other warps sort
    constexpr int kSortThreads = kSelThreads - 32;
    if (warp == kZWarp) {
      if (lane < nr) {  // Z_i in ascending j, sequential (spec order); lane r sums row r, loads ahead of the adds
        const double* wr = w + lane * sortN;
        double Z = 0.0;
        int j = 0;
        for (; j + 8 <= Ck; j += 8) {
          double v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) v[u] = wr[j + u];
#pragma unroll
          for (int u = 0; u < 8; ++u) Z = Z + v[u];
        }
        for (; j < Ck; ++j) Z = Z + wr[j];
        Z_sh[lane] = Z;
      }
    } else {
      // segmented bitonic sort of (w desc, j asc): R independent segments of sortN (a power of two >= Ck).  Each
      // thread takes pairs (t, t + jj) directly (no idle half of the index space) and exchanges them without
      // branches; the sorting warps synchronise among themselves (named barrier 1).
      const int half = R * sortN / 2;
      for (int k = 2; k <= sortN; k <<= 1) {
        for (int jj = k >> 1; jj > 0; jj >>= 1) {
          named_barrier_sync(1, kSortThreads);
          for (int pi = tid; pi < half; pi += kSortThreads) {
            const int t = ((pi & ~(jj - 1)) << 1) | (pi & (jj - 1)), u = t + jj;  // jj < sortN: same segment
            const bool up = ((t & (sortN - 1)) & k) == 0;  // direction from the position inside the segment
            const double wt = ws[t], wu = ws[u];
            const int it = idx[t], iu = idx[u];
            const bool sw = up ? before(wu, iu, wt, it) : before(wt, it, wu, iu);
            ws[t] = sw ? wu : wt;
            ws[u] = sw ? wt : wu;
            idx[t] = sw ? iu : it;
            idx[u] = sw ? it : iu;
          }
        }
      }
    }
    __syncthreads();
    if (lane == 0 && warp < nr) {  // the top-p walk of row `warp` in sorted order (R11)
      const double* wr = ws + warp * sortN;
      const int* ir = idx + warp * sortN;
      uint8_t* sr_sel = sel + warp * Ck;
      const double target = top_p * Z_sh[warp];
      double cum = 0.0;
      long long keys = 0;
      bool done = false;
      for (int r0 = 0; r0 < Ck && !done; r0 += 8) {
        double wv[8];
        int jv[8], sv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {  // sortN >= r0 + 8 whenever Ck > r0 (sortN is a power of two >= 8)
          wv[u] = wr[r0 + u];
          jv[u] = ir[r0 + u];
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) sv[u] = (r0 + u < Ck) ? sks[jv[u]] : 0;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (done || r0 + u >= Ck || wv[u] <= 0.0 || !(cum < target)) {
            done = true;
          } else {
            sr_sel[jv[u]] = 1;
            keys += sv[u];
            cum = cum + wv[u];
          }
        }
      }
      keys_sh[warp] = keys;
    }
    __syncthreads();
  }
  for (int e = tid; e < nr * Ck; e += kSelThreads) {
    const int r = e / Ck, j = e - r * Ck;
    mask[(size_t(bh) * Cq + i0 + r) * Ck + j] = sel[e];
  }
  if (tid < nr && pairs) {
    const long long contrib = (long long)__ldg(sq + size_t(bh) * Cq + i0 + tid) * keys_sh[tid];
    atomicAdd(pairs + bh, (unsigned long long)contrib);  // integer: order-free
  }
}

}  // namespace

cudaError_t launch_select_topp(const float* cq, const float* ck, const int32_t* sq, const int32_t* sk, int BH, int Cq,
                               int Ck, int d, float scale, double top_p, uint8_t* mask, int64_t* pairs,
                               cudaStream_t s) {
  int sortN = 8;
  while (sortN < Ck) sortN <<= 1;
  auto smem_of = [&](int R) {
    return size_t(R) * sortN * (2 * sizeof(double) + sizeof(int)) + size_t(R) * d * sizeof(double) +
           size_t(Ck) * sizeof(int) + size_t(R) * Ck;
  };
  int R = kRows;
  while (R > 1 && smem_of(R) > 200 * 1024) --R;
  const size_t smem = smem_of(R);
  // per launch (the attribute is per device; a process-wide flag would miss a second GPU and race across threads)
  cudaFuncSetAttribute(k_select, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  if (pairs) cudaMemsetAsync(pairs, 0, size_t(BH) * sizeof(int64_t), s);
  k_select<<<dim3((Cq + R - 1) / R, BH), kSelThreads, smem, s>>>(cq, ck, sq, sk, Cq, Ck, d, double(scale), top_p,
                                                                  sortN, R, mask,
                                                                  reinterpret_cast<unsigned long long*>(pairs));
  return cudaGetLastError();
}

}  // namespace svg2

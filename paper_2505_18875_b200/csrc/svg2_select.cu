// svg2_select.cu — A7/A8: centroid-based top-p selection, one CTA per (b, h, query cluster i).
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

__device__ __forceinline__ bool before(double wa, int ja, double wb, int jb) {
  return wa > wb || (wa == wb && ja < jb);
}

// One CTA per (query cluster i, bh).  Eq. 1 per key cluster j by one thread: its sequential FMA chain over k, the key
// centroid row read straight from L2 with kEq1Unroll 16-byte loads in flight (no staging barriers), the query
// centroid broadcast from shared memory.  Eq. 2 weights, Z_i summed by one thread in ascending j with its loads
// issued ahead of the dependent adds, a shared-memory bitonic sort (w desc, j asc), and the top-p walk (R11) by one
// thread over prefetched chunks of the sorted order.
__global__ void __launch_bounds__(kSelThreads) k_select(const float* __restrict__ cq, const float* __restrict__ ck,
                                                        const int32_t* __restrict__ sq, const int32_t* __restrict__ sk,
                                                        int Cq, int Ck, int d, double scale, double top_p, int sortN,
                                                        uint8_t* __restrict__ mask,
                                                        unsigned long long* __restrict__ pairs) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* w = reinterpret_cast<double*>(smem);          // [sortN]
  double* crow = w + sortN;                             // [d]
  int* idx = reinterpret_cast<int*>(crow + d);          // [sortN]
  int* sks = idx + sortN;                               // [Ck] key-cluster sizes
  uint8_t* sel = reinterpret_cast<uint8_t*>(sks + Ck);  // [Ck]
  __shared__ double red[kSelThreads / 32];
  __shared__ double Z_sh;
  __shared__ long long keys_sh;
  const int i = blockIdx.x, bh = blockIdx.y, tid = threadIdx.x, lane = tid & 31;
  const float* cqi = cq + (size_t(bh) * Cq + i) * d;
  const float4* ckb = reinterpret_cast<const float4*>(ck + size_t(bh) * Ck * d);
  const int32_t* skb = sk + size_t(bh) * Ck;
  for (int k = tid; k < d; k += kSelThreads) crow[k] = double(cqi[k]);
  for (int j = tid; j < Ck; j += kSelThreads) {
    sel[j] = 0;
    sks[j] = __ldg(skb + j);
  }
  __syncthreads();
  // Eq. 1: S_ij = scale * (sequential fp64 FMA over k ascending)
  double m = -INFINITY;
  for (int j = tid; j < Ck; j += kSelThreads) {
    const float4* row = ckb + size_t(j) * (d / 4);
    double acc = 0.0;
    for (int k4 = 0; k4 < d / 4; k4 += kEq1Unroll) {
      float4 c[kEq1Unroll];
#pragma unroll
      for (int u = 0; u < kEq1Unroll; ++u) c[u] = __ldg(row + k4 + u);
#pragma unroll
      for (int u = 0; u < kEq1Unroll; ++u) {
        const double* q = crow + 4 * (k4 + u);
        acc = fma(q[0], double(c[u].x), acc);
        acc = fma(q[1], double(c[u].y), acc);
        acc = fma(q[2], double(c[u].z), acc);
        acc = fma(q[3], double(c[u].w), acc);
      }
    }
    const double S = scale * acc;
    w[j] = S;
    if (sks[j] > 0) m = fmax(m, S);
  }
  // block max over non-empty clusters (exact, order-free)
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0) red[tid >> 5] = m;
  __syncthreads();
  m = red[0];
  for (int t = 1; t < kSelThreads / 32; ++t) m = fmax(m, red[t]);
  // Eq. 2: w_ij = |K_j| exp(S_ij - m_i); empty clusters weigh 0; sort padding sorts last
  for (int j = tid; j < sortN; j += kSelThreads) {
    if (j < Ck) {
      const int s = sks[j];
      w[j] = s > 0 ? double(s) * exp(w[j] - m) : 0.0;
      idx[j] = j;
    } else {
      w[j] = -1.0;
      idx[j] = 0x7fffffff;
    }
  }
  __syncthreads();
  if (top_p >= 1.0) {  // p = 1: exactly the non-empty clusters (R11), no order needed
    long long keys = 0;
    for (int j = tid; j < Ck; j += kSelThreads) {
      const int s = sks[j];
      sel[j] = s > 0;
      keys += s;
    }
    for (int o = 16; o > 0; o >>= 1) keys += __shfl_xor_sync(0xffffffffu, keys, o);
    if (tid == 0) keys_sh = 0;
    __syncthreads();
    if (lane == 0) atomicAdd(reinterpret_cast<unsigned long long*>(&keys_sh), (unsigned long long)keys);
    __syncthreads();
  } else {
    if (tid == 0) {  // Z_i in ascending j, sequential (spec order); the loads run ahead of the dependent adds
      double Z = 0.0;
      int j = 0;
      for (; j + 8 <= Ck; j += 8) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = w[j + u];
#pragma unroll
        for (int u = 0; u < 8; ++u) Z = Z + v[u];
      }
      for (; j < Ck; ++j) Z = Z + w[j];
      Z_sh = Z;
    }
    // bitonic sort of (w desc, j asc) over sortN (power of two >= Ck)
    for (int k = 2; k <= sortN; k <<= 1) {
      for (int jj = k >> 1; jj > 0; jj >>= 1) {
        __syncthreads();
        for (int t = tid; t < sortN; t += kSelThreads) {
          const int u = t ^ jj;
          if (u > t) {
            const bool up = (t & k) == 0;
            const double wt = w[t], wu = w[u];
            const int it = idx[t], iu = idx[u];
            const bool sw = up ? before(wu, iu, wt, it) : before(wt, it, wu, iu);
            if (sw) {
              w[t] = wu;
              w[u] = wt;
              idx[t] = iu;
              idx[u] = it;
            }
          }
        }
      }
    }
    __syncthreads();
    if (tid == 0) {  // the top-p walk in sorted order (R11): take rank r while the mass before it is < p Z_i
      const double target = top_p * Z_sh;
      double cum = 0.0;
      long long keys = 0;
      bool done = false;
      for (int r0 = 0; r0 < Ck && !done; r0 += 8) {
        double wr[8];
        int jr[8], sr[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {  // sortN >= r0 + 8 whenever Ck > r0 (sortN is a power of two >= 8 here)
          wr[u] = w[r0 + u];
          jr[u] = idx[r0 + u];
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) sr[u] = (r0 + u < Ck) ? sks[jr[u]] : 0;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (done || r0 + u >= Ck || wr[u] <= 0.0 || !(cum < target)) {
            done = true;
          } else {
            sel[jr[u]] = 1;
            keys += sr[u];
            cum = cum + wr[u];
          }
        }
      }
      keys_sh = keys;
    }
    __syncthreads();
  }
  uint8_t* mrow = mask + (size_t(bh) * Cq + i) * Ck;
  for (int j = tid; j < Ck; j += kSelThreads) mrow[j] = sel[j];
  if (tid == 0 && pairs) {
    const long long contrib = (long long)__ldg(sq + size_t(bh) * Cq + i) * keys_sh;
    atomicAdd(pairs + bh, (unsigned long long)contrib);  // integer: order-free
  }
}

}  // namespace

cudaError_t launch_select_topp(const float* cq, const float* ck, const int32_t* sq, const int32_t* sk, int BH, int Cq,
                               int Ck, int d, float scale, double top_p, uint8_t* mask, int64_t* pairs,
                               cudaStream_t s) {
  int sortN = 8;
  while (sortN < Ck) sortN <<= 1;
  const size_t smem = size_t(sortN) * sizeof(double) + size_t(d) * sizeof(double) + size_t(sortN) * sizeof(int) +
                      size_t(Ck) * sizeof(int) + size_t(Ck);
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(k_select, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    attr_set = true;
  }
  if (pairs) cudaMemsetAsync(pairs, 0, size_t(BH) * sizeof(int64_t), s);
  k_select<<<dim3(Cq, BH), kSelThreads, smem, s>>>(cq, ck, sq, sk, Cq, Ck, d, double(scale), top_p, sortN, mask,
                                                   reinterpret_cast<unsigned long long*>(pairs));
  return cudaGetLastError();
}

}  // namespace svg2

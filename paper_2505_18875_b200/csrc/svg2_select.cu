// svg2_select.cu — A7/A8: centroid-based top-p selection, one CTA per (b, h, query cluster i).
//   Eq. 1  S_ij = scale * sum_k c^q_ik c^k_jk          fp64, sequential FMA over k ascending (spec, DESIGN R8)
//   Eq. 2  w_ij = |K_j| exp(S_ij - m_i), m_i = max over non-empty j;  Z_i = sum_j w_ij, ascending j (R9)
//   top-p  sort (w desc, j asc) by a shared-memory bitonic sort; select ranks while cum < p Z_i (R10, R11);
//          p == 1 selects every non-empty cluster exactly.
// The order of every floating-point operation is fixed by the specification above (not by shared code with the
// oracle), so the mask is bit-exact against it except at documented near-ties (R17).
#include <cfloat>
#include <climits>
#include "internal.h"

namespace svg2 {
namespace {

constexpr int kSelThreads = 256;
constexpr int kKChunk = 32;  // centroid columns staged per pass (rows padded to kKChunk + 1 floats)

__device__ __forceinline__ bool before(double wa, int ja, double wb, int jb) {
  return wa > wb || (wa == wb && ja < jb);
}

__global__ void __launch_bounds__(kSelThreads) k_select(const float* __restrict__ cq, const float* __restrict__ ck,
                                                        const int32_t* __restrict__ sq, const int32_t* __restrict__ sk,
                                                        int Cq, int Ck, int d, double scale, double top_p, int sortN,
                                                        uint8_t* __restrict__ mask,
                                                        unsigned long long* __restrict__ pairs) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* w = reinterpret_cast<double*>(smem);          // [sortN]
  double* crow = w + sortN;                             // [d]
  int* idx = reinterpret_cast<int*>(crow + d);          // [sortN]
  int* sks = idx + sortN;                                  // [Ck] key-cluster sizes (staged for the serial walk)
  uint8_t* sel = reinterpret_cast<uint8_t*>(sks + Ck);     // [Ck]
  float* stage = reinterpret_cast<float*>(sks + Ck + (Ck + 3) / 4 + 4);  // [kSelThreads][kKChunk + 1]
  __shared__ double red[kSelThreads / 32];
  __shared__ long long keys_sh;
  const int i = blockIdx.x, bh = blockIdx.y, tid = threadIdx.x;
  const float* cqi = cq + (size_t(bh) * Cq + i) * d;
  const float* ckb = ck + size_t(bh) * Ck * d;
  const int32_t* skb = sk + size_t(bh) * Ck;
  for (int k = tid; k < d; k += kSelThreads) crow[k] = double(cqi[k]);
  for (int j = tid; j < Ck; j += kSelThreads) {
    sel[j] = 0;
    sks[j] = __ldg(skb + j);
  }
  __syncthreads();
  // Eq. 1: the key centroids are staged kSelThreads rows x kKChunk columns at a time through padded shared memory
  // (coalesced global reads, conflict-free row reads); each thread keeps its own sequential FMA chain over k.
  double m = -INFINITY;
  for (int j0 = 0; j0 < Ck; j0 += kSelThreads) {
    const int j = j0 + tid;
    double acc = 0.0;
    for (int k0 = 0; k0 < d; k0 += kKChunk) {
      __syncthreads();
      for (int e = tid; e < kSelThreads * kKChunk; e += kSelThreads) {
        const int r = e / kKChunk, c = e - r * kKChunk;
        stage[r * (kKChunk + 1) + c] = (j0 + r < Ck) ? __ldg(ckb + size_t(j0 + r) * d + k0 + c) : 0.f;
      }
      __syncthreads();
      const float* srow = stage + tid * (kKChunk + 1);
#pragma unroll 8
      for (int k = 0; k < kKChunk; ++k) acc = fma(crow[k0 + k], double(srow[k]), acc);
    }
    if (j < Ck) {
      const double S = scale * acc;
      w[j] = S;
      if (sks[j] > 0) m = fmax(m, S);
    }
  }
  // block max (exact, order-free)
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((tid & 31) == 0) red[tid >> 5] = m;
  __syncthreads();
  m = red[0];
  for (int t = 1; t < kSelThreads / 32; ++t) m = fmax(m, red[t]);
  for (int j = tid; j < sortN; j += kSelThreads) {
    if (j < Ck) {
      const int s = __ldg(skb + j);
      w[j] = s > 0 ? double(s) * exp(w[j] - m) : 0.0;
      idx[j] = j;
    } else {
      w[j] = -1.0;
      idx[j] = INT_MAX;
    }
  }
  __syncthreads();
  if (top_p >= 1.0) {
    long long keys = 0;
    for (int j = tid; j < Ck; j += kSelThreads) {
      const int s = __ldg(skb + j);
      sel[j] = s > 0;
      keys += s;
    }
    for (int o = 16; o > 0; o >>= 1) keys += __shfl_xor_sync(0xffffffffu, keys, o);
    if (tid == 0) keys_sh = 0;
    __syncthreads();
    if ((tid & 31) == 0) atomicAdd(reinterpret_cast<unsigned long long*>(&keys_sh), (unsigned long long)keys);
    __syncthreads();
  } else {
    __shared__ double Z_sh;
    if (tid == 0) {  // Z_i in ascending j, sequential (spec order)
      double Z = 0.0;
      for (int j = 0; j < Ck; ++j) Z = Z + w[j];
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
    if (tid == 0) {
      const double target = top_p * Z_sh;
      double cum = 0.0;
      long long keys = 0;
      for (int r = 0; r < Ck; ++r) {
        const double wr = w[r];
        if (wr <= 0.0) break;
        if (!(cum < target)) break;
        sel[idx[r]] = 1;
        keys += sks[idx[r]];
        cum = cum + wr;
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
  int sortN = 1;
  while (sortN < Ck) sortN <<= 1;
  const size_t smem = size_t(sortN) * sizeof(double) + size_t(d) * sizeof(double) + size_t(sortN) * sizeof(int) +
                      size_t(Ck) * sizeof(int) + (size_t(Ck) / 4 + 5) * sizeof(int) +
                      size_t(kSelThreads) * (kKChunk + 1) * sizeof(float);
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

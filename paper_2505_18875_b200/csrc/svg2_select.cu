// svg2_select.cu — A7/A8: centroid-based top-p selection.
//   Eq. 1  S_ij = scale * sum_k c^q_ik c^k_jk          fp64, sequential FMA over k ascending (spec, DESIGN R8)
//   Eq. 2  w_ij = |K_j| exp(S_ij - m_i), m_i = max over non-empty j (R9);  Z_i = sum_j w_ij
//   top-p  sort j by (w desc, j asc); select the ranks whose preceding mass is < p Z_i (R10, R11); p == 1 selects
//          every non-empty cluster exactly.
// Two kernels: k_scores computes Eq. 1 for a tile of 8 query x 256 key clusters (each key-centroid row read once for 8
// rows) into an fp64 workspace; k_select does the rest per query cluster, without sorting: the selected ranks are
// the w at or above a threshold found bit by bit (k_select).  S, m and w are the specification's exactly; Z_i and the
// masses the threshold test uses are sums of the same fp64 terms in a fixed tree order (a row's thread-local runs,
// then shuffle and cross-warp trees) instead of the sequential order of the sorted walk: deterministic, and different
// from the sequential sums only by fp64 rounding (< 4096 ulps of Z_i), so a mask can differ from the oracle's only on
// an R17 near-tie (DESIGN R17, R27).
#include <cfloat>
#include "internal.h"

namespace svg2 {
namespace {

constexpr int kSelThreads = 256, kSelWarps = kSelThreads / 32;
constexpr int kEq1Unroll = 8;  // 16-byte key-centroid loads in flight per thread (the Eq. 1 loop is L2-latency-bound)

// Eq. 1 for 8 query clusters x 256 key clusters per CTA: thread j reads key centroid j once (kEq1Unroll 16-byte loads
// in flight), widens it to fp64 and runs the 8 sequential FMA chains (k ascending); S [BH, Cq, Ck] fp64.
constexpr int kScoreRows = 8;
__global__ void __launch_bounds__(kSelThreads) k_scores(const float* __restrict__ cq, const float* __restrict__ ck,
                                                        int Cq, int Ck, int d, double scale, double* __restrict__ S) {
  __shared__ double crow[kScoreRows * 128];
  const int i0 = blockIdx.x * kScoreRows, bh = blockIdx.z, tid = threadIdx.x;
  const int nr = min(kScoreRows, Cq - i0);
  for (int e = tid; e < kScoreRows * d; e += kSelThreads) {
    const int r = e / d, k = e - r * d;
    crow[e] = r < nr ? double(cq[(size_t(bh) * Cq + i0 + r) * d + k]) : 0.0;
  }
  __syncthreads();
  const int j = blockIdx.y * kSelThreads + tid;
  if (j >= Ck) return;
  const float4* row = reinterpret_cast<const float4*>(ck + (size_t(bh) * Ck + j) * d);
  double acc[kScoreRows];
#pragma unroll
  for (int r = 0; r < kScoreRows; ++r) acc[r] = 0.0;
  for (int k4 = 0; k4 < d / 4; k4 += kEq1Unroll) {
    float4 c[kEq1Unroll];
#pragma unroll
    for (int u = 0; u < kEq1Unroll; ++u) c[u] = __ldg(row + k4 + u);
#pragma unroll
    for (int u = 0; u < kEq1Unroll; ++u) {
      const double c0 = c[u].x, c1 = c[u].y, c2 = c[u].z, c3 = c[u].w;
      const int k = 4 * (k4 + u);
#pragma unroll
      for (int r = 0; r < kScoreRows; ++r) {
        const double* q = crow + r * d + k;
        acc[r] = fma(q[0], c0, acc[r]);
        acc[r] = fma(q[1], c1, acc[r]);
        acc[r] = fma(q[2], c2, acc[r]);
        acc[r] = fma(q[3], c3, acc[r]);
      }
    }
  }
  for (int r = 0; r < nr; ++r) S[(size_t(bh) * Cq + i0 + r) * Ck + j] = scale * acc[r];
}

// Team-wide fp64 sum of one value per thread, identical on every thread of the team (so every thread takes the same
// threshold decisions): shuffle-down tree inside each warp, broadcast of lane 0, then the team's warps in ascending
// order through shared memory (double-buffered by pass parity: one __syncthreads per call when TW > 1).
template <int TW>
__device__ __forceinline__ double team_sum(double v, double (*red)[kSelWarps], int& parity, int warp, int row) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  v = __shfl_sync(0xffffffffu, v, 0);
  if constexpr (TW == 1) {
    return v;
  } else {
    if ((threadIdx.x & 31) == 0) red[parity][warp] = v;
    __syncthreads();
    double t = 0.0;
#pragma unroll
    for (int k = 0; k < TW; ++k) t += red[parity][row * TW + k];
    parity ^= 1;
    return t;
  }
}
template <int TW>
__device__ __forceinline__ long long team_sum_ll(long long v, long long (*red)[kSelWarps], int& parity, int warp,
                                                 int row) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);  // integers: order-free
  if constexpr (TW == 1) {
    return v;
  } else {
    if ((threadIdx.x & 31) == 0) red[parity][warp] = v;
    __syncthreads();
    long long t = 0;
#pragma unroll
    for (int k = 0; k < TW; ++k) t += red[parity][row * TW + k];
    parity ^= 1;
    return t;
  }
}

// One CTA per (R query clusters, bh); row r is owned by a team of TW = 8 / R warps.  A row's entries live in
// registers, E per thread (entry j = team_thread * E + i, ascending j), 32 * TW * E >= Ck.
//   1) S of the entries (k_scores), row max over non-empty j (R9); w = |K_j| exp(S - m) (Eq. 2); Z by a fixed tree.
//   2) top-p without sorting (R27): with B(v) = sum of the w >= v, the ranks the sorted walk selects (mass before
//      the rank < p Z) are exactly the w >= w*, w* = max{v : B(v) >= p Z} -- the first rank whose inclusive mass
//      reaches p Z.  B is monotone in v and positive doubles order like their bit patterns, so w* is found bit by
//      bit from the top (63 team sums of the thread-local partial masses).  Entries equal to w* (only equal
//      centroids and sizes give such ties) are then ordered by ascending j as the sort would: the k-th of them is
//      selected iff B(> w*) + k w* < p Z.
template <int E, int R>
__global__ void __launch_bounds__(kSelThreads) k_select(const double* __restrict__ S, const int32_t* __restrict__ sq,
                                                        const int32_t* __restrict__ sk, int Cq, int Ck, double top_p,
                                                        uint8_t* __restrict__ mask,
                                                        unsigned long long* __restrict__ pairs) {
  constexpr int TW = kSelWarps / R;  // warps per row
  extern __shared__ __align__(16) unsigned char smem[];
  int* sks = reinterpret_cast<int*>(smem);                     // [Ck]
  uint8_t* sel = reinterpret_cast<uint8_t*>(sks + Ck);         // [R][Ck]
  __shared__ double red_w[2][kSelWarps];
  __shared__ long long red_k[2][kSelWarps];
  const int i0 = blockIdx.x * R, bh = blockIdx.y, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nr = min(R, Cq - i0);
  const int32_t* skb = sk + size_t(bh) * Ck;
  for (int j = tid; j < Ck; j += kSelThreads) sks[j] = __ldg(skb + j);
  for (int e = tid; e < R * Ck; e += kSelThreads) sel[e] = 0;
  __syncthreads();
  const int row = warp / TW, wt = warp % TW, tt = wt * 32 + lane;  // team thread 0..32*TW-1
  const double* Srow = S + (size_t(bh) * Cq + min(i0 + row, Cq - 1)) * Ck;
  int pw = 0, pk = 0;  // parities of the double / integer reduction buffers
  // S of this thread's entries; the row max over non-empty clusters (exact, order-free)
  double w[E];
  double mx = -INFINITY;
#pragma unroll
  for (int i = 0; i < E; ++i) {
    const int j = tt * E + i;
    w[i] = j < Ck ? __ldg(Srow + j) : 0.0;
    if (j < Ck && sks[j] > 0) mx = fmax(mx, w[i]);
  }
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (TW > 1) {
    if (lane == 0) red_w[pw][warp] = mx;
    __syncthreads();
    mx = red_w[pw][row * TW];
    for (int t = 1; t < TW; ++t) mx = fmax(mx, red_w[pw][row * TW + t]);
    pw ^= 1;
  }
  // ---- Eq. 2 weights (0 for empty clusters and padding entries: never selected, add nothing)
#pragma unroll
  for (int i = 0; i < E; ++i) {
    const int j = tt * E + i;
    const int s = j < Ck ? sks[j] : 0;
    w[i] = s > 0 ? double(s) * exp(w[i] - mx) : 0.0;
  }
  long long keys = 0;
  if (top_p >= 1.0) {  // p = 1: exactly the non-empty clusters (R11)
#pragma unroll
    for (int i = 0; i < E; ++i) {
      const int j = tt * E + i;
      if (w[i] > 0.0) {
        sel[row * Ck + j] = 1;
        keys += sks[j];
      }
    }
  } else {
    // Z: thread-local run in ascending j, then the fixed tree
    double z = 0.0;
#pragma unroll
    for (int i = 0; i < E; ++i) z += w[i];
    const double target = top_p * team_sum<TW>(z, red_w, pw, warp, row);
    // ---- w* bit by bit: t = max{v : B(v) >= target}; stays 0 (select every w > 0) if no v reaches it
    unsigned long long t = 0;
    for (int b = 62; b >= 0; --b) {
      const unsigned long long cand = t | (1ull << b);
      double part0 = 0.0, part1 = 0.0;
#pragma unroll
      for (int i = 0; i < E; i += 2) {
        part0 += (unsigned long long)__double_as_longlong(w[i]) >= cand ? w[i] : 0.0;
        if (i + 1 < E) part1 += (unsigned long long)__double_as_longlong(w[i + 1]) >= cand ? w[i + 1] : 0.0;
      }
      if (team_sum<TW>(part0 + part1, red_w, pw, warp, row) >= target) t = cand;
    }
    // ---- entries equal to w*: the sort orders them by ascending j
    const double wstar = __longlong_as_double((long long)t);
    int nt = 0;
#pragma unroll
    for (int i = 0; i < E; ++i) nt += (w[i] > 0.0 && w[i] == wstar) ? 1 : 0;
    const long long ties = team_sum_ll<TW>(nt, red_k, pk, warp, row);
    // mass strictly above w* and each tied entry's rank among the ties (team exclusive scan); computed by every
    // team (the reductions synchronise the CTA) but used only when w* is tied
    double above = 0.0;
#pragma unroll
    for (int i = 0; i < E; ++i) above += (unsigned long long)__double_as_longlong(w[i]) > t ? w[i] : 0.0;
    above = team_sum<TW>(above, red_w, pw, warp, row);
    int incl = nt;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    long long rank = incl - nt;
    if (TW > 1) {
      __syncthreads();
      if (lane == 31) red_k[pk][warp] = incl;
      __syncthreads();
      for (int u = 0; u < wt; ++u) rank += red_k[pk][row * TW + u];
    }
#pragma unroll
    for (int i = 0; i < E; ++i) {
      const int j = tt * E + i;
      const unsigned long long bits = (unsigned long long)__double_as_longlong(w[i]);
      bool take = w[i] > 0.0 && bits > t;
      if (w[i] > 0.0 && bits == t) {
        take = ties <= 1 || above + double(rank) * wstar < target;
        ++rank;
      }
      if (take) {
        sel[row * Ck + j] = 1;
        keys += sks[j];
      }
    }
  }
  // selected keys of the row (integers: order-free), then the mask rows and the pair count
  for (int o = 16; o > 0; o >>= 1) keys += __shfl_xor_sync(0xffffffffu, keys, o);
  __syncthreads();
  if (lane == 0) red_k[0][warp] = keys;
  __syncthreads();
  for (int e = tid; e < nr * Ck; e += kSelThreads) {
    const int r = e / Ck, j = e - r * Ck;
    mask[(size_t(bh) * Cq + i0 + r) * Ck + j] = sel[e];
  }
  if (wt == 0 && lane == 0 && row < nr && pairs) {
    long long rk = 0;
    for (int t = 0; t < TW; ++t) rk += red_k[0][row * TW + t];
    const long long contrib = (long long)__ldg(sq + size_t(bh) * Cq + i0 + row) * rk;
    atomicAdd(pairs + bh, (unsigned long long)contrib);  // integer: order-free
  }
}

template <int E, int R>
cudaError_t launch_select(const double* S, const int32_t* sq, const int32_t* sk, int BH, int Cq, int Ck, double top_p,
                          uint8_t* mask, int64_t* pairs, cudaStream_t s) {
  const size_t smem = size_t(Ck) * sizeof(int) + size_t(R) * Ck;
  // per launch (the attribute is per device; a process-wide flag would miss a second GPU and race across threads)
  cudaFuncSetAttribute(k_select<E, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  k_select<E, R><<<dim3((Cq + R - 1) / R, BH), kSelThreads, smem, s>>>(
      S, sq, sk, Cq, Ck, top_p, mask, reinterpret_cast<unsigned long long*>(pairs));
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_select_topp(const float* cq, const float* ck, const int32_t* sq, const int32_t* sk, int BH, int Cq,
                               int Ck, int d, float scale, double top_p, uint8_t* mask, int64_t* pairs, double* S,
                               cudaStream_t s) {
  if (pairs) cudaMemsetAsync(pairs, 0, size_t(BH) * sizeof(int64_t), s);
  k_scores<<<dim3((Cq + kScoreRows - 1) / kScoreRows, (Ck + kSelThreads - 1) / kSelThreads, BH), kSelThreads, 0, s>>>(
      cq, ck, Cq, Ck, d, double(scale), S);
  // entries per row = 256 / R threads x E: one warp per row up to 512 (8 rows per CTA), then 2 / 4 / 8 warps per row
  if (Ck <= 32) return launch_select<1, 8>(S, sq, sk, BH, Cq, Ck, top_p, mask, pairs, s);
  if (Ck <= 64) return launch_select<2, 8>(S, sq, sk, BH, Cq, Ck, top_p, mask, pairs, s);
  if (Ck <= 128) return launch_select<4, 8>(S, sq, sk, BH, Cq, Ck, top_p, mask, pairs, s);
  if (Ck <= 256) return launch_select<8, 8>(S, sq, sk, BH, Cq, Ck, top_p, mask, pairs, s);
  if (Ck <= 512) return launch_select<16, 8>(S, sq, sk, BH, Cq, Ck, top_p, mask, pairs, s);
  if (Ck <= 1024) return launch_select<16, 4>(S, sq, sk, BH, Cq, Ck, top_p, mask, pairs, s);
  if (Ck <= 2048) return launch_select<16, 2>(S, sq, sk, BH, Cq, Ck, top_p, mask, pairs, s);
  return launch_select<16, 1>(S, sq, sk, BH, Cq, Ck, top_p, mask, pairs, s);
}

}  // namespace svg2

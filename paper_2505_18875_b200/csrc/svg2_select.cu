// svg2_select.cu — A7/A8: centroid-based top-p selection.
//   Eq. 1  S_ij = scale * sum_k c^q_ik c^k_jk          fp64, sequential FMA over k ascending (spec, DESIGN R8)
//   Eq. 2  w_ij = |K_j| exp(S_ij - m_i), m_i = max over non-empty j (R9);  Z_i = sum_j w_ij
//   top-p  sort j by (w desc, j asc); select the ranks whose preceding mass is < p Z_i (R10, R11); p == 1 selects
//          every non-empty cluster exactly.
// Two kernels: k_scores computes Eq. 1 for a tile of 8 query x 256 key clusters (each key-centroid row read once for 8
// rows) into an fp64 workspace; k_select does the rest per query cluster.  S, m, w and the sorted order are the
// specification's exactly.  Z_i and the preceding masses are sums of the same
// fp64 terms in a fixed tree order (a row's thread-local runs, then shuffle and cross-warp trees) instead of the
// sequential order: deterministic, and different from the sequential sums only by fp64 rounding (< 4096 ulps of
// Z_i), so a mask can differ from the oracle's only on an R17 near-tie (DESIGN R17, R27).
#include <cfloat>
#include "internal.h"

namespace svg2 {
namespace {

constexpr int kSelThreads = 256, kSelWarps = kSelThreads / 32;
constexpr int kEq1Unroll = 8;  // 16-byte key-centroid loads in flight per thread (the Eq. 1 loop is L2-latency-bound)
constexpr int kMaxRows = 8;    // query clusters per CTA (one warp per row up to 512 sorted entries)

__device__ __forceinline__ bool before(double wa, int ja, double wb, int jb) {
  return wa > wb || (wa == wb && ja < jb);
}

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

// One bitonic stage with partners jj < E apart inside a thread's E consecutive entries (e = tt * E + i).
template <int E, int JJ>
__device__ __forceinline__ void sort_in_thread(double (&w)[E], int (&ix)[E], int tt, int k) {
  if (JJ >= E) return;
#pragma unroll
  for (int i = 0; i < E; ++i) {
    if (i & JJ) continue;
    const int u = i | JJ;
    const bool up = ((tt * E + i) & k) == 0;
    const bool sw = up ? before(w[u], ix[u], w[i], ix[i]) : before(w[i], ix[i], w[u], ix[u]);
    const double a = w[i], b = w[u];
    const int ia = ix[i], ib = ix[u];
    w[i] = sw ? b : a;
    w[u] = sw ? a : b;
    ix[i] = sw ? ib : ia;
    ix[u] = sw ? ia : ib;
  }
}

// One CTA per (R query clusters, bh); row r is owned by a team of TW = 8 / R warps.  A row's entries live in
// registers, E per thread (entry e = team_thread * E + i), sortN = 32 * TW * E >= Ck entries (padding sorts last).
//   1) Eq. 1 for the R rows by all 256 threads, one key cluster per thread at a time (its centroid row read from L2
//      once and widened to fp64 for R sequential FMA chains) -> S in shared memory; row max over non-empty j.
//   2) each team: w = |K_j| exp(S - m) into registers; Z by a fixed tree.
//   3) bitonic sort of (w desc, j asc): partners inside a thread in registers, inside a warp by shuffles, across
//      the team's warps through shared memory.
//   4) exclusive scan of the sorted weights (fixed tree) -> select rank r iff w_r > 0 and mass before r < p Z.
template <int E, int R>
__global__ void __launch_bounds__(kSelThreads) k_select(const double* __restrict__ S, const int32_t* __restrict__ sq,
                                                        const int32_t* __restrict__ sk, int Cq, int Ck, double top_p,
                                                        uint8_t* __restrict__ mask,
                                                        unsigned long long* __restrict__ pairs) {
  constexpr int TW = kSelWarps / R;        // warps per row
  constexpr int TT = 32 * TW;              // threads per row
  constexpr int kSortN = TT * E;           // entries per row
  extern __shared__ __align__(16) unsigned char smem[];
  double* Xs = reinterpret_cast<double*>(smem);               // [R][kSortN] cross-warp exchange of weights
  int* Ish = reinterpret_cast<int*>(Xs + R * kSortN);         // [R][kSortN] cross-warp exchange of indices
  int* sks = Ish + R * kSortN;                                // [Ck]
  uint8_t* sel = reinterpret_cast<uint8_t*>(sks + Ck);        // [R][Ck]
  __shared__ double red_w[kSelWarps];
  __shared__ long long red_k[kSelWarps];
  const int i0 = blockIdx.x * R, bh = blockIdx.y, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nr = min(R, Cq - i0);
  const int32_t* skb = sk + size_t(bh) * Ck;
  for (int j = tid; j < Ck; j += kSelThreads) sks[j] = __ldg(skb + j);
  for (int e = tid; e < R * Ck; e += kSelThreads) sel[e] = 0;
  __syncthreads();
  const int row = warp / TW, wt = warp % TW, tt = wt * 32 + lane;  // team thread 0..TT-1
  const double* Srow = S + (size_t(bh) * Cq + min(i0 + row, Cq - 1)) * Ck;
  // S of this thread's entries; the row max over non-empty clusters (exact, order-free)
  double w[E];
  int ix[E];
  double mx = -INFINITY;
#pragma unroll
  for (int i = 0; i < E; ++i) {
    const int j = tt * E + i;
    w[i] = j < Ck ? __ldg(Srow + j) : 0.0;
    if (j < Ck && sks[j] > 0) mx = fmax(mx, w[i]);
  }
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 0) red_w[warp] = mx;
  __syncthreads();
  mx = red_w[row * TW];
  for (int t = 1; t < TW; ++t) mx = fmax(mx, red_w[row * TW + t]);
  __syncthreads();
  // ---- Eq. 2 weights
#pragma unroll
  for (int i = 0; i < E; ++i) {
    const int j = tt * E + i;
    if (j < Ck) {
      const int s = sks[j];
      w[i] = s > 0 ? double(s) * exp(w[i] - mx) : 0.0;
      ix[i] = j;
    } else {
      w[i] = -1.0;  // padding: sorts after every real entry
      ix[i] = 0x7fffffff;
    }
  }
  const bool row_valid = row < nr;
  long long keys = 0;
  if (top_p >= 1.0) {  // p = 1: exactly the non-empty clusters (R11), no order needed
#pragma unroll
    for (int i = 0; i < E; ++i) {
      if (ix[i] < Ck && sks[ix[i]] > 0) {
        sel[row * Ck + ix[i]] = 1;
        keys += sks[ix[i]];
      }
    }
  } else {
    // Z: thread-local run, then a shuffle tree, then the team's warps in order
    double z = 0.0;
#pragma unroll
    for (int i = 0; i < E; ++i) z += fmax(w[i], 0.0);
    for (int o = 16; o > 0; o >>= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
    if (lane == 0) red_w[warp] = z;
    __syncthreads();
    double Z = 0.0;
    for (int t = 0; t < TW; ++t) Z += red_w[row * TW + t];
    // ---- 3) bitonic sort of the team's kSortN entries by (w desc, j asc)
    for (int k = 2; k <= kSortN; k <<= 1) {
      for (int jj = k >> 1; jj > 0; jj >>= 1) {
        if (jj < E) {  // partner in the same thread (compile-time register indices)
          switch (jj) {
            case 8: sort_in_thread<E, 8>(w, ix, tt, k); break;
            case 4: sort_in_thread<E, 4>(w, ix, tt, k); break;
            case 2: sort_in_thread<E, 2>(w, ix, tt, k); break;
            default: sort_in_thread<E, 1>(w, ix, tt, k); break;
          }
        } else if (jj < 32 * E) {  // partner in another lane of the warp, same slot
          const int lm = jj / E;
          const bool lower = (lane & lm) == 0;
#pragma unroll
          for (int i = 0; i < E; ++i) {
            const int e = tt * E + i;
            const bool up = (e & k) == 0;
            const double pw = __shfl_xor_sync(0xffffffffu, w[i], lm);
            const int pi = __shfl_xor_sync(0xffffffffu, ix[i], lm);
            // the lower position keeps the entry that comes first in this segment's direction
            const bool mine_first = before(w[i], ix[i], pw, pi);
            const bool keep = (lower == up) ? mine_first : !mine_first;
            if (!keep) {
              w[i] = pw;
              ix[i] = pi;
            }
          }
        } else {  // partner in another warp of the team: exchange through shared memory
          double* xs = Xs + row * kSortN;
          int* xi = Ish + row * kSortN;
          __syncthreads();
          // slot-major layout (entry tt * E + i at i * TT + tt): consecutive threads, consecutive words
#pragma unroll
          for (int i = 0; i < E; ++i) {
            xs[i * TT + tt] = w[i];
            xi[i * TT + tt] = ix[i];
          }
          __syncthreads();
          const int pt = tt ^ (jj / E);  // partner thread, same slot
          const bool lower = (tt & (jj / E)) == 0;
#pragma unroll
          for (int i = 0; i < E; ++i) {
            const int e = tt * E + i;
            const bool up = (e & k) == 0;
            const double pw = xs[i * TT + pt];
            const int pi = xi[i * TT + pt];
            const bool mine_first = before(w[i], ix[i], pw, pi);
            const bool keep = (lower == up) ? mine_first : !mine_first;
            if (!keep) {
              w[i] = pw;
              ix[i] = pi;
            }
          }
        }
      }
    }
    // ---- 4) exclusive scan of the sorted weights (padding counts 0): thread run, warp shuffle scan, team warps
    double run = 0.0;
#pragma unroll
    for (int i = 0; i < E; ++i) run += fmax(w[i], 0.0);
    double incl = run;
    for (int o = 1; o < 32; o <<= 1) {
      const double y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    __syncthreads();
    if (lane == 31) red_w[warp] = incl;
    __syncthreads();
    double cum = incl - run;
    for (int t = 0; t < wt; ++t) cum += red_w[row * TW + t];
    const double target = top_p * Z;
#pragma unroll
    for (int i = 0; i < E; ++i) {
      if (w[i] > 0.0 && cum < target) {
        sel[row * Ck + ix[i]] = 1;
        keys += sks[ix[i]];
      }
      cum += fmax(w[i], 0.0);
    }
  }
  // selected keys of the row (integers: order-free), then the mask rows and the pair count
  for (int o = 16; o > 0; o >>= 1) keys += __shfl_xor_sync(0xffffffffu, keys, o);
  __syncthreads();
  if (lane == 0) red_k[warp] = keys;
  __syncthreads();
  for (int e = tid; e < nr * Ck; e += kSelThreads) {
    const int r = e / Ck, j = e - r * Ck;
    mask[(size_t(bh) * Cq + i0 + r) * Ck + j] = sel[e];
  }
  if (wt == 0 && lane == 0 && row_valid && pairs) {
    long long rk = 0;
    for (int t = 0; t < TW; ++t) rk += red_k[row * TW + t];
    const long long contrib = (long long)__ldg(sq + size_t(bh) * Cq + i0 + row) * rk;
    atomicAdd(pairs + bh, (unsigned long long)contrib);  // integer: order-free
  }
}

template <int E, int R>
cudaError_t launch_select(const double* S, const int32_t* sq, const int32_t* sk, int BH, int Cq, int Ck, double top_p,
                          uint8_t* mask, int64_t* pairs, cudaStream_t s) {
  constexpr int kSortN = (kSelThreads / R) * E;
  const size_t smem = size_t(R) * kSortN * (sizeof(double) + sizeof(int)) + size_t(Ck) * sizeof(int) + size_t(R) * Ck;
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

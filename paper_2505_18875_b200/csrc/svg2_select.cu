// svg2_select.cu — A7/A8: centroid-based top-p selection.
//   Eq. 1  S_ij = scale * sum_k c^q_ik c^k_jk          fp64, sequential FMA over k ascending (spec, DESIGN R8)
//   Eq. 2  w_ij = |K_j| exp(S_ij - m_i), m_i = max over non-empty j (R9);  Z_i = sum_j w_ij
//   top-p  sort j by (w desc, j asc); select the ranks whose preceding mass is < p Z_i (R10, R11); p == 1 selects
//          every non-empty cluster exactly.
// Two kernels: k_scores computes Eq. 1 for a tile of 32 query x 128 key clusters (centroid tiles staged in shared
// memory) into an fp64 workspace; k_select does the rest per query cluster, without sorting: the selected ranks are
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
// top-p threshold lists of at most this many weights are resolved directly (O(L^2 / 32) adds per lane), longer ones
// are narrowed 8 bits at a time first
constexpr int kShortList = 64;

// Eq. 1 for a tile of 32 query x 128 key clusters per CTA: both centroid tiles pass through shared memory in chunks
// of 32 dimensions (coalesced loads, widened to fp64 once); thread (ty, tx) owns rows 4ty..4ty+3 and keys tx + 32u
// (u < 4) and runs their 16 sequential FMA chains (k ascending, the specification's order); S [BH, Cq, Ck] fp64.
constexpr int kScQ = 32, kScK = 128, kScD = 32;
__global__ void __launch_bounds__(kSelThreads) k_scores(const float* __restrict__ cq, const float* __restrict__ ck,
                                                        int Cq, int Ck, int d, double scale, double* __restrict__ S) {
  __shared__ double qs[kScD][kScQ];      // [k][query row]
  __shared__ double cs[kScD][kScK + 1];  // [k][key] (+1: the transposing stores spread over banks)
  const int i0 = blockIdx.x * kScQ, j0 = blockIdx.y * kScK, bh = blockIdx.z, tid = threadIdx.x;
  const int tx = tid & 31, ty = tid >> 5;
  double acc[4][4];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int u = 0; u < 4; ++u) acc[r][u] = 0.0;
  const float* cqb = cq + size_t(bh) * Cq * d;
  const float* ckb = ck + size_t(bh) * Ck * d;
  for (int k0 = 0; k0 < d; k0 += kScD) {
    __syncthreads();
    // 32 rows x 32 dims of the query centroids and 128 x 32 of the key centroids: lane = dimension (128-byte rows)
    for (int e = tid; e < kScQ * kScD; e += kSelThreads) {
      const int r = e / kScD, k = e % kScD;
      qs[k][r] = i0 + r < Cq ? double(__ldg(cqb + size_t(i0 + r) * d + k0 + k)) : 0.0;
    }
    for (int e = tid; e < kScK * kScD; e += kSelThreads) {
      const int jj = e / kScD, k = e % kScD;
      cs[k][jj] = j0 + jj < Ck ? double(__ldg(ckb + size_t(j0 + jj) * d + k0 + k)) : 0.0;
    }
    __syncthreads();
#pragma unroll 4
    for (int k = 0; k < kScD; ++k) {
      double qv[4], cv[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) qv[r] = qs[k][4 * ty + r];
#pragma unroll
      for (int u = 0; u < 4; ++u) cv[u] = cs[k][tx + 32 * u];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int u = 0; u < 4; ++u) acc[r][u] = fma(qv[r], cv[u], acc[r][u]);
    }
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int i = i0 + 4 * ty + r;
    if (i >= Cq) continue;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int j = j0 + tx + 32 * u;
      if (j < Ck) S[(size_t(bh) * Cq + i) * Ck + j] = scale * acc[r][u];
    }
  }
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

// Team-wide exclusive scan of per-thread counts in team-thread order (warp shuffle scan, then the team's warps in
// order); *total = the team's sum.  Every thread of the CTA must call it (block barriers when TW > 1).
template <int TW>
__device__ __forceinline__ int team_excl_scan(int v, int* total, long long (*red)[kSelWarps], int& parity, int warp,
                                              int row) {
  const int lane = threadIdx.x & 31;
  int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  int pos = incl - v;
  *total = __shfl_sync(0xffffffffu, incl, 31);
  if constexpr (TW > 1) {
    if (lane == 31) red[parity][warp] = incl;
    __syncthreads();
    int tot = 0;
    const int wt = warp % TW;
#pragma unroll
    for (int u = 0; u < TW; ++u) {
      const int c = int(red[parity][row * TW + u]);
      if (u < wt) pos += c;
      tot += c;
    }
    *total = tot;
    parity ^= 1;
  }
  return pos;
}

// One CTA per (R query clusters, bh); row r is owned by a team of TW = 8 / R warps.  A row's entries live in
// registers, E per thread (entry j = team_thread * E + i, ascending j), 32 * TW * E >= Ck.
//   1) S of the entries (k_scores), row max over non-empty j (R9); w = |K_j| exp(S - m) (Eq. 2); Z by a fixed tree.
//   2) top-p without sorting (R27): with B(v) = sum of the w >= v, the ranks the sorted walk selects (mass before
//      the rank < p Z) are exactly the w >= w*, w* = max{v : B(v) >= p Z} -- the first rank whose inclusive mass
//      reaches p Z.  B is monotone in v and positive doubles order like their bit patterns, so w* is found bit by
//      bit from the top: 11 team sums over all entries fix its binade, whose weights are compacted into shared memory
//      and narrowed 8 bits per level while more than kShortList remain; a short list is resolved directly (see the
//      code).  Entries equal to w* (only equal centroids and sizes give such ties) are then ordered by ascending j as
//      the sort would: the k-th of them is selected iff B(> w*) + k w* < p Z.
template <int E, int R>
__global__ void __launch_bounds__(kSelThreads) k_select(const double* __restrict__ S, const int32_t* __restrict__ sq,
                                                        const int32_t* __restrict__ sk, int Cq, int Ck, double top_p,
                                                        uint8_t* __restrict__ mask,
                                                        unsigned long long* __restrict__ pairs) {
  constexpr int TW = kSelWarps / R;  // warps per row
  constexpr int TT = 32 * TW;        // threads per row
  extern __shared__ __align__(16) unsigned char smem[];
  double* wlist = reinterpret_cast<double*>(smem);             // [R][TT * E] the binade's weights (top-p search)
  double* wlist2 = wlist + R * TT * E;                         // [R][TT * E] its next compaction
  int* sks = reinterpret_cast<int*>(wlist2 + R * TT * E);      // [Ck]
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
    // ---- w* bit by bit: t = max{v : B(v) >= target}; stays 0 (select every w > 0) if no v reaches it.  The sign and
    // exponent bits (62..52) take team passes over every entry (high words compared); that fixes the binade
    // [t, t + 2^52) holding w*.
    unsigned long long t = 0;
    for (int b = 62; b >= 52; --b) {
      const unsigned int ch = unsigned((t | (1ull << b)) >> 32);
      double part0 = 0.0, part1 = 0.0;
#pragma unroll
      for (int i = 0; i < E; i += 2) {
        part0 += unsigned(__double2hiint(w[i])) >= ch ? w[i] : 0.0;
        if (i + 1 < E) part1 += unsigned(__double2hiint(w[i + 1])) >= ch ? w[i + 1] : 0.0;
      }
      if (team_sum<TW>(part0 + part1, red_w, pw, warp, row) >= target) t |= 1ull << b;
    }
    // Narrowing: the interval [t, t + 2^lo) holds w*; `above` is the mass of the entries above it and the list in
    // shared memory its entries (in a fixed order).  While a list is long (weights within a factor of 2 of each other),
    // the team takes 8 more bits in passes over the list, spread evenly over its threads, and compacts it again; a
    // short list (the usual case after the exponent) is resolved directly: w* is the largest entry v whose
    // B(v) = above + (list entries >= v, in list order) reaches the target.
    int lo = 52;
    double above = 0.0;
    int nlist = 0;
    double* lst = wlist + row * (TT * E);
    {
      const unsigned long long thi = t + (1ull << lo);
      int nin = 0;
#pragma unroll
      for (int i = 0; i < E; ++i) {
        const unsigned long long bits = (unsigned long long)__double_as_longlong(w[i]);
        if (w[i] > 0.0 && bits >= thi) above += w[i];
        nin += (w[i] > 0.0 && bits >= t && bits < thi) ? 1 : 0;
      }
      above = team_sum<TW>(above, red_w, pw, warp, row);
      int pos = team_excl_scan<TW>(nin, &nlist, red_k, pk, warp, row);
#pragma unroll
      for (int i = 0; i < E; ++i) {
        const unsigned long long bits = (unsigned long long)__double_as_longlong(w[i]);
        if (w[i] > 0.0 && bits >= t && bits < thi) lst[pos++] = w[i];
      }
      __syncthreads();
    }
    double* nxt = wlist2 + row * (TT * E);  // the compacted list goes to the other buffer (ping-pong)
    while (__syncthreads_or(nlist > kShortList && lo > 0)) {  // CTA-uniform: the team reductions synchronise the CTA
      const bool act = nlist > kShortList && lo > 0;
      const int nb = act ? min(8, lo) : 0;
#pragma unroll 1
      for (int q = 1; q <= 8; ++q) {
        const bool live = q <= nb;
        const unsigned long long cand = live ? t | (1ull << (lo - q)) : ~0ull;
        double p0 = 0.0, p1 = 0.0;
        int k = tt;
        for (; k + TT < nlist; k += 2 * TT) {  // this thread's list entries tt + TT m
          const double x0 = lst[k], x1 = lst[k + TT];
          p0 += (unsigned long long)__double_as_longlong(x0) >= cand ? x0 : 0.0;
          p1 += (unsigned long long)__double_as_longlong(x1) >= cand ? x1 : 0.0;
        }
        if (k < nlist) p0 += (unsigned long long)__double_as_longlong(lst[k]) >= cand ? lst[k] : 0.0;
        const double bsum = team_sum<TW>(p0 + p1, red_w, pw, warp, row);
        if (live && above + bsum >= target) t = cand;
      }
      lo -= nb;
      const unsigned long long thi = act ? t + (1ull << lo) : ~0ull;
      double ab = 0.0;
      int nin = 0;
      for (int k = tt; k < nlist; k += TT) {
        const double x = lst[k];
        const unsigned long long bits = (unsigned long long)__double_as_longlong(x);
        if (act && bits >= thi) ab += x;
        nin += (act && bits >= t && bits < thi) ? 1 : 0;
      }
      ab = team_sum<TW>(ab, red_w, pw, warp, row);
      int nnew;
      int pos = team_excl_scan<TW>(nin, &nnew, red_k, pk, warp, row);
      if (act) {
        above += ab;
        for (int k = tt; k < nlist; k += TT) {
          const double x = lst[k];
          const unsigned long long bits = (unsigned long long)__double_as_longlong(x);
          if (bits >= t && bits < thi) nxt[pos++] = x;
        }
        nlist = nnew;
        double* tmp = lst;
        lst = nxt;
        nxt = tmp;
      }
      __syncthreads();
    }
    if (lo > 0) {  // every warp of the team resolves the short list itself (same entries, same order: same t)
      unsigned long long best = 0;
      for (int i = lane; i < nlist; i += 32) {
        const unsigned long long bi = (unsigned long long)__double_as_longlong(lst[i]);
        double s0 = 0.0, s1 = 0.0;
        int k = 0;
        for (; k + 1 < nlist; k += 2) {
          const double x0 = lst[k], x1 = lst[k + 1];
          s0 += (unsigned long long)__double_as_longlong(x0) >= bi ? x0 : 0.0;
          s1 += (unsigned long long)__double_as_longlong(x1) >= bi ? x1 : 0.0;
        }
        if (k < nlist) s0 += (unsigned long long)__double_as_longlong(lst[k]) >= bi ? lst[k] : 0.0;
        if (above + (s0 + s1) >= target) best = max(best, bi);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
      t = max(t, best);
    }
    // ---- entries equal to w*: the sort orders them by ascending j
    const double wstar = __longlong_as_double((long long)t);
    int nt = 0;
#pragma unroll
    for (int i = 0; i < E; ++i) nt += (w[i] > 0.0 && w[i] == wstar) ? 1 : 0;
    const long long ties = team_sum_ll<TW>(nt, red_k, pk, warp, row);
    // mass strictly above w* and each tied entry's rank among the ties (team exclusive scan); computed by every
    // team (the reductions synchronise the CTA) but used only when w* is tied
    double above_t = 0.0;
#pragma unroll
    for (int i = 0; i < E; ++i) above_t += (unsigned long long)__double_as_longlong(w[i]) > t ? w[i] : 0.0;
    above_t = team_sum<TW>(above_t, red_w, pw, warp, row);
    int ntot;
    long long rank = team_excl_scan<TW>(nt, &ntot, red_k, pk, warp, row);
#pragma unroll
    for (int i = 0; i < E; ++i) {
      const int j = tt * E + i;
      const unsigned long long bits = (unsigned long long)__double_as_longlong(w[i]);
      bool take = w[i] > 0.0 && bits > t;
      if (w[i] > 0.0 && bits == t) {
        take = ties <= 1 || above_t + double(rank) * wstar < target;
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
  const size_t smem = 2 * size_t(kSelThreads) * E * sizeof(double) + size_t(Ck) * sizeof(int) + size_t(R) * Ck;
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
  k_scores<<<dim3((Cq + kScQ - 1) / kScQ, (Ck + kScK - 1) / kScK, BH), kSelThreads, 0, s>>>(
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

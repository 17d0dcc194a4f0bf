// internal.h — launchers and workspace layout shared by the svg2 CUDA translation units (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <cstddef>
#include <cstdint>

namespace svg2 {

constexpr int kSortTile = 2048;      // labels per histogram / stable-scatter tile
constexpr int kMaxClusters = 4096;   // C limit (a select_topp row of Ck weights lives in one CTA)
constexpr int kQTile = 128;          // query rows per tcgen05 M=128 tile
constexpr int kKTile = 128;          // keys per S tile (N of the QK^T MMA, K of the PV MMA)
constexpr int kItemRows = 2 * kQTile;  // one attention work item = two Q tiles of one query cluster
// Work item int4 = {first flat row of Q', rows_a | rows_b << 16, stream index, bh | flags}.  kItemSplit marks an
// item with one Q tile and >= 2 key tiles: the attention kernels give its even key tiles to one softmax warpgroup and
// the odd ones to the other and merge the two partial softmax states.
constexpr int kItemSplit = 1 << 30;
constexpr int kItemBhMask = kItemSplit - 1;

// A [B, H, N, d] bf16 tensor (Q, K or V of the fused call) with d contiguous and element strides (sB, sH, sN): head
// bh = b * H + h, token n.  The contiguous layout is (H N d, N d, d); the token-major buffer of a Ulysses all-to-all
// [B, N, H, d] is (N H d, d, H d) and is read in place.
struct XView {
  const void* p = nullptr;
  long long sB = 0, sH = 0, sN = 0;
  int H = 1;
  __host__ __device__ const uint16_t* row(int bh, long long n) const {
    return static_cast<const uint16_t*>(p) + (bh / H) * sB + (bh % H) * sH + n * sN;
  }
  __host__ __device__ bool contiguous(int N, int d) const { return sN == d && sH == (long long)N * d && sB == H * sH; }
};
inline XView contiguous_view(const void* p, int B, int H, int N, int d) {
  (void)B;
  XView v;
  v.p = p;
  v.sN = d;
  v.sH = (long long)N * d;
  v.sB = (long long)H * N * d;
  v.H = H;
  return v;
}

// Where the attention writes output row (bh, token n): the fused A10 scatter, optionally straight into the
// token-sharded output buffers of a sequence-parallel caller (the reverse Ulysses all-to-all fused into the epilogue:
// shard s holds tokens [s * shard_tokens, (s + 1) * shard_tokens); peers' shards are IPC / symmetric-memory mappings).
constexpr int kMaxShards = 16;
struct OutView {
  void* shard[kMaxShards] = {};
  int n_shards = 1;
  int shard_tokens = 0;
  long long sB = 0, sH = 0, sN = 0;  // element strides inside a shard
  int H = 1;                         // heads of the call (bh -> b, h)
  int head_offset = 0;               // added to h (this call's heads inside the shard's head dimension)
  __host__ __device__ uint16_t* row(int bh, long long n) const {
    const int s = n_shards == 1 ? 0 : int(n / shard_tokens);
    const long long local = n - (long long)s * shard_tokens;
    return static_cast<uint16_t*>(shard[s]) + (bh / H) * sB + (bh % H + head_offset) * sH + local * sN;
  }
};
inline OutView contiguous_out(void* O, int H, int N, int d) {
  OutView o;
  o.shard[0] = O;
  o.shard_tokens = N;
  o.sN = d;
  o.sH = (long long)N * d;
  o.sB = (long long)H * N * d;
  o.H = H;
  return o;
}

inline int sort_tiles(int N) { return (N + kSortTile - 1) / kSortTile; }
inline int items_cap_per_bh(int Nq, int Cq) { return (Nq + kItemRows - 1) / kItemRows + Cq; }

// Bump allocator over the caller's workspace: the same code computes the size (base == nullptr) and the
// pointers, so the two can never disagree.
struct Carver {
  char* base;
  size_t off = 0;
  explicit Carver(void* b) : base(static_cast<char*>(b)) {}
  template <typename T>
  T* take(size_t count) {
    off = (off + 255) & ~size_t(255);
    T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off += count * sizeof(T);
    return p;
  }
};

struct SortWs {  // histogram/scan/stable-scatter scratch
  int32_t* tile_counts;  // [BH, T, C]
};
inline SortWs carve_sort(Carver& c, int BH, int N, int C) {
  SortWs w;
  w.tile_counts = c.take<int32_t>(size_t(BH) * sort_tiles(N) * C);
  return w;
}

constexpr int kCentChunk = 128;  // centroids per tcgen05 N-chunk in the assign kernel
inline int cent_pad(int C) { return (C + kCentChunk - 1) / kCentChunk * kCentChunk; }

struct KmeansWs {
  SortWs sort;
  int32_t* perm;      // [BH, N]   (used when the caller does not want perm)
  int32_t* offsets;   // [BH, C+1]
  uint16_t* c_hi;     // [BH, Cpad, d] bf16 hi part of the centroids (assign operand)
  uint16_t* c_lo;     // [BH, Cpad, d] bf16 lo part: c - hi
  float* c_norm;      // [BH, Cpad]  ||c||^2 (f32), +inf for padding centroids
  double* c_sum;      // [BH, C, d]  fp64 sums of the clusters that lie inside one update chunk
  double* c_part;     // [BH, ceil(N/kUpdRows), 2, d]  fp64 chunk partials of clusters crossing chunk boundaries
  double* c_sq;       // [BH, C]  (objective) sum ||x||^2 per cluster, as c_sum
  double* c_sqpart;   // [BH, ceil(N/kUpdRows), 2]
  double* j_part;     // [BH, C, 2]  (objective) per-cluster J before / after the update
  void* pp;           // k-means++ seeding scratch (kmeanspp_ws_bytes)
};
constexpr int kUpdRows = 32;  // rows per chunk (one warp) of the segmented centroid reduction
constexpr int kPPMaxBlocks = 64;  // k-means++: CTAs per head
size_t kmeanspp_ws_bytes(int BH, int N);
inline KmeansWs carve_kmeans(Carver& c, int BH, int N, int C, int d = 128) {
  KmeansWs w;
  w.sort = carve_sort(c, BH, N, C);
  w.perm = c.take<int32_t>(size_t(BH) * N);
  w.offsets = c.take<int32_t>(size_t(BH) * (C + 1));
  w.c_hi = c.take<uint16_t>(size_t(BH) * cent_pad(C) * d);
  w.c_lo = c.take<uint16_t>(size_t(BH) * cent_pad(C) * d);
  w.c_norm = c.take<float>(size_t(BH) * cent_pad(C));
  w.c_sum = c.take<double>(size_t(BH) * C * d);
  const size_t nch = (size_t(N) + kUpdRows - 1) / kUpdRows;
  w.c_part = c.take<double>(size_t(BH) * nch * 2 * d);
  w.c_sq = c.take<double>(size_t(BH) * C);
  w.c_sqpart = c.take<double>(size_t(BH) * nch * 2);
  w.j_part = c.take<double>(size_t(BH) * C * 2);
  w.pp = c.take<uint8_t>(kmeanspp_ws_bytes(BH, N));
  return w;
}

// Key stream of one query cluster = its selected key clusters' rows in K'/V', adjacent clusters merged into runs,
// every run padded to whole 8-row groups.  A group = (first row in the flattened [BH*Nk] key tensor, #valid rows
// 0..8).  The stream is padded to an even number of groups so every tile has N = 16*k keys.  Tile t = groups
// [gpt t, gpt t + gpt) (gpt = attn_groups_per_tile: 10 or 16); its valid counts are also packed 4 bits each into one
// 64-bit tile word for the softmax mask.  tile_cap covers the smallest tile (kMinGroupsPerTile groups).
constexpr int kMinGroupsPerTile = 8;
inline size_t group_cap(int Nk, int Ck) { return size_t(Nk) / 8 + size_t(Ck) + 2; }
inline size_t tile_cap(int Nk, int Ck) { return group_cap(Nk, Ck) / kMinGroupsPerTile + 1; }

struct AttnWs {
  int2* groups;        // [BH, Cq, group_cap]
  uint64_t* tilew;     // [BH, Cq, tile_cap]
  int32_t* ngroups;    // [BH, Cq]
  int32_t* order;      // [BH, Cq] query clusters of each head in work-list order (longest key stream first)
  int4* items;         // [BH * cap] flattened
  int32_t* n_items;    // [3]: item count, dynamic-scheduler counter, query rows with an empty key stream
  long long* keys;     // [BH, Cq] selected key rows of each query cluster's stream
  uint8_t* owned;      // [BH, Cq] query cluster belongs to this call's part (QPart)
  size_t gcap, tcap;
};
inline AttnWs carve_attn(Carver& c, int BH, int Nq, int Nk, int Cq, int Ck) {
  AttnWs w;
  const size_t cap = items_cap_per_bh(Nq, Cq);
  w.gcap = group_cap(Nk, Ck);
  w.tcap = tile_cap(Nk, Ck);
  w.groups = c.take<int2>(size_t(BH) * Cq * w.gcap);
  w.tilew = c.take<uint64_t>(size_t(BH) * Cq * w.tcap);
  w.ngroups = c.take<int32_t>(size_t(BH) * Cq);
  w.order = c.take<int32_t>(size_t(BH) * Cq);
  w.items = c.take<int4>(size_t(BH) * cap);
  w.n_items = c.take<int32_t>(3);
  w.keys = c.take<long long>(size_t(BH) * Cq);
  w.owned = c.take<uint8_t>(size_t(BH) * Cq);
  return w;
}

// ---- launchers (return cudaGetLastError() of their launches)
cudaError_t launch_stable_sort(const int32_t* labels, int BH, int N, int C, SortWs ws, int32_t* perm,
                               int32_t* offsets, int32_t* sizes, cudaStream_t s);
cudaError_t launch_gather_rows(const int32_t* perm, int BH, int N, int d, const void* X0, void* X0p,
                               const void* X1, void* X1p, cudaStream_t s);
cudaError_t launch_scatter_rows(const void* Op, const int32_t* perm, int BH, int N, int d, void* O, cudaStream_t s);
// FP8 PV: per-(head, channel) |x| max (amax [BH, d], f32 bits) and the gather of X[perm] rounded to e4m3 with channel
// scales 448 / amax_c
// FP8 PV (R26): per-(b,h,channel) max |V| into amax (zeroed here), then V' = V[perm] in e4m3 with channel scales
cudaError_t launch_absmax(int BH, int N, int d, XView X, uint32_t* amax, cudaStream_t s);
cudaError_t launch_gather_rows_e4m3(const int32_t* perm, int BH, int N, int d, XView X, void* Xq,
                                    const uint32_t* amax, cudaStream_t s);
// k-means cold-start options (DESIGN R2, R25): strided rows, or k-means++ with the R25 generator
struct KmeansInit {
  bool kmeanspp = false;
  uint32_t seed = 0;
  int role = 0;     // 0 = Q, 1 = K (part of the generator's stream id)
  int bh_base = 0;  // global (b,h) index of the first head of this launch (chunked calls keep the stream ids)
};
// Optional gather fused into the last update pass: Xp = pi X and Yp = pi Y (rows permuted by the final labels).
struct KmeansGather {
  void* Xp = nullptr;
  XView Y;  // Y.p == nullptr: no second tensor
  void* Yp = nullptr;
  cudaEvent_t wait_y = nullptr;  // Y may still be arriving (host pipeline): the gather pass waits for this event
};
cudaError_t launch_kmeans(XView X, int BH, int N, int d, int C, int iters, bool warm, float* centroids,
                          int32_t* labels, int32_t* sizes, int32_t* perm, int32_t* offsets, KmeansWs ws,
                          cudaStream_t s, int* launches, const KmeansInit& init = KmeansInit(),
                          const KmeansGather& g = KmeansGather(), double* objective = nullptr);
// S: fp64 workspace [BH, Cq, Ck] (select_ws_bytes) for the Eq. 1 scores
inline size_t select_ws_elems(int BH, int Cq, int Ck) { return size_t(BH) * Cq * Ck; }
cudaError_t launch_select_topp(const float* cq, const float* ck, const int32_t* sq, const int32_t* sk, int BH,
                               int Cq, int Ck, int d, float scale, double top_p, uint8_t* mask, int64_t* pairs,
                               double* S, cudaStream_t s);
// The attention's output rows, for the NaN fill of query clusters with an empty key stream (k_items)
struct OrphanFill {
  const int32_t* q_perm;  // nullable: rows in permuted order (then out.shard[0] is O [BH, Nq, d])
  OutView out;
  float* lse;             // nullable
  int d;
};
// Query-cluster partition of the attention (multi-GPU split of a head): only the clusters of parts
// [begin, end) of `count` get work items; parts are cut by the cumulative selected-pair cost |Q_i| * keys_i of the head.
struct QPart {
  int begin = 0, end = 1, count = 1;
};
// key-stream tile size (8-row groups) the attention pipeline for (d, FP8 PV) runs on: the work list must match it
int attn_groups_per_tile(int d, bool fp8);
cudaError_t launch_build_worklist(const int32_t* q_offsets, const int32_t* k_offsets, const uint8_t* mask, int BH,
                                  int Nq, int Nk, int Cq, int Ck, int gpt, AttnWs ws, OrphanFill of, cudaStream_t s,
                                  QPart part = QPart());
cudaError_t launch_varblock_attention(const void* Qp, const void* Kp, const void* Vp, int BH, int Nq, int Nk, int d,
                                      float scale, const int32_t* q_perm, const OutView& out, float* lse, AttnWs ws,
                                      cudaStream_t s, const uint32_t* v_amax = nullptr);
// top_p = 1: every query cluster selects every non-empty key cluster, so the attention of a head is one query range
// [0, Nq) over the whole key stream: q_offsets [BH, 2] = {0, Nq}, mask [BH, Ck] = 1 (no per-cluster Q-tile padding)
cudaError_t launch_dense_stream(int BH, int Nq, int Ck, int32_t* q_offsets, uint8_t* mask, cudaStream_t s);
int kmeans_launch_count(int iters, bool warm, bool objective = false);
cudaError_t launch_kmeanspp(XView X, int BH, int N, int d, int C, uint32_t seed, int role, int bh_base,
                            float* cent, void* ws, cudaStream_t s);
int kmeanspp_launch_count(int BH, int N, int d);
constexpr int kSortLaunches = 3, kWorklistLaunches = 3;

}  // namespace svg2

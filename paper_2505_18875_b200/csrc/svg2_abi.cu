// svg2_abi.cu — the extern "C" boundary declared in include/svg2.h: synchronous validation (no launch, no output
// touched on error), workspace carving, and the enqueue of the kernels of svg2_*.cu on the caller's stream.
#include <cuda_runtime.h>
#include <cmath>
#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: stage ranges for nsys / ncu --nvtx (no-ops without a tool)
#include "../../include/svg2.h"
#include "internal.h"

using namespace svg2;

namespace {

constexpr long long kMaxN = 1ll << 24;
constexpr int kMaxHostChunks = 64;
// host pipeline: device staging slots (chunk ci uses slot ci % kHostSlots) and compute streams (<= kHostSlots)
constexpr int kHostSlots = 3, kHostComputeStreams = 3;  // e2e HunyuanVideo: 62.7 / 57.9 / 57.5 ms with 1 / 2 / 3
// middle chunks of the host pipeline (e2e, HunyuanVideo, one compute stream: 67.1 / 63.4 / 63.1 / 61.7 ms with
// 2 / 3 / 4 / 6 middle chunks + ramp, 64.6 ms with 6 equal chunks; two compute streams: 59.7 / 57.5 / 58.4 ms with
// 4 / 6 / 9)
constexpr int kHostChunks = 6;
// chunk sizes (heads) before and after the middle chunks: only the first chunk's upload and the last chunk's download
// are not overlapped with computation
// (e2e, HunyuanVideo, interleaved A/B on one box: 1,1,2,2 | 6 | 2,1 -> 52.98 ms mean of 4 vs 53.72 for 1,2 | 6 | 2,1;
// 1,1,2 | 6 | 1 53.8-54.2, 1,2 | 8 | 1 53.4-53.6, 1,1,1,2 | 5 | 1,1 54.0-56.0)
constexpr int kRampUp[] = {1, 1, 2, 2}, kRampDown[] = {2, 1};
static_assert(kHostChunks + 16 <= kMaxHostChunks, "host chunks");

svg2_status_t check_device() {
  int dev = 0, major = 0, minor = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return SVG2_ERR_CUDA;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  if (major != 10 || minor != 0) return SVG2_ERR_UNSUPPORTED_DEVICE;
  return SVG2_OK;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

svg2_status_t check_bhnd(long long B, long long H, long long N, long long d) {
  if (B <= 0 || H <= 0 || N <= 0) return SVG2_ERR_INVALID_SHAPE;
  if (d != 64 && d != 128) return SVG2_ERR_INVALID_SHAPE;
  if (N > kMaxN || B * H * N >= (1ll << 31)) return SVG2_ERR_INVALID_SHAPE;
  return SVG2_OK;
}

svg2_status_t check_clusters(long long C, long long N) {
  if (C < 1 || C > N || C > kMaxClusters) return SVG2_ERR_INVALID_PARAM;
  return SVG2_OK;
}

svg2_status_t from_cuda(cudaError_t e) { return e == cudaSuccess ? SVG2_OK : SVG2_ERR_CUDA; }

// Sticky or pending errors from earlier asynchronous work are reported (and cleared) before new work.
svg2_status_t pending_error() { return from_cuda(cudaGetLastError()); }

float resolve_scale(float scale, int d) { return scale > 0.f ? scale : float(1.0 / std::sqrt(double(d))); }

struct AuxStream {  // a caller-owned stream and two events for the K-role fork (svg2_layout_t.aux_*)
  cudaStream_t stream = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};

struct FusedWs {
  int32_t *lab_q, *lab_k, *perm_q, *perm_k, *off_q, *off_k, *size_q, *size_k;
  void *Qp, *Kp, *Vp;
  uint8_t* mask;
  double* scores;    // [BH, Cq, Ck] fp64 Eq. 1 scores of the selection
  int32_t* dense_qoff;  // top_p = 1: [BH, 2] one query range per head
  uint8_t* dense_mask;  // top_p = 1: [BH, Ck] all key clusters
  uint32_t* v_amax;  // FP8 PV: per-(head, channel) max |V| (f32 bits) [BH, d]
  KmeansWs km_q, km_k;  // per-role k-means scratch: the two roles may run concurrently
  AttnWs attn;
};

FusedWs carve_fused(Carver& c, const svg2_dims_t& dm, const svg2_config_t& cfg) {
  const size_t BH = size_t(dm.B) * dm.H;
  FusedWs w;
  w.lab_q = c.take<int32_t>(BH * dm.Nq);
  w.lab_k = c.take<int32_t>(BH * dm.Nk);
  w.perm_q = c.take<int32_t>(BH * dm.Nq);
  w.perm_k = c.take<int32_t>(BH * dm.Nk);
  w.off_q = c.take<int32_t>(BH * (cfg.Cq + 1));
  w.off_k = c.take<int32_t>(BH * (cfg.Ck + 1));
  w.size_q = c.take<int32_t>(BH * cfg.Cq);
  w.size_k = c.take<int32_t>(BH * cfg.Ck);
  w.Qp = c.take<uint16_t>(BH * dm.Nq * dm.d);
  w.Kp = c.take<uint16_t>(BH * dm.Nk * dm.d);
  w.Vp = c.take<uint16_t>(BH * dm.Nk * dm.d);
  w.mask = c.take<uint8_t>(BH * cfg.Cq * cfg.Ck);
  w.scores = c.take<double>(select_ws_elems(int(BH), cfg.Cq, cfg.Ck));
  w.dense_qoff = c.take<int32_t>(BH * 2);
  w.dense_mask = c.take<uint8_t>(BH * cfg.Ck);
  w.v_amax = c.take<uint32_t>(BH * dm.d);
  w.km_q = carve_kmeans(c, int(BH), dm.Nq, cfg.Cq);
  w.km_k = carve_kmeans(c, int(BH), dm.Nk, cfg.Ck);
  w.attn = carve_attn(c, int(BH), dm.Nq, dm.Nk, cfg.Cq, cfg.Ck);
  return w;
}

svg2_status_t validate_fused(const svg2_dims_t& dm, const svg2_config_t* cfg) {
  if (!cfg) return SVG2_ERR_NULL_POINTER;
  svg2_status_t st = check_bhnd(dm.B, dm.H, dm.Nq, dm.d);
  if (st != SVG2_OK) return st;
  if ((st = check_bhnd(dm.B, dm.H, dm.Nk, dm.d)) != SVG2_OK) return st;
  if ((st = check_clusters(cfg->Cq, dm.Nq)) != SVG2_OK) return st;
  if ((st = check_clusters(cfg->Ck, dm.Nk)) != SVG2_OK) return st;
  if (cfg->iters < 1) return SVG2_ERR_INVALID_PARAM;
  if (!(cfg->top_p > 0.0 && cfg->top_p <= 1.0)) return SVG2_ERR_INVALID_PARAM;
  if (!(cfg->scale >= 0.f) || std::isinf(cfg->scale)) return SVG2_ERR_INVALID_PARAM;
  if (cfg->flags & ~(SVG2_WARM_START | SVG2_INIT_KMEANSPP | SVG2_FP8_PV)) return SVG2_ERR_INVALID_PARAM;
  if ((cfg->flags & SVG2_FP8_PV) && dm.d != 128) return SVG2_ERR_INVALID_PARAM;
  return SVG2_OK;
}

// The whole fused call for the heads of `dm` on stream s (arguments validated by the caller).  bh_base = global
// (b,h) index of the first head (k-means++ stream ids of chunked calls, R25).
// Q, K, V as strided views, the output rows through `out`, the attention restricted to query-cluster part `part`.
cudaError_t run_fused(const XView& Q, const XView& K, const XView& V, const svg2_dims_t& dm, const svg2_config_t* cfg,
                      float* q_centroids, float* k_centroids, const OutView& out, int64_t* selected_pairs,
                      const svg2_debug_t* dbg, FusedWs w, cudaStream_t s, int bh_base,
                      const cudaEvent_t* arrive = nullptr, QPart part = QPart(), const AuxStream* aux = nullptr) {
  // arrive (host pipeline): events of Q, K and V landing in device memory; each role waits only for its own tensor,
  // V only before the pass that gathers it
  if (dbg) {  // intermediates requested: write them straight into the caller's buffers
    if (dbg->q_labels) w.lab_q = dbg->q_labels;
    if (dbg->k_labels) w.lab_k = dbg->k_labels;
    if (dbg->q_perm) w.perm_q = dbg->q_perm;
    if (dbg->k_perm) w.perm_k = dbg->k_perm;
    if (dbg->q_offsets) w.off_q = dbg->q_offsets;
    if (dbg->k_offsets) w.off_k = dbg->k_offsets;
    if (dbg->mask) w.mask = dbg->mask;
  }
  // stage boundaries: the caller's timing events (dbg) and NVTX ranges around each stage's enqueue
  static const char* const kStageNames[7] = {"svg2 kmeans K (forked stream)", "svg2 kmeans Q", "svg2 permute V (fp8)",
                                             "svg2 select_topp", "svg2 worklist", "svg2 varblock_attention", ""};
  auto mark = [&](int k) {
    if (dbg && dbg->events[k]) cudaEventRecord(static_cast<cudaEvent_t>(dbg->events[k]), s);
    if (k > 0 && k < 7) nvtxRangePop();
    if (k < 6) nvtxRangePushA(kStageNames[k]);
  };
  const int BH = dm.B * dm.H;
  const bool warm = cfg->flags & SVG2_WARM_START;
  const float scale = resolve_scale(cfg->scale, dm.d);
  cudaError_t e = cudaSuccess;
  mark(0);
  KmeansInit init_q, init_k;
  init_q.kmeanspp = init_k.kmeanspp = (cfg->flags & SVG2_INIT_KMEANSPP) != 0;
  init_q.seed = init_k.seed = cfg->seed;
  init_q.role = 0;
  init_k.role = 1;
  init_q.bh_base = init_k.bh_base = bh_base;
  // A6 rides on the last Lloyd update: that pass already reads every row through the final permutation, so it also
  // writes Q' = pi_q Q, K' = pi_k K and (bf16 PV) V' = pi_k V
  const bool fp8 = (cfg->flags & SVG2_FP8_PV) != 0;
  KmeansGather gq, gk;
  gq.Xp = w.Qp;
  gk.Xp = w.Kp;
  if (!fp8) {
    gk.Y = V;
    gk.Yp = w.Vp;
  }
  // The K role (the longer one: C_k > C_q) on a forked stream of the highest priority, enqueued first, so that its
  // kernels win the SMs whenever both roles have work ready; the Q role on s.  The k-means++ cold start (cooperative
  // launches) stays on one stream.
  cudaStream_t s2 = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  const bool pp_cold = !warm && init_q.kmeanspp;
  const bool own = !(aux && aux->stream);  // the caller may lend a stream and two events (no per-call creation)
  cudaStreamCaptureStatus capture = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(s, &capture);  // capturing: only a lent stream forks (event fork / join is capture-legal)
  if (!pp_cold && !own) {
    s2 = aux->stream;
    ev_fork = aux->fork;
    ev_join = aux->join;
    if (cudaEventRecord(ev_fork, s) != cudaSuccess || cudaStreamWaitEvent(s2, ev_fork, 0) != cudaSuccess) {
      s2 = nullptr;
      (void)cudaGetLastError();
    }
  } else if (!pp_cold && capture == cudaStreamCaptureStatusNone) {
    int prio_low = 0, prio_high = 0;
    cudaDeviceGetStreamPriorityRange(&prio_low, &prio_high);
    if (cudaStreamCreateWithPriority(&s2, cudaStreamNonBlocking, prio_high) !=
            cudaSuccess ||
        cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventRecord(ev_fork, s) != cudaSuccess || cudaStreamWaitEvent(s2, ev_fork, 0) != cudaSuccess) {
      if (s2) cudaStreamDestroy(s2);
      s2 = nullptr;
      (void)cudaGetLastError();
    }
  }
  cudaStream_t sk = s2 ? s2 : s;  // K role
  if (arrive) {
    cudaStreamWaitEvent(sk, arrive[1], 0);
    if (gk.Yp) gk.wait_y = arrive[2];
  }
  e = launch_kmeans(K, BH, dm.Nk, dm.d, cfg->Ck, cfg->iters, warm, k_centroids, w.lab_k, w.size_k, w.perm_k, w.off_k,
                    w.km_k, sk, nullptr, init_k, gk, dbg ? dbg->k_objective : nullptr);
  mark(1);  // with two streams: the fork point (stage "kmeans_k" then covers both roles)
  if (arrive) cudaStreamWaitEvent(s, arrive[0], 0);
  if (e == cudaSuccess)
    e = launch_kmeans(Q, BH, dm.Nq, dm.d, cfg->Cq, cfg->iters, warm, q_centroids, w.lab_q, w.size_q, w.perm_q,
                      w.off_q, w.km_q, s, nullptr, init_q, gq, dbg ? dbg->q_objective : nullptr);
  // FP8 PV: the |V| channel maxima depend on V alone, so they run on the Q-role stream while the (longer) K role is
  // still clustering; only the e4m3 gather through pi_k waits for the join
  if (e == cudaSuccess && fp8) {
    if (arrive) cudaStreamWaitEvent(s, arrive[2], 0);
    e = launch_absmax(BH, dm.Nk, dm.d, V, w.v_amax, s);
  }
  if (s2) {  // join (always, so no work is left behind on s2 even after an error) and release (deferred by CUDA)
    cudaEventRecord(ev_join, s2);
    cudaStreamWaitEvent(s, ev_join, 0);
    if (own) cudaStreamDestroy(s2);
  }
  if (own && ev_fork) cudaEventDestroy(ev_fork);
  if (own && ev_join) cudaEventDestroy(ev_join);
  mark(2);
  if (arrive && !gk.wait_y) cudaStreamWaitEvent(s, arrive[2], 0);  // V gathered by a separate pass (FP8 PV)
  // FP8 PV (R26): V' in e4m3 with a per-head scale, written into the first half of the bf16 V' buffer
  if (e == cudaSuccess && fp8) e = launch_gather_rows_e4m3(w.perm_k, BH, dm.Nk, dm.d, V, w.Vp, w.v_amax, s);
  mark(3);
  if (e == cudaSuccess)
    e = launch_select_topp(q_centroids, k_centroids, w.size_q, w.size_k, BH, cfg->Cq, cfg->Ck, dm.d, scale,
                           cfg->top_p, w.mask, selected_pairs, w.scores, s);
  mark(4);
  // top_p = 1 (and no query-cluster split): every query cluster selects every non-empty key cluster (R11), so the
  // attention runs each head as one query range over the whole key stream -- the same key order and the same result
  // up to the lazy-rescale points, without the per-cluster Q-tile padding (W480p: tile work 1.19 -> 1.00)
  const bool dense = cfg->top_p >= 1.0 && part.count == 1;
  if (e == cudaSuccess && dense) e = launch_dense_stream(BH, dm.Nq, cfg->Ck, w.dense_qoff, w.dense_mask, s);
  if (e == cudaSuccess)
    e = launch_build_worklist(dense ? w.dense_qoff : w.off_q, w.off_k, dense ? w.dense_mask : w.mask, BH, dm.Nq,
                              dm.Nk, dense ? 1 : cfg->Cq, cfg->Ck, attn_groups_per_tile(dm.d, fp8), w.attn,
                              OrphanFill{w.perm_q, out, nullptr, dm.d}, s, part);
  mark(5);
  if (e == cudaSuccess)
    e = launch_varblock_attention(w.Qp, w.Kp, w.Vp, BH, dm.Nq, dm.Nk, dm.d, scale, w.perm_q, out, nullptr, w.attn, s,
                                  fp8 ? w.v_amax : nullptr);
  mark(6);
  mark(7);
  return e;
}

// Host-buffer pipeline (svg2_sparse_attention_host): heads in chunks, double-buffered device staging.
struct HostPlan {
  int BH, hc, nchunks;      // hc = the largest chunk (staging size)
  int start[kMaxHostChunks + 1];  // chunk c = heads [start[c], start[c+1])
};
// Head chunks of the host pipeline.  Only the first chunk's upload and the last chunk's download are not overlapped
// with computation, so the chunks ramp up (kRampUp: each upload shorter than the computation of the chunks before
// it) and down (kRampDown) around equal middle chunks (kHostChunks of them); small problems get one chunk per head.
HostPlan host_plan(const svg2_dims_t& dm) {
  HostPlan p;
  p.BH = dm.B * dm.H;
  int sizes[kMaxHostChunks], n = 0;
  const int mid_chunks = kHostChunks;
  int rest = p.BH;
  const int* up = kRampUp;
  const int* down = kRampDown;
  constexpr int nup = sizeof(kRampUp) / sizeof(int), ndown = sizeof(kRampDown) / sizeof(int);
  int ramp_heads = 0;
  for (int i = 0; i < nup; ++i) ramp_heads += up[i];
  for (int i = 0; i < ndown; ++i) ramp_heads += down[i];
  const bool use_ramp = p.BH >= ramp_heads + mid_chunks;
  if (use_ramp) {
    for (int i = 0; i < nup; ++i) sizes[n++] = up[i];
    rest -= ramp_heads;
  }
  const int m = rest < mid_chunks ? (rest > 0 ? rest : 1) : mid_chunks;
  for (int i = 0; i < m && rest > 0; ++i) {  // equal middle chunks (the first ones one head larger if uneven)
    const int sz = rest / (m - i) + (rest % (m - i) ? 1 : 0);
    sizes[n++] = sz;
    rest -= sz;
  }
  if (use_ramp)
    for (int i = 0; i < ndown; ++i) sizes[n++] = down[i];
  p.nchunks = n;
  p.hc = 1;
  p.start[0] = 0;
  for (int c = 0; c < n; ++c) {
    p.start[c + 1] = p.start[c] + sizes[c];
    p.hc = sizes[c] > p.hc ? sizes[c] : p.hc;
  }
  return p;
}
struct HostWs {
  void *Q[kHostSlots], *K[kHostSlots], *V[kHostSlots], *O[kHostSlots];
  FusedWs fused[kHostSlots];  // one per compute stream: consecutive chunks run concurrently
};
HostWs carve_host(Carver& c, const svg2_dims_t& dm, const svg2_config_t& cfg, const HostPlan& p) {
  HostWs w;
  const size_t q = size_t(p.hc) * dm.Nq * dm.d, k = size_t(p.hc) * dm.Nk * dm.d;
  for (int i = 0; i < kHostSlots; ++i) {
    w.Q[i] = c.take<uint16_t>(q);
    w.K[i] = c.take<uint16_t>(k);
    w.V[i] = c.take<uint16_t>(k);
    w.O[i] = c.take<uint16_t>(q);
  }
  const svg2_dims_t chunk{1, p.hc, dm.Nq, dm.Nk, dm.d};
  for (int i = 0; i < kHostSlots; ++i) w.fused[i] = carve_fused(c, chunk, cfg);
  return w;
}
}  // namespace

extern "C" {

const char* svg2_status_string(svg2_status_t s) {
  switch (s) {
    case SVG2_OK: return "SVG2_OK";
    case SVG2_ERR_NULL_POINTER: return "SVG2_ERR_NULL_POINTER";
    case SVG2_ERR_INVALID_SHAPE: return "SVG2_ERR_INVALID_SHAPE";
    case SVG2_ERR_INVALID_PARAM: return "SVG2_ERR_INVALID_PARAM";
    case SVG2_ERR_MISALIGNED: return "SVG2_ERR_MISALIGNED";
    case SVG2_ERR_WORKSPACE_TOO_SMALL: return "SVG2_ERR_WORKSPACE_TOO_SMALL";
    case SVG2_ERR_UNSUPPORTED_DEVICE: return "SVG2_ERR_UNSUPPORTED_DEVICE";
    case SVG2_ERR_CUDA: return "SVG2_ERR_CUDA";
    case SVG2_ERR_NOT_IMPLEMENTED: return "SVG2_ERR_NOT_IMPLEMENTED";
  }
  return "SVG2_UNKNOWN_STATUS";
}

int svg2_abi_version(void) { return SVG2_ABI_VERSION; }

size_t svg2_workspace_size(svg2_entry_t entry, svg2_dims_t dm, const svg2_config_t* cfg) {
  if (!cfg) return 0;
  const long long BH = (long long)dm.B * dm.H;
  Carver c(nullptr);
  switch (entry) {
    case SVG2_ENTRY_KMEANS:
      if (check_bhnd(dm.B, dm.H, dm.Nq, dm.d) != SVG2_OK || check_clusters(cfg->Cq, dm.Nq) != SVG2_OK) return 0;
      carve_kmeans(c, int(BH), dm.Nq, cfg->Cq);
      return c.off + 256;
    case SVG2_ENTRY_PERMUTE:
      if (check_bhnd(dm.B, dm.H, dm.Nq, dm.d) != SVG2_OK || check_clusters(cfg->Cq, dm.Nq) != SVG2_OK) return 0;
      carve_sort(c, int(BH), dm.Nq, cfg->Cq);
      return c.off + 256;
    case SVG2_ENTRY_SELECT_TOPP:
      if (BH <= 0 || cfg->Cq < 1 || cfg->Ck < 1 || cfg->Cq > kMaxClusters || cfg->Ck > kMaxClusters) return 0;
      c.take<double>(select_ws_elems(int(BH), cfg->Cq, cfg->Ck));
      return c.off + 256;
    case SVG2_ENTRY_UNPERMUTE:
      return 0;
    case SVG2_ENTRY_VARBLOCK_ATTENTION:
      if (check_bhnd(dm.B, dm.H, dm.Nq, dm.d) != SVG2_OK || check_bhnd(dm.B, dm.H, dm.Nk, dm.d) != SVG2_OK ||
          check_clusters(cfg->Cq, dm.Nq) != SVG2_OK || check_clusters(cfg->Ck, dm.Nk) != SVG2_OK)
        return 0;
      carve_attn(c, int(BH), dm.Nq, dm.Nk, cfg->Cq, cfg->Ck);
      return c.off + 256;
    case SVG2_ENTRY_SPARSE_ATTENTION:
      if (validate_fused(dm, cfg) != SVG2_OK) return 0;
      carve_fused(c, dm, *cfg);
      return c.off + 256;
    case SVG2_ENTRY_SPARSE_ATTENTION_HOST:
      if (validate_fused(dm, cfg) != SVG2_OK) return 0;
      carve_host(c, dm, *cfg, host_plan(dm));
      return c.off + 256;
  }
  return 0;
}

svg2_status_t svg2_kmeans(const void* X, int32_t B, int32_t H, int32_t N, int32_t d, int32_t C, int32_t iters,
                          uint32_t flags, uint32_t seed, int32_t role, float* centroids, int32_t* labels,
                          int32_t* sizes, int32_t* perm, int32_t* offsets, double* objective, void* ws,
                          size_t ws_bytes, void* stream) {
  if (!X || !centroids || !labels || !sizes || (!ws && ws_bytes)) return SVG2_ERR_NULL_POINTER;
  svg2_status_t st = check_bhnd(B, H, N, d);
  if (st != SVG2_OK) return st;
  if ((st = check_clusters(C, N)) != SVG2_OK) return st;
  if (iters < 1 || (flags & ~(SVG2_WARM_START | SVG2_INIT_KMEANSPP)) || role < 0 || role > 1)
    return SVG2_ERR_INVALID_PARAM;
  if (!aligned16(X) || !aligned16(centroids)) return SVG2_ERR_MISALIGNED;
  svg2_config_t cfg{C, C, iters, 1.0, 0.f, flags, seed};
  svg2_dims_t dm{B, H, N, N, d};
  if (ws_bytes < svg2_workspace_size(SVG2_ENTRY_KMEANS, dm, &cfg)) return SVG2_ERR_WORKSPACE_TOO_SMALL;
  if ((st = check_device()) != SVG2_OK) return st;
  if ((st = pending_error()) != SVG2_OK) return st;
  Carver c(ws);
  KmeansWs kw = carve_kmeans(c, B * H, N, C);
  KmeansInit init;
  init.kmeanspp = (flags & SVG2_INIT_KMEANSPP) != 0;
  init.seed = seed;
  init.role = role;
  return from_cuda(launch_kmeans(contiguous_view(X, B, H, N, d), B * H, N, d, C, iters, flags & SVG2_WARM_START,
                                 centroids, labels, sizes, perm,
                                 offsets, kw, static_cast<cudaStream_t>(stream), nullptr, init, KmeansGather(),
                                 objective));
}

svg2_status_t svg2_permute(const int32_t* labels, int32_t B, int32_t H, int32_t N, int32_t d, int32_t C,
                           const void* X0, void* X0p, const void* X1, void* X1p, int32_t* perm, int32_t* offsets,
                           void* ws, size_t ws_bytes, void* stream) {
  if (!labels || !perm || !offsets || (!ws && ws_bytes)) return SVG2_ERR_NULL_POINTER;
  if ((X0 == nullptr) != (X0p == nullptr) || (X1 == nullptr) != (X1p == nullptr)) return SVG2_ERR_NULL_POINTER;
  svg2_status_t st = check_bhnd(B, H, N, d);
  if (st != SVG2_OK) return st;
  if ((st = check_clusters(C, N)) != SVG2_OK) return st;
  if ((X0 && (!aligned16(X0) || !aligned16(X0p))) || (X1 && (!aligned16(X1) || !aligned16(X1p))))
    return SVG2_ERR_MISALIGNED;
  svg2_config_t cfg{C, C, 1, 1.0, 0.f, 0};
  svg2_dims_t dm{B, H, N, N, d};
  if (ws_bytes < svg2_workspace_size(SVG2_ENTRY_PERMUTE, dm, &cfg)) return SVG2_ERR_WORKSPACE_TOO_SMALL;
  if ((st = check_device()) != SVG2_OK) return st;
  if ((st = pending_error()) != SVG2_OK) return st;
  Carver c(ws);
  SortWs sw = carve_sort(c, B * H, N, C);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e = launch_stable_sort(labels, B * H, N, C, sw, perm, offsets, nullptr, s);
  if (e == cudaSuccess && (X0 || X1)) e = launch_gather_rows(perm, B * H, N, d, X0, X0p, X1, X1p, s);
  return from_cuda(e);
}

svg2_status_t svg2_select_topp(const float* q_centroids, const float* k_centroids, const int32_t* q_sizes,
                               const int32_t* k_sizes, int32_t B, int32_t H, int32_t Cq, int32_t Ck, int32_t d,
                               float scale, double top_p, uint8_t* mask, int64_t* selected_pairs, void* ws,
                               size_t ws_bytes, void* stream) {
  if (!q_centroids || !k_centroids || !q_sizes || !k_sizes || !mask || !ws) return SVG2_ERR_NULL_POINTER;
  if (B <= 0 || H <= 0 || (d != 64 && d != 128)) return SVG2_ERR_INVALID_SHAPE;
  if (Cq < 1 || Ck < 1 || Cq > kMaxClusters || Ck > kMaxClusters) return SVG2_ERR_INVALID_PARAM;
  if (!(top_p > 0.0 && top_p <= 1.0) || !(scale >= 0.f) || std::isinf(scale)) return SVG2_ERR_INVALID_PARAM;
  svg2_config_t cfg{Cq, Ck, 1, top_p, scale, 0u, 0u};
  svg2_dims_t dm{B, H, 1, 1, d};
  if (ws_bytes < svg2_workspace_size(SVG2_ENTRY_SELECT_TOPP, dm, &cfg)) return SVG2_ERR_WORKSPACE_TOO_SMALL;
  svg2_status_t st;
  if ((st = check_device()) != SVG2_OK) return st;
  if ((st = pending_error()) != SVG2_OK) return st;
  Carver c(ws);
  double* S = c.take<double>(select_ws_elems(B * H, Cq, Ck));
  return from_cuda(launch_select_topp(q_centroids, k_centroids, q_sizes, k_sizes, B * H, Cq, Ck, d,
                                      resolve_scale(scale, d), top_p, mask, selected_pairs, S,
                                      static_cast<cudaStream_t>(stream)));
}

svg2_status_t svg2_varblock_attention(const void* Qp, const void* Kp, const void* Vp, svg2_dims_t dm,
                                      const int32_t* q_offsets, const int32_t* k_offsets, const uint8_t* mask,
                                      int32_t Cq, int32_t Ck, float scale, const int32_t* q_perm, void* O,
                                      float* lse, void* ws, size_t ws_bytes, void* stream) {
  if (!Qp || !Kp || !Vp || !q_offsets || !k_offsets || !mask || !O || !ws) return SVG2_ERR_NULL_POINTER;
  svg2_status_t st = check_bhnd(dm.B, dm.H, dm.Nq, dm.d);
  if (st != SVG2_OK) return st;
  if ((st = check_bhnd(dm.B, dm.H, dm.Nk, dm.d)) != SVG2_OK) return st;
  if ((st = check_clusters(Cq, dm.Nq)) != SVG2_OK) return st;
  if ((st = check_clusters(Ck, dm.Nk)) != SVG2_OK) return st;
  if (!(scale >= 0.f) || std::isinf(scale)) return SVG2_ERR_INVALID_PARAM;
  if (!aligned16(Qp) || !aligned16(Kp) || !aligned16(Vp) || !aligned16(O)) return SVG2_ERR_MISALIGNED;
  svg2_config_t cfg{Cq, Ck, 1, 1.0, scale, 0};
  if (ws_bytes < svg2_workspace_size(SVG2_ENTRY_VARBLOCK_ATTENTION, dm, &cfg)) return SVG2_ERR_WORKSPACE_TOO_SMALL;
  if ((st = check_device()) != SVG2_OK) return st;
  if ((st = pending_error()) != SVG2_OK) return st;
  Carver c(ws);
  const int BH = dm.B * dm.H;
  AttnWs aw = carve_attn(c, BH, dm.Nq, dm.Nk, Cq, Ck);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e = launch_build_worklist(q_offsets, k_offsets, mask, BH, dm.Nq, dm.Nk, Cq, Ck,
                                        attn_groups_per_tile(dm.d, false), aw,
                                        OrphanFill{q_perm, contiguous_out(O, dm.H, dm.Nq, dm.d), lse, dm.d}, s);
  if (e == cudaSuccess)
    e = launch_varblock_attention(Qp, Kp, Vp, BH, dm.Nq, dm.Nk, dm.d, resolve_scale(scale, dm.d), q_perm,
                                  contiguous_out(O, dm.H, dm.Nq, dm.d), lse, aw, s);
  return from_cuda(e);
}

svg2_status_t svg2_unpermute(const void* Op, const int32_t* perm, int32_t B, int32_t H, int32_t N, int32_t d,
                             void* O, void* stream) {
  if (!Op || !perm || !O) return SVG2_ERR_NULL_POINTER;
  svg2_status_t st = check_bhnd(B, H, N, d);
  if (st != SVG2_OK) return st;
  if (!aligned16(Op) || !aligned16(O)) return SVG2_ERR_MISALIGNED;
  if ((st = check_device()) != SVG2_OK) return st;
  if ((st = pending_error()) != SVG2_OK) return st;
  return from_cuda(launch_scatter_rows(Op, perm, B * H, N, d, O, static_cast<cudaStream_t>(stream)));
}

int32_t svg2_sparse_attention_launch_count(svg2_dims_t dm, const svg2_config_t* cfg) {
  (void)dm;
  if (!cfg) return 0;
  const bool warm = cfg->flags & SVG2_WARM_START;
  // the Q / K / V gathers are fused into the last k-means update (no launches of their own)
  int n = 2 * kmeans_launch_count(cfg->iters, warm) + 2 /*scores + select*/ + kWorklistLaunches + 1 /*attn*/;
  if (cfg->top_p >= 1.0) n += 1;  // the dense stream's query offsets (the mask is a memset)
  if (cfg->flags & SVG2_FP8_PV) n += 2;  // |V| max per head + the e4m3 gather
  if (!warm && (cfg->flags & SVG2_INIT_KMEANSPP))
    n += kmeanspp_launch_count(dm.B * dm.H, dm.Nq, dm.d) + kmeanspp_launch_count(dm.B * dm.H, dm.Nk, dm.d) - 2;
  return n;
}

svg2_status_t svg2_sparse_attention(const void* Q, const void* K, const void* V, svg2_dims_t dm,
                                    const svg2_config_t* cfg, float* q_centroids, float* k_centroids, void* O,
                                    int64_t* selected_pairs, const svg2_debug_t* dbg, void* ws, size_t ws_bytes,
                                    void* stream) {
  return svg2_sparse_attention_ex(Q, K, V, dm, cfg, q_centroids, k_centroids, O, selected_pairs, dbg, nullptr, ws,
                                  ws_bytes, stream);
}

svg2_status_t svg2_sparse_attention_ex(const void* Q, const void* K, const void* V, svg2_dims_t dm,
                                       const svg2_config_t* cfg, float* q_centroids, float* k_centroids, void* O,
                                       int64_t* selected_pairs, const svg2_debug_t* dbg, void* const* input_ready,
                                       void* ws, size_t ws_bytes, void* stream) {
  return svg2_sparse_attention_layout(Q, K, V, dm, cfg, nullptr, q_centroids, k_centroids, O, selected_pairs, dbg,
                                      input_ready, ws, ws_bytes, stream);
}

namespace {
bool strides_ok(const int64_t* st, int d) {  // (sB, sH, sN): positive multiples of 8 elements (16-byte TMA rows)
  for (int i = 0; i < 3; ++i)
    if (st[i] <= 0 || st[i] % 8) return false;
  return st[2] >= d;
}
XView view_of(const void* p, const svg2_dims_t& dm, int N, const int64_t* st) {
  if (!st || (st[0] == 0 && st[1] == 0 && st[2] == 0)) return contiguous_view(p, dm.B, dm.H, N, dm.d);
  XView v;
  v.p = p;
  v.sB = st[0];
  v.sH = st[1];
  v.sN = st[2];
  v.H = dm.H;
  return v;
}
bool zero3(const int64_t* st) { return st[0] == 0 && st[1] == 0 && st[2] == 0; }
}  // namespace

svg2_status_t svg2_sparse_attention_layout(const void* Q, const void* K, const void* V, svg2_dims_t dm,
                                           const svg2_config_t* cfg, const svg2_layout_t* lay, float* q_centroids,
                                           float* k_centroids, void* O, int64_t* selected_pairs,
                                           const svg2_debug_t* dbg, void* const* input_ready, void* ws,
                                           size_t ws_bytes, void* stream) {
  if (input_ready && (!input_ready[0] || !input_ready[1] || !input_ready[2])) return SVG2_ERR_NULL_POINTER;
  const bool sharded = lay && lay->o_shards;
  if (!Q || !K || !V || !cfg || !q_centroids || !k_centroids || (!O && !sharded) || !ws) return SVG2_ERR_NULL_POINTER;
  svg2_status_t st = validate_fused(dm, cfg);
  if (st != SVG2_OK) return st;
  if (!aligned16(Q) || !aligned16(K) || !aligned16(V) || (!sharded && !aligned16(O)) || !aligned16(q_centroids) ||
      !aligned16(k_centroids))
    return SVG2_ERR_MISALIGNED;
  QPart part;
  OutView out = contiguous_out(O, dm.H, dm.Nq, dm.d);
  AuxStream aux;
  if (lay && lay->aux_stream) {
    if (!lay->aux_events[0] || !lay->aux_events[1]) return SVG2_ERR_NULL_POINTER;
    aux.stream = static_cast<cudaStream_t>(lay->aux_stream);
    aux.fork = static_cast<cudaEvent_t>(lay->aux_events[0]);
    aux.join = static_cast<cudaEvent_t>(lay->aux_events[1]);
  }
  if (lay) {
    const int64_t* strs[3] = {lay->q_strides, lay->k_strides, lay->v_strides};
    for (int t = 0; t < 3; ++t)
      if (!zero3(strs[t]) && !strides_ok(strs[t], dm.d)) return SVG2_ERR_INVALID_SHAPE;
    if (lay->part_count != 0 || lay->part_begin != 0 || lay->part_end != 0) {
      if (lay->part_count < 1 || lay->part_count > kMaxClusters || lay->part_begin < 0 ||
          lay->part_end <= lay->part_begin || lay->part_end > lay->part_count)
        return SVG2_ERR_INVALID_PARAM;
      part.begin = lay->part_begin;
      part.end = lay->part_end;
      part.count = lay->part_count;
    }
    if (sharded) {
      if (lay->n_shards < 1 || lay->n_shards > kMaxShards || lay->shard_tokens < 1 ||
          (long long)lay->n_shards * lay->shard_tokens < dm.Nq || lay->o_head_offset < 0 || !strides_ok(lay->o_strides, dm.d))
        return SVG2_ERR_INVALID_SHAPE;
      out.n_shards = lay->n_shards;
      out.shard_tokens = lay->shard_tokens;
      for (int i = 0; i < lay->n_shards; ++i) {
        if (!lay->o_shards[i]) return SVG2_ERR_NULL_POINTER;
        if (!aligned16(lay->o_shards[i])) return SVG2_ERR_MISALIGNED;
        out.shard[i] = lay->o_shards[i];
      }
      out.sB = lay->o_strides[0];
      out.sH = lay->o_strides[1];
      out.sN = lay->o_strides[2];
      out.head_offset = lay->o_head_offset;
    }
  }
  if (ws_bytes < svg2_workspace_size(SVG2_ENTRY_SPARSE_ATTENTION, dm, cfg)) return SVG2_ERR_WORKSPACE_TOO_SMALL;
  if ((st = check_device()) != SVG2_OK) return st;
  if ((st = pending_error()) != SVG2_OK) return st;

  Carver c(ws);
  FusedWs w = carve_fused(c, dm, *cfg);
  cudaEvent_t ready[3];
  if (input_ready)
    for (int i = 0; i < 3; ++i) ready[i] = static_cast<cudaEvent_t>(input_ready[i]);
  const XView qv = view_of(Q, dm, dm.Nq, lay ? lay->q_strides : nullptr);
  const XView kv = view_of(K, dm, dm.Nk, lay ? lay->k_strides : nullptr);
  const XView vv = view_of(V, dm, dm.Nk, lay ? lay->v_strides : nullptr);
  return from_cuda(run_fused(qv, kv, vv, dm, cfg, q_centroids, k_centroids, out, selected_pairs, dbg, w,
                             static_cast<cudaStream_t>(stream), 0, input_ready ? ready : nullptr, part, &aux));
}

svg2_status_t svg2_sparse_attention_host(const void* Qh, const void* Kh, const void* Vh, svg2_dims_t dm,
                                         const svg2_config_t* cfg, float* q_centroids, float* k_centroids, void* Oh,
                                         int64_t* selected_pairs, void* ws, size_t ws_bytes, void* stream) {
  if (!Qh || !Kh || !Vh || !cfg || !q_centroids || !k_centroids || !Oh || !ws) return SVG2_ERR_NULL_POINTER;
  svg2_status_t st = validate_fused(dm, cfg);
  if (st != SVG2_OK) return st;
  if (!aligned16(Qh) || !aligned16(Kh) || !aligned16(Vh) || !aligned16(Oh) || !aligned16(q_centroids) ||
      !aligned16(k_centroids))
    return SVG2_ERR_MISALIGNED;
  if (ws_bytes < svg2_workspace_size(SVG2_ENTRY_SPARSE_ATTENTION_HOST, dm, cfg)) return SVG2_ERR_WORKSPACE_TOO_SMALL;
  if ((st = check_device()) != SVG2_OK) return st;
  if ((st = pending_error()) != SVG2_OK) return st;
  const HostPlan plan = host_plan(dm);
  Carver c(ws);
  HostWs w = carve_host(c, dm, *cfg, plan);
  cudaStream_t caller = static_cast<cudaStream_t>(stream);
  // internal streams: copies in, up to kHostSlots compute streams (chunk ci on stream ci % ncomp: the next chunks'
  // k-means, selection and first attention items fill the SMs the current chunk's attention tail leaves idle), copies
  // out; events order them per chunk and slot.  The k-means++ cold start (cooperative launches) keeps one compute
  // stream.
  const bool pp_cold = !(cfg->flags & SVG2_WARM_START) && (cfg->flags & SVG2_INIT_KMEANSPP);
  const int ncomp = pp_cold ? 1 : kHostComputeStreams;
  cudaStream_t sin = nullptr, scomp[kHostSlots] = {}, sout = nullptr;
  cudaEvent_t start = nullptr;
  cudaError_t e = cudaStreamCreateWithFlags(&sin, cudaStreamNonBlocking);
  for (int i = 0; i < ncomp && e == cudaSuccess; ++i) e = cudaStreamCreateWithFlags(&scomp[i], cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&sout, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&start, cudaEventDisableTiming);
  const int n = plan.nchunks;
  cudaEvent_t* ev = new cudaEvent_t[3 * n]();  // per chunk: inputs in (V, the last copy), computed, output out
  cudaEvent_t* evqk = new cudaEvent_t[2 * n]();  // per chunk: Q in, K in
  for (int i = 0; e == cudaSuccess && i < 3 * n; ++i) e = cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming);
  for (int i = 0; e == cudaSuccess && i < 2 * n; ++i) e = cudaEventCreateWithFlags(&evqk[i], cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventRecord(start, caller);  // after the caller's earlier work
  if (e == cudaSuccess) e = cudaStreamWaitEvent(sin, start, 0);
  for (int i = 0; i < ncomp && e == cudaSuccess; ++i) e = cudaStreamWaitEvent(scomp[i], start, 0);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(sout, start, 0);
  const size_t qrow = size_t(dm.Nq) * dm.d * 2, krow = size_t(dm.Nk) * dm.d * 2;  // bytes per head
  for (int ci = 0; e == cudaSuccess && ci < n; ++ci) {
    const int bh0 = plan.start[ci], nh = plan.start[ci + 1] - bh0, slot = ci % kHostSlots, cs = ci % ncomp;
    cudaStream_t sc = scomp[cs];
    cudaEvent_t in = ev[3 * ci], done = ev[3 * ci + 1], out = ev[3 * ci + 2];
    if (ci >= kHostSlots) e = cudaStreamWaitEvent(sin, ev[3 * (ci - kHostSlots) + 1], 0);  // slot's inputs consumed
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(w.Q[slot], static_cast<const uint8_t*>(Qh) + bh0 * qrow, nh * qrow, cudaMemcpyHostToDevice, sin);
    if (e == cudaSuccess) e = cudaEventRecord(evqk[2 * ci], sin);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(w.K[slot], static_cast<const uint8_t*>(Kh) + bh0 * krow, nh * krow, cudaMemcpyHostToDevice, sin);
    if (e == cudaSuccess) e = cudaEventRecord(evqk[2 * ci + 1], sin);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(w.V[slot], static_cast<const uint8_t*>(Vh) + bh0 * krow, nh * krow, cudaMemcpyHostToDevice, sin);
    if (e == cudaSuccess) e = cudaEventRecord(in, sin);
    if (e == cudaSuccess && ci >= kHostSlots)
      e = cudaStreamWaitEvent(sc, ev[3 * (ci - kHostSlots) + 2], 0);  // slot's output read
    if (e == cudaSuccess) {
      const svg2_dims_t cd{1, nh, dm.Nq, dm.Nk, dm.d};
      const cudaEvent_t arrive[3] = {evqk[2 * ci], evqk[2 * ci + 1], in};  // the computation starts on Q alone
      e = run_fused(contiguous_view(w.Q[slot], 1, nh, dm.Nq, dm.d), contiguous_view(w.K[slot], 1, nh, dm.Nk, dm.d),
                    contiguous_view(w.V[slot], 1, nh, dm.Nk, dm.d), cd, cfg, q_centroids + size_t(bh0) * cfg->Cq * dm.d,
                    k_centroids + size_t(bh0) * cfg->Ck * dm.d, contiguous_out(w.O[slot], nh, dm.Nq, dm.d),
                    selected_pairs ? selected_pairs + bh0 : nullptr, nullptr, w.fused[cs], sc, bh0,
                    arrive);
    }
    if (e == cudaSuccess) e = cudaEventRecord(done, sc);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(sout, done, 0);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(static_cast<uint8_t*>(Oh) + bh0 * qrow, w.O[slot], nh * qrow, cudaMemcpyDeviceToHost, sout);
    if (e == cudaSuccess) e = cudaEventRecord(out, sout);
  }
  // the last copy out ends the call (sout is in order and each copy waited for its chunk); the last two chunks'
  // compute events as well, so no work of either compute stream outlives the call
  if (e == cudaSuccess) e = cudaStreamWaitEvent(caller, ev[3 * (n - 1) + 2], 0);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(caller, ev[3 * (n - 1) + 1], 0);
  for (int k = 2; k <= ncomp && k <= n && e == cudaSuccess; ++k) e = cudaStreamWaitEvent(caller, ev[3 * (n - k) + 1], 0);
  for (int i = 0; i < 3 * n; ++i)
    if (ev[i]) cudaEventDestroy(ev[i]);
  for (int i = 0; i < 2 * n; ++i)
    if (evqk[i]) cudaEventDestroy(evqk[i]);
  delete[] ev;
  delete[] evqk;
  if (start) cudaEventDestroy(start);
  if (sin) cudaStreamDestroy(sin);  // released once their queued work completes
  for (int i = 0; i < kHostSlots; ++i)
    if (scomp[i]) cudaStreamDestroy(scomp[i]);
  if (sout) cudaStreamDestroy(sout);
  return from_cuda(e);
}

}  // extern "C"

/*
 * svg2.h — C ABI of the B200-native SVG2 sparse-attention hot path (arXiv 2505.18875, "Sparse VideoGen2").
 *
 * One shared library, libsvg2.so, hand-written CUDA for sm_100a.  Every entry point takes plain device
 * pointers and sizes, validates synchronously (nothing is enqueued and no output is touched on error), then
 * enqueues its kernels on `stream` (a cudaStream_t passed as void*; NULL = legacy default stream) and
 * returns without synchronising.  Kernel faults surface as SVG2_ERR_CUDA from a later call or from the
 * caller's stream synchronisation (the CUDA convention).  The library allocates no device memory and keeps
 * no mutable global state: the caller owns every buffer, including the workspace sized by
 * svg2_workspace_size().  Calls are reentrant; concurrent calls on different streams need distinct
 * workspaces.
 *
 * Layout conventions.
 *   Q, K, V, O        bf16 [B, H, N, d], contiguous, d in {64, 128}, 16-byte aligned.
 *   labels, perm      int32 [B, H, N].  perm[p] = original token index of permuted position p (pi as an index map).
 *   offsets           int32 [B, H, C+1]: cluster j owns permuted positions [offsets[j], offsets[j+1]).
 *   sizes             int32 [B, H, C]   (= offsets[j+1] - offsets[j]).
 *   centroids         float32 [B, H, C, d]  (the centroid cache of PAPER.md:325-326; exact means of the
 *                     returned clusters, rounded to f32; fp64 accumulation inside).
 *   mask              uint8 [B, H, Cq, Ck]: 1 = key cluster j is selected for query cluster i.
 *   selected_pairs    int64 [B, H]: sum_i |Q_i| * sum_{j selected} |K_j| (density = pairs / (Nq*Nk)).
 * Limits: 1 <= C <= min(N, 4096); N <= 2^24; B*H*N < 2^31; 0 < top_p <= 1; iters >= 1.
 *
 * Citations are PAPER.md line numbers of /root/reference (the paper's LaTeX); DESIGN.md lists every reading
 * of an ambiguous passage (R1..R23).
 */
#ifndef SVG2_H_
#define SVG2_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SVG2_ABI_VERSION 3

#if defined(__GNUC__)
#define SVG2_API __attribute__((visibility("default")))
#else
#define SVG2_API
#endif

typedef enum {
  SVG2_OK = 0,
  SVG2_ERR_NULL_POINTER = 1,       /* a required pointer is NULL */
  SVG2_ERR_INVALID_SHAPE = 2,      /* B,H,N <= 0, d not in {64,128}, sizes beyond the limits above */
  SVG2_ERR_INVALID_PARAM = 3,      /* C < 1 or C > N or C > 4096, top_p outside (0,1], iters < 1, bad flags, role */
  SVG2_ERR_MISALIGNED = 4,         /* a tensor pointer is not 16-byte aligned (TMA requirement) */
  SVG2_ERR_WORKSPACE_TOO_SMALL = 5,/* ws_bytes < svg2_workspace_size(...) */
  SVG2_ERR_UNSUPPORTED_DEVICE = 6, /* current device is not compute capability 10.0 (sm_100) */
  SVG2_ERR_CUDA = 7,               /* a CUDA runtime error (launch failure or an earlier asynchronous fault) */
  SVG2_ERR_NOT_IMPLEMENTED = 8
} svg2_status_t;

typedef struct {
  int32_t B, H, Nq, Nk, d; /* Q: [B,H,Nq,d]; K, V: [B,H,Nk,d] */
} svg2_dims_t;

/* flags */
#define SVG2_WARM_START 1u /* k-means starts from the caller's centroids (the centroid cache);
                              otherwise a cold init: the deterministic strided rows c_j = x[floor(j*N/C)] (R2),
                              or k-means++ with SVG2_INIT_KMEANSPP */
#define SVG2_INIT_KMEANSPP 2u /* cold init by k-means++ seeding with the generator of
                                 DESIGN.md R25: Philox4x32-10 keyed (seed, 2*(b*H+h) + role), role 0 = Q, 1 = K;
                                 picks reproducible bit for bit.  Ignored with SVG2_WARM_START.  Costs C passes over
                                 X (the expense the centroid cache avoids). */
#define SVG2_FP8_PV 4u /* the "+FP8" variant as DESIGN.md R26 reads it: P and V enter the PV
                          product as e4m3 -- V with per-(b,h, channel) scales 448 / max_n |V_nc| undone in the epilogue,
                          P with a per-row power-of-two scale (2^6 over the running max, lazy rescale at +2) that
                          cancels in O / l -- fp32 accumulation; QK^T, the softmax and the output stay bf16 / fp32.
                          d = 128 only. */

typedef struct {
  int32_t Cq, Ck;  /* query / key cluster counts (paper default 100 / 500) */
  int32_t iters;   /* Lloyd iterations, exactly (R3) */
  double top_p;    /* top-p target in (0, 1] */
  float scale;     /* softmax scale; 0 => 1/sqrt(d) */
  uint32_t flags;  /* SVG2_WARM_START | SVG2_INIT_KMEANSPP | SVG2_FP8_PV */
  uint32_t seed;   /* k-means++ generator seed (R25); unused otherwise */
} svg2_config_t;

/* Optional intermediates of the fused call (device pointers, each NULL or sized as in the layout block above)
 * plus up to 8 cudaEvent_t handles recorded on `stream` at stage boundaries:
 *   events[0] start, [1] after k-means(Q), [2] after k-means(K), [3] after permute (Q', K', V'),
 *   [4] after select_topp, [5] after run/work-list build, [6] after varblock attention (+ fused unpermute),
 *   [7] end.  Used for the per-stage breakdown and the roofline measurement of bench.py. */
typedef struct {
  int32_t *q_labels, *k_labels, *q_perm, *k_perm, *q_offsets, *k_offsets;
  uint8_t* mask;
  void* events[8];
  double *q_objective, *k_objective; /* NULL or [iters, B, H, 2]: the Lloyd objective of each role per iteration,
                                        as svg2_kmeans' `objective` (an extra launch per iteration when set) */
} svg2_debug_t;

SVG2_API const char* svg2_status_string(svg2_status_t status);
SVG2_API int svg2_abi_version(void);

/* Entry ids for svg2_workspace_size. */
typedef enum {
  SVG2_ENTRY_KMEANS = 0,
  SVG2_ENTRY_PERMUTE = 1,
  SVG2_ENTRY_SELECT_TOPP = 2,
  SVG2_ENTRY_VARBLOCK_ATTENTION = 3,
  SVG2_ENTRY_UNPERMUTE = 4,
  SVG2_ENTRY_SPARSE_ATTENTION = 5,
  SVG2_ENTRY_SPARSE_ATTENTION_HOST = 6
} svg2_entry_t;

/* Bytes of workspace the entry needs for these dims/config (dims.Nq is N for SVG2_ENTRY_KMEANS/PERMUTE;
 * config->Cq is C there).  Returns 0 for invalid arguments. */
SVG2_API size_t svg2_workspace_size(svg2_entry_t entry, svg2_dims_t dims, const svg2_config_t* config);

/* ---- A1-A5: Lloyd k-means on one role (warm start PAPER.md:322-326).
 * X [B,H,N,d] bf16.  Per (b,h), `iters` iterations of: assign label_n = argmin_j ||x_n - c_j||^2 (ties -> lowest
 * j), then c_j = mean of its tokens (fp64 sums, stored f32; an empty cluster keeps its centroid, R6).
 * centroids [B,H,C,d] f32: input iff flags & SVG2_WARM_START, always output (exact means of the final labels).
 * Cold start: strided rows, or k-means++ (flags & SVG2_INIT_KMEANSPP) with generator key (seed, 2*(b*H+h) + role),
 * role 0 for queries, 1 for keys (R25).
 * labels [B,H,N] out (last assign).  sizes [B,H,C] out.  perm / offsets: optional (NULL) outputs = the stable
 * permutation of the final labels, identical to what svg2_permute would compute.
 * objective: optional (NULL) output [iters, B, H, 2] fp64, the Lloyd objective J = sum_n ||x_n - c_{label_n}||^2
 * of iteration t: [t,b,h,0] = J_assign(t) with the centroids the assign step used, [t,b,h,1] =
 * J_post(t) with the updated (f32) centroids, so J_assign(t) >= J_post(t) >= J_assign(t+1) up to rounding and
 * near-ties.  Evaluated per cluster as sum ||x||^2 - 2 c.S + n ||c||^2 in fp64 (S = the cluster's fp64 sum).
 * The centroid sums are a fixed-order segmented reduction: results are deterministic for any input. */
SVG2_API svg2_status_t svg2_kmeans(const void* X, int32_t B, int32_t H, int32_t N, int32_t d, int32_t C, int32_t iters,
                                   uint32_t flags, uint32_t seed, int32_t role, float* centroids, int32_t* labels,
                                   int32_t* sizes, int32_t* perm, int32_t* offsets, double* objective, void* ws,
                                   size_t ws_bytes, void* stream);

/* ---- A3, A4, A6: semantic-aware permutation.
 * Stable counting sort of the tokens by (label, index): perm [B,H,N] and offsets [B,H,C+1] out.  Then gathers
 * up to two bf16 tensors through the same permutation (K and V share pi_k):
 * X0p[b,h,p,:] = X0[b,h,perm[p],:], likewise X1 -> X1p.  X0/X0p and X1/X1p may be NULL (then no gather). */
SVG2_API svg2_status_t svg2_permute(const int32_t* labels, int32_t B, int32_t H, int32_t N, int32_t d, int32_t C,
                           const void* X0, void* X0p, const void* X1, void* X1p, int32_t* perm, int32_t* offsets,
                           void* ws, size_t ws_bytes, void* stream);

/* ---- A7, A8: centroid-based top-p selection (Eq. 1, Eq. 2, top-p
 * PAPER.md:314-315).  Per (b,h,i), in fp64: S_ij = scale * sum_k c^q_ik c^k_jk (sequential FMA, k ascending);
 * w_ij = |K_j| exp(S_ij - max_{j:|K_j|>0} S_ij); Z_i = sum_j w_ij; sort j by w_ij descending (ties: ascending j)
 * and select the ranks whose preceding mass is < top_p * Z_i (non-empty clusters only); top_p == 1 selects every
 * non-empty key cluster.  The library takes this decision without sorting: the selected ranks are the w_ij >= w*,
 * w* = the largest w whose mass of weights >= w reaches top_p * Z_i (ties at w* in ascending j); Z_i and those
 * masses are fp64 sums in a fixed tree order (deterministic; equal to the sequential sums up to rounding, DESIGN R27).  mask [B,H,Cq,Ck] out; selected_pairs [B,H] out (nullable).
 * ws: svg2_workspace_size(SVG2_ENTRY_SELECT_TOPP, {B,H,*,*,d}, {Cq,Ck,...}) bytes (the fp64 score table). */
SVG2_API svg2_status_t svg2_select_topp(const float* q_centroids, const float* k_centroids, const int32_t* q_sizes,
                                        const int32_t* k_sizes, int32_t B, int32_t H, int32_t Cq, int32_t Ck,
                                        int32_t d, float scale, double top_p, uint8_t* mask,
                                        int64_t* selected_pairs, void* ws, size_t ws_bytes, void* stream);

/* ---- A9 (+ optional A10): dynamic-block-size sparse attention over permuted, cluster-contiguous tokens
 * (PAPER.md:329-334).  For every query row p of cluster i (rows [q_offsets[i], q_offsets[i+1]) of Qp):
 * O[p] = softmax over the keys of all selected key clusters j (rows [k_offsets[j], k_offsets[j+1]) of Kp),
 * renormalised over that set (R12), times the matching rows of Vp.  bf16 in, fp32 accumulation (tcgen05/TMEM),
 * bf16 out.  If q_perm is non-NULL the output row is scattered to original order, O[q_perm[p]] (the inverse
 * permutation pi_q^T of PAPER.md:277 fused into the epilogue); otherwise O is written in permuted order.
 * lse [B,H,Nq] f32 (natural log-sum-exp of the scaled scores, same row order as O), nullable.
 * Precondition: every non-empty query cluster selects at least one non-empty key cluster (the fused call guarantees
 * it, R11).  A cluster that violates it gets no attention work: its O rows are filled with bf16 NaN and its lse
 * entries with NaN, so the violation is visible (the call still returns SVG2_OK: the mask is device data). */
SVG2_API svg2_status_t svg2_varblock_attention(const void* Qp, const void* Kp, const void* Vp, svg2_dims_t dims,
                                      const int32_t* q_offsets, const int32_t* k_offsets, const uint8_t* mask,
                                      int32_t Cq, int32_t Ck, float scale, const int32_t* q_perm, void* O,
                                      float* lse, void* ws, size_t ws_bytes, void* stream);

/* ---- A10: inverse permutation of the output: O[b,h,perm[p],:] = Op[b,h,p,:]. */
SVG2_API svg2_status_t svg2_unpermute(const void* Op, const int32_t* perm, int32_t B, int32_t H, int32_t N, int32_t d,
                             void* O, void* stream);

/* ---- A1-A11 fused: the whole SVG2 attention call for Q, K, V [B,H,N,d].
 * k-means(Q; Cq) and k-means(K; Ck) with the centroid cache (q_centroids [B,H,Cq,d], k_centroids [B,H,Ck,d]
 * f32, read iff config->flags & SVG2_WARM_START, always written back), permutation, selection, variable-block
 * attention with the unpermute fused into its epilogue.  O [B,H,Nq,d] bf16 out in original token order.
 * selected_pairs [B,H] int64 out (nullable).  dbg: NULL or intermediates / stage events (see svg2_debug_t).
 * Streams: the K-role k-means runs on a (high-priority) stream forked from `stream` for the duration of the call
 * (event fork / join; the stream and events are created and released per call unless the caller lends them through
 * svg2_layout_t.aux_*; without lent ones the call stays on `stream` while `stream` is being captured into a CUDA
 * graph); all work is ordered after, and joined back into, `stream`. */
SVG2_API svg2_status_t svg2_sparse_attention(const void* Q, const void* K, const void* V, svg2_dims_t dims,
                                    const svg2_config_t* config, float* q_centroids, float* k_centroids, void* O,
                                    int64_t* selected_pairs, const svg2_debug_t* dbg, void* ws, size_t ws_bytes,
                                    void* stream);

/* ---- The fused call with inputs still arriving (e.g. the Ulysses all-to-all of Q, K, V running on another stream):
 * as svg2_sparse_attention, plus input_ready = NULL or three cudaEvent_t (as void*) recorded when Q, K and V are
 * complete in device memory.  The Q-role k-means waits for Q's event, the K-role for K's, and V is waited for only
 * before the pass that gathers it, so the computation overlaps the transfer of the later tensors.  A NULL event in a
 * non-NULL input_ready is SVG2_ERR_NULL_POINTER.  svg2_sparse_attention(...) == svg2_sparse_attention_ex(..., NULL,
 * ...). */
SVG2_API svg2_status_t svg2_sparse_attention_ex(const void* Q, const void* K, const void* V, svg2_dims_t dims,
                                                const svg2_config_t* config, float* q_centroids, float* k_centroids,
                                                void* O, int64_t* selected_pairs, const svg2_debug_t* dbg,
                                                void* const* input_ready, void* ws, size_t ws_bytes, void* stream);

/* ---- Memory layouts and the multi-GPU split of the fused call (SURVEY 8(b) strides, 8(e), 8(f) row 4).
 *   q/k/v_strides  element strides (sB, sH, sN) of Q, K, V ([B,H,N,d] logical, d contiguous); {0,0,0} = contiguous.
 *                  Positive multiples of 8 elements, sN >= d.  E.g. the token-major [B, N, H, d] buffer a Ulysses
 *                  all-to-all produces is (N*H*d, d, H*d): read in place, no transpose pass.
 *   o_shards       NULL: O is the call's contiguous [B,H,Nq,d] argument.  Otherwise n_shards (<= 16) device pointers
 *                  (this process's mappings -- peers' buffers through CUDA IPC or symmetric memory): output token n
 *                  of head h goes to shard s = n / shard_tokens, row n - s*shard_tokens, at element offset
 *                  b*o_strides[0] + (h + o_head_offset)*o_strides[1] + row*o_strides[2].  The attention epilogue
 *                  stores there directly: the inverse permutation (A10) and the reverse Ulysses all-to-all in one
 *                  store per row.  The O argument is then unused (may be NULL).
 *   part_begin / part_end / part_count  the query-cluster split of a head across ranks (K/V replicated): every rank
 *                  runs the same k-means and selection (deterministic, so identical), but the attention covers only
 *                  the query clusters of parts [part_begin, part_end) of part_count -- per head, cluster i with cost
 *                  c_i = |Q_i| * keys_i (its selected pairs) and preceding cost P_i belongs to part
 *                  floor((2 P_i + c_i) part_count / (2 T)), T the head's total -- and writes only their rows.
 *                  {0, 0, 0} = all clusters.  selected_pairs and the centroid caches are always the whole head's.
 *   aux_stream / aux_events  optional resources for the forked K-role stream (see svg2_sparse_attention). */
typedef struct {
  int64_t q_strides[3], k_strides[3], v_strides[3];
  void* const* o_shards;
  int32_t n_shards, shard_tokens, o_head_offset, part_begin;
  int64_t o_strides[3];
  int32_t part_end, part_count;
  void* aux_stream;     /* NULL, or a caller-owned cudaStream_t (high priority recommended) for the K-role k-means */
  void* aux_events[2];  /* with aux_stream: two caller-owned cudaEvent_t (fork, join); then the call creates no stream
                           or event of its own, and the role overlap also works inside CUDA graph capture */
} svg2_layout_t;

/* The fused call with a layout (NULL layout == svg2_sparse_attention_ex). */
SVG2_API svg2_status_t svg2_sparse_attention_layout(const void* Q, const void* K, const void* V, svg2_dims_t dims,
                                                    const svg2_config_t* config, const svg2_layout_t* layout,
                                                    float* q_centroids, float* k_centroids, void* O,
                                                    int64_t* selected_pairs, const svg2_debug_t* dbg,
                                                    void* const* input_ready, void* ws, size_t ws_bytes,
                                                    void* stream);

/* ---- The fused call on HOST buffers (offload / end-to-end use).  Qh, Kh, Vh [B,H,N,d] bf16 and Oh [B,H,Nq,d] bf16
 * in host memory (page-locked for the copies to overlap; pageable memory works but serialises).  Same math and
 * results as svg2_sparse_attention, bit for bit.  The (b,h) heads are processed in chunks (small first and last ones,
 * then 6 equal middle ones): the copy of
 * chunk c+1 to the device and of chunk c-1 back to the host overlap the computation of chunk c, consecutive chunks
 * compute on three rotating streams, and each role of a chunk waits only for its own tensor's upload (internal
 * streams, three device staging slots and three fused-call workspaces in the workspace,
 * SVG2_ENTRY_SPARSE_ATTENTION_HOST).  The centroid caches and
 * selected_pairs are DEVICE buffers as in svg2_sparse_attention.  The work is ordered after the work already queued
 * on `stream`, and later work on `stream` waits for it; Oh is complete when `stream` has synchronised. */
SVG2_API svg2_status_t svg2_sparse_attention_host(const void* Qh, const void* Kh, const void* Vh, svg2_dims_t dims,
                                                  const svg2_config_t* config, float* q_centroids,
                                                  float* k_centroids, void* Oh, int64_t* selected_pairs, void* ws,
                                                  size_t ws_bytes, void* stream);

/* Number of kernels the fused call launches for these dims/config (for launch accounting in benchmarks). */
SVG2_API int32_t svg2_sparse_attention_launch_count(svg2_dims_t dims, const svg2_config_t* config);

#ifdef __cplusplus
}
#endif

#endif /* SVG2_H_ */

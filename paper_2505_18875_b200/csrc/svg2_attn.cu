// svg2_attn.cu — A9 (+ fused A10): variable-block sparse attention over the permuted, cluster-contiguous tokens
// (PAPER.md:329-334), written for sm_100a; and the work list (per-query-cluster key streams, work items) it runs on.
//
// Work item = two 128-row Q tiles of one query cluster i (contiguous rows of Q' after the permutation) sharing ONE
// packed key stream: the selected key clusters' row ranges of K'/V' (adjacent selected clusters merged into runs),
// each run padded to whole 8-row groups.  The paper loads K/V "sparsely per token via address offsets into
// contiguous shared memory"; here a key tile of the stream (kGpt groups) is assembled from TMA box
// loads straight into the 128B-swizzled layout the MMA descriptors expect: consecutive groups of one run merge into
// power-of-two boxes of 8..128 rows.  Padding rows of a run's last group are masked in the softmax (a 4-bit valid
// count per group, packed per tile into one 64-bit word).
//
// Pipeline.  The chain S(t) -> softmax(t) -> PV(t) -> S(t+1) -> softmax(t+1) of a Q tile is cut at
// S: each Q tile g has an S buffer and a SEPARATE P buffer in TMEM, and the softmax releases S(t) as soon as it has
// the scores in registers, so S(t+1) is computed while softmax(t) runs its exponentials and softmax(t+1) starts the
// moment softmax(t) hands P(t) over.  The softmax warpgroups then run back to back and the tensor pipe, not the
// softmax round trip, sets the pace.  Budget (512 TMEM columns): S_a, S_b (kN fp32 each), P_a, P_b (kN/2 packed
// bf16), O_a, O_b (D fp32), hence kN = 80 keys per tile for d = 128 and 128 for d = 64.
//
// Warp roles (384 threads, 1 CTA per SM, persistent; items fetched dynamically with an atomic counter, in the work-list
// order k_parts / k_items build: heads in order, each head's query clusters longest key stream first, so the launch
// ends on short items and the long streams of a head, which share most key clusters, run together in L2):
//   warps 0-3   softmax warpgroup of Q tile a; warps 4-7 of Q tile b.  One thread = one query row = one TMEM lane
//               (warp w owns lanes 32(w%4)..+31): tcgen05.ld S, release S, online softmax in registers (exp2 domain,
//               lazy rescale of O in TMEM when the running max grows by > 8, after the previous PV completed), P
//               (bf16) stored into the P buffer once the previous PV has read it; epilogue O / l -> bf16 -> global,
//               scattered to original token order through pi_q (fused A10).
//   warp 8      scheduler + TMA producer: fetches the next item, broadcasts it through a 2-slot smem ring, loads the
//               Q tiles and the K/V tiles (box loads) into kStages-deep rings
//   warp 9      TMEM allocator (512 columns)
//   warps 10/11 MMA issuers for Q tile a / b (whole warp convergent, elect.sync issues inside the asm), each in its
//               own order S(t0), [S(t+1), PV(t)] for t = t0.. — two warps so that neither tile's S waits behind the
//               other tile's P hand-over.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include "internal.h"
#include "ptx.cuh"
#include "tmap.h"

namespace svg2 {
namespace {

constexpr int kThreads = 384;
constexpr int kBoxKinds = 5;  // box heights 8, 16, 32, 64, 128 rows
// Lazy rescale threshold (log2 units): O and l are rescaled only when a row's tile max exceeds the max in use by more
// than this, so P <= 2^8 between rescales (bf16 P keeps its relative precision; O and l accumulate in fp32).
constexpr float kRescaleThreshold = 8.0f;
// setmaxnreg budget: the launch reserves 168 regs x 384 threads; the control warpgroup (warps 8-11) shrinks to 88 and
// the two softmax warpgroups grow to 208.  The sum must not exceed the reservation or .inc never returns.
constexpr int kRegsCtl = 88, kRegsSoftmax = 208, kRegsLaunch = 168;
static_assert(128 * kRegsCtl + 256 * kRegsSoftmax <= kRegsLaunch * kThreads, "setmaxnreg budget exceeds launch");
// warp 8: scheduler + Q and K loads; warp 9: TMEM allocator, then V loads; warps 10, 11: MMA issuers
constexpr int kWarpProducer = 8, kWarpTmem = 9, kWarpProducerV = 9, kWarpMma0 = 10;
constexpr int kItemConsumers = 1 + 2 + 8;  // the V producer, the two MMA warps and 8 softmax warps arrive on item_empty
// In every 8-pair chunk of a row's exponentials kPolyPairs pairs may take 2^x on the FMA pipe (ex2_poly2) instead of
// MUFU.  With the exponential phases of the two warps of an SMSP alternating (kBarTurnA), MUFU alone is fastest
// (attention, HunyuanVideo, interleaved A/B on one box: 46.2-46.5 / 46.7 / 47.3 / 48.1 / 49.6 / 51.6 / 54.8 ms at
// 0 / 1 / 2 / 3 / 4 / 5 / 6 pairs; without the alternation 1 pair: 50.2 ms, gpurun_out -> profiles/r02_micro).
#ifndef SVG2_POLY_PAIRS
#define SVG2_POLY_PAIRS 0
#endif
constexpr int kPolyPairs = SVG2_POLY_PAIRS;  // measurement builds override it with -DSVG2_POLY_PAIRS
// Exponential-phase hand-over between the two softmax warpgroups: warp w of tile a and warp w + 4 of
// tile b share an SMSP and its MUFU unit, so their exponential phases alternate strictly (a, b, a, b, ...): named
// barrier kBarTurnA + (w & 3) = "a may start", kBarTurnB + (w & 3) = "b may start", 64 threads each.  While one warp
// runs its exponentials the other loads S, takes the row max and stores P.  Split items deal the even key tiles to a
// and start with a (if it is b's turn, b hands the turn over first), so the alternation never waits for an
// exponential phase that does not exist;
// both warpgroups track that turn identically from the item sequence.
constexpr int kBarMerge = 1, kBarTurnA = 2, kBarTurnB = 6;
#ifndef SVG2_EXP_TURNS
#define SVG2_EXP_TURNS 1
#endif
constexpr bool kExpTurns = SVG2_EXP_TURNS != 0;  // measurement builds: -DSVG2_EXP_TURNS=0 lets both run freely

template <int D>
struct Cfg {
  static constexpr int kN = D == 128 ? 80 : 128;          // keys per S tile (N of QK^T, K of PV)
  static constexpr int kGpt = kN / 8;                      // 8-row groups per tile
  static constexpr int kBlocks = D / 64;                   // 64-column (128-byte) swizzle blocks per row
  static constexpr uint32_t kQBlockBytes = 128 * 128;      // one block of a 128-row Q tile
  static constexpr uint32_t kQTileBytes = kBlocks * kQBlockBytes;
  static constexpr uint32_t kKBlockBytes = kN * 128;       // one block of a kN-row K or V tile
  static constexpr uint32_t kKTileBytes = kBlocks * kKBlockBytes;
  static constexpr uint32_t kGroupBytes = 8 * 2 * D;       // 8 rows x D bf16
  static constexpr int kStages = D == 128 ? 4 : 6;         // K/V ring depth
  static constexpr uint32_t kSmemBytes = 2 * kQTileBytes + 2 * kStages * kKTileBytes + 1024;
  // P is held in registers until the previous PV has read the P buffer (d = 128); with 128-key tiles (d = 64) the
  // scores + P would not fit, so the softmax waits for that PV before its exponentials and stores P as it goes.
  static constexpr bool kHoldP = kN <= 96;
  // TMEM columns (every tcgen05.ld / st below is aligned to its own width)
  __device__ static constexpr uint32_t col_s(int g) { return g ? 128u : 0u; }
  __device__ static constexpr uint32_t col_p(int g) { return D == 128 ? (g ? 208u : 80u) : (g ? 320u : 256u); }
  __device__ static constexpr uint32_t col_o(int g) { return D == 128 ? (g ? 384u : 256u) : (g ? 448u : 384u); }
};
static_assert(Cfg<128>::kSmemBytes <= 227 * 1024 - 2048 && Cfg<64>::kSmemBytes <= 227 * 1024 - 2048, "smem");

struct Bars {
  uint64_t q_full, q_empty;
  uint64_t k_full[8], k_empty[8], v_full[8], v_empty[8];
  uint64_t s_full[2], s_free[2], p_full[2], pv_done[2], o_empty[2];
  uint64_t item_full[2], item_empty[2];
};

struct KVMaps {
  CUtensorMap k[kBoxKinds], v[kBoxKinds];  // box = 64 columns x (8 << kind) rows
};

struct Params {
  const int4* items;
  int32_t* n_items;  // [0] = count, [1] = dynamic-scheduler counter (zeroed by k_items), [2] = orphan rows
  const int2* groups;
  const uint64_t* tilew;
  const int32_t* ngroups;
  size_t gcap, tcap;
  const int32_t* q_perm;
  __nv_bfloat16* O;  // permuted-order output (q_perm == nullptr)
  OutView out;       // original-order output rows (q_perm set): the fused A10 scatter
  float* lse;
  int Nq;
  float scale_log2;
};

// Measurement build only (-DSVG2_TRACE, tools/trace_attn.py): clock64 per event and key tile of the first item of
// CTA 0, printed at kernel exit.  The product build compiles no trace code.
#ifdef SVG2_CTA_TIMES
// measurement build only (-DSVG2_CTA_TIMES, tools/cta_times.py): per CTA the globaltimer at start and exit and the
// number of items it processed
__device__ unsigned long long g_cta_times[1024][3];
#endif
#ifdef SVG2_TRACE
constexpr int kTrT = 48, kTrEv = 24;
__device__ long long g_trace[kTrEv][kTrT];
#define TRACE(ev, t)                                                                       \
  do {                                                                                     \
    if (blockIdx.x == 0 && tr_first && (t) < kTrT && (threadIdx.x & 31) == 0) g_trace[ev][t] = clock64(); \
  } while (0)
#else
#define TRACE(ev, t) \
  do {               \
  } while (0)
#endif

// Loads one tile (ngt <= kGpt groups) of the item's key stream into a K or V stage.  Lanes 0..ngt-1 hold one group
// each; a lane whose group does not continue the previous lane's full group starts a run segment and issues
// power-of-two boxes covering it.  The stage's mbarrier receives ngt x 8 rows x D x 2 bytes.
template <int D>
__device__ __forceinline__ void load_kv_tile(const CUtensorMap* maps, uint8_t* stage, uint64_t* bar, int ngt, int lane,
                                             int2 gw, uint64_t policy) {
  using C = Cfg<D>;
  const int prev_row = __shfl_up_sync(0xffffffffu, gw.x, 1);
  const int prev_nv = __shfl_up_sync(0xffffffffu, gw.y, 1);
  const bool in = lane < ngt;
  const bool cont = in && lane > 0 && gw.x == prev_row + 8 && prev_nv == 8;
  const bool start = in && !cont;
  const unsigned starts = __ballot_sync(0xffffffffu, start);
  if (start) {
    const unsigned above = starts & ~((2u << lane) - 1u);
    const int end = above ? (__ffs(above) - 1) : ngt;
    int pos = lane, len = end - lane, row = gw.x;
    while (len > 0) {
      const int kind = 31 - __clz(min(len, 16));  // largest power of two <= len, capped at 16 groups (128 rows)
      const int pw = 1 << kind;
#pragma unroll
      for (int b = 0; b < C::kBlocks; ++b)
        tma_load_2d_hint(stage + b * C::kKBlockBytes + pos * 1024, &maps[kind], bar, 64 * b, row, policy);
      pos += pw;
      len -= pw;
      row += 8 * pw;
    }
  }
}

template <int N>
__device__ __forceinline__ uint32_t (&sub32(uint32_t (&a)[N], int off))[32] {
  return *reinterpret_cast<uint32_t(*)[32]>(a + off);
}
template <int N>
__device__ __forceinline__ uint32_t (&sub16(uint32_t (&a)[N], int off))[16] {
  return *reinterpret_cast<uint32_t(*)[16]>(a + off);
}
template <int N>
__device__ __forceinline__ uint32_t (&sub8(uint32_t (&a)[N], int off))[8] {
  return *reinterpret_cast<uint32_t(*)[8]>(a + off);
}

template <int D>
__global__ void __launch_bounds__(kThreads, 1)
    k_varblock_attn(const __grid_constant__ CUtensorMap mapQ, const __grid_constant__ KVMaps kv, const Params p) {
  using C = Cfg<D>;
  constexpr int kN = C::kN, kGpt = C::kGpt, kSt = C::kStages;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;                            // [2][Q tile]
  uint8_t* sK = smem + 2 * C::kQTileBytes;       // [kSt][K tile]
  uint8_t* sV = sK + kSt * C::kKTileBytes;       // [kSt][V tile]
  __shared__ Bars bars;
  __shared__ uint32_t tmem_slot;
  __shared__ int4 item_slot[2];
  __shared__ float2 merge_ml[kQTile];  // split items: (m, l) of warpgroup b's rows
  __shared__ float zero_slot;          // 0.0f: the exponentials depend on a load of it after the turn barrier

  const int warp = __shfl_sync(0xffffffffu, int(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  if (warp == kWarpProducer && lane == 0) {
    tma_prefetch_desc(&mapQ);
    mbar_init(&bars.q_full, 1);
    mbar_init(&bars.q_empty, 2);  // one arrival per MMA warp
    for (int s = 0; s < kSt; ++s) {
      mbar_init(&bars.k_full[s], 1);
      mbar_init(&bars.k_empty[s], 2);  // two arrivals per tile: one per MMA warp using it, or two from its only user
      mbar_init(&bars.v_full[s], 1);
      mbar_init(&bars.v_empty[s], 2);
    }
    for (int g = 0; g < 2; ++g) {
      mbar_init(&bars.s_full[g], 1);
      mbar_init(&bars.s_free[g], 4);
      mbar_init(&bars.p_full[g], 4);
      mbar_init(&bars.pv_done[g], 1);
      mbar_init(&bars.o_empty[g], 4);
      mbar_init(&bars.item_full[g], 1);
      mbar_init(&bars.item_empty[g], kItemConsumers);
    }
    fence_mbar_init();
  }
  if (warp == kWarpTmem) tmem_alloc<512>(&tmem_slot);
  if (threadIdx.x == 0) zero_slot = 0.f;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = __shfl_sync(0xffffffffu, tmem_slot, 0);
  const int n_items = __ldg(p.n_items);
#ifdef SVG2_CTA_TIMES
  if (threadIdx.x == 0) {
    g_cta_times[blockIdx.x][0] = globaltimer_ns();
    g_cta_times[blockIdx.x][2] = 0;
  }
#endif

  if (warp >= 8) {
    reg_dealloc<kRegsCtl>();
    if (warp == kWarpProducer || warp == kWarpProducerV) {
      // ===================== scheduler + TMA producers (warp 8: Q and K tiles, warp 9: V tiles) =====================
      // Issuing a tile's box loads costs hundreds of cycles (each box's operands go through uniform registers), so
      // K and V have a warp each: the K/V rings then refill twice as fast.
      const bool vrole = warp == kWarpProducerV;
      const CUtensorMap* maps = vrole ? kv.v : kv.k;
      uint8_t* ring = vrole ? sV : sK;
      uint64_t* full = vrole ? bars.v_full : bars.k_full;
      uint64_t* empty = vrole ? bars.v_empty : bars.k_empty;
      uint32_t qph = 0, ks = 0, kph = 0, islot = 0, iph = 0;
      // L2 policies: K' / V' rows are re-read by every query cluster of the head that selects them (keep them),
      // Q' rows are read once (let them go first)
      const uint64_t pol_kv = l2_policy_evict_last(), pol_q = l2_policy_evict_first();
      bool tr_first = true;
      (void)tr_first;
      while (true) {
        int4 it;
        if (!vrole) {
          int item = 0;
          if (lane == 0) item = atomicAdd(p.n_items + 1, 1);
          item = __shfl_sync(0xffffffffu, item, 0);
#ifdef SVG2_CTA_TIMES
          if (lane == 0 && item < n_items) g_cta_times[blockIdx.x][2] += 1;
#endif
          it = item < n_items ? __ldg(p.items + item) : make_int4(-1, 0, 0, 0);
          mbar_wait(&bars.item_empty[islot], iph ^ 1);
          if (lane == 0) {
            item_slot[islot] = it;
            mbar_arrive(&bars.item_full[islot]);  // release: the slot write is visible to the waiting consumers
          }
        } else {
          mbar_wait(&bars.item_full[islot], iph);
          it = item_slot[islot];
          __syncwarp();
          if (lane == 0) mbar_arrive(&bars.item_empty[islot]);
        }
        if (++islot == 2) {
          islot = 0;
          iph ^= 1;
        }
        if (it.x < 0) break;
        const int nb = it.y >> 16;
        const int ng = __ldg(p.ngroups + it.z);
        const int2* grp = p.groups + size_t(it.z) * p.gcap;
        if (!vrole) {
          mbar_wait(&bars.q_empty, qph ^ 1);
          if (lane == 0) {
            mbar_arrive_expect_tx(&bars.q_full, (nb > 0 ? 2u : 1u) * C::kQTileBytes);
            for (int b = 0; b < C::kBlocks; ++b) {
              tma_load_2d_hint(sQ + b * C::kQBlockBytes, &mapQ, &bars.q_full, 64 * b, it.x, pol_q);
              if (nb > 0)
                tma_load_2d_hint(sQ + C::kQTileBytes + b * C::kQBlockBytes, &mapQ, &bars.q_full, 64 * b, it.x + 128,
                                 pol_q);
            }
          }
          qph ^= 1;
        }
        const int T = (ng + kGpt - 1) / kGpt;
        int2 gw = lane < min(kGpt, ng) ? __ldg(grp + lane) : make_int2(0, 0);
        for (int t = 0; t < T; ++t) {
          const int ngt = min(kGpt, ng - t * kGpt);
          // prefetch the next tile's group words while this tile's loads are being issued
          const int nxt = (t + 1) * kGpt + lane;
          const int2 gw_next = (t + 1 < T && lane < kGpt && nxt < ng) ? __ldg(grp + nxt) : make_int2(0, 0);
          mbar_wait(&empty[ks], kph ^ 1);
          if (lane == 0) mbar_arrive_expect_tx(&full[ks], uint32_t(ngt) * C::kGroupBytes);
          __syncwarp();
          load_kv_tile<D>(maps, ring + ks * C::kKTileBytes, &full[ks], ngt, lane, gw, pol_kv);
          TRACE(vrole ? 1 : 0, t);
          gw = gw_next;
          if (++ks == kSt) {
            ks = 0;
            kph ^= 1;
          }
        }
        tr_first = false;
      }
    } else if (warp >= kWarpMma0) {
      // ============================ MMA issuers (warp 10: Q tile a, warp 11: Q tile b) ============================
      const int g = warp - kWarpMma0;
      uint32_t qph = 0, islot = 0, iph = 0, ktile = 0;  // ktile: ring position of the item's first K/V tile
      uint32_t n_s = 0, n_p = 0, n_o = 0;               // S issued, PV waited for, items started (o_empty)
      const uint32_t idesc_pv = idesc_bf16_f32(128, D, true);
      const uint64_t dq0 = desc_kmajor_sw128(smem_u32(sQ)), dq1 = desc_kmajor_sw128(smem_u32(sQ + C::kQTileBytes));
      // ring stage s = the stage-0 descriptor + s tiles in the start-address field (16-byte units)
      const uint64_t dk0 = desc_kmajor_sw128(smem_u32(sK));
      const uint64_t dv0 = desc_mnmajor_sw128(smem_u32(sV), C::kKBlockBytes);
      const uint32_t tS = tmem + C::col_s(g), tP = tmem + C::col_p(g), tO = tmem + C::col_o(g);
      bool tr_first = true;
      (void)tr_first;
      while (true) {
        mbar_wait_warp(&bars.item_full[islot], iph);
        const int4 it = item_slot[islot];
        __syncwarp();
        mbar_arrive_warp(&bars.item_empty[islot]);
        if (++islot == 2) {
          islot = 0;
          iph ^= 1;
        }
        if (__all_sync(0xffffffffu, it.x < 0)) break;
        const bool has_b = (it.y >> 16) > 0;
        const bool split = (it.w & kItemSplit) != 0;  // one Q tile, key tiles dealt alternately to a and b
        const int ng = __ldg(p.ngroups + it.z);
        const int T = (ng + kGpt - 1) / kGpt;
        // this warp's key tiles: split -> g, g + 2, ...; otherwise all of them (tile a, and tile b if present)
        const int t0 = split ? g : 0, ts = split ? 2 : 1;
        const bool active = split ? g < T : (g == 0 || has_b);
        const bool shared = !split && has_b;  // both warps read every K/V tile: one release arrival each
        const uint64_t qd = (g == 1 && !split) ? dq1 : dq0;
        mbar_wait_warp(&bars.q_full, qph);
        qph ^= 1;
        if (!active) {
          mma_commit_warp(&bars.q_empty);
          ktile += T;
          continue;
        }
        auto stage = [&](int t) { return (ktile + uint32_t(t)) % uint32_t(kSt); };
        auto parity = [&](int t) { return ((ktile + uint32_t(t)) / uint32_t(kSt)) & 1u; };
        auto tile_n = [&](int t) { return uint32_t(min(kGpt, ng - t * kGpt)) * 8u; };
        auto issue_s = [&](int t) {
          const uint32_t st = stage(t);
          mbar_wait_warp(&bars.k_full[st], parity(t));
          mbar_wait_warp(&bars.s_free[g], (n_s & 1) ^ 1);  // the softmax holds S(t - 1) in registers
          ++n_s;
          tc_fence_after();
          TRACE(2 + g, t);
          const uint32_t idesc = idesc_bf16_f32(128, tile_n(t), false);
          const uint64_t kd = dk0 + uint64_t(st) * (C::kKTileBytes >> 4);
#pragma unroll
          for (int k = 0; k < D / 16; ++k) {
            const uint64_t qo = uint64_t(((k >> 2) * C::kQBlockBytes + (k & 3) * 32) >> 4);
            const uint64_t ko = uint64_t(((k >> 2) * C::kKBlockBytes + (k & 3) * 32) >> 4);
            mma_ss_warp(tS, qd + qo, kd + ko, idesc, k > 0);
          }
          mma_commit_warp(&bars.s_full[g]);
          mma_commit_warp(&bars.k_empty[st]);
          if (!shared) mma_commit_warp(&bars.k_empty[st]);
        };
        auto issue_pv = [&](int t, bool first) {
          const uint32_t st = stage(t);
          mbar_wait_warp(&bars.v_full[st], parity(t));
          mbar_wait_warp(&bars.p_full[g], n_p & 1);
          ++n_p;
          if (first) {  // the previous item's epilogue has read O
            mbar_wait_warp(&bars.o_empty[g], (n_o & 1) ^ 1);
            ++n_o;
          }
          tc_fence_after();
          TRACE(4 + g, t);
          const uint64_t vd = dv0 + uint64_t(st) * (C::kKTileBytes >> 4);
          const int ksteps = int(tile_n(t)) / 16;
#pragma unroll 1
          for (int k = 0; k < ksteps; ++k)
            mma_ts_warp(tO, tP + 8 * k, vd + uint64_t((k * 16 * 128) >> 4), idesc_pv, (!first || k > 0) ? 1u : 0u);
          mma_commit_warp(&bars.pv_done[g]);
          mma_commit_warp(&bars.v_empty[st]);
          if (!shared) mma_commit_warp(&bars.v_empty[st]);
        };
        issue_s(t0);
        if (t0 + ts >= T) mma_commit_warp(&bars.q_empty);
        for (int t = t0; t < T; t += ts) {
          if (t + ts < T) {
            issue_s(t + ts);  // S(t+1) before PV(t): it only needs the softmax to have read S(t)
            if (t + 2 * ts >= T) mma_commit_warp(&bars.q_empty);
          }
          issue_pv(t, t == t0);
        }
        ktile += T;
        tr_first = false;
      }
    }
  } else {
    reg_alloc<kRegsSoftmax>();
    // ============================ softmax warpgroups ============================
    const int g = warp >> 2;                        // 0: tile a, 1: tile b
    const int rloc = ((warp & 3) << 5) + lane;      // row in the tile == TMEM lane
    const uint32_t lane_addr = uint32_t((warp & 3) * 32) << 16;
    const uint32_t tS = tmem + lane_addr + C::col_s(g);
    const uint32_t tP = tmem + lane_addr + C::col_p(g);
    const uint32_t tO = tmem + lane_addr + C::col_o(g);
    const float sl2 = p.scale_log2;
    uint32_t n_sf = 0, n_pv = 0, islot = 0, iph = 0;  // s_full / pv_done phases consumed
    const int bar_mine = (g == 0 ? kBarTurnA : kBarTurnB) + (warp & 3);
    const int bar_other = (g == 0 ? kBarTurnB : kBarTurnA) + (warp & 3);
    bool turn_a = true;
    if (kExpTurns && g == 1) named_bar_arrive(bar_other, 64);  // tile a's warps go first
    bool tr_first = true;
    (void)tr_first;
    auto wait_pv = [&] {
      mbar_wait(&bars.pv_done[g], n_pv & 1);
      ++n_pv;
      tc_fence_after();
    };
    while (true) {
      mbar_wait(&bars.item_full[islot], iph);
      const int4 it = item_slot[islot];
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars.item_empty[islot]);
      if (++islot == 2) {
        islot = 0;
        iph ^= 1;
      }
      if (it.x < 0) break;
      const bool split = (it.w & kItemSplit) != 0;  // both warpgroups on Q tile a, alternate key tiles
      const bool paired = kExpTurns && (split || (it.y >> 16) > 0);  // both warpgroups work: exponentials alternate
      const int nrows = (g == 0 || split) ? (it.y & 0xFFFF) : (it.y >> 16);
      if (nrows <= 0) continue;
      const int ng = __ldg(p.ngroups + it.z);
      const uint64_t* tw = p.tilew + size_t(it.z) * p.tcap;
      const int T = (ng + kGpt - 1) / kGpt;
      const int t_first = split ? g : 0, t_step = split ? 2 : 1;
      if (kExpTurns && split) {
        // a split item's exponentials start with tile a's warps (even tiles, a fixed deal: the merge is then
        // bitwise reproducible); if it is b's turn, b passes the turn on without an exponential phase
        if (!turn_a && g == 1) {
          named_bar_sync(bar_mine, 64);
          named_bar_arrive(bar_other, 64);
        }
        turn_a = (T & 1) == 0;  // the last exponential phase of the item is a's iff T is odd
      }
      float m_used = -INFINITY, l = 0.f;
      uint64_t word_next = __ldg(tw + t_first);
      for (int t = t_first; t < T; t += t_step) {
        const uint64_t word = word_next;  // 4-bit valid counts of the tile's groups (0 beyond the stream)
        if (t + t_step < T) word_next = __ldg(tw + t + t_step);
        mbar_wait(&bars.s_full[g], n_sf & 1);
        ++n_sf;
        tc_fence_after();
        if ((warp & 3) == 0) TRACE(6 + g, t);
        uint32_t s[kN];
#pragma unroll
        for (int c = 0; c < kN / 32; ++c) tmem_ld32(tS + 32 * c, sub32(s, 32 * c));
        if constexpr (kN % 32 != 0) tmem_ld16(tS + kN - 16, sub16(s, kN - 16));
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars.s_free[g]);  // S(t+1) may now overwrite the S buffer
        if ((warp & 3) == 0) TRACE(8 + g, t);
        // Padding rows of partial 8-row groups get -inf scores.  The word is the same for every lane, so each
        // group's test is a uniform branch and only partial groups pay for the selects.
        if (word != (0x8888888888888888ull >> (64 - 4 * kGpt))) {
#pragma unroll
          for (int q = 0; q < kGpt; ++q) {
            const uint32_t nv = uint32_t(word >> (4 * q)) & 15u;
            if (nv < 8u) {
#pragma unroll
              for (int e = 0; e < 8; ++e)
                if (uint32_t(e) >= nv) s[8 * q + e] = __float_as_uint(-INFINITY);
            }
          }
        }
        // row max on the raw scores (scale > 0 preserves order)
        float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
        for (int e = 0; e < kN; e += 4) {
          mx0 = fmaxf(mx0, fmaxf(__uint_as_float(s[e]), __uint_as_float(s[e + 2])));
          mx1 = fmaxf(mx1, fmaxf(__uint_as_float(s[e + 1]), __uint_as_float(s[e + 3])));
        }
        const float mt = fmaxf(mx0, mx1) * sl2;
        if ((warp & 3) == 0) TRACE(14 + g, t);
        bool pv_waited = t == t_first;  // no PV of this item in flight before its first tile
        if (t == t_first) {
          m_used = mt;
        } else if (__any_sync(0xffffffffu, rloc < nrows && mt > m_used + kRescaleThreshold)) {
          // only rows of the cluster vote: the tile's padding rows hold whatever follows the cluster in Q' (another
          // cluster or head) and must not change how the cluster's rows are rounded.  Warp-uniform branch
          // (tcgen05.ld/st are .sync.aligned); rows whose max did not grow get alpha = 1.  O is complete up to PV(t-1).
          wait_pv();
          pv_waited = true;
          const float m_new = fmaxf(m_used, mt);
          const float alpha = ex2_approx(m_used - m_new);
          l *= alpha;
#pragma unroll 1
          for (int c = 0; c < D / 32; ++c) {
            uint32_t o[32];
            tmem_ld32(tO + 32 * c, o);
            tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
            tmem_st32(tO + 32 * c, o);
          }
          m_used = m_new;
        }
        if (!C::kHoldP && !pv_waited) {
          wait_pv();
          pv_waited = true;
        }
        // p = 2^(s * scale*log2e - m): FFMA2 on pairs, MUFU ex2 per element (kPolyPairs of 8 pairs on the FMA pipe),
        // FADD2 row sums, bf16x2 packs
        float negm = -m_used;
        if (paired) {  // the partner warp on this SMSP has finished its exponentials
          named_bar_sync(bar_mine, 64);
          negm += ld_shared_volatile(&zero_slot);  // every exponential depends on a load after the barrier
        }
        const uint64_t sl2x2 = f2(sl2, sl2), negm2 = f2(negm, negm);
        if (g == 0) TRACE(20 + (warp & 3), t);  // exponential phase start, each warp of tile a
        uint64_t lsum2 = f2(0.f, 0.f);
        uint32_t pk[kN / 2];
#pragma unroll
        for (int e = 0; e < kN / 2; ++e) {
          float x0, x1;
          f2_split(ffma2(f2(__uint_as_float(s[2 * e]), __uint_as_float(s[2 * e + 1])), sl2x2, negm2), x0, x1);
          float p0, p1;
          if ((e % 8) < kPolyPairs) {
            f2_split(ex2_poly2(f2(x0, x1)), p0, p1);
          } else {
            p0 = ex2_approx(x0);
            p1 = ex2_approx(x1);
          }
          lsum2 = fadd2(lsum2, f2(p0, p1));
          pk[e] = pack_bf16x2(p0, p1);
          if (!C::kHoldP && e % 16 == 15) tmem_st16(tP + (e - 15), sub16(pk, e - 15));
        }
        if (paired) named_bar_arrive_after(bar_other, 64, lsum2);  // after the last exponential
        if ((warp & 3) == 0) TRACE(10 + g, t);
        if (C::kHoldP) {
          if (!pv_waited) wait_pv();  // PV(t-1) has read the P buffer
#pragma unroll
          for (int c = 0; c < kN / 32; ++c) tmem_st16(tP + 16 * c, sub16(pk, 16 * c));
          if constexpr (kN % 32 != 0) tmem_st8(tP + kN / 2 - 8, sub8(pk, kN / 2 - 8));
        }
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars.p_full[g]);
        if ((warp & 3) == 0) TRACE(12 + g, t);
        if (g == 0) TRACE(16 + (warp & 3), t);  // P stored, each warp of tile a
        float ls0, ls1;
        f2_split(lsum2, ls0, ls1);
        l += ls0 + ls1;
      }
      // ---- epilogue: O / l  -> bf16 -> original token order (fused pi_q^T)
      wait_pv();  // the last PV of this warpgroup's tiles
      tr_first = false;
      if (split) {
        // Merge the two partial softmax states of the same rows (flash-decoding style): warpgroup b hands (m, l)
        // over through shared memory, warpgroup a reads O_a and O_b from TMEM and writes
        //   O = (2^(m_a-m) O_a + 2^(m_b-m) O_b) / (2^(m_a-m) l_a + 2^(m_b-m) l_b),  m = max(m_a, m_b).
        // Warpgroup a releases both O accumulators (o_empty counts 4 arrivals, one per warp of a).
        if (g == 1) merge_ml[rloc] = make_float2(m_used, l);
        tc_fence_before();
        named_bar_sync(kBarMerge, 256);
        float2 mlb = make_float2(0.f, 0.f);
        if (g == 0) mlb = merge_ml[rloc];
        // warpgroup b may write merge_ml again only after a has read it (the o_full / o_empty chain already orders
        // this; the second barrier makes it explicit at the cost of one 256-thread sync per split item)
        named_bar_sync(kBarMerge, 256);
        if (g == 1) continue;
        tc_fence_after();
        const float m = fmaxf(m_used, mlb.x);
        const float wa = ex2_approx(m_used - m), wb = ex2_approx(mlb.x - m);
        const float lt = l * wa + mlb.y * wb;
        const float ca = wa / lt, cb = wb / lt;
        const long long row_flat = (long long)it.x + rloc;
        long long dst = row_flat;
        uint4* orow = reinterpret_cast<uint4*>(p.O + dst * D);
        if (rloc < nrows && p.q_perm) {
          const int bh = it.w & kItemBhMask;
          const int n = __ldg(p.q_perm + row_flat);
          dst = (long long)bh * p.Nq + n;
          orow = reinterpret_cast<uint4*>(p.out.row(bh, n));
        }
        const uint32_t tOb = tmem + lane_addr + C::col_o(1);
#pragma unroll 1
        for (int c = 0; c < D / 32; ++c) {
          uint32_t oa[32], ob[32];
          tmem_ld32(tO + 32 * c, oa);
          tmem_ld32(tOb + 32 * c, ob);
          tmem_wait_ld();
          if (rloc < nrows) {
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              float r[8];
#pragma unroll
              for (int e = 0; e < 8; ++e)
                r[e] = __uint_as_float(oa[8 * v + e]) * ca + __uint_as_float(ob[8 * v + e]) * cb;
              __stcs(orow + 4 * c + v, make_uint4(pack_bf16x2(r[0], r[1]), pack_bf16x2(r[2], r[3]),
                                                  pack_bf16x2(r[4], r[5]), pack_bf16x2(r[6], r[7])));
            }
          }
        }
        if (rloc < nrows && p.lse) p.lse[dst] = (m + __log2f(lt)) * 0.69314718055994531f;
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&bars.o_empty[0]);
          mbar_arrive(&bars.o_empty[1]);
        }
        continue;
      }
      const float inv_l = 1.f / l;
      const long long row_flat = (long long)it.x + g * kQTile + rloc;
      long long dst = row_flat;
      uint4* orow = reinterpret_cast<uint4*>(p.O + dst * D);
      if (rloc < nrows && p.q_perm) {
        const int bh = it.w & kItemBhMask;
        const int n = __ldg(p.q_perm + row_flat);
        dst = (long long)bh * p.Nq + n;
        orow = reinterpret_cast<uint4*>(p.out.row(bh, n));
      }
#pragma unroll
      for (int c = 0; c < D / 32; ++c) {
        uint32_t o[32];
        tmem_ld32(tO + 32 * c, o);
        tmem_wait_ld();
        if (rloc < nrows) {
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            uint4 u;
            u.x = pack_bf16x2(__uint_as_float(o[8 * v + 0]) * inv_l, __uint_as_float(o[8 * v + 1]) * inv_l);
            u.y = pack_bf16x2(__uint_as_float(o[8 * v + 2]) * inv_l, __uint_as_float(o[8 * v + 3]) * inv_l);
            u.z = pack_bf16x2(__uint_as_float(o[8 * v + 4]) * inv_l, __uint_as_float(o[8 * v + 5]) * inv_l);
            u.w = pack_bf16x2(__uint_as_float(o[8 * v + 6]) * inv_l, __uint_as_float(o[8 * v + 7]) * inv_l);
            __stcs(orow + 4 * c + v, u);  // streamed: O is not re-read by this kernel
          }
        }
      }
      if (rloc < nrows && p.lse) p.lse[dst] = (m_used + __log2f(l)) * 0.69314718055994531f;
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars.o_empty[g]);
    }
  }
  tc_fence_before();
  __syncthreads();
#ifdef SVG2_CTA_TIMES
  if (threadIdx.x == 0) g_cta_times[blockIdx.x][1] = globaltimer_ns();
#endif
  if (warp == kWarpTmem) tmem_dealloc<512>(tmem);
}

template <int D>
cudaError_t run_attn(const void* Qp, const void* Kp, const void* Vp, int BH, int Nq, int Nk, float scale,
                     const int32_t* q_perm, const OutView& out, float* lse, AttnWs ws, cudaStream_t s) {
  using C = Cfg<D>;
  CUtensorMap mq;
  KVMaps kv;
  if (!make_tmap_bf16(&mq, Qp, uint64_t(BH) * Nq, D, 128)) return cudaErrorInvalidValue;
  for (int k = 0; k < kBoxKinds; ++k)
    if (!make_tmap_bf16(&kv.k[k], Kp, uint64_t(BH) * Nk, D, 8u << k) ||
        !make_tmap_bf16(&kv.v[k], Vp, uint64_t(BH) * Nk, D, 8u << k))
      return cudaErrorInvalidValue;
  Params p;
  p.items = ws.items;
  p.n_items = ws.n_items;
  p.groups = ws.groups;
  p.tilew = ws.tilew;
  p.ngroups = ws.ngroups;
  p.gcap = ws.gcap;
  p.tcap = ws.tcap;
  p.q_perm = q_perm;
  p.O = static_cast<__nv_bfloat16*>(out.shard[0]);
  p.out = out;
  p.lse = lse;
  p.Nq = Nq;
  p.scale_log2 = scale * 1.4426950408889634f;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaFuncSetAttribute(k_varblock_attn<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::kSmemBytes));
  k_varblock_attn<D><<<sms, kThreads, C::kSmemBytes, s>>>(mq, kv, p);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- work-list builder
// block-wide exclusive scan (NT threads, one value each); *total receives the block sum
template <int NT, typename T>
__device__ T build_scan(T v, T* total) {
  __shared__ T wsum[NT / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  T x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const T y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[w] = x;
  __syncthreads();
  T before = 0, tot = 0;
#pragma unroll
  for (int k = 0; k < NT / 32; ++k) {
    before += k < w ? wsum[k] : 0;
    tot += wsum[k];
  }
  __syncthreads();
  *total = tot;
  return before + x - v;
}

// One CTA per (b,h,i): the key stream of query cluster i = its selected, non-empty key clusters in ascending j,
// contiguous clusters merged into runs, runs cut into 8-row groups (the last one partial), the stream padded to an
// even group count; plus the packed 4-bit valid counts per gpt-group tile.  Three block scans (selected clusters with
// their key rows packed into one 64-bit scan, run starts, groups per run) make every step parallel; NT = 512 threads
// for C_k > 1024 so a mask row takes few scan rounds.
template <int NT>
__global__ void __launch_bounds__(NT) k_build_streams(const int32_t* __restrict__ k_off,
                                                                 const uint8_t* __restrict__ mask, int Nk, int Cq,
                                                                 int Ck, int gpt, AttnWs ws) {
  extern __shared__ int sbuf[];
  int* sel_s = sbuf;           // [Ck] start row (within head) of the k-th selected non-empty cluster
  int* sel_e = sel_s + Ck;     // [Ck] end row
  int* run_s = sel_e + Ck;     // [Ck] run start
  int* run_e = run_s + Ck;     // [Ck] run end
  int* run_g = run_e + Ck;     // [Ck+1] first group of the run
  const int i = blockIdx.x, bh = blockIdx.y, tid = threadIdx.x;
  const size_t li = size_t(bh) * Cq + i;
  const uint8_t* mrow = mask + li * Ck;
  const int32_t* ko = k_off + size_t(bh) * (Ck + 1);
  // 1) compact the selected, non-empty clusters (ascending j); count the stream's key rows
  int base = 0;
  long long nkeys = 0;
  for (int j0 = 0; j0 < Ck; j0 += NT) {
    const int j = j0 + tid;
    int s = 0, e = 0, f = 0;
    if (j < Ck && mrow[j]) {
      s = __ldg(ko + j);
      e = __ldg(ko + j + 1);
      f = e > s;
    }
    long long tot;  // (key rows << 20) | selected clusters: one scan for both (<= NT clusters per round)
    const int pos = base + int(build_scan<NT, long long>((static_cast<long long>(e - s) << 20) | f, &tot) & 0xFFFFF);
    if (f) {
      sel_s[pos] = s;
      sel_e[pos] = e;
    }
    base += int(tot & 0xFFFFF);
    nkeys += tot >> 20;
  }
  if (tid == 0) ws.keys[li] = int(nkeys);
  const int nsel = base;
  __syncthreads();
  // 2) runs: a selected cluster starts a run unless it begins exactly where the previous one ends
  base = 0;
  for (int k0 = 0; k0 < nsel; k0 += NT) {
    const int k = k0 + tid;
    const int f = (k < nsel) && (k == 0 || sel_s[k] != sel_e[k - 1]);
    int tot;
    const int r = base + build_scan<NT, int>(f, &tot);
    if (f) run_s[r] = sel_s[k];
    base += tot;
  }
  const int nrun = base;
  __syncthreads();
  for (int k = tid; k < nsel; k += NT) {  // the last cluster of each run writes the run end
    const bool last = (k == nsel - 1) || (sel_s[k + 1] != sel_e[k]);
    if (last) {
      int lo = 0, hi = nrun - 1;  // the run containing cluster k: last run start <= its start
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (run_s[mid] <= sel_s[k]) lo = mid; else hi = mid - 1;
      }
      run_e[lo] = sel_e[k];
    }
  }
  __syncthreads();
  // 3) groups per run -> group offsets
  base = 0;
  for (int r0 = 0; r0 < nrun; r0 += NT) {
    const int r = r0 + tid;
    const int gr = r < nrun ? (run_e[r] - run_s[r] + 7) / 8 : 0;
    int tot;
    const int g0 = base + build_scan<NT, int>(gr, &tot);
    if (r < nrun) run_g[r] = g0;
    base += tot;
  }
  const int ng_real = base;
  const int ng = ng_real + (ng_real & 1);  // even group count: every MMA has N = 16 k keys
  if (tid == 0) {
    run_g[nrun] = ng_real;
    ws.ngroups[li] = ng;
  }
  __syncthreads();
  const int rowbase = int(size_t(bh) * Nk);
  int2* grp = ws.groups + li * ws.gcap;
  // one thread per gpt-group tile: locate the tile's first group by binary search, then walk the runs forward,
  // writing the group words and packing the tile's 4-bit valid counts in the same pass
  uint64_t* tw = ws.tilew + li * ws.tcap;
  const int ntiles = (ng + gpt - 1) / gpt;
  for (int t = tid; t < ntiles; t += NT) {
    const int g0 = t * gpt, g1 = min(ng, g0 + gpt);
    int r = 0;
    if (g0 < ng_real) {
      int lo = 0, hi = nrun - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (run_g[mid] <= g0) lo = mid; else hi = mid - 1;
      }
      r = lo;
    }
    uint64_t word = 0;
    for (int gi = g0; gi < g1; ++gi) {
      int2 gw;
      if (gi >= ng_real) {
        gw = make_int2(rowbase + run_s[0], 0);  // the padding group: valid rows, all masked
      } else {
        while (run_g[r + 1] <= gi) ++r;  // run_g[nrun] = ng_real > gi
        const int row = run_s[r] + 8 * (gi - run_g[r]);
        gw = make_int2(rowbase + row, min(8, run_e[r] - row));
      }
      grp[gi] = gw;
      word |= uint64_t(gw.y) << (4 * (gi - g0));
    }
    tw[t] = word;
  }
}

// Query-cluster partition (QPart): per head, cluster i costs c_i = |Q_i| * keys_i (its attention pairs); with P_i the
// cost of clusters 0..i-1 and T the head's total, cluster i belongs to part floor((2 P_i + c_i) * count / (2 T)) --
// the part its cost midpoint falls in, so the parts' costs differ by at most one cluster; owned = part in
// [begin, end).  One CTA per head.
__global__ void __launch_bounds__(1024) k_parts(const int32_t* __restrict__ q_off, int Cq, QPart part, AttnWs ws) {
  __shared__ long long wsum[32];
  const int bh = blockIdx.x, tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  constexpr int kPer = (kMaxClusters + 1023) / 1024;  // clusters per thread (contiguous)
  long long c[kPer], run = 0;
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    const int i = tid * kPer + u;
    c[u] = 0;
    if (i < Cq) {
      const long long sq = q_off[size_t(bh) * (Cq + 1) + i + 1] - q_off[size_t(bh) * (Cq + 1) + i];
      c[u] = sq * ws.keys[size_t(bh) * Cq + i];
    }
    run += c[u];
  }
  long long x = run;
  for (int o = 1; o < 32; o <<= 1) {
    const long long y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[w] = x;
  __syncthreads();
  long long before = 0, T = 0;
  for (int k = 0; k < 32; ++k) {
    before += k < w ? wsum[k] : 0;
    T += wsum[k];
  }
  long long P = before + x - run;
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    const int i = tid * kPer + u;
    if (i < Cq) {
      const long long pi = T > 0 ? (2 * P + c[u]) * part.count / (2 * T) : 0;
      ws.owned[size_t(bh) * Cq + i] = pi >= part.begin && pi < part.end;
    }
    P += c[u];
  }
  // the work-list order of this head's clusters: longest key stream first (ties: lower index), k_items lists the
  // items in this order so the persistent attention launch ends on short items
  __shared__ int ng_s[kMaxClusters];
  const int32_t* ng = ws.ngroups + size_t(bh) * Cq;
  for (int i = tid; i < Cq; i += 1024) ng_s[i] = ng[i];
  __syncthreads();
  for (int i = tid; i < Cq; i += 1024) {
    const int gi = ng_s[i];
    int rank = 0;
    for (int k = 0; k < Cq; ++k) {
      const int gk = ng_s[k];
      rank += (gk > gi || (gk == gi && k < i)) ? 1 : 0;
    }
    ws.order[size_t(bh) * Cq + rank] = i;
  }
}

// Work items in (b,h)-major order, clusters of a head in k_parts' order (longest key stream first): ceil(|Q_i| / 256) pairs of 128-row Q
// tiles per non-empty query cluster with a non-empty key stream.  One CTA scans all B*H*Cq clusters; also resets the dynamic-scheduler counter.  A
// query cluster whose mask row selects no non-empty key cluster (a contract violation of svg2_varblock_attention,
// include/svg2.h; impossible in the fused call, where every row selects >= 1 non-empty cluster) gets no item: its
// output rows (and lse) are filled with NaN here, so the violation is visible instead of leaving memory unwritten,
// and n_items[2] counts those rows.
__global__ void __launch_bounds__(1024) k_items(const int32_t* __restrict__ q_off, int BH, int Nq, int Cq, int gpt,
                                                AttnWs ws, OrphanFill of) {
  __shared__ int wsum[32];
  __shared__ int n_orphan;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid == 0) n_orphan = 0;
  const int total_clusters = BH * Cq;
  __syncthreads();
  int base = 0;
  for (int c0 = 0; c0 < total_clusters; c0 += 1024) {
    int c = c0 + tid;
    int n = 0, q0 = 0, sq = 0, bh = 0;
    if (c < total_clusters) {
      bh = c / Cq;
      c = bh * Cq + ws.order[c];  // the cluster at this position of the head's order (k_parts)
      const int i = c - bh * Cq;
      q0 = q_off[size_t(bh) * (Cq + 1) + i];
      sq = q_off[size_t(bh) * (Cq + 1) + i + 1] - q0;
      if (!ws.owned[c]) {
        // another part's query cluster (multi-GPU split of the head): no items, no output rows here
      } else if (ws.ngroups[c] > 0) {
        n = (sq + kItemRows - 1) / kItemRows;
      } else if (sq > 0) {
        atomicAdd(&n_orphan, sq);
        const uint4 nan4 = make_uint4(0x7FC07FC0u, 0x7FC07FC0u, 0x7FC07FC0u, 0x7FC07FC0u);  // bf16 NaN
        for (int r = 0; r < sq; ++r) {
          const long long row_flat = (long long)bh * Nq + q0 + r;
          const long long dst = of.q_perm ? (long long)bh * Nq + of.q_perm[row_flat] : row_flat;
          uint4* orow = reinterpret_cast<uint4*>(of.q_perm ? of.out.row(bh, of.q_perm[row_flat])
                                                           : static_cast<uint16_t*>(of.out.shard[0]) + dst * of.d);
          for (int v = 0; v < of.d / 8; ++v) orow[v] = nan4;
          if (of.lse) of.lse[dst] = __int_as_float(0x7FC00000);
        }
      }
    }
    int x = n;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    int before = 0, tot = 0;
    for (int k = 0; k < 32; ++k) {
      before += k < w ? wsum[k] : 0;
      tot += wsum[k];
    }
    __syncthreads();
    int slot = base + before + x - n;
    for (int u = 0; u < n; ++u) {
      const int rem = sq - u * kItemRows;
      const int na = min(kQTile, rem), nb = max(0, min(kQTile, rem - kQTile));
      // a lone Q tile with >= 2 key tiles is split over both softmax warpgroups (even / odd key tiles)
      const int split = (nb == 0 && ws.ngroups[c] > gpt) ? kItemSplit : 0;
      ws.items[slot++] = make_int4(int(size_t(bh) * Nq) + q0 + u * kItemRows, na | (nb << 16), c, bh | split);
    }
    base += tot;
  }
  __syncthreads();
  if (tid == 0) {
    ws.n_items[0] = base;
    ws.n_items[1] = 0;  // dynamic scheduler counter of the next attention launch
    ws.n_items[2] = n_orphan;
  }
}

}  // namespace

__global__ void k_dense_qoff(int BH, int Nq, int32_t* __restrict__ q_offsets) {
  const int bh = blockIdx.x * blockDim.x + threadIdx.x;
  if (bh < BH) {
    q_offsets[2 * bh] = 0;
    q_offsets[2 * bh + 1] = Nq;
  }
}

static_assert(Cfg<128>::kGpt >= kMinGroupsPerTile && Cfg<64>::kGpt >= kMinGroupsPerTile, "tile_cap");
int attn_groups_per_tile(int d, bool fp8) { return fp8 ? kKTile / 8 : (d == 128 ? Cfg<128>::kGpt : Cfg<64>::kGpt); }

cudaError_t launch_dense_stream(int BH, int Nq, int Ck, int32_t* q_offsets, uint8_t* mask, cudaStream_t s) {
  k_dense_qoff<<<(BH + 127) / 128, 128, 0, s>>>(BH, Nq, q_offsets);
  cudaMemsetAsync(mask, 1, size_t(BH) * Ck, s);
  return cudaGetLastError();
}

cudaError_t launch_build_worklist(const int32_t* q_offsets, const int32_t* k_offsets, const uint8_t* mask, int BH,
                                  int Nq, int Nk, int Cq, int Ck, int gpt, AttnWs ws, OrphanFill of, cudaStream_t s,
                                  QPart part) {
  const size_t smem = (5 * size_t(Ck) + 1) * sizeof(int);
  if (Ck > 1024) {
    cudaFuncSetAttribute(k_build_streams<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    k_build_streams<512><<<dim3(Cq, BH), 512, smem, s>>>(k_offsets, mask, Nk, Cq, Ck, gpt, ws);
  } else {
    cudaFuncSetAttribute(k_build_streams<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    k_build_streams<128><<<dim3(Cq, BH), 128, smem, s>>>(k_offsets, mask, Nk, Cq, Ck, gpt, ws);
  }
  k_parts<<<BH, 1024, 0, s>>>(q_offsets, Cq, part, ws);
  k_items<<<1, 1024, 0, s>>>(q_offsets, BH, Nq, Cq, gpt, ws, of);
  return cudaGetLastError();
}

// svg2_attn_fp8.cu: the FP8 PV pipeline (DESIGN R26), 128-key tiles
cudaError_t launch_varblock_attention_fp8(const void* Qp, const void* Kp, const void* Vp, int BH, int Nq, int Nk,
                                          int d, float scale, const int32_t* q_perm, const OutView& out, float* lse,
                                          AttnWs ws, cudaStream_t s, const uint32_t* v_amax);

cudaError_t launch_varblock_attention(const void* Qp, const void* Kp, const void* Vp, int BH, int Nq, int Nk, int d,
                                      float scale, const int32_t* q_perm, const OutView& out, float* lse, AttnWs ws,
                                      cudaStream_t s, const uint32_t* v_amax) {
  if (v_amax) return launch_varblock_attention_fp8(Qp, Kp, Vp, BH, Nq, Nk, d, scale, q_perm, out, lse, ws, s, v_amax);
  if (d == 128) return run_attn<128>(Qp, Kp, Vp, BH, Nq, Nk, scale, q_perm, out, lse, ws, s);
  return run_attn<64>(Qp, Kp, Vp, BH, Nq, Nk, scale, q_perm, out, lse, ws, s);
}

}  // namespace svg2

#ifdef SVG2_CTA_TIMES
extern "C" __attribute__((visibility("default"))) int svg2_cta_times_dump(unsigned long long* out) {
  return int(cudaMemcpyFromSymbol(out, svg2::g_cta_times, sizeof(svg2::g_cta_times)));
}
#endif
#ifdef SVG2_TRACE
// measurement build only: the cycle trace of the last attention launch, [kTrEv][kTrT] clock64 values
extern "C" __attribute__((visibility("default"))) int svg2_trace_dump(long long* out) {
  return int(cudaMemcpyFromSymbol(out, svg2::g_trace, sizeof(svg2::g_trace)));
}
#endif

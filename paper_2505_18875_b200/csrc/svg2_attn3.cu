// svg2_attn3.cu — A9 (+ fused A10): dynamic-block-size sparse attention over the permuted, cluster-contiguous
// tokens, written for sm_100a.
//
// Work item = two 128-row Q tiles of one query cluster i (contiguous rows of Q' after the permutation) sharing ONE
// packed key stream: the selected key clusters' row ranges of K'/V' (adjacent selected clusters merged into runs),
// each run padded to whole 8-row groups.  The paper loads K/V "sparsely per token via address offsets into
// contiguous shared memory"; here a 128-key tile of the stream (16 groups) is assembled from TMA box
// loads straight into the 128B-swizzled layout the MMA descriptors expect: consecutive groups of one run merge into
// power-of-two boxes of 8..128 rows, so a tile typically costs 1-3 box loads per 64-column half.  Padding rows of a
// run's last group are masked in the softmax (a 4-bit valid count per group, packed per tile).
//
// Pipeline granularity is a half tile of 64 keys ("step" n = 2 t + h).  Each Q tile g has two S/P buffers in TMEM
// (one per half h), so the MMA computes S_g(n+1) while the softmax works on S_g(n), and PV_g(n) runs while the
// softmax works on S_g(n+1): the softmax warpgroups stream through steps back to back instead of waiting for the
// S -> softmax -> PV -> next S round trip.  TMEM: S_a0 | S_a1 | S_b0 | S_b1 (64 columns each) | O_a | O_b (128 each).
//
// Warp roles (384 threads, 1 CTA per SM, persistent; items fetched dynamically with an atomic counter).  The warp
// scheduler favours high warp ids, so the latency-critical MMA issuer gets the highest one:
//   warps 0-3   softmax warpgroup for Q tile a; warps 4-7 for Q tile b.  One thread = one query row = one TMEM
//               lane (warp w owns lanes 32(w%4)..+31): tcgen05.ld S, online softmax in registers (exp2 domain, lazy
//               rescale of O in TMEM when the running max grows by > 8, after the previous PV has completed), P (bf16)
//               written back over S with tcgen05.st; epilogue O / l -> bf16 -> global, scattered to original token
//               order through pi_q (fused A10).
//   warp 8      scheduler + TMA producer: fetches the next item, broadcasts it through a 2-slot smem ring, loads the
//               Q tiles and the K/V tiles (box loads) into 2-stage rings of 128-key tiles
//   warp 9      TMEM allocator (512 columns)
//   warp 11     MMA issuer (whole warp convergent, elect.sync issues inside the asm): per step n and Q tile g,
//               PV_g(n) then S_g(n+2) into the buffer PV_g(n) just read (in-order tensor pipe).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cstdlib>
#include "internal.h"
#include "ptx.cuh"
#include "tmap.h"

namespace svg2 {
namespace {

constexpr int kThreads = 384;
constexpr int kStages = 2;
constexpr int kGroupsPerTile = kKTile / 8;  // 16 groups of 8 keys per 128-key K/V tile
constexpr int kGroupsPerStep = 8;           // 64 keys per pipeline step (half tile)
constexpr int kBoxKinds = 5;                // box heights 8, 16, 32, 64, 128 rows
constexpr float kRescaleThreshold = 8.0f;   // log2 units: P <= 256 between rescales
constexpr uint32_t kFullHalfWord = 0x88888888u;
// setmaxnreg budget: the launch reserves 168 regs x 384 threads; the control warpgroup (warps 8-11) shrinks to 88
// and the two softmax warpgroups grow to 208.  The sum must not exceed the reservation or .inc never returns.
constexpr int kRegsCtl = 88, kRegsSoftmax = 208, kRegsLaunch = 168;
static_assert(128 * kRegsCtl + 256 * kRegsSoftmax <= kRegsLaunch * kThreads, "setmaxnreg budget exceeds launch");
constexpr int kWarpProducer = 8, kWarpTmem = 9, kWarpMma = 11;  // warp 10 idle
constexpr int kItemConsumers = 1 + 8;  // the MMA warp + 8 softmax warps arrive on item_empty
constexpr int kDefaultPolyStride = 0;
// v2 (128-key S tiles, svg2_attn2.cu) measured faster than v3 on B200 (HunyuanVideo: 50.5 vs 55.4 ms, same run):
// at N = 64 the S MMAs cost nearly as much per instruction as at N = 128.
constexpr int kDefaultAttnVariant = 2;

template <int D>
struct Cfg {
  static constexpr int kBlocks = D / 64;               // 64-column (128-byte) swizzle blocks per row
  static constexpr uint32_t kBlockBytes = 128 * 128;   // one 64-column block of a 128-row tile
  static constexpr uint32_t kTileBytes = kBlocks * kBlockBytes;
  static constexpr uint32_t kGroupBytes = 8 * 2 * D;   // 8 rows x D bf16
  static constexpr uint32_t kSmemBytes = (2 + 2 * kStages) * kTileBytes + 1024;
  // TMEM columns: S/P buffer h of Q tile g, and O of Q tile g
  __host__ __device__ static constexpr uint32_t col_s(int g, int h) { return uint32_t(g * 128 + h * 64); }
  __host__ __device__ static constexpr uint32_t col_o(int g) { return g ? 384u : 256u; }
};

struct Bars {
  uint64_t q_full, q_empty;
  uint64_t k_full[kStages], k_empty[kStages], v_full[kStages], v_empty[kStages];
  uint64_t s_full[2][2], p_full[2][2];  // [Q tile][S/P buffer]
  uint64_t pv_done[2];                  // one phase per PV step of Q tile g (for the O rescale)
  uint64_t o_full[2], o_empty[2];
  uint64_t item_full[2], item_empty[2];
};

struct KVMaps {
  CUtensorMap k[kBoxKinds], v[kBoxKinds];  // box = 64 columns x (8 << kind) rows
};

struct Params {
  const int4* items;
  int32_t* n_items;  // [0] = count, [1] = dynamic-scheduler counter (zeroed by k_items)
  const int2* groups;
  const uint64_t* tilew;
  const int32_t* ngroups;
  size_t gcap, tcap;
  const int32_t* q_perm;
  __nv_bfloat16* O;
  float* lse;
  int Nq;
  float scale_log2;
  int debug_mode;  // measurement only (env SVG2_DEBUG_MODE): 1 = softmax skips max/exp (P = 0), 2 = cycle trace
};

// Cycle trace of the first item of CTA 0 (SVG2_DEBUG_MODE=2 with the SVG2_TRACE_PRINT build, measurement only):
// clock64 per step and event, printed at kernel exit.  Events: 0/2 MMA saw P of a/b, 1/3 MMA issued PV+S of a/b,
// 4/6 softmax a/b got S, 5/7 softmax a/b handed P over, 8/9 producer issued K/V (per tile: even steps only).
constexpr int kTraceSteps = 64, kTraceEvents = 10;
#define TRACE(ev, n)                                                                                      \
  do {                                                                                                    \
    if (p.debug_mode == 2 && blockIdx.x == 0 && n_done == 0 && (n) < kTraceSteps && (threadIdx.x & 31) == 0) \
      trace_buf[(ev)*kTraceSteps + (n)] = clock64();                                                      \
  } while (0)

// Loads one 16-group tile of the item's key stream into a K or V stage.  Lanes 0..ngt-1 hold one group each; a
// lane whose group does not continue the previous lane's full group starts a run segment and issues power-of-two
// boxes covering it.  The stage's mbarrier receives ngt x 8 rows x D x 2 bytes.
template <int D>
__device__ __forceinline__ void load_kv_tile(const CUtensorMap* maps, uint8_t* stage, uint64_t* bar, int ngt, int lane,
                                             int2 gw) {
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
      for (int b = 0; b < C::kBlocks; ++b)
        tma_load_2d(stage + b * C::kBlockBytes + pos * 1024, &maps[kind], bar, 64 * b, row);
      pos += pw;
      len -= pw;
      row += 8 * pw;
    }
  }
}

// kPolyStride > 0: one pair of elements in every kPolyStride takes exp2 on the FMA pipes (ex2_poly) instead of
// MUFU (FA4's partial software exp2).
template <int D, int kPolyStride>
__global__ void __launch_bounds__(kThreads, 1)
    k_varblock_attn(const __grid_constant__ CUtensorMap mapQ, const __grid_constant__ KVMaps kv, const Params p) {
  using C = Cfg<D>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;                                // [2][tile]
  uint8_t* sK = smem + 2 * C::kTileBytes;            // [kStages][tile]
  uint8_t* sV = sK + kStages * C::kTileBytes;        // [kStages][tile]
  __shared__ Bars bars;
  __shared__ uint32_t tmem_slot;
  __shared__ int4 item_slot[2];
  __shared__ long long trace_buf[kTraceEvents * kTraceSteps];
  __shared__ int trace_H;

  // warp index broadcast from lane 0: ptxas then knows role branches are warp-uniform (uniform-register MMA issue)
  const int warp = __shfl_sync(0xffffffffu, int(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  int n_done = 0;  // items finished by this role (the trace covers the first one)
  if (warp == kWarpProducer && lane == 0) {
    tma_prefetch_desc(&mapQ);
    mbar_init(&bars.q_full, 1);
    mbar_init(&bars.q_empty, 1);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&bars.k_full[s], 1);
      mbar_init(&bars.k_empty[s], 1);
      mbar_init(&bars.v_full[s], 1);
      mbar_init(&bars.v_empty[s], 1);
    }
    for (int g = 0; g < 2; ++g) {
      for (int h = 0; h < 2; ++h) {
        mbar_init(&bars.s_full[g][h], 1);
        mbar_init(&bars.p_full[g][h], 4);
      }
      mbar_init(&bars.pv_done[g], 1);
      mbar_init(&bars.o_full[g], 1);
      mbar_init(&bars.o_empty[g], 4);
      mbar_init(&bars.item_full[g], 1);
      mbar_init(&bars.item_empty[g], kItemConsumers);
    }
    fence_mbar_init();
  }
  if (warp == kWarpTmem) tmem_alloc<512>(&tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = __shfl_sync(0xffffffffu, tmem_slot, 0);
  const int n_items = __ldg(p.n_items);

  if (warp >= 8) {
    reg_dealloc<kRegsCtl>();
    if (warp == kWarpProducer) {
      // ============================ scheduler + TMA producer ============================
      uint32_t qph = 0, ks = 0, kph = 0, islot = 0, iph = 0;
      while (true) {
        int item = 0;
        if (lane == 0) item = atomicAdd(p.n_items + 1, 1);
        item = __shfl_sync(0xffffffffu, item, 0);
        const int4 it = item < n_items ? __ldg(p.items + item) : make_int4(-1, 0, 0, 0);
        mbar_wait(&bars.item_empty[islot], iph ^ 1, 16);
        if (lane == 0) {
          item_slot[islot] = it;
          mbar_arrive(&bars.item_full[islot]);  // release: the slot write is visible to the waiting consumers
        }
        if (++islot == 2) {
          islot = 0;
          iph ^= 1;
        }
        if (it.x < 0) break;
        const int nb = it.y >> 16;
        const int ng = __ldg(p.ngroups + it.z);
        const int2* grp = p.groups + size_t(it.z) * p.gcap;
        mbar_wait(&bars.q_empty, qph ^ 1, 1);
        if (lane == 0) {
          mbar_arrive_expect_tx(&bars.q_full, (nb > 0 ? 2u : 1u) * C::kTileBytes);
          for (int b = 0; b < C::kBlocks; ++b) {
            tma_load_2d(sQ + b * C::kBlockBytes, &mapQ, &bars.q_full, 64 * b, it.x);
            if (nb > 0)
              tma_load_2d(sQ + C::kTileBytes + b * C::kBlockBytes, &mapQ, &bars.q_full, 64 * b, it.x + 128);
          }
        }
        qph ^= 1;
        const int T = (ng + kGroupsPerTile - 1) / kGroupsPerTile;
        int2 gw = lane < min(kGroupsPerTile, ng) ? __ldg(grp + lane) : make_int2(0, 0);
        for (int t = 0; t < T; ++t) {
          const int ngt = min(kGroupsPerTile, ng - t * kGroupsPerTile);
          const uint32_t bytes = uint32_t(ngt) * C::kGroupBytes;
          const int nxt = (t + 1) * kGroupsPerTile + lane;  // prefetch the next tile's group words
          const int2 gw_next = (t + 1 < T && nxt < ng) ? __ldg(grp + nxt) : make_int2(0, 0);
          mbar_wait(&bars.k_empty[ks], kph ^ 1, 2);
          if (lane == 0) mbar_arrive_expect_tx(&bars.k_full[ks], bytes);
          __syncwarp();
          load_kv_tile<D>(kv.k, sK + ks * C::kTileBytes, &bars.k_full[ks], ngt, lane, gw);
          TRACE(8, 2 * t);
          mbar_wait(&bars.v_empty[ks], kph ^ 1, 3);
          if (lane == 0) mbar_arrive_expect_tx(&bars.v_full[ks], bytes);
          __syncwarp();
          load_kv_tile<D>(kv.v, sV + ks * C::kTileBytes, &bars.v_full[ks], ngt, lane, gw);
          TRACE(9, 2 * t);
          gw = gw_next;
          if (++ks == kStages) {
            ks = 0;
            kph ^= 1;
          }
        }
        if (n_done == 0 && blockIdx.x == 0 && lane == 0) trace_H = (ng + kGroupsPerStep - 1) / kGroupsPerStep;
        ++n_done;
      }
    } else if (warp == kWarpMma) {
      // ============================ MMA issuer ============================
      uint32_t qph = 0, ks = 0, kph = 0, vs = 0, vph = 0, islot = 0, iph = 0;
      uint32_t oeph = 0, pph = 0;  // phase bits: o_empty[g] at bit g, p_full[g][h] at bit 2g+h
      const uint32_t idesc_pv = idesc_bf16_f32(128, D, true);
      const uint64_t dq0 = desc_kmajor_sw128(smem_u32(sQ)), dq1 = desc_kmajor_sw128(smem_u32(sQ + C::kTileBytes));
      const uint64_t dk0 = desc_kmajor_sw128(smem_u32(sK)), dk1 = desc_kmajor_sw128(smem_u32(sK + C::kTileBytes));
      const uint64_t dv0 = desc_mnmajor_sw128(smem_u32(sV), C::kBlockBytes);
      const uint64_t dv1 = desc_mnmajor_sw128(smem_u32(sV + C::kTileBytes), C::kBlockBytes);
      while (true) {
        mbar_wait_warp(&bars.item_full[islot], iph);
        const int4 it = item_slot[islot];
        __syncwarp();
        mbar_arrive_warp(&bars.item_empty[islot]);
        if (++islot == 2) {
          islot = 0;
          iph ^= 1;
        }
        if (__all_sync(0xffffffffu, it.x < 0)) break;  // uniform exit
        const int G = (it.y >> 16) > 0 ? 2 : 1;  // Q tiles in this item
        const int ng = __ldg(p.ngroups + it.z);
        const int H = (ng + kGroupsPerStep - 1) / kGroupsPerStep;  // 64-key steps
        auto step_keys = [&](int n) { return uint32_t(min(kGroupsPerStep, ng - n * kGroupsPerStep)) * 8u; };
        // S_g(n) = Q_g K(n)^T, N = keys of step n, K stage of tile n/2 (row offset 64 (n%2) inside the tile)
        auto issue_s = [&](int n, int g, uint32_t kstage) {
          const uint32_t idesc = idesc_bf16_f32(128, step_keys(n), false);
          const uint64_t kd = (kstage ? dk1 : dk0) + uint64_t((n & 1) * 64 * 128 >> 4), qd = g ? dq1 : dq0;
          const uint32_t d = tmem + C::col_s(g, n & 1);
#pragma unroll
          for (int k = 0; k < D / 16; ++k) {
            const uint64_t off = uint64_t(((k >> 2) * C::kBlockBytes + (k & 3) * 32) >> 4);
            mma_ss_warp(d, qd + off, kd + off, idesc, k > 0);
          }
        };
        // O_g += P_g(n) V(n): K-steps of 16 keys, V rows 64 (n%2) + 16 k of the V stage
        auto issue_pv = [&](int n, int g, uint32_t vstage) {
          const int ksteps = int(step_keys(n)) / 16;
          const uint64_t vd = (vstage ? dv1 : dv0) + uint64_t((n & 1) * 64 * 128 >> 4);
          const uint32_t ps = tmem + C::col_s(g, n & 1), d = tmem + C::col_o(g);
#pragma unroll 1
          for (int k = 0; k < ksteps; ++k)
            mma_ts_warp(d, ps + 8 * k, vd + uint64_t((k * 16 * 128) >> 4), idesc_pv, (n > 0 || k > 0) ? 1u : 0u);
        };
        mbar_wait_warp(&bars.q_full, qph);
        qph ^= 1;
        // prologue: S(0) and S(1) (both halves of tile 0) for every Q tile
        mbar_wait_warp(&bars.k_full[ks], kph);
        tc_fence_after();
        for (int n = 0; n < min(2, H); ++n)
          for (int g = 0; g < G; ++g) {
            issue_s(n, g, ks);
            mma_commit_warp(&bars.s_full[g][n & 1]);
          }
        mma_commit_warp(&bars.k_empty[ks]);  // tile 0's K fully consumed
        if (H <= 2) mma_commit_warp(&bars.q_empty);
        uint32_t kcur = ks;  // K stage of the tile of step n+2
        if (++ks == kStages) {
          ks = 0;
          kph ^= 1;
        }
        for (int n = 0; n < H; ++n) {
          const bool more = n + 2 < H;
          if ((n & 1) == 0) mbar_wait_warp(&bars.v_full[vs], vph);  // V of tile n/2
          if (more && ((n + 2) & 1) == 0) {                        // S(n+2) starts a new tile: its K
            mbar_wait_warp(&bars.k_full[ks], kph);
            kcur = ks;
          }
          for (int g = 0; g < G; ++g) {
            const uint32_t pbit = 1u << (2 * g + (n & 1));
            mbar_wait_warp(&bars.p_full[g][n & 1], (pph & pbit) ? 1u : 0u);
            pph ^= pbit;
            if (n == 0) {
              mbar_wait_warp(&bars.o_empty[g], ((oeph >> g) & 1u) ^ 1u);
              oeph ^= 1u << g;
            }
            tc_fence_after();
            issue_pv(n, g, vs);
            mma_commit_warp(&bars.pv_done[g]);
            if (more) {
              issue_s(n + 2, g, kcur);
              mma_commit_warp(&bars.s_full[g][n & 1]);
            } else if (n == H - 1) {
              mma_commit_warp(&bars.o_full[g]);
            }
          }
          if ((n & 1) == 1 || n == H - 1) {  // V of tile n/2 fully consumed
            mma_commit_warp(&bars.v_empty[vs]);
            if (++vs == kStages) {
              vs = 0;
              vph ^= 1;
            }
          }
          if (more && (((n + 2) & 1) == 1 || n + 2 == H - 1)) {  // last S of the tile of step n+2 issued
            mma_commit_warp(&bars.k_empty[kcur]);
            if (++ks == kStages) {
              ks = 0;
              kph ^= 1;
            }
          }
          if (more && n + 2 == H - 1) mma_commit_warp(&bars.q_empty);  // the item's last S has been issued
        }
        ++n_done;
      }
    }
  } else {
    reg_alloc<kRegsSoftmax>();
    // ============================ softmax warpgroups ============================
    const int g = warp >> 2;                        // 0: tile a, 1: tile b
    const int rloc = ((warp & 3) << 5) + lane;      // row in the tile == TMEM lane
    const uint32_t lane_addr = uint32_t((warp & 3) * 32) << 16;
    const uint32_t tO = tmem + lane_addr + C::col_o(g);
    const float sl2 = p.scale_log2;
    uint32_t sph = 0, oph = 0, islot = 0, iph = 0;  // sph: s_full[g][h] phase at bit h
    uint32_t pv_count = 0;  // PV steps of this Q tile issued over the whole launch (pv_done phases)
    while (true) {
      mbar_wait(&bars.item_full[islot], iph, 18);
      const int4 it = item_slot[islot];
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars.item_empty[islot]);
      if (++islot == 2) {
        islot = 0;
        iph ^= 1;
      }
      if (it.x < 0) break;
      const int nrows = g == 0 ? (it.y & 0xFFFF) : (it.y >> 16);
      if (nrows <= 0) continue;
      const int ng = __ldg(p.ngroups + it.z);
      const uint64_t* tw = p.tilew + size_t(it.z) * p.tcap;
      const int H = (ng + kGroupsPerStep - 1) / kGroupsPerStep;
      float m_used = -INFINITY, l = 0.f;
      for (int n = 0; n < H; ++n, ++pv_count) {
        const int h = n & 1;
        // 4-bit valid counts of the step's 8 groups (0 beyond the stream)
        const uint32_t word = uint32_t(__ldg(tw + (n >> 1)) >> (32 * h));
        const uint32_t tS = tmem + lane_addr + C::col_s(g, h);
        mbar_wait(&bars.s_full[g][h], (sph >> h) & 1u, 12 + g);
        sph ^= 1u << h;
        if ((warp & 3) == 0) TRACE(4 + 2 * g, n);
        tc_fence_after();
        uint32_t s0[32], s1[32];
        tmem_ld32(tS + 0, s0);
        tmem_ld32(tS + 32, s1);
        tmem_wait_ld();
        if (p.debug_mode == 1) {  // measurement: the MMA/TMA pipeline without the softmax math
          uint32_t z[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) z[e] = s0[e] & 0u;
          tmem_st16(tS + 0, z);
          tmem_st16(tS + 16, z);
          l = 1.f;
          m_used = 0.f;
          tmem_wait_st();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&bars.p_full[g][h]);
          continue;
        }
        // row max on the raw scores (scale > 0 preserves order); only steps with padding rows need the mask
        if (word != kFullHalfWord) {
          // word is lane-uniform: one uniform test per 8-row group, selects only inside partial groups
          auto apply_mask = [&](uint32_t(&a)[32], int c0) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const uint32_t nv = (word >> (4 * ((c0 >> 3) + q))) & 15u;
              if (nv < 8u) {
#pragma unroll
                for (int e = 0; e < 8; ++e)
                  if (uint32_t(e) >= nv) a[8 * q + e] = __float_as_uint(-INFINITY);
              }
            }
          };
          apply_mask(s0, 0);
          apply_mask(s1, 32);
        }
        float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
        for (int e = 0; e < 32; e += 2) {
          mx0 = fmaxf(mx0, fmaxf(__uint_as_float(s0[e]), __uint_as_float(s1[e])));
          mx1 = fmaxf(mx1, fmaxf(__uint_as_float(s0[e + 1]), __uint_as_float(s1[e + 1])));
        }
        const float mt = fmaxf(mx0, mx1) * sl2;
        if (n == 0) {
          m_used = mt;
        } else if (__any_sync(0xffffffffu, rloc < nrows && mt > m_used + kRescaleThreshold)) {
          // only rows of the cluster vote: the tile's padding rows hold whatever follows the cluster in Q'
          // (another cluster or head), and must not change how the cluster's rows are rounded
          // warp-uniform branch (tcgen05.ld/st are .sync.aligned); rows whose max did not grow get alpha = 1.
          // O may only be touched once the previous PV of this tile has completed (PV(n) waits for our P(n)).
          mbar_wait(&bars.pv_done[g], (pv_count - 1) & 1, 19);
          tc_fence_after();
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
        // p = 2^(s * scale*log2e - m): FFMA2 on pairs, MUFU ex2 per element, FADD2 row sums, bf16x2 packs
        const uint64_t sl2x2 = f2(sl2, sl2), negm2 = f2(-m_used, -m_used);
        uint64_t lsum2 = f2(0.f, 0.f);
        auto exp_store = [&](const uint32_t(&a)[32], int c) {
          uint32_t pk[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            float x0, x1;
            f2_split(ffma2(f2(__uint_as_float(a[2 * e]), __uint_as_float(a[2 * e + 1])), sl2x2, negm2), x0, x1);
            const bool poly = kPolyStride > 0 && (e % (kPolyStride > 0 ? kPolyStride : 1)) == 0;
            const float p0 = poly ? ex2_poly(x0) : ex2_approx(x0);
            const float p1 = poly ? ex2_poly(x1) : ex2_approx(x1);
            lsum2 = fadd2(lsum2, f2(p0, p1));
            pk[e] = pack_bf16x2(p0, p1);
          }
          tmem_st16(tS + 16 * c, pk);
        };
        exp_store(s0, 0);
        exp_store(s1, 1);
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars.p_full[g][h]);
        if ((warp & 3) == 0) TRACE(5 + 2 * g, n);
        float ls0, ls1;
        f2_split(lsum2, ls0, ls1);
        l += ls0 + ls1;
      }
      // ---- epilogue: O / l  -> bf16 -> original token order (fused pi_q^T)
      mbar_wait(&bars.o_full[g], oph, 14 + g);
      oph ^= 1;
      tc_fence_after();
      const float inv_l = 1.f / l;
      const long long row_flat = (long long)it.x + g * kQTile + rloc;
      long long dst = row_flat;
      if (rloc < nrows && p.q_perm) {
        const long long bh = it.w & kItemBhMask;
        dst = bh * p.Nq + __ldg(p.q_perm + row_flat);
      }
      uint4* orow = reinterpret_cast<uint4*>(p.O + dst * D);
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
            orow[4 * c + v] = u;
          }
        }
      }
      if (rloc < nrows && p.lse) p.lse[dst] = (m_used + __log2f(l)) * 0.69314718055994531f;
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars.o_empty[g]);
      ++n_done;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kWarpTmem) tmem_dealloc<512>(tmem);
#ifdef SVG2_TRACE_PRINT
  if (p.debug_mode == 2 && blockIdx.x == 0 && threadIdx.x == 0) {
    const long long t0 = trace_buf[8 * kTraceSteps];
    printf("svg2 trace: H=%d (cycles relative to the first K issue)\n", trace_H);
    for (int n = 0; n < min(trace_H, kTraceSteps); ++n) {
      printf("svg2 trace n=%2d", n);
      for (int e = 0; e < kTraceEvents; ++e) printf(" %8lld", trace_buf[e * kTraceSteps + n] - t0);
      printf("\n");
    }
  }
#endif
}

// ---------------------------------------------------------------- work-list builder
constexpr int kBuildThreads = 128;

// block-wide exclusive scan (kBuildThreads threads, one value each); *total receives the block sum
__device__ int build_scan(int v, int* total) {
  __shared__ int wsum[kBuildThreads / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[w] = x;
  __syncthreads();
  int before = 0, tot = 0;
#pragma unroll
  for (int k = 0; k < kBuildThreads / 32; ++k) {
    before += k < w ? wsum[k] : 0;
    tot += wsum[k];
  }
  __syncthreads();
  *total = tot;
  return before + x - v;
}

// One CTA per (b,h,i): the key stream of query cluster i = its selected, non-empty key clusters in ascending j,
// contiguous clusters merged into runs, runs cut into 8-row groups (the last one partial), the stream padded to an
// even group count; plus the packed 4-bit valid counts per 16-group tile.  Three block scans (selected clusters,
// run starts, groups per run) make every step parallel.
__global__ void __launch_bounds__(kBuildThreads) k_build_streams(const int32_t* __restrict__ k_off,
                                                                 const uint8_t* __restrict__ mask, int Nk, int Cq,
                                                                 int Ck, AttnWs ws) {
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
  // 1) compact the selected, non-empty clusters (ascending j)
  int base = 0;
  for (int j0 = 0; j0 < Ck; j0 += kBuildThreads) {
    const int j = j0 + tid;
    int s = 0, e = 0, f = 0;
    if (j < Ck && mrow[j]) {
      s = __ldg(ko + j);
      e = __ldg(ko + j + 1);
      f = e > s;
    }
    int tot;
    const int pos = base + build_scan(f, &tot);
    if (f) {
      sel_s[pos] = s;
      sel_e[pos] = e;
    }
    base += tot;
  }
  const int nsel = base;
  __syncthreads();
  // 2) runs: a selected cluster starts a run unless it begins exactly where the previous one ends
  base = 0;
  for (int k0 = 0; k0 < nsel; k0 += kBuildThreads) {
    const int k = k0 + tid;
    const int f = (k < nsel) && (k == 0 || sel_s[k] != sel_e[k - 1]);
    int tot;
    const int r = base + build_scan(f, &tot);
    if (f) run_s[r] = sel_s[k];
    base += tot;
  }
  const int nrun = base;
  __syncthreads();
  for (int k = tid; k < nsel; k += kBuildThreads) {  // the last cluster of each run writes the run end
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
  for (int r0 = 0; r0 < nrun; r0 += kBuildThreads) {
    const int r = r0 + tid;
    const int gr = r < nrun ? (run_e[r] - run_s[r] + 7) / 8 : 0;
    int tot;
    const int g0 = base + build_scan(gr, &tot);
    if (r < nrun) run_g[r] = g0;
    base += tot;
  }
  const int ng_real = base;
  const int ng = ng_real + (ng_real & 1);  // even group count: every step has N = 16 k keys
  if (tid == 0) {
    run_g[nrun] = ng_real;
    ws.ngroups[li] = ng;
  }
  __syncthreads();
  const int rowbase = int(size_t(bh) * Nk);
  int2* grp = ws.groups + li * ws.gcap;
  // one thread per 16-group tile: locate the tile's first group by binary search, then walk the runs forward,
  // writing the group words and packing the tile's 4-bit valid counts in the same pass
  uint64_t* tw = ws.tilew + li * ws.tcap;
  const int ntiles = (ng + kGroupsPerTile - 1) / kGroupsPerTile;
  for (int t = tid; t < ntiles; t += kBuildThreads) {
    const int g0 = t * kGroupsPerTile, g1 = min(ng, g0 + kGroupsPerTile);
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

// Work items in (b,h)-major, cluster order: ceil(|Q_i| / 256) pairs of 128-row Q tiles per non-empty query cluster
// with a non-empty key stream.  One CTA scans all B*H*Cq clusters; also resets the dynamic-scheduler counter.
__global__ void __launch_bounds__(1024) k_items(const int32_t* __restrict__ q_off, int BH, int Nq, int Cq,
                                                AttnWs ws, int allow_split) {
  __shared__ int wsum[32];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int total_clusters = BH * Cq;
  int base = 0;
  for (int c0 = 0; c0 < total_clusters; c0 += 1024) {
    const int c = c0 + tid;
    int n = 0, q0 = 0, sq = 0, bh = 0;
    if (c < total_clusters) {
      bh = c / Cq;
      const int i = c - bh * Cq;
      q0 = q_off[size_t(bh) * (Cq + 1) + i];
      sq = q_off[size_t(bh) * (Cq + 1) + i + 1] - q0;
      if (ws.ngroups[c] > 0) n = (sq + kItemRows - 1) / kItemRows;
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
      const int split = (allow_split && nb == 0 && ws.ngroups[c] > kKTile / 8) ? kItemSplit : 0;
      ws.items[slot++] = make_int4(int(size_t(bh) * Nq) + q0 + u * kItemRows, na | (nb << 16), c, bh | split);
    }
    base += tot;
  }
  if (tid == 0) {
    ws.n_items[0] = base;
    ws.n_items[1] = 0;  // dynamic scheduler counter of the next attention launch
  }
}

template <int D>
cudaError_t run_attn(const void* Qp, const void* Kp, const void* Vp, int BH, int Nq, int Nk, float scale,
                     const int32_t* q_perm, void* O, float* lse, AttnWs ws, cudaStream_t s) {
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
  p.O = static_cast<__nv_bfloat16*>(O);
  p.lse = lse;
  p.Nq = Nq;
  p.scale_log2 = scale * 1.4426950408889634f;
  static const int debug_mode = [] {
    const char* e = getenv("SVG2_DEBUG_MODE");
    return e ? atoi(e) : 0;
  }();
  p.debug_mode = debug_mode;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // exp2 split between MUFU and the FMA pipes (env SVG2_EXP_POLY_STRIDE overrides, for measurements)
  static const int poly = [] {
    const char* e = getenv("SVG2_EXP_POLY_STRIDE");
    return e ? atoi(e) : kDefaultPolyStride;
  }();
  auto launch = [&](auto kernel) {
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<D>::kSmemBytes);
    kernel<<<sms, kThreads, Cfg<D>::kSmemBytes, s>>>(mq, kv, p);
  };
  if (poly == 2) launch(k_varblock_attn<D, 2>);
  else if (poly == 4) launch(k_varblock_attn<D, 4>);
  else if (poly == 8) launch(k_varblock_attn<D, 8>);
  else launch(k_varblock_attn<D, 0>);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_build_worklist(const int32_t* q_offsets, const int32_t* k_offsets, const uint8_t* mask, int BH,
                                  int Nq, int Nk, int Cq, int Ck, AttnWs ws, cudaStream_t s) {
  const size_t smem = (5 * size_t(Ck) + 1) * sizeof(int);
  cudaFuncSetAttribute(k_build_streams, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  k_build_streams<<<dim3(Cq, BH), kBuildThreads, smem, s>>>(k_offsets, mask, Nk, Cq, Ck, ws);
  static const int allow_split = [] {  // env SVG2_SPLIT_ITEMS=0 disables split items (measurements)
    const char* e = getenv("SVG2_SPLIT_ITEMS");
    return e ? atoi(e) : 1;
  }();
  k_items<<<1, 1024, 0, s>>>(q_offsets, BH, Nq, Cq, ws, allow_split);
  return cudaGetLastError();
}

cudaError_t launch_varblock_attention_v3(const void* Qp, const void* Kp, const void* Vp, int BH, int Nq, int Nk, int d,
                                         int Cq, int Ck, float scale, const int32_t* q_perm, void* O, float* lse,
                                         AttnWs ws, cudaStream_t s) {
  (void)Cq;
  (void)Ck;
  if (d == 128) return run_attn<128>(Qp, Kp, Vp, BH, Nq, Nk, scale, q_perm, O, lse, ws, s);
  return run_attn<64>(Qp, Kp, Vp, BH, Nq, Nk, scale, q_perm, O, lse, ws, s);
}

// svg2_attn2.cu: the 128-key-tile design (single S/P buffer per Q tile)
cudaError_t launch_varblock_attention_v2(const void* Qp, const void* Kp, const void* Vp, int BH, int Nq, int Nk, int d,
                                         int Cq, int Ck, float scale, const int32_t* q_perm, void* O, float* lse,
                                         AttnWs ws, cudaStream_t s, const uint32_t* v_amax);
cudaError_t launch_varblock_attention_v4(const void* Qp, const void* Kp, const void* Vp, int BH, int Nq, int Nk, int d,
                                         int Cq, int Ck, float scale, const int32_t* q_perm, void* O, float* lse,
                                         AttnWs ws, cudaStream_t s);

// The pipeline designs share the work list and produce identical math; env SVG2_ATTN_VARIANT=2|3|4 selects one for
// measurements, kDefaultAttnVariant otherwise.
cudaError_t launch_varblock_attention(const void* Qp, const void* Kp, const void* Vp, int BH, int Nq, int Nk, int d,
                                      int Cq, int Ck, float scale, const int32_t* q_perm, void* O, float* lse,
                                      AttnWs ws, cudaStream_t s, const uint32_t* v_amax) {
  static const int variant = [] {
    const char* e = getenv("SVG2_ATTN_VARIANT");
    return e ? atoi(e) : kDefaultAttnVariant;
  }();
  // the FP8 PV path (V' in e4m3, v_amax = per-head |V| max) exists in design v2 only
  if (variant == 2 || v_amax)
    return launch_varblock_attention_v2(Qp, Kp, Vp, BH, Nq, Nk, d, Cq, Ck, scale, q_perm, O, lse, ws, s, v_amax);
  if (variant == 4)
    return launch_varblock_attention_v4(Qp, Kp, Vp, BH, Nq, Nk, d, Cq, Ck, scale, q_perm, O, lse, ws, s);

  return launch_varblock_attention_v3(Qp, Kp, Vp, BH, Nq, Nk, d, Cq, Ck, scale, q_perm, O, lse, ws, s);
}

}  // namespace svg2

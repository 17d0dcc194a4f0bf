// svg2_attn_fp8.cu — A9 (+ fused A10) with the PV product in e4m3 (the "+FP8" variant of PAPER.md:414, 418; DESIGN
// R26), written for sm_100a.  Same work list as svg2_attn.cu (key streams of 8-row groups), 128-key tiles.
//
// Work item = two 128-row Q tiles of one query cluster sharing one packed key stream (svg2_attn.cu).  V' arrives in
// e4m3 (scale 448 / amax per head, computed by the permute step), P is packed to e4m3 in TMEM and PV runs as
// kind::f8f6f4 MMAs (K = 32 keys each, half the instructions of bf16); QK^T, the softmax statistics and O stay
// bf16 / fp32.  d = 128 only.
//
// Warp roles (384 threads, 1 CTA per SM, persistent; items fetched dynamically with an atomic counter):
//   warps 0-3   softmax warpgroup for Q tile a; warps 4-7 for Q tile b.  One thread = one query row = one TMEM
//               lane: tcgen05.ld S, online softmax in registers (exp2 domain, lazy rescale when the running max grows
//               by > 8), P (e4m3) written back over S with tcgen05.st, O rescaled in TMEM when needed; epilogue
//               O / l -> bf16 -> global, scattered to original token order through pi_q (fused A10).
//   warp 8      scheduler + TMA producer (Q tiles, K tiles and e4m3 V tiles into 3-stage rings)
//   warp 9      TMEM allocator (512 columns: S_a | S_b | O_a | O_b)
//   warp 11     MMA issuer (whole warp convergent, elect.sync issues; highest priority), for both Q tiles in turn:
//               S = Q K^T (SS) into TMEM, then per key tile O += P V (TS: P read from TMEM, V MN-major)
//               followed by the next S, which overwrites P only after the PV that reads it (in-order tensor pipe).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include "internal.h"
#include "ptx.cuh"
#include "tmap.h"

namespace svg2 {
namespace {
// (its helpers live in this file's anonymous namespace; the bf16 pipeline is svg2_attn.cu)

constexpr int kThreads = 384;
constexpr int kStages = 2;     // K/V ring depth (bf16)
constexpr int kStagesFp8 = 3;  // with e4m3 V tiles (16 KB) a third stage fits: prefetch two tiles ahead
constexpr int kStagesMax = 3;
constexpr int kGroupsPerTile = kKTile / 8;  // 16
constexpr int kBoxKinds = 5;                // box heights 8, 16, 32, 64, 128 rows
// Lazy rescale threshold (log2 units): O and l are rescaled only when a row's tile max exceeds the max in use by
// more than this, so P <= 2^threshold between rescales.  P is bf16 (relative precision at any magnitude) and O / l
// accumulate in fp32, so 2^20 leaves > 10^20 headroom for 10^5 keys.
constexpr float kRescaleThreshold = 8.0f;
// FP8 PV: the per-row P scale.  P enters e4m3 as p' = 2^(s*scale*log2e - m_used + kPShift), with the lazy rescale
// threshold lowered to kRescaleThresholdFp8 so that p' <= 2^(threshold + shift) = 256 <= 448 (e4m3 max): weights
// down to 2^-(6+shift) = 2^-12 of the running max stay normal e4m3 (3-bit mantissa) instead of 2^-6, and only weights
// below 2^-16 of it flush to zero (unscaled P lost everything under 2^-10).  l sums the same scaled p', so
// the shift cancels in O / l; lse subtracts it.
constexpr float kRescaleThresholdFp8 = 2.0f, kPShift = 6.0f;
static_assert(kRescaleThresholdFp8 + kPShift <= 8.0f, "scaled P must stay <= 256 < 448 (e4m3 max)");
constexpr uint64_t kFullTileWord = 0x8888888888888888ull;
// setmaxnreg budget: the launch reserves 168 regs x 384 threads; the control warpgroup (warps 8-11) shrinks to 72
// and the two softmax warpgroups grow to 216.  The sum must not exceed the reservation or .inc never returns.
constexpr int kRegsCtl = 88, kRegsSoftmax = 208, kRegsLaunch = 168;
static_assert(128 * kRegsCtl + 256 * kRegsSoftmax <= kRegsLaunch * kThreads, "setmaxnreg budget exceeds launch");
constexpr int kWarpProducer = 8, kWarpTmem = 9, kWarpMma = 11;  // warp 10 idle
constexpr int kItemConsumers = 1 + 8;  // the MMA warp + 8 softmax warps arrive on item_empty
constexpr int kDefaultPoly = 4;  // measured (interleaved, HunyuanVideo): 49.0 / 49.9 / 51.2 / 54.4 ms at 4 / 6 / 8 / 10

template <int D>
struct Cfg {
  static constexpr int kBlocks = D / 64;               // 64-column (128-byte) swizzle blocks per row
  static constexpr uint32_t kBlockBytes = 128 * 128;   // one 64-column block of a 128-row tile
  static constexpr uint32_t kTileBytes = kBlocks * kBlockBytes;
  static constexpr uint32_t kGroupBytes = 8 * 2 * D;   // 8 rows x D bf16
  static constexpr uint32_t kSmemBytes = (2 + 2 * kStages) * kTileBytes + 1024;
  // FP8 PV: kStagesFp8 K tiles and kStagesFp8 half-size (e4m3) V tiles
  static constexpr uint32_t kSmemBytesFp8 = (2 + kStagesFp8) * kTileBytes + kStagesFp8 * (kTileBytes / 2) + 1024;
  // TMEM columns: S of Q tile g at col_s(g) (P aliases it as bf16), O at col_o(g)
  __host__ __device__ static constexpr uint32_t col_s(int g) { return g ? 128u : 0u; }
  __host__ __device__ static constexpr uint32_t col_o(int g) { return g ? 384u : 256u; }
};

struct Bars {
  uint64_t q_full, q_empty;
  uint64_t k_full[kStagesMax], k_empty[kStagesMax], v_full[kStagesMax], v_empty[kStagesMax];
  uint64_t s_full[2], p_full[2], o_full[2], o_empty[2];
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
  __nv_bfloat16* O;  // permuted-order output (q_perm == nullptr)
  OutView out;       // original-order output rows (q_perm set): the fused A10 scatter
  float* lse;
  int Nq;
  float scale_log2;
  const uint32_t* v_amax;  // kFp8: per-(head, channel) max |V| [BH, D] (f32 bits); O channel c is scaled by amax_c / 448
};

// Loads one 16-group tile of the item's key stream into a K or V stage.  Lanes 0..ngt-1 hold one group each; a
// lane whose group does not continue the previous lane's full group starts a run segment and issues power-of-two
// boxes covering it.  The stage's mbarrier receives ngt x 8 rows x D x 2 bytes.
template <int D>
__device__ __forceinline__ void load_kv_tile(const CUtensorMap* maps, uint8_t* stage, uint64_t* bar, int ngt, int lane,
                                             int2 gw, int nblk = Cfg<D>::kBlocks) {
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
      for (int b = 0; b < nblk; ++b)  // 128-byte column blocks (64 bf16, or all 128 e4m3 of a V row)
        tma_load_2d(stage + b * C::kBlockBytes + pos * 1024, &maps[kind], bar, 64 * b, row);
      pos += pw;
      len -= pw;
      row += 8 * pw;
    }
  }
}

// kPoly: in every 16-pair chunk of a row's 128 exponentials, kPoly pairs take 2^x on the FMA/ALU pipes (ex2_poly2)
// instead of MUFU, which otherwise bounds the softmax (16 ex2/clk/SM; tools/xu_micro.cu).
// kFp8: the FP8 PV path (DESIGN R26) — V' arrives in e4m3 (scale 448 / amax per head), P is packed to e4m3 in
// TMEM and PV runs as kind::f8f6f4 MMAs (K = 32 keys each, half the instructions of bf16); d = 128 only.
template <int D, int kPoly, bool kFp8 = false>
__global__ void __launch_bounds__(kThreads, 1)
    k_varblock_attn(const __grid_constant__ CUtensorMap mapQ, const __grid_constant__ KVMaps kv, const Params p) {
  using C = Cfg<D>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;                                // [2][tile]
  constexpr int kSt = kFp8 ? kStagesFp8 : kStages;                  // K/V ring depth
  constexpr uint32_t kVTile = kFp8 ? C::kTileBytes / 2 : C::kTileBytes;  // one V stage (e4m3: 1 byte / element)
  uint8_t* sK = smem + 2 * C::kTileBytes;            // [kSt][tile]
  uint8_t* sV = sK + kSt * C::kTileBytes;            // [kSt][kVTile]
  __shared__ Bars bars;
  __shared__ uint32_t tmem_slot;
  __shared__ int4 item_slot[2];
  __shared__ float2 merge_ml[kQTile];  // split items: (m, l) of warpgroup b's rows

  const int warp = __shfl_sync(0xffffffffu, int(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  if (warp == kWarpProducer && lane == 0) {
    tma_prefetch_desc(&mapQ);
    mbar_init(&bars.q_full, 1);
    mbar_init(&bars.q_empty, 1);
    for (int s = 0; s < kSt; ++s) {
      mbar_init(&bars.k_full[s], 1);
      mbar_init(&bars.k_empty[s], 1);
      mbar_init(&bars.v_full[s], 1);
      mbar_init(&bars.v_empty[s], 1);
    }
    for (int g = 0; g < 2; ++g) {
      mbar_init(&bars.s_full[g], 1);
      mbar_init(&bars.p_full[g], 4);
      mbar_init(&bars.o_full[g], 1);
      mbar_init(&bars.o_empty[g], 4);
      mbar_init(&bars.item_full[g], 1);
      mbar_init(&bars.item_empty[g], kItemConsumers);
    }
    fence_mbar_init();
  }
  if (warp == kWarpTmem) tmem_alloc<512>(&tmem_slot);
  if (kFp8) {  // a tile of 16 (mod 32) keys ends in a K = 32 step whose last 16 V rows are stale: keep them finite
    for (int i = threadIdx.x; i < int(kSt * kVTile / 16); i += kThreads)
      reinterpret_cast<uint4*>(sV)[i] = make_uint4(0, 0, 0, 0);
    fence_async_smem();
  }
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
          // prefetch the next tile's group words while this tile's loads are being issued
          const int nxt = (t + 1) * kGroupsPerTile + lane;
          const int2 gw_next = (t + 1 < T && nxt < ng) ? __ldg(grp + nxt) : make_int2(0, 0);
          mbar_wait(&bars.k_empty[ks], kph ^ 1, 2);
          if (lane == 0) mbar_arrive_expect_tx(&bars.k_full[ks], bytes);
          __syncwarp();
          load_kv_tile<D>(kv.k, sK + ks * C::kTileBytes, &bars.k_full[ks], ngt, lane, gw);
          mbar_wait(&bars.v_empty[ks], kph ^ 1, 3);
          if (lane == 0) mbar_arrive_expect_tx(&bars.v_full[ks], kFp8 ? uint32_t(ngt) * 8u * D : bytes);
          __syncwarp();
          load_kv_tile<D>(kv.v, sV + ks * kVTile, &bars.v_full[ks], ngt, lane, gw, kFp8 ? 1 : C::kBlocks);
          gw = gw_next;
          if (++ks == kSt) {
            ks = 0;
            kph ^= 1;
          }
        }
      }
    } else if (warp == kWarpMma) {
      // ============================ MMA issuer ============================
      // Whole warp runs this code convergently; elect.sync inside the asm picks the issuing lane, so descriptors
      // stay in uniform registers and the MMAs issue back to back.  Order per key tile t (ping-pong):
      //   PV_a(t), S_a(t+1) | PV_b(t), S_b(t+1)  -- softmax of tile a overlaps tile b's MMAs and vice versa.
      uint32_t qph = 0, ks = 0, kph = 0, vs = 0, vph = 0, islot = 0, iph = 0;
      uint32_t oeph[2] = {0, 0}, pph[2] = {0, 0};
      const uint32_t idesc_pv = kFp8 ? idesc_e4m3_f32_bmn(128, D) : idesc_bf16_f32(128, D, true);
      const uint64_t dq0 = desc_kmajor_sw128(smem_u32(sQ)), dq1 = desc_kmajor_sw128(smem_u32(sQ + C::kTileBytes));
      // ring stage s = the stage-0 descriptor + s tiles in the start-address field (16-byte units)
      const uint64_t dk0 = desc_kmajor_sw128(smem_u32(sK));
      const uint64_t dv0 = desc_mnmajor_sw128(smem_u32(sV), C::kBlockBytes);
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
        const int T = (ng + kGroupsPerTile - 1) / kGroupsPerTile;
        auto tile_n = [&](int t) { return uint32_t(min(kGroupsPerTile, ng - t * kGroupsPerTile)) * 8u; };
        auto issue_s = [&](int t, int g, uint32_t kstage) {
          const uint32_t idesc = idesc_bf16_f32(128, tile_n(t), false);
          const uint64_t kd = dk0 + uint64_t(kstage) * (C::kTileBytes >> 4), qd = (g && !split) ? dq1 : dq0;
          const uint32_t d = tmem + C::col_s(g);
#pragma unroll
          for (int k = 0; k < D / 16; ++k) {
            const uint64_t off = uint64_t(((k >> 2) * C::kBlockBytes + (k & 3) * 32) >> 4);
            mma_ss_warp(d, qd + off, kd + off, idesc, k > 0);
          }
        };
        auto issue_pv = [&](int t, int g, uint32_t vstage, bool first) {
          const uint64_t vd = dv0 + uint64_t(vstage) * (kVTile >> 4);
          const uint32_t ps = tmem + C::col_s(g), d = tmem + C::col_o(g);
          if (kFp8) {  // K = 32 keys per MMA: 8 TMEM columns of e4m3 P, 32 V rows (4 KB) of the stage
            const int ksteps = (int(tile_n(t)) + 31) / 32;
#pragma unroll 1
            for (int k = 0; k < ksteps; ++k)
              mma_ts8_warp(d, ps + 8 * k, vd + uint64_t((k * 32 * 128) >> 4), idesc_pv, (!first || k > 0) ? 1u : 0u);
          } else {
            const int ksteps = int(tile_n(t)) / 16;
#pragma unroll 1
            for (int k = 0; k < ksteps; ++k)
              mma_ts_warp(d, ps + 8 * k, vd + uint64_t((k * 16 * 128) >> 4), idesc_pv, (!first || k > 0) ? 1u : 0u);
          }
        };
        auto next_k = [&] {
          if (++ks == kSt) {
            ks = 0;
            kph ^= 1;
          }
        };
        mbar_wait_warp(&bars.q_full, qph);
        qph ^= 1;
        if (split) {
          // Lone Q tile with T >= 2 key tiles: tile u goes to softmax warpgroup g = u & 1 (both hold the same Q rows
          // with their own m, l and O; warpgroup a merges them in the epilogue).  Tile order on the K/V rings is
          // unchanged.  Chain per warpgroup: PV_g(u) then S_g(u + 2).
          for (int u = 0; u < 2; ++u) {
            mbar_wait_warp(&bars.k_full[ks], kph);
            tc_fence_after();
            issue_s(u, u, ks);
            mma_commit_warp(&bars.s_full[u]);
            mma_commit_warp(&bars.k_empty[ks]);
            if (u == T - 1) mma_commit_warp(&bars.q_empty);
            next_k();
          }
          for (int u = 0; u < T; ++u) {
            const int g = u & 1;
            mbar_wait_warp(&bars.v_full[vs], vph);
            mbar_wait_warp(&bars.p_full[g], pph[g]);
            pph[g] ^= 1;
            if (u < 2) {
              mbar_wait_warp(&bars.o_empty[g], oeph[g] ^ 1);
              oeph[g] ^= 1;
            }
            tc_fence_after();
            issue_pv(u, g, vs, u < 2);
            if (u + 2 < T) {
              mbar_wait_warp(&bars.k_full[ks], kph);
              tc_fence_after();
              issue_s(u + 2, g, ks);
              mma_commit_warp(&bars.s_full[g]);
              mma_commit_warp(&bars.k_empty[ks]);
              if (u + 2 == T - 1) mma_commit_warp(&bars.q_empty);
              next_k();
            } else {
              mma_commit_warp(&bars.o_full[g]);
            }
            mma_commit_warp(&bars.v_empty[vs]);
            if (++vs == kSt) {
              vs = 0;
              vph ^= 1;
            }
          }
          continue;
        }
        // prologue: S(0)
        mbar_wait_warp(&bars.k_full[ks], kph);
        tc_fence_after();
        issue_s(0, 0, ks);
        mma_commit_warp(&bars.s_full[0]);
        if (has_b) {
          issue_s(0, 1, ks);
          mma_commit_warp(&bars.s_full[1]);
        }
        mma_commit_warp(&bars.k_empty[ks]);
        if (T == 1) mma_commit_warp(&bars.q_empty);
        if (++ks == kSt) {
          ks = 0;
          kph ^= 1;
        }
        for (int t = 0; t < T; ++t) {
          const bool more = t + 1 < T;
          mbar_wait_warp(&bars.v_full[vs], vph);
          if (more) mbar_wait_warp(&bars.k_full[ks], kph);
#pragma unroll
          for (int g = 0; g < 2; ++g) {
            if (g == 1 && !has_b) break;
            mbar_wait_warp(&bars.p_full[g], pph[g]);
            pph[g] ^= 1;
            if (t == 0) {
              mbar_wait_warp(&bars.o_empty[g], oeph[g] ^ 1);
              oeph[g] ^= 1;
            }
            tc_fence_after();
            issue_pv(t, g, vs, t == 0);
            if (more) {
              issue_s(t + 1, g, ks);
              mma_commit_warp(&bars.s_full[g]);
            } else {
              mma_commit_warp(&bars.o_full[g]);
            }
          }
          mma_commit_warp(&bars.v_empty[vs]);
          if (more) {
            mma_commit_warp(&bars.k_empty[ks]);
            if (t + 2 == T) mma_commit_warp(&bars.q_empty);
          }
          if (++vs == kSt) {
            vs = 0;
            vph ^= 1;
          }
          if (more && ++ks == kSt) {
            ks = 0;
            kph ^= 1;
          }
        }
      }
    }
  } else {
    reg_alloc<kRegsSoftmax>();
    // ============================ softmax warpgroups ============================
    const int g = warp >> 2;                        // 0: tile a, 1: tile b
    const int rloc = ((warp & 3) << 5) + lane;      // row in the tile == TMEM lane
    const uint32_t lane_addr = uint32_t((warp & 3) * 32) << 16;
    const uint32_t tS = tmem + lane_addr + C::col_s(g);
    const uint32_t tO = tmem + lane_addr + C::col_o(g);
    const float sl2 = p.scale_log2;
    uint32_t sph = 0, oph = 0, islot = 0, iph = 0;
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
      const bool split = (it.w & kItemSplit) != 0;  // both warpgroups on Q tile a, alternate key tiles
      const int nrows = (g == 0 || split) ? (it.y & 0xFFFF) : (it.y >> 16);
      if (nrows <= 0) continue;
      const int ng = __ldg(p.ngroups + it.z);
      const uint64_t* tw = p.tilew + size_t(it.z) * p.tcap;
      const int T = (ng + kGroupsPerTile - 1) / kGroupsPerTile;
      const int t_first = split ? g : 0, t_step = split ? 2 : 1;
      float m_used = -INFINITY, l = 0.f;
      uint64_t word_next = __ldg(tw + t_first);
      for (int t = t_first; t < T; t += t_step) {
        const uint64_t word = word_next;  // 4-bit valid counts of the tile's 16 groups (0 beyond the stream)
        if (t + t_step < T) word_next = __ldg(tw + t + t_step);
        mbar_wait(&bars.s_full[g], sph, 12 + g);
        sph ^= 1;
        tc_fence_after();
        uint32_t s0[32], s1[32], s2[32], s3[32];
        const bool full = word == kFullTileWord;
        // Padding rows of partial 8-row groups get -inf scores.  The word is the same for every lane, so each
        // group's test is a uniform branch and only partial groups pay for the selects.
        auto apply_mask = [&](uint32_t(&a)[32], int c0) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const uint32_t nv = uint32_t(word >> (4 * ((c0 >> 3) + q))) & 15u;
            if (nv < 8u) {
#pragma unroll
              for (int e = 0; e < 8; ++e)
                if (uint32_t(e) >= nv) a[8 * q + e] = __float_as_uint(-INFINITY);
            }
          }
        };
        tmem_ld32(tS + 0, s0);
        tmem_ld32(tS + 32, s1);
        tmem_ld32(tS + 64, s2);
        tmem_ld32(tS + 96, s3);
        tmem_wait_ld();
        // row max on the raw scores (scale > 0 preserves order); only tiles with padding rows need the mask
        if (!full) {
          apply_mask(s0, 0);
          apply_mask(s1, 32);
          apply_mask(s2, 64);
          apply_mask(s3, 96);
        }
        float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
        for (int e = 0; e < 32; e += 2) {
          mx0 = fmaxf(mx0, fmaxf(__uint_as_float(s0[e]), __uint_as_float(s1[e])));
          mx1 = fmaxf(mx1, fmaxf(__uint_as_float(s0[e + 1]), __uint_as_float(s1[e + 1])));
          mx0 = fmaxf(mx0, fmaxf(__uint_as_float(s2[e]), __uint_as_float(s3[e])));
          mx1 = fmaxf(mx1, fmaxf(__uint_as_float(s2[e + 1]), __uint_as_float(s3[e + 1])));
        }
        const float mt = fmaxf(mx0, mx1) * sl2;
        if (t == t_first) {
          m_used = mt;
        } else if (__any_sync(0xffffffffu,
                              rloc < nrows && mt > m_used + (kFp8 ? kRescaleThresholdFp8 : kRescaleThreshold))) {
          // only rows of the cluster vote: the tile's padding rows hold whatever follows the cluster in Q'
          // (another cluster or head), and must not change how the cluster's rows are rounded
          // warp-uniform branch (tcgen05.ld/st are .sync.aligned); rows whose max did not grow get alpha = 1
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
        const float pshift = kFp8 ? kPShift : 0.f;
        const uint64_t sl2x2 = f2(sl2, sl2), negm2 = f2(pshift - m_used, pshift - m_used);
        uint64_t lsum2 = f2(0.f, 0.f);
        auto exp_store = [&](const uint32_t(&a)[32], int c) {
          uint32_t pk[16];
          uint32_t pk8[8];  // kFp8: four e4m3 per column, key 4i + j in byte j
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            float x0, x1;
            f2_split(ffma2(f2(__uint_as_float(a[2 * e]), __uint_as_float(a[2 * e + 1])), sl2x2, negm2), x0, x1);
            float p0, p1;
            if (kPoly > 0 && (e % 8) < kPoly / 2) {  // spread the FMA-pipe pairs evenly over the chunk
              f2_split(ex2_poly2(f2(x0, x1)), p0, p1);
            } else {
              p0 = ex2_approx(x0);
              p1 = ex2_approx(x1);
            }
            lsum2 = fadd2(lsum2, f2(p0, p1));
            if (kFp8) {
              const uint32_t h16 = pack_e4m3x2(p0, p1);
              pk8[e >> 1] = (e & 1) ? (pk8[e >> 1] | (h16 << 16)) : h16;
            } else {
              pk[e] = pack_bf16x2(p0, p1);
            }
          }
          if (kFp8)
            tmem_st8(tS + 8 * c, pk8);
          else
            tmem_st16(tS + 16 * c, pk);
        };
        exp_store(s0, 0);
        exp_store(s1, 1);
        exp_store(s2, 2);
        exp_store(s3, 3);
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars.p_full[g]);
        float ls0, ls1;
        f2_split(lsum2, ls0, ls1);
        l += ls0 + ls1;
      }
      // ---- epilogue: O / l  -> bf16 -> original token order (fused pi_q^T)
      mbar_wait(&bars.o_full[g], oph, 14 + g);
      oph ^= 1;
      tc_fence_after();
      if (split) {
        // Merge the two partial softmax states of the same rows (flash-decoding style): warpgroup b hands (m, l)
        // over through shared memory, warpgroup a reads O_a and O_b from TMEM and writes
        //   O = (2^(m_a-m) O_a + 2^(m_b-m) O_b) / (2^(m_a-m) l_a + 2^(m_b-m) l_b),  m = max(m_a, m_b).
        // Warpgroup a releases both O accumulators (o_empty counts 4 arrivals, one per warp of a).
        if (g == 1) merge_ml[rloc] = make_float2(m_used, l);
        named_bar_sync(1, 256);
        float2 mlb = make_float2(0.f, 0.f);
        if (g == 0) mlb = merge_ml[rloc];
        named_bar_sync(1, 256);  // b writes merge_ml again only after a has read it
        if (g == 1) {
          continue;
        }
        const float m = fmaxf(m_used, mlb.x);
        const float wa = ex2_approx(m_used - m), wb = ex2_approx(mlb.x - m);
        const float lt = l * wa + mlb.y * wb;
        const float ca = wa / lt, cb = wb / lt;
        const uint32_t* vam = kFp8 ? p.v_amax + size_t(it.w & kItemBhMask) * D : nullptr;
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
              for (int e = 0; e < 8; ++e) {
                r[e] = __uint_as_float(oa[8 * v + e]) * ca + __uint_as_float(ob[8 * v + e]) * cb;
                if (kFp8) r[e] *= __uint_as_float(__ldg(vam + 32 * c + 8 * v + e)) * (1.f / 448.f);
              }
              orow[4 * c + v] = make_uint4(pack_bf16x2(r[0], r[1]), pack_bf16x2(r[2], r[3]), pack_bf16x2(r[4], r[5]),
                                           pack_bf16x2(r[6], r[7]));
            }
          }
        }
        if (rloc < nrows && p.lse) p.lse[dst] = (m - (kFp8 ? kPShift : 0.f) + __log2f(lt)) * 0.69314718055994531f;
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&bars.o_empty[0]);
          mbar_arrive(&bars.o_empty[1]);
        }
        continue;
      }
      const float inv_l = 1.f / l;
      const uint32_t* vam = kFp8 ? p.v_amax + size_t(it.w & kItemBhMask) * D : nullptr;
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
        if (kFp8) {  // per-channel V scale: o_c *= amax_c / 448
#pragma unroll
          for (int e = 0; e < 32; ++e)
            o[e] = __float_as_uint(__uint_as_float(o[e]) * (__uint_as_float(__ldg(vam + 32 * c + e)) * (1.f / 448.f)));
        }
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
      if (rloc < nrows && p.lse)
        p.lse[dst] = (m_used - (kFp8 ? kPShift : 0.f) + __log2f(l)) * 0.69314718055994531f;
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars.o_empty[g]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kWarpTmem) tmem_dealloc<512>(tmem);
}

cudaError_t run_attn_fp8(const void* Qp, const void* Kp, const void* Vp, int BH, int Nq, int Nk, float scale,
                         const int32_t* q_perm, const OutView& out, float* lse, AttnWs ws, cudaStream_t s,
                         const uint32_t* v_amax) {
  constexpr int D = 128;
  CUtensorMap mq;
  KVMaps kv;
  if (!make_tmap_bf16(&mq, Qp, uint64_t(BH) * Nq, D, 128)) return cudaErrorInvalidValue;
  for (int k = 0; k < kBoxKinds; ++k)
    if (!make_tmap_bf16(&kv.k[k], Kp, uint64_t(BH) * Nk, D, 8u << k) ||
        !make_tmap_u8(&kv.v[k], Vp, uint64_t(BH) * Nk, D, 8u << k))
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
  p.v_amax = v_amax;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  auto kernel = k_varblock_attn<D, kDefaultPoly, true>;
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(Cfg<D>::kSmemBytesFp8));
  kernel<<<sms, kThreads, Cfg<D>::kSmemBytesFp8, s>>>(mq, kv, p);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_varblock_attention_fp8(const void* Qp, const void* Kp, const void* Vp, int BH, int Nq, int Nk,
                                          int d, float scale, const int32_t* q_perm, const OutView& out, float* lse,
                                          AttnWs ws, cudaStream_t s, const uint32_t* v_amax) {
  if (d != 128 || !v_amax) return cudaErrorNotSupported;
  return run_attn_fp8(Qp, Kp, Vp, BH, Nq, Nk, scale, q_perm, out, lse, ws, s, v_amax);
}

}  // namespace svg2

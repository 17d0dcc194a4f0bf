// svg2_attn4.cu — A9 (+ fused A10), design v4: dynamic-block-size sparse attention over the permuted,
// cluster-contiguous tokens for sm_100a, with P staged in shared memory so that the next score
// tile never waits for the previous PV.
//
// Same work items, key streams and TMA box loads as design v2 (svg2_attn2.cu): an item is two 128-row Q
// tiles of one query cluster sharing one packed key stream of 8-row groups, 128 keys per tile.  What changes is the
// hand-over between the softmax and the tensor core.  In v2 P is written back over S in TMEM, so S(t+1) can only be
// computed after PV(t) has read P(t): each Q tile's chain is softmax -> PV -> S -> softmax and the softmax
// warpgroups idle for the MMA half of it.  Measured on B200 (tools/tmem_micro.cu): TMEM loads run at ~100 B/clk/SM,
// so reading one 128x128 fp32 S tile costs ~650 cycles, and one warpgroup alone (load, then 16K exp2 at 16/clk/SM)
// needs ~1260 cycles per tile while two warpgroups running together overlap each other's load and MUFU phases
// (~1080 cycles per tile).  Here P goes to a 32 KB shared-memory tile per Q tile (K-major, 128B swizzle, the A
// operand of an SS MMA), so:
//   * S_g(t+1) is issued as soon as the softmax warps of tile g have read S_g(t) into registers (s_free), and is
//     ready before they finish tile t: both softmax warpgroups run back to back;
//   * PV_g(t) runs whenever P_g(t) is in shared memory (p_full); its completion (p_free) gates the next P write and
//     the (rare) O rescale.
// Shared memory (d = 128): Q 2 x 32 KB | K 1 stage 32 KB | V 2 stages 64 KB | P 2 x 32 KB = 224 KB.  One K stage
// suffices because S is computed a whole tile ahead.  TMEM: S_a | S_b | O_a | O_b (512 columns).
//
// Warp roles (384 threads, 1 CTA per SM, persistent, dynamic item scheduler as in v2):
//   warps 0-3 / 4-7  softmax for Q tile a / b (one thread = one row = one TMEM lane)
//   warp 8           scheduler + TMA producer;  warp 9: TMEM allocator;  warp 11: MMA issuer (convergent)
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdlib>
#include "internal.h"
#include "ptx.cuh"
#include "tmap.h"

namespace svg2 {
namespace {

constexpr int kThreads = 384;
constexpr int kVStages = 2;
constexpr int kGroupsPerTile = kKTile / 8;  // 16
constexpr int kBoxKinds = 5;                // box heights 8, 16, 32, 64, 128 rows
constexpr float kRescaleThreshold = 8.0f;   // log2 units (see svg2_attn2.cu)
constexpr uint64_t kFullTileWord = 0x8888888888888888ull;
constexpr int kRegsCtl = 88, kRegsSoftmax = 208, kRegsLaunch = 168;
static_assert(128 * kRegsCtl + 256 * kRegsSoftmax <= kRegsLaunch * kThreads, "setmaxnreg budget exceeds launch");
constexpr int kWarpProducer = 8, kWarpTmem = 9, kWarpMma = 11;  // warp 10 idle
constexpr int kItemConsumers = 1 + 8;
constexpr uint32_t kPBlockBytes = 128 * 128;        // 64 keys x 128 rows of bf16 P
constexpr uint32_t kPBytes = 2 * kPBlockBytes;      // one 128 x 128 P tile

template <int D>
struct Cfg {
  static constexpr int kBlocks = D / 64;
  static constexpr uint32_t kBlockBytes = 128 * 128;
  static constexpr uint32_t kTileBytes = kBlocks * kBlockBytes;
  static constexpr uint32_t kGroupBytes = 8 * 2 * D;
  static constexpr uint32_t kSmemBytes = (2 + 1 + kVStages) * kTileBytes + 2 * kPBytes + 1024;
  __host__ __device__ static constexpr uint32_t col_s(int g) { return g ? 128u : 0u; }
  __host__ __device__ static constexpr uint32_t col_o(int g) { return g ? 384u : 256u; }
};

struct Bars {
  uint64_t q_full, q_empty, k_full, k_empty;
  uint64_t v_full[kVStages], v_empty[kVStages];
  uint64_t s_full[2], s_free[2], p_full[2], p_free[2], o_full[2], o_empty[2];
  uint64_t item_full[2], item_empty[2];
};

struct KVMaps {
  CUtensorMap k[kBoxKinds], v[kBoxKinds];
};

struct Params {
  const int4* items;
  int32_t* n_items;
  const int2* groups;
  const uint64_t* tilew;
  const int32_t* ngroups;
  size_t gcap, tcap;
  const int32_t* q_perm;
  __nv_bfloat16* O;
  float* lse;
  int Nq;
  float scale_log2;
  float rescale_thr;
  int debug_mode;  // 2 = cycle trace (SVG2_TRACE_PRINT build only)
};

#ifdef SVG2_TRACE_PRINT
// Events per tile of CTA 0's first item: 0/2 MMA issued PV a/b, 1/3 MMA issued S(t+1) a/b, 4/6 softmax a/b got S,
// 5/7 softmax a/b handed P over, 8/9 producer issued K/V.
constexpr int kTraceTiles = 8, kTraceEvents = 10;  // small: the smem budget is nearly full
#define TRACE(ev, t)                                                                                          \
  do {                                                                                                        \
    if (p.debug_mode == 2 && blockIdx.x == 0 && n_done == 0 && (t) < kTraceTiles && (threadIdx.x & 31) == 0) \
      trace_buf[(ev)*kTraceTiles + (t)] = clock64();                                                          \
  } while (0)
#else
#define TRACE(ev, t) \
  do {               \
  } while (0)
#endif

__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}

// One 16-group tile of the key stream into a K or V stage (power-of-two TMA boxes per run segment; see v2).
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
      const int kind = 31 - __clz(min(len, 16));
      const int pw = 1 << kind;
      for (int b = 0; b < C::kBlocks; ++b)
        tma_load_2d(stage + b * C::kBlockBytes + pos * 1024, &maps[kind], bar, 64 * b, row);
      pos += pw;
      len -= pw;
      row += 8 * pw;
    }
  }
}

template <int D>
__global__ void __launch_bounds__(kThreads, 1)
    k_varblock_attn4(const __grid_constant__ CUtensorMap mapQ, const __grid_constant__ KVMaps kv, const Params p) {
  using C = Cfg<D>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;                          // [2][tile]
  uint8_t* sK = sQ + 2 * C::kTileBytes;        // [1][tile]
  uint8_t* sV = sK + C::kTileBytes;            // [kVStages][tile]
  uint8_t* sP = sV + kVStages * C::kTileBytes; // [2][kPBytes]
  __shared__ Bars bars;
  __shared__ uint32_t tmem_slot;
  __shared__ int4 item_slot[2];
#ifdef SVG2_TRACE_PRINT
  __shared__ long long trace_buf[kTraceEvents * kTraceTiles];
  __shared__ int trace_T;
#endif

  const int warp = __shfl_sync(0xffffffffu, int(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  int n_done = 0;
  (void)n_done;
  if (warp == kWarpProducer && lane == 0) {
    tma_prefetch_desc(&mapQ);
    mbar_init(&bars.q_full, 1);
    mbar_init(&bars.q_empty, 1);
    mbar_init(&bars.k_full, 1);
    mbar_init(&bars.k_empty, 1);
    for (int s = 0; s < kVStages; ++s) {
      mbar_init(&bars.v_full[s], 1);
      mbar_init(&bars.v_empty[s], 1);
    }
    for (int g = 0; g < 2; ++g) {
      mbar_init(&bars.s_full[g], 1);
      mbar_init(&bars.s_free[g], 4);
      mbar_init(&bars.p_full[g], 4);
      mbar_init(&bars.p_free[g], 1);
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
      uint32_t qph = 0, kph = 0, vs = 0, vph = 0, islot = 0, iph = 0;
      while (true) {
        int item = 0;
        if (lane == 0) item = atomicAdd(p.n_items + 1, 1);
        item = __shfl_sync(0xffffffffu, item, 0);
        const int4 it = item < n_items ? __ldg(p.items + item) : make_int4(-1, 0, 0, 0);
        mbar_wait(&bars.item_empty[islot], iph ^ 1, 16);
        if (lane == 0) {
          item_slot[islot] = it;
          mbar_arrive(&bars.item_full[islot]);
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
          const int nxt = (t + 1) * kGroupsPerTile + lane;
          const int2 gw_next = (t + 1 < T && nxt < ng) ? __ldg(grp + nxt) : make_int2(0, 0);
          mbar_wait(&bars.k_empty, kph ^ 1, 2);
          if (lane == 0) mbar_arrive_expect_tx(&bars.k_full, bytes);
          __syncwarp();
          load_kv_tile<D>(kv.k, sK, &bars.k_full, ngt, lane, gw);
          kph ^= 1;
          TRACE(8, t);
          mbar_wait(&bars.v_empty[vs], vph ^ 1, 3);
          if (lane == 0) mbar_arrive_expect_tx(&bars.v_full[vs], bytes);
          __syncwarp();
          load_kv_tile<D>(kv.v, sV + vs * C::kTileBytes, &bars.v_full[vs], ngt, lane, gw);
          TRACE(9, t);
          gw = gw_next;
          if (++vs == kVStages) {
            vs = 0;
            vph ^= 1;
          }
        }
#ifdef SVG2_TRACE_PRINT
        if (n_done == 0 && blockIdx.x == 0 && lane == 0) trace_T = T;
#endif
        ++n_done;
      }
    } else if (warp == kWarpMma) {
      // ============================ MMA issuer ============================
      // Per key tile t: S_a(t+1), S_b(t+1) as soon as the softmax warps released S(t) (and K(t+1) landed), then
      // PV_a(t), PV_b(t) as soon as P(t) is in shared memory.  Whole warp convergent; elect.sync issues.
      uint32_t qph = 0, kph = 0, vs = 0, vph = 0, islot = 0, iph = 0;
      uint32_t oeph[2] = {0, 0}, pph[2] = {0, 0}, sfph[2] = {0, 0};
      const uint32_t idesc_pv = idesc_bf16_f32(128, D, true);
      const uint64_t dq0 = desc_kmajor_sw128(smem_u32(sQ)), dq1 = desc_kmajor_sw128(smem_u32(sQ + C::kTileBytes));
      const uint64_t dk = desc_kmajor_sw128(smem_u32(sK));
      const uint64_t dv0 = desc_mnmajor_sw128(smem_u32(sV), C::kBlockBytes);
      const uint64_t dv1 = desc_mnmajor_sw128(smem_u32(sV + C::kTileBytes), C::kBlockBytes);
      const uint64_t dp0 = desc_kmajor_sw128(smem_u32(sP)), dp1 = desc_kmajor_sw128(smem_u32(sP + kPBytes));
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
        const int ng = __ldg(p.ngroups + it.z);
        const int T = (ng + kGroupsPerTile - 1) / kGroupsPerTile;
        auto tile_n = [&](int t) { return uint32_t(min(kGroupsPerTile, ng - t * kGroupsPerTile)) * 8u; };
        auto issue_s = [&](int t, int g) {
          const uint32_t idesc = idesc_bf16_f32(128, tile_n(t), false);
          const uint64_t qd = g ? dq1 : dq0;
          const uint32_t d = tmem + C::col_s(g);
#pragma unroll
          for (int k = 0; k < D / 16; ++k) {
            const uint64_t off = uint64_t(((k >> 2) * C::kBlockBytes + (k & 3) * 32) >> 4);
            mma_ss_warp(d, qd + off, dk + off, idesc, k > 0);
          }
        };
        auto issue_pv = [&](int t, int g, uint32_t vstage) {
          const int ksteps = int(tile_n(t)) / 16;
          const uint64_t vd = vstage ? dv1 : dv0, pd = g ? dp1 : dp0;
          const uint32_t d = tmem + C::col_o(g);
#pragma unroll 1
          for (int k = 0; k < ksteps; ++k) {
            const uint64_t aoff = uint64_t(((k >> 2) * kPBlockBytes + (k & 3) * 32) >> 4);
            mma_ss_warp(d, pd + aoff, vd + uint64_t((k * 16 * 128) >> 4), idesc_pv, (t > 0 || k > 0) ? 1u : 0u);
          }
        };
        // S(t) for both Q tiles; waits for the softmax warps to have read the previous S of that tile
        auto issue_s_both = [&](int t) {
          mbar_wait_warp(&bars.k_full, kph);
          kph ^= 1;
#pragma unroll
          for (int g = 0; g < 2; ++g) {
            if (g == 1 && !has_b) break;
            mbar_wait_warp(&bars.s_free[g], sfph[g] ^ 1);
            sfph[g] ^= 1;
            tc_fence_after();
            issue_s(t, g);
            mma_commit_warp(&bars.s_full[g]);
            TRACE(1 + 2 * g, t);
          }
          mma_commit_warp(&bars.k_empty);
          if (t + 1 == T) mma_commit_warp(&bars.q_empty);
        };
        mbar_wait_warp(&bars.q_full, qph);
        qph ^= 1;
        issue_s_both(0);
        for (int t = 0; t < T; ++t) {
          if (t + 1 < T) issue_s_both(t + 1);
          mbar_wait_warp(&bars.v_full[vs], vph);
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
            issue_pv(t, g, vs);
            mma_commit_warp(&bars.p_free[g]);
            if (t + 1 == T) mma_commit_warp(&bars.o_full[g]);
            TRACE(2 * g, t);
          }
          mma_commit_warp(&bars.v_empty[vs]);
          if (++vs == kVStages) {
            vs = 0;
            vph ^= 1;
          }
        }
        ++n_done;
      }
    }
  } else {
    reg_alloc<kRegsSoftmax>();
    // ============================ softmax warpgroups ============================
    const int g = warp >> 2;
    const int rloc = ((warp & 3) << 5) + lane;
    const uint32_t lane_addr = uint32_t((warp & 3) * 32) << 16;
    const uint32_t tS = tmem + lane_addr + C::col_s(g);
    const uint32_t tO = tmem + lane_addr + C::col_o(g);
    // this row of the P tile: 8-row swizzle atom (rloc >> 3), row within it (rloc & 7); 16-byte chunk c of a
    // 64-key block lives at chunk (c ^ (rloc & 7)) -- the 128B swizzle the MMA's K-major descriptor expects
    const uint32_t prow = smem_u32(sP + g * kPBytes) + (rloc >> 3) * 1024 + (rloc & 7) * 128;
    const uint32_t psw = rloc & 7;
    const float sl2 = p.scale_log2;
    uint32_t sph = 0, pfph = 0, oph = 0, islot = 0, iph = 0;
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
      const int T = (ng + kGroupsPerTile - 1) / kGroupsPerTile;
      float m_used = -INFINITY, l = 0.f;
      uint64_t word_next = __ldg(tw);
      for (int t = 0; t < T; ++t) {
        const uint64_t word = word_next;
        if (t + 1 < T) word_next = __ldg(tw + t + 1);
        mbar_wait(&bars.s_full[g], sph, 12 + g);
        sph ^= 1;
        if ((warp & 3) == 0) TRACE(4 + 2 * g, t);
        tc_fence_after();
        uint32_t s0[32], s1[32], s2[32], s3[32];
        tmem_ld32(tS + 0, s0);
        tmem_ld32(tS + 32, s1);
        tmem_ld32(tS + 64, s2);
        tmem_ld32(tS + 96, s3);
        tmem_wait_ld();
        // S_g is in registers: the tensor core may overwrite it with the next tile's scores
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars.s_free[g]);
        if (word != kFullTileWord) {
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
        bool pv_done = false;  // PV_g(t-1) known complete (p_free consumed for this tile)
        if (t == 0) {
          m_used = mt;
        } else if (__any_sync(0xffffffffu, rloc < nrows && mt > m_used + p.rescale_thr)) {
          // only rows of the cluster vote: the tile's padding rows hold whatever follows the cluster in Q'
          // (another cluster or head), and must not change how the cluster's rows are rounded
          // O_g must hold all of PV_g(t-1) before it is rescaled
          mbar_wait(&bars.p_free[g], pfph ^ 1, 20 + g);
          pfph ^= 1;
          pv_done = true;
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
          tmem_wait_st();
          m_used = m_new;
        }
        // p = 2^(s * scale*log2e - m) packed to bf16 pairs; kept in registers until the P buffer is free
        const uint64_t sl2x2 = f2(sl2, sl2), negm2 = f2(-m_used, -m_used);
        uint64_t lsum2 = f2(0.f, 0.f);
        uint32_t pk[64];
        auto exps = [&](const uint32_t(&a)[32], int c) {
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            float x0, x1;
            f2_split(ffma2(f2(__uint_as_float(a[2 * e]), __uint_as_float(a[2 * e + 1])), sl2x2, negm2), x0, x1);
            const float p0 = ex2_approx(x0), p1 = ex2_approx(x1);
            lsum2 = fadd2(lsum2, f2(p0, p1));
            pk[16 * c + e] = pack_bf16x2(p0, p1);
          }
        };
        exps(s0, 0);
        exps(s1, 1);
        exps(s2, 2);
        exps(s3, 3);
        if (!pv_done) {  // PV_g(t-1) has finished reading the P buffer
          mbar_wait(&bars.p_free[g], pfph ^ 1, 20 + g);
          pfph ^= 1;
        }
#pragma unroll
        for (int j = 0; j < 16; ++j)
          st_shared_v4(prow + (j >> 3) * kPBlockBytes + ((uint32_t(j & 7) ^ psw) << 4), pk[4 * j], pk[4 * j + 1],
                       pk[4 * j + 2], pk[4 * j + 3]);
        fence_async_smem();  // generic-proxy stores -> visible to the tensor core (async proxy)
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars.p_full[g]);
        if ((warp & 3) == 0) TRACE(5 + 2 * g, t);
        float ls0, ls1;
        f2_split(lsum2, ls0, ls1);
        l += ls0 + ls1;
      }
      // ---- epilogue: O / l -> bf16 -> original token order (fused pi_q^T)
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
    const long long t0 = trace_buf[8 * kTraceTiles];
    printf("svg2 trace: T=%d (cycles relative to the first K issue)\n", trace_T);
    for (int t = 0; t < min(trace_T, kTraceTiles); ++t) {
      printf("svg2 trace t=%2d", t);
      for (int e = 0; e < kTraceEvents; ++e) printf(" %8lld", trace_buf[e * kTraceTiles + t] - t0);
      printf("\n");
    }
  }
#endif
}

template <int D>
cudaError_t run_attn4(const void* Qp, const void* Kp, const void* Vp, int BH, int Nq, int Nk, float scale,
                      const int32_t* q_perm, void* O, float* lse, const AttnWs& ws, cudaStream_t s) {
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
  static const float rescale_thr = [] {
    const char* e = getenv("SVG2_RESCALE_LOG2");
    return e ? float(atof(e)) : kRescaleThreshold;
  }();
  p.rescale_thr = rescale_thr;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaFuncSetAttribute(k_varblock_attn4<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<D>::kSmemBytes);
  k_varblock_attn4<D><<<sms, kThreads, Cfg<D>::kSmemBytes, s>>>(mq, kv, p);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_varblock_attention_v4(const void* Qp, const void* Kp, const void* Vp, int BH, int Nq, int Nk, int d,
                                         int Cq, int Ck, float scale, const int32_t* q_perm, void* O, float* lse,
                                         AttnWs ws, cudaStream_t s) {
  (void)Cq;
  (void)Ck;
  if (d == 128) return run_attn4<128>(Qp, Kp, Vp, BH, Nq, Nk, scale, q_perm, O, lse, ws, s);
  return run_attn4<64>(Qp, Kp, Vp, BH, Nq, Nk, scale, q_perm, O, lse, ws, s);
}

}  // namespace svg2
